"""Loader for tests/golden/golden_v1.npz (produced by tests/golden/make_golden.py
from the real reference)."""
import functools
import json
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


class Golden:
    def __init__(self, z):
        self.z = z
        self.buf = z["wire_buf"]
        self.off = z["wire_off"]

    def wire(self, i) -> bytes:
        return self.buf[int(self.off[i]):int(self.off[i + 1])].tobytes()

    def __getitem__(self, k):
        v = self.z[k]
        if v.dtype.kind in "US":
            return json.loads(str(v))
        return v


@functools.lru_cache(maxsize=1)
def load() -> Golden:
    return Golden(np.load(PATH))
