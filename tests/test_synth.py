"""Workload generator sanity (CPU): every synthetic image decodes under the
oracle's reference-exact validator, and the configs have their stated shape."""
import struct

import numpy as np

from oracle import oracle as orc
import workloads as synth


def _types(buf, offs):
    t = np.zeros(4, dtype=np.int64)
    for i in range(len(offs) - 1):
        w = buf[int(offs[i]):int(offs[i + 1])].tobytes()
        orc.check(w)
        (c,) = struct.unpack_from("<I", w, 4)
        for k in range(c):
            t[w[8 + 8 * k + 2]] += 1
    return t


def test_config1_shape():
    buf, offs = synth.config1()
    assert _types(buf, offs)[1] == 128  # 2 bitmaps x 64 array chunks
    for i in range(2):
        assert orc.cardinality(buf[int(offs[i]):int(offs[i + 1])].tobytes()) == 100_000


def test_config2_all_bitsets():
    buf, offs = synth.config2(npairs=4)
    t = _types(buf, offs)
    assert t[2] == 8 * 256 and t[1] == 0 and t[3] == 0


def test_config3_zipf_sizes():
    buf, offs = synth.config3(npairs=20000)
    lens = np.diff(offs.astype(np.int64)) - 16
    n = lens[:20000] // 2
    m = lens[20000:] // 2
    assert n.min() >= 1 and n.max() <= 4096
    assert 0.12 < np.mean(n == 4096) < 0.22          # clipped Zipf(1.2) tail
    assert 10 <= np.median(n) <= 40
    assert np.all((m == n) | (m == np.maximum(1, n // 64)))


def test_config4_mixed_types():
    buf, offs = synth.config4(nbitmaps=3)
    t = _types(buf, offs)
    assert t[1] > 0 and t[2] > 0 and t[3] > 0
    assert 1800 <= t[1:].sum() / 3 <= 2000


def test_config5_clusters():
    buf, offs = synth.config5(nbitmaps=3)
    t = _types(buf, offs)
    assert t[1] > 0 and t[2] > 0


def test_generator_is_deterministic():
    a = synth.config4(nbitmaps=2, nkeys=50)
    b = synth.config4(nbitmaps=2, nkeys=50)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
