"""Oracle digests of every result of the five BASELINE.json configs at full size.

    python tools/make_config_digests.py [--configs 1,2,3,4,5]

Runs the C oracle (oracle/, the restatement pinned to the reference by
tests/golden) over the seeded workloads (workloads/, deterministic for any
thread count) and writes tests/golden/config_digests.json: per config and op,
fold_digests of the per-result content digests (every result bitmap / result
container) and of the counts.  bench.py checks the GPU's full results against
these -- rs_batch_digests on the device, so nothing moves to the host -- and
tests/test_gpu_fullscale.py reuses them.  Test infrastructure only.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_1709_07821_b200.batch import fold_digests  # noqa: E402  (pure numpy helper)
import workloads as synth  # noqa: E402

OPS = ("and", "or", "andnot", "xor")
OUT = os.path.join(ROOT, "tests", "golden", "config_digests.json")


def hx(x: int) -> str:
    return f"{x:016x}"


def pairs_digests(SA, SB, ia, ib, kind_op, kind_count):
    out = {}
    for op in OPS:
        d = SA.digests(op, kind_op, SB, ia, ib)
        c = SA.run(op, kind_count, SB, ia, ib)
        out[op] = hx(fold_digests(d))
        out[op + "_count"] = hx(fold_digests(c.astype(np.uint64)))
    return out


def c1():
    buf, offs = synth.config1()
    S = orc.Session(buf, offs)
    return {"workload": "config1()", **pairs_digests(S, S, [0], [1], "op", "op_cardinality")}


def c2():
    n = 1024
    buf, offs = synth.config2()
    S = orc.Session(buf, offs)
    ia = np.arange(n)
    return {"workload": "config2()", **pairs_digests(S, S, ia, ia + n, "op", "op_cardinality")}


def c3():
    n = 1_000_000
    buf, offs = synth.config3()
    S = orc.Session(buf, offs)
    ia = np.arange(n)
    return {"workload": "config3()", **pairs_digests(S, S, ia, ia + n, "container_pairwise",
                                                        "container_pairwise_cardinality")}


def c4():
    nb = 200
    buf, offs = synth.config4()
    S = orc.Session(buf, offs)
    ia = np.arange(nb - 1)
    out = {"workload": "config4()", **pairs_digests(S, S, ia, ia + 1, "op", "op_cardinality")}
    out["union_many"] = hx(fold_digests([S.union_digest()]))
    return out


def c5():
    nb = 512
    buf, offs = synth.config5()
    pi, pj = np.triu_indices(nb, 1)
    inter = orc.all_pairs_and(buf, offs, pi, pj)
    card = np.array([orc.cardinality(buf[int(offs[i]):int(offs[i + 1])].tobytes()) for i in range(nb)], np.int64)
    uni = card[pi] + card[pj] - inter
    return {"workload": "config5()", "inter": hx(fold_digests(inter.astype(np.uint64))),
            "union": hx(fold_digests(uni.astype(np.uint64)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    args = ap.parse_args()
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    fns = {"1": c1, "2": c2, "3": c3, "4": c4, "5": c5}
    for c in args.configs.split(","):
        t0 = time.time()
        res["C" + c] = fns[c]()
        print(f"C{c}: {time.time() - t0:.1f} s", flush=True)
        json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
