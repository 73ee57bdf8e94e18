"""Per-config measurements for all five BASELINE.json configs (C1..C5).

bench.py is the driver's single headline line (C2).  This script measures every
config the same way -- oracle-checked warm-up, CUDA-event timing on the library
stream with inputs resident, the oracle port timed beside it on the host cores
-- and writes one JSON object per config (profiles/configs_<tag>.json).

    python bench_configs.py [--configs 1,2,3,4,5] [--steps 5] [--tag r01]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

OPS = ("and", "or", "andnot", "xor")


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, steps, warmup=2):
    from paper_1709_07821_b200 import _lib
    for _ in range(warmup):
        fn()
    _lib.synchronize()
    e0 = _lib.Event()
    for _ in range(steps):
        fn()
    e1 = _lib.Event()
    _lib.synchronize()
    return e0.elapsed_ms(e1) / steps


def cpu_time(fn, min_seconds=2.0, max_reps=50):
    reps, t0 = 0, time.perf_counter()
    while reps < max_reps:
        fn()
        reps += 1
        if time.perf_counter() - t0 > min_seconds:
            break
    return (time.perf_counter() - t0) / reps


def wires(buf, offs, idx):
    return [buf[int(offs[i]):int(offs[i + 1])].tobytes() for i in idx]


def c1(steps):
    import paper_1709_07821_b200 as rb
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config1()
    B = rb.BitmapBatch.from_wire((buf, offs))
    w = wires(buf, offs, [0, 1])
    for op in OPS:  # oracle-checked warm-up
        assert B.pairwise(op, B, [0], [1]).to_wire_list()[0] == orc.op(op, w[0], w[1])
        assert int(B.pairwise_cardinality(op, B, [0], [1])[0]) == orc.op_cardinality(op, w[0], w[1])

    def step():
        for op in OPS:
            B.pairwise(op, B, [0], [1])
        for op in OPS:
            B.pairwise_cardinality(op, B, [0], [1])
    ms = timed(step, steps * 10)
    units = 8 * 64
    S = orc.Session(buf, offs)
    cpu = cpu_time(lambda: [S.run(op, k, S, [0], [1], 1) for op in OPS for k in ("op", "op_cardinality")])
    return {"config": "C1: one pair of 100k-value bitmaps in [0,2^22) (64 array chunks), 4 ops + 4 counts",
            "units_per_step": units, "ms_per_step": ms, "container_pairs_per_s": units / (ms * 1e-3),
            "note": "latency-bound: ~200 KB per op; synchronous API calls", "parity": "oracle-checked warm-up: 8/8",
            "cpu_port": {"container_pairs_per_s": units / cpu, "cores": 1, "ms_per_step": cpu * 1e3}}


def c2(steps):
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200 import _lib
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config2()
    n = 1024
    A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
    B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
    wa, wb = wires(buf, offs, [0, 1]), wires(buf, offs, [n, n + 1])
    res = {}
    for op in OPS:
        R = A.pairwise(op, B)
        got = R.select([0, 1]).to_wire_list()
        assert got == [orc.op(op, wa[k], wb[k]) for k in range(2)]
        pb, db, tc = R.stats()
        res[op] = pb + db
    in_bytes = n * 256 * 2 * 8200
    _lib.profile_reset()
    _lib.profile(True)
    per_op = {}
    for op in OPS:
        per_op[op] = timed(lambda: A.pairwise(op, B), steps)
    for op in OPS:
        per_op[op + "_count"] = timed(lambda: A.pairwise_cardinality(op, B), steps)
    _lib.profile(False)
    units = n * 256
    out = {"config": "C2: 1024 pairs x 256 bitset chunks (4.3 GB)", "per_op": {}}
    for op in OPS:
        ms = per_op[op]
        out["per_op"][op] = {"ms": ms, "container_pairs_per_s": units / (ms * 1e-3),
                             "algorithmic_GBps": (in_bytes + res[op]) / (ms * 1e-3) / 1e9}
        ms = per_op[op + "_count"]
        out["per_op"][op + "_count"] = {"ms": ms, "container_pairs_per_s": units / (ms * 1e-3),
                                        "algorithmic_GBps": (in_bytes + 8 * n) / (ms * 1e-3) / 1e9}
    S = orc.Session(buf, offs)
    ia = np.arange(64)
    cpu = cpu_time(lambda: [S.run(op, k, S, ia, ia + n, 0) for op in OPS for k in ("op", "op_cardinality")], 5.0, 3)
    out["cpu_port"] = {"container_pairs_per_s": 8 * 64 * 256 / cpu, "cores": orc.num_threads(),
                       "sample": "64 bitmap pairs x 8 ops"}
    return out


def c3(steps, npairs=1_000_000):
    import paper_1709_07821_b200 as rb
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config3(npairs=npairs)
    ia_, ib_ = synth.slice_images(buf, offs, 0, npairs), synth.slice_images(buf, offs, npairs, 2 * npairs)
    A, B = rb.BitmapBatch.from_wire(ia_), rb.BitmapBatch.from_wire(ib_)
    SA, SB = orc.Session(*ia_), orc.Session(*ib_)
    import torch
    dev_out = torch.empty(npairs, dtype=torch.int64, device="cuda")
    sample = np.arange(0, npairs, max(1, npairs // 2000))
    in_bytes = A.stats()[0] + B.stats()[0] + 16 * npairs
    out = {"config": f"C3: {npairs} array x array container pairs, Zipf(1.2) sizes", "per_op": {}}
    for op in OPS:
        R = A.container_pairwise(op, B)
        card = R.cardinalities()
        assert np.array_equal(card[sample].astype(np.int64), SA.run(op, "container_pairwise", SB, sample, sample))
        c = A.container_pairwise_cardinality(op, B)
        assert np.array_equal(c.astype(np.int64), card.astype(np.int64))
        pb, db, _ = R.stats()
        ms = timed(lambda: A.container_pairwise(op, B), steps)
        msc = timed(lambda: A.container_pairwise_cardinality_device(op, B, dev_out.data_ptr(), npairs), steps)
        out["per_op"][op] = {"ms": ms, "container_pairs_per_s": npairs / (ms * 1e-3),
                             "algorithmic_GBps": (in_bytes + pb + db) / (ms * 1e-3) / 1e9}
        out["per_op"][op + "_count"] = {"ms": msc, "container_pairs_per_s": npairs / (msc * 1e-3),
                                        "algorithmic_GBps": (in_bytes + 8 * npairs) / (msc * 1e-3) / 1e9}
    cs = np.arange(20000)
    cpu = cpu_time(lambda: [SA.run(op, k, SB, cs, cs, 0) for op in OPS
                            for k in ("container_pairwise", "container_pairwise_cardinality")], 5.0, 3)
    out["cpu_port"] = {"container_pairs_per_s": 8 * len(cs) / cpu, "cores": orc.num_threads(),
                       "sample": f"{len(cs)} pairs x 8 ops"}
    out["parity"] = f"cardinalities of every pair vs count-only; {len(sample)} sampled pairs vs oracle"
    return out


def descriptors(buf, offs, i):
    """(keys, container bytes incl. 8 B descriptor) of wire image i."""
    b = buf[int(offs[i]):int(offs[i + 1])]
    n = int(b[4:8].view("<u4")[0])
    d = b[8:8 + 8 * n].reshape(n, 8)
    keys = d[:, 0:2].copy().view("<u2").ravel().astype(np.int64)
    tag = d[:, 2]
    card = d[:, 4:8].copy().view("<u4").ravel().astype(np.int64)
    size = np.where(tag == 1, 2 * card, np.where(tag == 2, 8192, 0)).astype(np.int64) + 8
    # run payload sizes need the run counts: walk the payload section
    if (tag == 3).any():
        off = 8 + 8 * n
        sizes = np.empty(n, dtype=np.int64)
        for k in range(n):
            if tag[k] == 1:
                sizes[k] = 2 * card[k]
            elif tag[k] == 2:
                sizes[k] = 8192
            else:
                nr = int(b[off:off + 2].view("<u2")[0])
                sizes[k] = 2 + 4 * nr
            off += sizes[k]
        size = sizes + 8
    return keys, size


def c4(steps, nbitmaps=200):
    import paper_1709_07821_b200 as rb
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config4(nbitmaps=nbitmaps)
    Bt = rb.BitmapBatch.from_wire((buf, offs))
    S = orc.Session(buf, offs)
    ia, ib = np.arange(nbitmaps - 1), np.arange(1, nbitmaps)
    desc = [descriptors(buf, offs, i) for i in range(nbitmaps)]
    matched_in = copied = 0
    n_matched = 0
    for a, b in zip(ia, ib):
        (ka, sa), (kb, sb) = desc[a], desc[b]
        ma, mb = np.isin(ka, kb), np.isin(kb, ka)
        matched_in += int(sa[ma].sum() + sb[mb].sum())
        copied += int(sa[~ma].sum() + sb[~mb].sum())
        n_matched += int(ma.sum())
    out = {"config": f"C4: {nbitmaps} mixed-container bitmaps, successive AND/OR + union_many", "per_op": {},
           "matched_container_pairs": n_matched}
    hbm = peak()
    for op in ("and", "or"):
        R = Bt.pairwise(op, Bt, ia, ib)
        assert np.array_equal(R.cardinalities().astype(np.int64), S.run(op, "op", S, ia, ib))
        pb, db, _ = R.stats()
        # inputs read (matched both sides; OR also reads + copies the
        # unmatched ones) + result containers written
        byts = matched_in + (copied if op == "or" else 0) + pb + db
        ms = timed(lambda: Bt.pairwise(op, Bt, ia, ib), steps)
        out["per_op"][op] = {"ms": ms, "bitmap_pairs_per_s": len(ia) / (ms * 1e-3),
                             "container_pairs_per_s": n_matched / (ms * 1e-3),
                             "algorithmic_GBps": byts / (ms * 1e-3) / 1e9, "frac_of_hbm": byts / (ms * 1e-3) / 1e9 / hbm}
    # the north_star's "mixed-container batched AND/OR pipeline": both ops'
    # algorithmic bytes over both ops' device time
    po = out["per_op"]
    pipe_bytes = sum(po[o]["algorithmic_GBps"] * 1e9 * po[o]["ms"] * 1e-3 for o in ("and", "or"))
    pipe_ms = po["and"]["ms"] + po["or"]["ms"]
    out["and_or_pipeline"] = {"ms": pipe_ms, "algorithmic_GBps": pipe_bytes / (pipe_ms * 1e-3) / 1e9,
                              "frac_of_hbm": pipe_bytes / (pipe_ms * 1e-3) / 1e9 / hbm}
    U = Bt.union_many()
    w = wires(buf, offs, range(nbitmaps)) if nbitmaps <= 200 else None
    if w is not None:
        assert U.to_wire_list()[0] == orc.union_many(w)
    ms = timed(lambda: Bt.union_many(), steps)
    nc = int(Bt.container_counts().sum())
    out["union_many"] = {"ms": ms, "input_containers_per_s": nc / (ms * 1e-3), "result_containers": int(U.info()[1])}
    cpu = cpu_time(lambda: [S.run(op, "op", S, ia, ib, 0) for op in ("and", "or")], 5.0, 3)
    out["cpu_port"] = {"and+or_ms": cpu * 1e3, "cores": orc.num_threads()}
    t0 = time.perf_counter()
    orc.union_many(w)
    out["cpu_port"]["union_many_ms_1core_incl_decode"] = (time.perf_counter() - t0) * 1e3
    out["parity"] = "AND/OR cardinalities of all pairs vs oracle; union_many wire bytes vs oracle"
    return out


def c5(steps, nbitmaps=512):
    import paper_1709_07821_b200 as rb
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config5(nbitmaps=nbitmaps)
    Bt = rb.BitmapBatch.from_wire((buf, offs))
    inter, uni = Bt.all_pairs_cardinality()
    pi, pj = np.triu_indices(nbitmaps, 1)
    samp = np.arange(0, len(pi), max(1, len(pi) // 4000))
    want = orc.all_pairs_and(buf, offs, pi[samp], pj[samp])
    assert np.array_equal(inter[samp].astype(np.int64), want)
    ms = timed(lambda: Bt.all_pairs_cardinality(), max(1, steps // 2), 1)
    t0 = time.perf_counter()
    orc.all_pairs_and(buf, offs, pi[:20000], pj[:20000])
    cpu = (time.perf_counter() - t0) / 20000
    return {"config": f"C5: all {len(pi)} pairs of {nbitmaps} clustered bitmaps, |A∩B| and |A∪B|",
            "ms": ms, "bitmap_pairs_per_s": len(pi) / (ms * 1e-3),
            "cpu_port": {"bitmap_pairs_per_s": 1.0 / cpu, "cores": orc.num_threads(), "sample": "20000 pairs"},
            "parity": f"{len(samp)} sampled pairs vs oracle"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--tag", default="r01")
    args = ap.parse_args()
    fns = {"1": c1, "2": c2, "3": c3, "4": c4, "5": c5}
    results = {}
    for c in args.configs.split(","):
        t0 = time.perf_counter()
        try:
            results["C" + c] = fns[c](args.steps)
        except Exception as e:  # keep going; report the failure
            results["C" + c] = {"error": f"{type(e).__name__}: {e}"}
        results["C" + c]["wall_s"] = time.perf_counter() - t0
        print(json.dumps({"C" + c: results["C" + c]}), flush=True)
    results["hbm_peak_GBps"] = peak()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"configs_{args.tag}.json"), "w") as fh:
        json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
