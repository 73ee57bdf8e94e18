"""Per-config measurements of the five BASELINE.json configs (C1..C5).

bench.py embeds these in its JSON line under "configs"; run standalone to
measure one or more configs:

    python bench_configs.py [--configs 1,2,3,4,5] [--tag r02]

Protocol per config (the reference harness's, bench/harness.py:114-123,
205-239): build the seeded inputs (workloads/), a warm-up whose FULL results
are checked against the oracle's -- per-result content digests computed on
the device (rs_batch_digests) folded into one u64 and compared with
tests/golden/config_digests.json (tools/make_config_digests.py, the C oracle
over the same inputs), counts likewise -- then the median of >= 5 timed
repetitions (CUDA events on the library stream, inputs resident in HBM), and
the oracle port timed on a bounded sample on the host cores beside it.
Algorithmic bytes follow SURVEY 8(d): a container costs its 8-byte
descriptor plus its payload; an op reads both inputs' matched containers
(and, for OR/XOR/ANDNOT, the unmatched ones it copies) and writes its
result; a count reads the matched inputs and writes 8 B.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

OPS = ("and", "or", "andnot", "xor")
UNIT = "container-pairs/s"
DIGESTS = os.path.join(ROOT, "tests", "golden", "config_digests.json")


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cached_digests():
    try:
        return json.load(open(DIGESTS))
    except Exception:
        return {}


def hx(x: int) -> str:
    return f"{x:016x}"


def median_ms(fn, reps=5, warmup=2):
    """Median of `reps` CUDA-event-timed calls of fn (library stream)."""
    from paper_1709_07821_b200 import _lib
    for _ in range(warmup):
        fn()
    _lib.synchronize()
    ts = []
    for _ in range(reps):
        e0 = _lib.Event()
        fn()
        e1 = _lib.Event()
        ts.append(e0.elapsed_ms(e1))
    return statistics.median(ts), ts


def cpu_rate(fn, units_per_call, min_seconds=2.0, max_calls=200):
    """Oracle-port throughput: repeat fn for at least min_seconds."""
    calls, t0 = 0, time.perf_counter()
    while calls < max_calls:
        fn()
        calls += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    return units_per_call * calls / dt, dt, calls


class Parity:
    """Full-result digests (device) vs the oracle's cached digests."""

    def __init__(self, config: str):
        self.want = cached_digests().get(config, {})
        self.checked, self.bad = [], []

    def check(self, name: str, got: int):
        want = self.want.get(name)
        if want is None:
            self.bad.append(f"{name}: no cached oracle digest")
            return
        self.checked.append(name)
        if hx(got) != want:
            self.bad.append(f"{name}: {hx(got)} != oracle {want}")

    def result(self, what: str):
        return {"status": "match" if self.checked and not self.bad else "MISMATCH", "checked": self.checked,
                "what": what, "mismatches": self.bad,
                "oracle": "tests/golden/config_digests.json (tools/make_config_digests.py)"}


def batch_bytes(B) -> int:
    pb, db, _ = B.stats()
    return pb + db


def descriptors(buf, offs, i):
    """(keys, bytes incl. the 8-byte descriptor) of each container of image i."""
    b = buf[int(offs[i]):int(offs[i + 1])]
    n = int(b[4:8].view("<u4")[0])
    d = b[8:8 + 8 * n].reshape(n, 8)
    keys = d[:, 0:2].copy().view("<u2").ravel().astype(np.int64)
    tag = d[:, 2]
    card = d[:, 4:8].copy().view("<u4").ravel().astype(np.int64)
    sizes = np.where(tag == 1, 2 * card, 8192).astype(np.int64)
    if (tag == 3).any():
        off = 8 + 8 * n
        for k in range(n):
            if tag[k] == 3:
                nr = int(b[off:off + 2].view("<u2")[0])
                sizes[k] = 2 + 4 * nr
            off += int(sizes[k])
    return keys, sizes + 8


# ------------------------------------------------------------------ configs

def c1(cpu_seconds=2.0):
    """C1: one pair of 100k-value bitmaps, 4 ops + 4 counts (8 API calls)."""
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200.batch import fold_digests
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config1()
    B = rb.BitmapBatch.from_wire((buf, offs))
    par = Parity("C1")
    in_bytes = int(offs[2])  # both wire images: descriptors + payloads
    out_bytes = 0
    for op in OPS:
        R = B.pairwise(op, B, [0], [1])
        par.check(op, fold_digests(R.digests()))
        par.check(op + "_count", fold_digests(B.pairwise_cardinality(op, B, [0], [1])))
        out_bytes += batch_bytes(R)

    def step():
        for op in OPS:
            B.pairwise(op, B, [0], [1])
        for op in OPS:
            B.pairwise_cardinality(op, B, [0], [1])
    ms, ts = median_ms(step, reps=21, warmup=5)
    units = 8 * 64
    S = orc.Session(buf, offs, 1)
    cpu, dt, calls = cpu_rate(lambda: [S.run(op, k, S, [0], [1], 1) for op in OPS for k in ("op", "op_cardinality")],
                              units, cpu_seconds)
    hbm, pk = peak()
    gbps = (8 * in_bytes + out_bytes) / (ms * 1e-3) / 1e9
    return {"workload": "C1: one pair of 100k-value bitmaps in [0,2^22) (64 array chunks each), "
                        "4 ops + 4 op_cardinality, synchronous RoaringBitmap-style calls",
            "units_per_step": units, "ms": ms, "ms_reps": ts, "value": units / (ms * 1e-3), "unit": UNIT,
            "algorithmic_GBps": gbps,
            "roofline": {"bound": "latency", "frac": gbps / hbm, "peak": hbm, "peak_kind": pk,
                         "note": "~0.4 MB per call: launch/host latency bound, not HBM"},
            "cpu_baseline": {"value": cpu, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": f"the full step x {calls} ({dt:.1f} s), oracle port, 1 thread "
                                       "(one pair: the reference algorithm is sequential)"},
            "parity": par.result("all 4 results (content digests) and 4 counts")}


def c2(cpu_seconds=3.0, reps=5):
    """C2 per op (bench.py's headline runs the same inputs as one step)."""
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200.batch import fold_digests
    import workloads as synth
    from oracle import oracle as orc
    n = 1024
    buf, offs = synth.config2()
    A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, n))
    B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, n, 2 * n))
    par = Parity("C2")
    in_bytes = n * 256 * 2 * 8200
    per_op, out_bytes = {}, {}
    for op in OPS:
        R = A.pairwise(op, B)
        par.check(op, fold_digests(R.digests()))
        par.check(op + "_count", fold_digests(A.pairwise_cardinality(op, B)))
        out_bytes[op] = batch_bytes(R)
        del R
    hbm, pk = peak()
    units = n * 256
    for op in OPS:
        ms, _ = median_ms(lambda: A.pairwise(op, B), reps)
        per_op[op] = {"ms": ms, "value": units / (ms * 1e-3),
                      "algorithmic_GBps": (in_bytes + out_bytes[op]) / (ms * 1e-3) / 1e9}
        per_op[op]["frac"] = per_op[op]["algorithmic_GBps"] / hbm
    import torch
    dev = torch.empty(n, dtype=torch.int64, device="cuda")
    for op in OPS:
        ms, _ = median_ms(lambda: A.pairwise_cardinality_device(op, B, dev.data_ptr(), n), reps)
        g = (in_bytes + 8 * n) / (ms * 1e-3) / 1e9
        per_op[op + "_count"] = {"ms": ms, "value": units / (ms * 1e-3), "algorithmic_GBps": g, "frac": g / hbm}
    tot_ms = sum(v["ms"] for v in per_op.values())
    tot_bytes = sum(v["algorithmic_GBps"] * v["ms"] * 1e6 for v in per_op.values())
    S = orc.Session(buf, offs)
    ia = np.arange(64)
    cpu, dt, calls = cpu_rate(lambda: [S.run(op, k, S, ia, ia + n) for op in OPS for k in ("op", "op_cardinality")],
                              8 * 64 * 256, cpu_seconds)
    return {"workload": "C2: 1024 bitmap pairs x 256 bitset chunks (4.3 GB of input), 4 ops + 4 counts",
            "units_per_step": 8 * units, "ms": tot_ms, "value": 8 * units / (tot_ms * 1e-3), "unit": UNIT,
            "algorithmic_GBps": tot_bytes / (tot_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "frac": tot_bytes / (tot_ms * 1e-3) / 1e9 / hbm, "peak": hbm,
                         "peak_kind": pk},
            "per_op": per_op,
            "cpu_baseline": {"value": cpu, "unit": UNIT, "cores": orc.num_threads(), "kind": "port",
                             "sample": f"64 of 1024 pairs x 8 ops, x{calls} ({dt:.1f} s), all host threads"},
            "parity": par.result("every result bitmap of all 1024 pairs x 4 ops (content digests) and all counts")}


def c3(cpu_seconds=3.0, reps=5, npairs=1_000_000):
    """C3: container-level array x array pairs (container_pairwise[_cardinality])."""
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200.batch import fold_digests
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config3(npairs=npairs)
    A = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, 0, npairs))
    B = rb.BitmapBatch.from_wire(synth.slice_images(buf, offs, npairs, 2 * npairs))
    par = Parity("C3")
    import torch
    dev = torch.empty(npairs, dtype=torch.int64, device="cuda")
    in_bytes = batch_bytes(A) + batch_bytes(B)
    hbm, pk = peak()
    per_op = {}
    for op in OPS:
        R = A.container_pairwise(op, B)
        par.check(op, fold_digests(R.digests()))
        par.check(op + "_count", fold_digests(A.container_pairwise_cardinality(op, B)))
        ob = batch_bytes(R)
        del R
        ms, _ = median_ms(lambda: A.container_pairwise(op, B), reps)
        g = (in_bytes + ob) / (ms * 1e-3) / 1e9
        per_op[op] = {"ms": ms, "value": npairs / (ms * 1e-3), "algorithmic_GBps": g, "frac": g / hbm}
        ms, _ = median_ms(lambda: A.container_pairwise_cardinality_device(op, B, dev.data_ptr(), npairs), reps)
        g = (in_bytes + 8 * npairs) / (ms * 1e-3) / 1e9
        per_op[op + "_count"] = {"ms": ms, "value": npairs / (ms * 1e-3), "algorithmic_GBps": g, "frac": g / hbm}
    tot_ms = sum(v["ms"] for v in per_op.values())
    tot_bytes = sum(v["algorithmic_GBps"] * v["ms"] * 1e6 for v in per_op.values())
    S = orc.Session(buf, offs)
    cs = np.arange(20000)
    cpu, dt, calls = cpu_rate(lambda: [S.run(op, k, S, cs, cs + npairs) for op in OPS
                                       for k in ("container_pairwise", "container_pairwise_cardinality")],
                              8 * len(cs), cpu_seconds)
    return {"workload": f"C3: {npairs} array x array container pairs, Zipf(1.2) sizes, "
                        "4 container_pairwise + 4 container_pairwise_cardinality",
            "units_per_step": 8 * npairs, "ms": tot_ms, "value": 8 * npairs / (tot_ms * 1e-3), "unit": UNIT,
            "algorithmic_GBps": tot_bytes / (tot_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "frac": tot_bytes / (tot_ms * 1e-3) / 1e9 / hbm, "peak": hbm,
                         "peak_kind": pk},
            "per_op": per_op,
            "cpu_baseline": {"value": cpu, "unit": UNIT, "cores": orc.num_threads(), "kind": "port",
                             "sample": f"20000 of {npairs} pairs x 8 ops, x{calls} ({dt:.1f} s), all host threads"},
            "parity": par.result(f"every result container of all {npairs} pairs x 4 ops and all counts")}


def c4(cpu_seconds=3.0, reps=5, nbitmaps=200):
    """C4: mixed-container collection: successive AND / OR pairs + union_many."""
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200.batch import fold_digests
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config4(nbitmaps=nbitmaps)
    Bt = rb.BitmapBatch.from_wire((buf, offs))
    par = Parity("C4")
    ia, ib = np.arange(nbitmaps - 1), np.arange(1, nbitmaps)
    desc = [descriptors(buf, offs, i) for i in range(nbitmaps)]
    matched_in = copied_a = copied_b = n_matched = 0
    for a, b in zip(ia, ib):
        (ka, sa), (kb, sb) = desc[a], desc[b]
        ma, mb = np.isin(ka, kb), np.isin(kb, ka)
        matched_in += int(sa[ma].sum() + sb[mb].sum())
        copied_a += int(sa[~ma].sum())
        copied_b += int(sb[~mb].sum())
        n_matched += int(ma.sum())
    hbm, pk = peak()
    per_op = {}
    for op in OPS:
        R = Bt.pairwise(op, Bt, ia, ib)
        par.check(op, fold_digests(R.digests()))
        par.check(op + "_count", fold_digests(Bt.pairwise_cardinality(op, Bt, ia, ib)))
        copies = {"and": 0, "or": copied_a + copied_b, "xor": copied_a + copied_b, "andnot": copied_a}[op]
        byts = matched_in + 2 * copies + batch_bytes(R) - copies  # copies: read once + written (in R's bytes)
        del R
        ms, _ = median_ms(lambda: Bt.pairwise(op, Bt, ia, ib), reps)
        g = byts / (ms * 1e-3) / 1e9
        per_op[op] = {"ms": ms, "value": n_matched / (ms * 1e-3), "bitmap_pairs_per_s": len(ia) / (ms * 1e-3),
                      "algorithmic_GBps": g, "frac": g / hbm, "bytes": byts}
    U = Bt.union_many()
    par.check("union_many", fold_digests(U.digests()))
    ub = batch_bytes(U)
    del U
    in_all = int(offs[-1]) - 8 * nbitmaps
    ms_u, _ = median_ms(lambda: Bt.union_many(), reps)
    per_op["union_many"] = {"ms": ms_u, "input_containers_per_s": int(Bt.container_counts().sum()) / (ms_u * 1e-3),
                            "algorithmic_GBps": (in_all + ub) / (ms_u * 1e-3) / 1e9,
                            "frac": (in_all + ub) / (ms_u * 1e-3) / 1e9 / hbm}
    pipe_ms = per_op["and"]["ms"] + per_op["or"]["ms"]
    pipe_b = per_op["and"]["bytes"] + per_op["or"]["bytes"]
    S = orc.Session(buf, offs)
    cpu, dt, calls = cpu_rate(lambda: [S.run(op, "op", S, ia, ib) for op in ("and", "or")], 2 * n_matched,
                              cpu_seconds)
    return {"workload": f"C4: {nbitmaps} mixed-container bitmaps (~2000 keys each; arrays, bitsets, runs), "
                        "199 successive pairs x 4 ops + union_many over all",
            "units_per_step": 2 * n_matched, "ms": pipe_ms, "value": 2 * n_matched / (pipe_ms * 1e-3),
            "unit": UNIT + " (matched container pairs of the AND + OR pipeline)",
            "algorithmic_GBps": pipe_b / (pipe_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "frac": pipe_b / (pipe_ms * 1e-3) / 1e9 / hbm, "peak": hbm,
                         "peak_kind": pk},
            "and_or_pipeline": {"ms": pipe_ms, "algorithmic_GBps": pipe_b / (pipe_ms * 1e-3) / 1e9,
                                "frac": pipe_b / (pipe_ms * 1e-3) / 1e9 / hbm,
                                "target": "north_star: mixed-container batched AND/OR pipeline >= 40% of HBM"},
            "per_op": per_op, "matched_container_pairs": n_matched,
            "cpu_baseline": {"value": cpu, "unit": UNIT, "cores": orc.num_threads(), "kind": "port",
                             "sample": f"AND + OR over all 199 pairs x{calls} ({dt:.1f} s), all host threads"},
            "parity": par.result("every result bitmap of 199 pairs x 4 ops, all counts, and union_many")}


def c5(cpu_seconds=3.0, reps=5, nbitmaps=512):
    """C5: all-pairs |A and B| and |A or B| (Jaccard) over 512 clustered bitmaps."""
    import paper_1709_07821_b200 as rb
    from paper_1709_07821_b200 import _lib
    from paper_1709_07821_b200.batch import fold_digests
    import workloads as synth
    from oracle import oracle as orc
    buf, offs = synth.config5(nbitmaps=nbitmaps)
    Bt = rb.BitmapBatch.from_wire((buf, offs))
    par = Parity("C5")
    inter, uni = Bt.all_pairs_cardinality()
    par.check("inter", fold_digests(inter))
    par.check("union", fold_digests(uni))
    del inter, uni
    npairs = nbitmaps * (nbitmaps - 1) // 2
    _lib.profile_reset()
    _lib.profile(True)
    ms, _ = median_ms(lambda: Bt.all_pairs_cardinality(), reps)
    um_ms, um_n, _ = _lib.profile_query("allpairs_umma")
    _lib.profile(False)
    hbm, pk = peak()
    compulsory = int(offs[-1])  # every bitmap read once
    pi, pj = np.triu_indices(nbitmaps, 1)
    samp = np.arange(0, npairs, 4)[:8192]
    S = orc.Session(buf, offs)  # in-memory bitmaps: |A and B| is op_cardinality (the union follows from it)
    rate, dt, calls = cpu_rate(lambda: S.run("and", "op_cardinality", S, pi[samp], pj[samp]), len(samp),
                               cpu_seconds)
    return {"workload": f"C5: all {npairs} pairs of {nbitmaps} clustered bitmaps on [0,2^26), |A and B| and "
                        "|A or B| (rs_all_pairs_cardinality: key grouping, densify, tcgen05 Gram tiles)",
            "units_per_step": npairs, "ms": ms, "value": npairs / (ms * 1e-3), "unit": "bitmap pairs/s",
            "algorithmic_GBps": compulsory / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "tensor", "frac_of_hbm_compulsory": compulsory / (ms * 1e-3) / 1e9 / hbm,
                         "peak": hbm, "peak_kind": pk,
                         "umma_kernel_ms": um_ms / um_n if um_n else None,
                         "note": "all-pairs intersections are a Gram matrix per chunk key (tcgen05 kind::mxf4); "
                                 "compulsory bytes = every bitmap read once"},
            "cpu_baseline": {"value": rate, "unit": "bitmap pairs/s", "cores": orc.num_threads(),
                             "kind": "port",
                             "sample": f"{len(samp)} of {npairs} pairs x{calls} ({dt:.1f} s), all host threads"},
            "parity": par.result(f"all {npairs} intersection and union counts")}


FNS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def measure(names, cpu_seconds=3.0):
    out = {}
    for name in names:
        t0 = time.perf_counter()
        try:
            out[name] = FNS[name](cpu_seconds=cpu_seconds)
        except Exception as e:  # report, keep going
            out[name] = {"error": f"{type(e).__name__}: {e}"}
        out[name]["wall_s"] = time.perf_counter() - t0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--tag", default="r02")
    args = ap.parse_args()
    names = ["C" + c for c in args.configs.split(",")]
    res = {}
    for n in names:
        res.update(measure([n], args.cpu_seconds))
        print(json.dumps({n: res[n]}), flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"configs_{args.tag}.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
