"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
entry point include/roaring_b200.h declares; without a GPU it fails loudly
(no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "roaring_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("rs_batch_from_wire", "rs_batch_from_u32", "rs_pairwise", "rs_pairwise_cardinality",
              "rs_container_pairwise", "rs_container_pairwise_cardinality", "rs_union_many",
              "rs_all_pairs_cardinality", "rs_batch_to_wire", "rs_batch_to_u32", "rs_batch_run_optimize"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1709_07821_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1709_07821_b200 import BitmapBatch, RoaringCudaError
    with pytest.raises(RoaringCudaError):
        BitmapBatch.from_wire([b"ROAR\x00\x00\x00\x00"])


def test_unknown_op_is_value_error_before_any_device_work():
    from paper_1709_07821_b200.containers import op_index
    with pytest.raises(ValueError, match="unknown op 'nand'"):
        op_index("nand")


def test_sm100a_cubin_in_library():
    import subprocess
    from paper_1709_07821_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the CPU arm the driver times beside the GPU
    arm) prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    for k in ("metric", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
