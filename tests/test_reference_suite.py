"""The reference's OWN test suite, run against the GPU package through the
``roaringset`` import shim (tests/dropin/roaringset): the direct proof that the
package is a drop-in for the hot path.

The reference tests (/root/reference/pkg/tests, copied with the pod-local
reference install into the git-ignored baseline/_ref/tests) run unmodified in
a subprocess whose ``import roaringset`` is the shim.  Files that exercise
the drop-in (bitmap, containers, wire format, acceptance criteria, and the
harness / CLI, which now build and time GPU bitmaps) run here.  Not run:
test_kernels.py and test_kernels_differential.py -- they test the reference's
per-container numpy/scalar kernel backends (kernels/scalar.py,
kernels/accelerated.py), a seam this library deliberately does not replace
(SURVEY.md 8(b)); under the shim they would only re-test the reference.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "dropin")


def reference_tests():
    for cand in (os.environ.get("RS_REFERENCE_TESTS"), os.path.join(ROOT, "baseline", "_ref", "tests"),
                 "/root/reference/pkg/tests"):
        if cand and os.path.isfile(os.path.join(cand, "test_bitmap.py")):
            return cand
    return None


FILES = ["test_bitmap.py", "test_containers.py", "test_serde.py", "test_acceptance.py", "test_bench.py",
         "test_cli.py"]


def run_reference_file(name, extra=()):
    tdir = reference_tests()
    if tdir is None:
        pytest.skip("reference tests not present (install them with tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT] + [p for p in env.get("PYTHONPATH", "").split(os.pathsep) if p])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-rs", "-p", "no:cacheprovider", "--rootdir", tdir,
           os.path.join(tdir, name), *extra]
    r = subprocess.run(cmd, cwd=tdir, env=env, capture_output=True, text=True, timeout=1800)
    log_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log_dir):
        with open(os.path.join(log_dir, f"reference_suite_{name[:-3]}.log"), "w") as fh:
            fh.write(r.stdout + r.stderr)
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_reference_suite_file(name):
    r = run_reference_file(name)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, f"reference {name} under the shim failed:\n{tail}"
    # the shim must really have routed the hot path to the GPU package
    assert "passed" in r.stdout


def test_shim_routes_hot_path_to_gpu_package():
    """CPU check: the shim resolves the hot-path modules to this package and
    the out-of-scope subsystems to the reference's own code."""
    if reference_tests() is None and not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference source not present")
    code = ("import roaringset, roaringset.containers as ct, paper_1709_07821_b200 as g;"
            "from roaringset.bench import harness;"
            "assert roaringset.RoaringBitmap is g.RoaringBitmap;"
            "assert harness.RoaringBitmap is g.RoaringBitmap;"
            "assert ct.container_pairwise is g.container_pairwise;"
            "assert roaringset.deserialize is g.deserialize;"
            "assert roaringset.kernels.__file__.startswith(roaringset.__path__[0]);"
            "print('ok')")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT])
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
