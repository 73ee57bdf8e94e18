"""Drop-in shim: ``import roaringset`` resolves to the GPU package for the hot path.

Test infrastructure only (tests/test_reference_suite.py).  It is what a
maintainer's integration looks like when the reference package
(/root/reference/pkg/src/roaringset) switches its hot path to this library:

* ``roaringset.bitmap`` / ``roaringset.containers`` ARE the GPU package's
  modules (paper_1709_07821_b200.bitmap / .containers): RoaringBitmap,
  container_pairwise[_cardinality], container_normalize/add/remove/contains,
  the container classes;
* ``roaringset.serialize`` / ``deserialize`` / ``DecodeError`` are the GPU wire
  codec (rs_batch_to_wire / rs_batch_from_wire);
* everything SURVEY.md section 2 marks out of scope stays the reference's own
  code -- the per-container kernel backends (``roaringset.kernels``), the
  benchmark harness, baselines and CLI (``roaringset.bench``), the text
  datasets and the ClusterData generator (``roaringset.serde``) -- loaded
  from the reference's source files under this package name, so their
  relative imports (``from ..bitmap import RoaringBitmap``) pick up the GPU
  classes: the harness benchmarks and validates GPU bitmaps.

The reference source is located through RS_REFERENCE_SRC, else the pod-local
install ``baseline/_ref/roaringset`` (pip --target, git-ignored), else
/root/reference/pkg/src/roaringset.
"""

from __future__ import annotations

import importlib.util
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(_HERE)))


def reference_src() -> str | None:
    for cand in (os.environ.get("RS_REFERENCE_SRC"),
                 os.path.join(_ROOT, "baseline", "_ref", "roaringset"),
                 "/root/reference/pkg/src/roaringset"):
        if cand and os.path.isfile(os.path.join(cand, "__init__.py")):
            return cand
    return None


_REF = reference_src()
if _REF is None:
    raise ImportError("reference roaringset source not found (baseline/_ref or /root/reference)")
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_1709_07821_b200 as _gpu  # noqa: E402
from paper_1709_07821_b200 import bitmap as _gpu_bitmap, containers as _gpu_containers  # noqa: E402

# this package's submodules are searched in the reference tree
__path__ = [_REF]


def _load(name: str, path: str, package: bool = False):
    spec = importlib.util.spec_from_file_location(
        name, os.path.join(path, "__init__.py") if package else path,
        submodule_search_locations=[path] if package else None)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


# 1. the hot path: the GPU modules under the reference's module names
sys.modules[__name__ + ".containers"] = _gpu_containers
sys.modules[__name__ + ".bitmap"] = _gpu_bitmap
containers, bitmap = _gpu_containers, _gpu_bitmap

# 2. out-of-scope subsystems: the reference's own modules
kernels = _load(__name__ + ".kernels", os.path.join(_REF, "kernels"), package=True)
serde = _load(__name__ + ".serde", os.path.join(_REF, "serde.py"))
serde.serialize = _gpu.serialize          # the wire codec is on the path
serde.deserialize = _gpu.deserialize
serde.DecodeError = _gpu.DecodeError
bench = _load(__name__ + ".bench", os.path.join(_REF, "bench"), package=True)

# 3. the reference's top-level names (roaringset/__init__.py:10-30)
RoaringBitmap = _gpu.RoaringBitmap
ArrayContainer, BitsetContainer, RunContainer = (_gpu.ArrayContainer, _gpu.BitsetContainer,
                                                 _gpu.RunContainer)
container_add, container_remove, container_contains = (_gpu.container_add, _gpu.container_remove,
                                                       _gpu.container_contains)
container_normalize = _gpu.container_normalize
container_pairwise, container_pairwise_cardinality = (_gpu.container_pairwise,
                                                      _gpu.container_pairwise_cardinality)
serialize, deserialize, DecodeError = _gpu.serialize, _gpu.deserialize, _gpu.DecodeError
Dataset, DatasetError = serde.Dataset, serde.DatasetError
load_dataset, write_dataset, gen_clusterdata = serde.load_dataset, serde.write_dataset, serde.gen_clusterdata
__version__ = "0.1.0+b200"
