"""paper_1709_07821_b200: B200-native (sm_100a) batched Roaring bitmap set operations.

Drop-in for the hot path of the reference package ``roaringset``
(/root/reference/pkg/src/roaringset/__init__.py:10-30): the same
``RoaringBitmap`` API (from_values, & | - ^, op, op_cardinality, union_many,
to_array, run_optimize, chunks, ==), the container-level
``container_pairwise[_cardinality]``, and the wire format, all computed by
hand-written CUDA kernels behind the C ABI of include/roaring_b200.h.
``BitmapBatch`` exposes the batched form that keeps the GPU busy.
"""

from .batch import BitmapBatch
from .bitmap import RoaringBitmap
from .containers import (ArrayContainer, BitsetContainer, RunContainer, container_add, container_contains,
                         container_normalize, container_pairwise, container_pairwise_cardinality,
                         container_remove)
from .serde import DecodeError, deserialize, serialize
from ._lib import RoaringCudaError

__version__ = "0.1.0"

__all__ = [
    "RoaringBitmap", "BitmapBatch",
    "ArrayContainer", "BitsetContainer", "RunContainer",
    "container_pairwise", "container_pairwise_cardinality",
    "container_add", "container_remove", "container_contains", "container_normalize",
    "serialize", "deserialize", "DecodeError", "RoaringCudaError",
    "__version__",
]
