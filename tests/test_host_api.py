"""Host-side API contracts that need no GPU: argument checks before the C ABI
is called, the reference's exception types, the container type rules."""
import ctypes as C
import gc
import weakref

import numpy as np
import pytest

from paper_1709_07821_b200 import _lib
from paper_1709_07821_b200.batch import BitmapBatch
from paper_1709_07821_b200.bitmap import RoaringBitmap
from paper_1709_07821_b200 import containers as ct


def test_pair_index_lengths_checked_before_the_abi():
    """rs_pairwise & co. read npairs u32 from both index arrays: unequal
    lengths, or an explicit n past either, are a ValueError here."""
    with pytest.raises(ValueError):
        BitmapBatch._npairs(None, None, [0, 1, 2], [0, 1])
    with pytest.raises(ValueError):
        BitmapBatch._npairs(None, None, [0, 1], [0, 1], n=3)
    assert BitmapBatch._npairs(None, None, [0, 1], [2, 3]) == 2
    assert BitmapBatch._npairs(None, None, [0, 1], None, n=1) == 1


def test_from_values_conversion_errors_match_the_reference():
    """bitmap.py:43-50: np.asarray(..., dtype=uint64) -- a negative Python int
    is an OverflowError, a value past 32 bits a ValueError."""
    with pytest.raises(OverflowError):
        RoaringBitmap.from_values([1, -1])
    with pytest.raises(ValueError):
        RoaringBitmap.from_values([1, 1 << 32])


def test_result_rule_table():
    """the result-type rule per declared input types."""
    A, B, R = ct.TAG_ARRAY, ct.TAG_BITSET, ct.TAG_RUN
    assert ct._result_rule(A, A, "or") == "card" and ct._result_rule(B, B, "and") == "card"
    assert ct._result_rule(A, B, "and") == "array" and ct._result_rule(B, A, "and") == "array"
    assert ct._result_rule(A, B, "andnot") == "array" and ct._result_rule(B, A, "andnot") == "card"
    assert ct._result_rule(A, B, "xor") == "card"
    assert all(ct._result_rule(R, R, op) == "run" for op in ct.OPS)
    assert ct._result_rule(R, A, "and") == "array" and ct._result_rule(R, A, "andnot") == "run"
    assert ct._result_rule(A, R, "andnot") == "array" and ct._result_rule(A, R, "or") == "run"
    assert ct._result_rule(R, B, "or") == "card" and ct._result_rule(B, R, "andnot") == "card"


def test_canonical_forms():
    assert not ct._canonical(ct.ArrayContainer())
    assert not ct._canonical(ct.bitset_from_positions(np.arange(10)))
    assert ct._canonical(ct.bitset_from_positions(np.arange(5000)))
    assert not ct._canonical(ct.ArrayContainer(np.arange(5000)))
    assert not ct._canonical(ct.RunContainer([[0, 1], [10, 1]]))     # 2 runs over 4 values
    assert ct._canonical(ct.RunContainer([[0, 999]]))
    ct.container_validate(ct.RunContainer([[0, 999]]))
    with pytest.raises(AssertionError):
        ct.container_validate(ct.bitset_from_positions(np.arange(10)))


def test_pinned_view_lifetime():
    """_PinnedPool: the pooled block is released only when the last view of
    the returned array dies (slices included)."""
    class FakeBuf:
        def __init__(self, n):
            self.raw = (C.c_uint8 * n)()
            self._p = C.c_void_p(C.addressof(self.raw))
    released = []
    owner = _lib._PinnedView(FakeBuf(4096), 4096)
    weakref.finalize(owner, lambda: released.append(1))
    arr = np.asarray(owner).view(np.uint64)
    del owner
    head = arr[:10]
    del arr
    gc.collect()
    assert not released
    head[:] = 7
    del head
    gc.collect()
    assert released == [1]
