// rs_single.h -- the one-launch single-pair path (rs_single.cu), called by
// rs_pairwise / rs_pairwise_cardinality for one pair of small bitmaps.
#pragma once
#include "rs_internal.cuh"

namespace rs {
// Result slots (8 KB each) of a single-pair op: a's containers for and /
// andnot, both sides' for or / xor.
uint32_t single_pair_slots(int op, uint32_t na, uint32_t nb);
// A[a] op B[b] into `out`, allocated by the caller with nb = 1, nc =
// single_pair_slots(...) and a pool of 8192 bytes per slot.  Host metadata of
// A and B must be valid.
int single_pair_op(int op, const rs_batch *A, const rs_batch *B, uint32_t a, uint32_t b, rs_batch *out);
// |A[a] op B[b]| written to out (device or page-locked host memory).
int single_pair_count(int op, const rs_batch *A, const rs_batch *B, uint32_t a, uint32_t b, uint64_t *out);
}  // namespace rs
