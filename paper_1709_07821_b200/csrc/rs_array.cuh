// rs_array.cuh -- array x array container pairs as a shared-memory merge path.
//
// The reference walks two sorted u16 arrays with two pointers
// (kernels/scalar.py:122-267; SIMD blocks in PAPER.md Alg. 1-3).  Here a
// group of GT threads owns one pair: both arrays are staged in smem, every
// thread takes VT consecutive items of the merged sequence (ties: A first)
// located by a merge-path binary search, and marks each item kept or not:
//   and:    A items present in B            (array_intersect)
//   or:     all A items + B items not in A  (array_union)
//   andnot: A items absent from B           (array_difference)
//   xor:    items present on one side only  (array_xor)
// A group scan of the per-thread kept counts gives output positions; the
// result is an array if it holds <= 4096 values, else a bitset
// (_container_from_values, containers.py:244-247).  Groups: a warp for
// na+nb <= 256, 128 threads for <= 2048, 256 threads for the rest.
#pragma once
#include "rs_internal.cuh"

namespace rsa {

template <int GT>
__device__ __forceinline__ void group_sync(int gid) {
  if constexpr (GT == 32) {
    __syncwarp();
  } else if constexpr (GT == 256) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(GT) : "memory");
  }
}

// exclusive scan over the group; `ws` holds GT/32 words of group smem
template <int GT>
__device__ __forceinline__ uint32_t group_scan(uint32_t x, uint32_t &total, uint32_t *ws, int gid) {
  const int lane = threadIdx.x & 31, w = (threadIdx.x % GT) >> 5;
  uint32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if constexpr (GT == 32) {
    total = __shfl_sync(0xffffffffu, v, 31);
    return v - x;
  } else {
    if (lane == 31) ws[w] = v;
    group_sync<GT>(gid);
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < GT / 32; k++) {
      uint32_t s = ws[k];
      pre += k < w ? s : 0;
      tot += s;
    }
    group_sync<GT>(gid);
    total = tot;
    return pre + v - x;
  }
}

__device__ __forceinline__ int merge_path(const uint16_t *A, int na, const uint16_t *B, int nb, int diag) {
  int lo = max(0, diag - nb), hi = min(diag, na);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Walk VT merged items from (i, j); call emit(value) for every kept item.
template <int VT, typename F>
__device__ __forceinline__ void merge_walk(int op, const uint16_t *A, int na, const uint16_t *B, int nb, int i, int j,
                                           F emit) {
  const int total = na + nb;
#pragma unroll 4
  for (int k = 0; k < VT; k++) {
    if (i + j >= total) break;
    bool takeA = j >= nb || (i < na && A[i] <= B[j]);
    if (takeA) {
      uint16_t v = A[i];
      bool both = j < nb && B[j] == v;
      bool keep = op == RS_OP_AND ? both : op == RS_OP_OR ? true : !both;
      if (keep) emit(v);
      i++;
    } else {
      uint16_t v = B[j];
      bool both = i > 0 && A[i - 1] == v;
      bool keep = (op == RS_OP_OR || op == RS_OP_XOR) && !both;
      if (keep) emit(v);
      j++;
    }
  }
}

// The same walk, fully unrolled, keeping the VT items' values and keep flags
// in registers (static indices), so a materialized pair walks once: the kept
// values go to their scanned positions straight from registers.
template <int VT>
__device__ __forceinline__ void merge_walk_reg(int op, const uint16_t *A, int na, const uint16_t *B, int nb, int i,
                                               int j, uint16_t (&kv)[VT], uint32_t &km) {
  const int total = na + nb;
  km = 0;
#pragma unroll
  for (int k = 0; k < VT; k++) {
    const bool valid = i + j < total;
    const bool takeA = j >= nb || (i < na && A[i] <= B[j]);
    uint16_t v;
    bool keep;
    if (takeA) {
      v = i < na ? A[i] : 0;
      const bool both = j < nb && B[j] == v;
      keep = op == RS_OP_AND ? both : op == RS_OP_OR ? true : !both;
    } else {
      v = B[j];
      const bool both = i > 0 && A[i - 1] == v;
      keep = (op == RS_OP_OR || op == RS_OP_XOR) && !both;
    }
    kv[k] = v;
    km |= (uint32_t)(valid && keep) << k;
    if (valid) {
      i += takeA;
      j += !takeA;
    }
  }
}

template <int GT, int VT>
struct alignas(16) AASmem {
  static constexpr int CAP = GT * VT;                       // merged items per group
  static constexpr int CAPA = CAP < 4096 ? CAP : 4096;      // one side
  static constexpr bool BITSET = CAP > 4096;                // result can exceed 4096 values
  uint16_t a[CAPA];
  uint16_t b[CAPA];
  union {
    uint16_t out[CAPA];
    uint32_t bits[BITSET ? 2048 : 1];
  };
  uint32_t ws[GT / 32];
};

// Load an array container's values into smem (16-byte vectors; pool payloads
// are 16-byte aligned and zero padded).
template <int GT>
__device__ __forceinline__ void stage(uint16_t *dst, const uint8_t *src, int n, int lt) {
  int nv = (2 * n + 15) >> 4;
  for (int k = lt; k < nv; k += GT) ((uint4 *)dst)[k] = ((const uint4 *)src)[k];
}

// One pair through the group.  count_only: returns the kept count, writes
// nothing.  Otherwise writes the result container at dst and returns its
// (type, card, n) through the out-parameters (identical on every thread).
// One tiny pair by ONE thread: the textbook two-pointer merge
// (kernels/scalar.py:122-267; the same keep rules as merge_walk) reading the
// values straight from the pools and writing the result array to dst with
// its 16-byte zero pad.  Returns the kept count (always an array result:
// at most na + nb values).
__device__ __forceinline__ uint32_t aa_pair_thread(int op, const uint16_t *A, uint32_t na, const uint16_t *B,
                                                   uint32_t nb, uint16_t *dst) {
  uint32_t i = 0, j = 0, k = 0;
  uint32_t a = na ? __ldg(A) : 0u, b = nb ? __ldg(B) : 0u;
  const bool keep_a = op != RS_OP_AND, keep_b = op == RS_OP_OR || op == RS_OP_XOR,
             keep_both = op == RS_OP_AND || op == RS_OP_OR;
  while (i < na || j < nb) {
    const bool take_a = j >= nb || (i < na && a < b), take_b = i >= na || (j < nb && b < a);
    uint32_t v;
    bool keep;
    if (take_a) { v = a; keep = keep_a; }
    else if (take_b) { v = b; keep = keep_b; }
    else { v = a; keep = keep_both; }
    if (keep) {
      if (dst) dst[k] = (uint16_t)v;
      k++;
    }
    if (!take_b) { i++; a = i < na ? __ldg(A + i) : 0u; }
    if (!take_a) { j++; b = j < nb ? __ldg(B + j) : 0u; }
  }
  if (dst)
    for (uint32_t p = k; p & 7; p++) dst[p] = 0;
  return k;
}

// OPC >= 0: the op as a compile-time constant (the caller's kernel is
// instantiated per op, so the keep rules fold away).
template <int GT, int VT, int OPC = -1>
__device__ uint32_t aa_pair(int op_rt, bool count_only, const uint8_t *pa, int na, const uint8_t *pb, int nb,
                            AASmem<GT, VT> &sm, int gid, uint8_t *dst, uint8_t &type, uint32_t &nout) {
  const int op = OPC >= 0 ? OPC : op_rt;
  const int lt = threadIdx.x % GT;
  stage<GT>(sm.a, pa, na, lt);
  stage<GT>(sm.b, pb, nb, lt);
  group_sync<GT>(gid);
  const int diag = min(lt * VT, na + nb);
  const int i0 = merge_path(sm.a, na, sm.b, nb, diag), j0 = diag - i0;
  if constexpr (!AASmem<GT, VT>::BITSET && VT <= 16) {  // one walk, kept items in registers
    uint16_t kv[VT];
    uint32_t km;
    merge_walk_reg<VT>(op, sm.a, na, sm.b, nb, i0, j0, kv, km);
    uint32_t total;
    uint32_t pos = group_scan<GT>((uint32_t)__popc(km), total, sm.ws, gid);
    type = RS_TAG_ARRAY;
    nout = total;
    if (count_only || total == 0) return total;
#pragma unroll
    for (int k = 0; k < VT; k++)
      if ((km >> k) & 1u) sm.out[pos++] = kv[k];
    group_sync<GT>(gid);
    const int nvec = (2 * (int)total + 15) >> 4;
    if (lt < 8 && (int)total + lt < nvec * 8) sm.out[total + lt] = 0;
    group_sync<GT>(gid);
    for (int k = lt; k < nvec; k += GT) ((uint4 *)dst)[k] = ((const uint4 *)sm.out)[k];
    return total;
  }
  uint32_t cnt = 0;
  merge_walk<VT>(op, sm.a, na, sm.b, nb, i0, j0, [&](uint16_t) { cnt++; });
  uint32_t total;
  uint32_t base = group_scan<GT>(cnt, total, sm.ws, gid);
  if (count_only || total == 0) {
    type = RS_TAG_ARRAY;
    nout = total;
    return total;
  }
  if (!AASmem<GT, VT>::BITSET || total <= RS_ARRAY_MAX) {
    merge_walk<VT>(op, sm.a, na, sm.b, nb, i0, j0, [&](uint16_t v) { sm.out[base++] = v; });
    group_sync<GT>(gid);
    int nvec = (2 * (int)total + 15) >> 4;
    if (lt < 8 && (int)total + lt < nvec * 8) sm.out[total + lt] = 0;
    group_sync<GT>(gid);
    for (int k = lt; k < nvec; k += GT) ((uint4 *)dst)[k] = ((const uint4 *)sm.out)[k];
    type = RS_TAG_ARRAY;
    nout = total;
  } else {
    if constexpr (AASmem<GT, VT>::BITSET) {
      for (int k = lt; k < 2048; k += GT) sm.bits[k] = 0;
      group_sync<GT>(gid);
      merge_walk<VT>(op, sm.a, na, sm.b, nb, i0, j0,
                     [&](uint16_t v) { atomicOr(&sm.bits[v >> 5], 1u << (v & 31)); });
      group_sync<GT>(gid);
      for (int k = lt; k < 512; k += GT) ((uint4 *)dst)[k] = ((const uint4 *)sm.bits)[k];
    }
    type = RS_TAG_BITSET;
    nout = RS_WORDS;
  }
  return total;
}

}  // namespace rsa
