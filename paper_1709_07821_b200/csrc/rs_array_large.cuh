// rs_array_large.cuh -- large array x array pairs (na + nb > 2048) through an
// 8 KB shared-memory bitset instead of a merge path.
//
// Same results as the two-pointer kernels (kernels/scalar.py:122-267) and
// _container_from_values (containers.py:244-247):
//   and     build X from A, keep the B values whose bit is set   (sorted: B order)
//   andnot  build X from B, keep the A values whose bit is clear (sorted: A order)
//   or/xor  build X from A, OR / XOR in B's bits (B values are distinct, so XOR
//           flips each bit at most once), then popcount -> bitset if > 4096
//           values, else extract the set bits in order.
// Building from a sorted array is run-length: each thread ORs its chunk's bits
// into a register word and issues one shared atomic per distinct word.  The
// CTA is persistent; one thread streams the next pairs' arrays (variable sizes,
// 16-byte padded) into a 2-stage smem ring with cp.async.bulk + mbarriers.
#pragma once
#include <cub/cub.cuh>
#include "rs_internal.cuh"
#include "rs_bitset.cuh"

namespace rsl {

constexpr int LT = 256;
constexpr int LSTAGES = 2;

struct LargeSmem {
  uint16_t a[LSTAGES][RS_ARRAY_MAX];
  uint16_t b[LSTAGES][RS_ARRAY_MAX];
  uint64_t X[RS_WORDS];
  uint64_t bar[LSTAGES];
  uint32_t meta[LSTAGES][3];  // na, nb, item
  typename cub::BlockScan<uint32_t, LT>::TempStorage scan;
  uint32_t red[2][LT / 32];
};

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int w = 0; w < LT / 32; w++) s += red[w];
  return s;
}

// OR (or XOR) the values v[lo, hi) of a sorted array into X with one native
// 32-bit shared atomic per touched half-word (64-bit shared atomics lower to
// CAS spin loops: ATOMS.CAST.SPIN.64)
template <bool XOR>
__device__ __forceinline__ void flush_word(uint32_t *X32, uint32_t w, uint32_t m) {
  if (!m) return;
  if (XOR) atomicXor(&X32[w], m);
  else atomicOr(&X32[w], m);
}

template <bool XOR>
__device__ __forceinline__ void set_bits_chunk(const uint16_t *v, uint32_t lo, uint32_t hi, uint64_t *X) {
  if (lo >= hi) return;
  uint32_t *X32 = (uint32_t *)X;
  uint32_t w = v[lo] >> 5;
  uint32_t m = 0;
  for (uint32_t k = lo; k < hi; k++) {
    uint32_t x = v[k];
    if ((x >> 5) != w) {
      flush_word<XOR>(X32, w, m);
      w = x >> 5;
      m = 0;
    }
    m |= 1u << (x & 31);
  }
  flush_word<XOR>(X32, w, m);
}

// Thread t owns values [16t, 16t+16) of an array (n <= 4096 = 256 x 16): two
// 128-bit shared loads put them in registers as 8 packed words, so the probes
// below are independent loads (ILP) instead of a dependent smem walk.
// Returns how many of the 16 are real.
__device__ __forceinline__ uint32_t load16(const uint16_t *v, uint32_t n, uint32_t w[8]) {
  const uint32_t base = 16 * threadIdx.x;
  if (base >= n) return 0;
  const uint4 *p = (const uint4 *)(v + base);
  const uint4 q0 = p[0], q1 = p[1];
  w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
  w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
  return min(16u, n - base);
}

__device__ __forceinline__ uint32_t val16(const uint32_t w[8], int k) { return (w[k >> 1] >> (16 * (k & 1))) & 0xFFFF; }

// OR / XOR the first c values (sorted) into X: one atomic per touched 32-bit word
template <bool XOR>
__device__ __forceinline__ void set_bits16(const uint32_t w8[8], uint32_t c, uint64_t *X) {
  if (!c) return;
  uint32_t *X32 = (uint32_t *)X;
  uint32_t w = val16(w8, 0) >> 5, m = 0;
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const uint32_t x = val16(w8, k);
    if ((uint32_t)k < c) {
      if ((x >> 5) != w) {
        flush_word<XOR>(X32, w, m);
        w = x >> 5;
        m = 0;
      }
      m |= 1u << (x & 31);
    }
  }
  flush_word<XOR>(X32, w, m);
}

// Result of one pair, computed from the staged arrays.  Writes the container
// at dst unless dst == nullptr (count only).  Returns card; type/n out.  On
// return every thread has passed a barrier after its last read of the stage.
// Copy `total` staged u16 values to dst with 128-bit stores (zero-padded to
// 16 bytes); the caller has put them in `stage` before a barrier.
__device__ __forceinline__ void flush_stage(uint16_t *stage, uint32_t total, uint8_t *dst) {
  const int t = threadIdx.x;
  const uint32_t nvec = (2 * total + 15) >> 4;
  if (t < 8 && total + t < nvec * 8) stage[total + t] = 0;
  __syncthreads();
  for (uint32_t v = t; v < nvec; v += LT) ((uint4 *)dst)[v] = ((const uint4 *)stage)[v];
}

// `stage` is the ring slot's A buffer: once every thread holds its values in
// registers (first barrier) it is free until the producer refills it after
// this pair, so it doubles as the output staging buffer.
__device__ uint32_t large_pair(LargeSmem &sm, int op, const uint16_t *A, uint32_t na, const uint16_t *B,
                               uint32_t nb, uint8_t *dst, int parity, uint8_t &type, uint32_t &nout,
                               uint16_t *stage) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; k++) sm.X[4 * t + k] = 0;
  uint32_t xa[8], xb[8];
  const uint32_t ca = load16(A, na, xa), cb = load16(B, nb, xb);
  __syncthreads();
  if (op == RS_OP_ANDNOT) set_bits16<false>(xb, cb, sm.X);
  else set_bits16<false>(xa, ca, sm.X);
  __syncthreads();
  const uint32_t *X32 = (const uint32_t *)sm.X;
  if (op == RS_OP_AND || op == RS_OP_ANDNOT) {
    // and: keep B values present in X(A); andnot: keep A values absent from X(B)
    const bool is_and = op == RS_OP_AND;
    uint32_t P[8];
#pragma unroll
    for (int k = 0; k < 8; k++) P[k] = is_and ? xb[k] : xa[k];
    const uint32_t cp = is_and ? cb : ca;
    const uint32_t want = is_and ? 1u : 0u;
    uint32_t keep = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const uint32_t x = val16(P, k);
      if ((uint32_t)k < cp && ((X32[x >> 5] >> (x & 31)) & 1u) == want) keep |= 1u << k;
    }
    uint32_t base, total;
    cub::BlockScan<uint32_t, LT>(sm.scan).ExclusiveSum((uint32_t)__popc(keep), base, total);
    type = RS_TAG_ARRAY;
    nout = total;
    if (dst && total) {
#pragma unroll
      for (int k = 0; k < 16; k++)
        if (keep >> k & 1) stage[base++] = (uint16_t)val16(P, k);
      flush_stage(stage, total, dst);
    }
    return total;
  }
  // or / xor: fold B into X(A); B values are distinct, so XOR flips each bit once
  if (op == RS_OP_OR) set_bits16<false>(xb, cb, sm.X);
  else set_bits16<true>(xb, cb, sm.X);
  __syncthreads();
  uint64_t r[4];
  uint32_t pc = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    r[k] = sm.X[4 * t + k];
    pc += __popcll(r[k]);
  }
  const uint32_t card = block_sum(pc, sm.red[parity]);
  if (!dst || card == 0) {
    type = RS_TAG_ARRAY;
    nout = card;
    return card;
  }
  if (card > RS_ARRAY_MAX) {
    uint4 *p = (uint4 *)dst + 2 * t;
    rsb::st_stream(p, make_uint4((uint32_t)r[0], (uint32_t)(r[0] >> 32), (uint32_t)r[1], (uint32_t)(r[1] >> 32)));
    rsb::st_stream(p + 1, make_uint4((uint32_t)r[2], (uint32_t)(r[2] >> 32), (uint32_t)r[3], (uint32_t)(r[3] >> 32)));
    type = RS_TAG_BITSET;
    nout = RS_WORDS;
    return card;
  }
  uint32_t base;
  cub::BlockScan<uint32_t, LT>(sm.scan).ExclusiveSum(pc, base);
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint64_t w = r[q];
    while (w) {
      stage[base++] = (uint16_t)((4 * t + q) * 64 + __ffsll((long long)w) - 1);
      w &= w - 1;
    }
  }
  flush_stage(stage, card, dst);
  type = RS_TAG_ARRAY;
  nout = card;
  return card;
}

// Persistent ring over items i = blockIdx.x + k*gridDim.x < count.
// src(i, pa, na, pb, nb) gives the operand arrays of item i;
// sink(i, card, type, n, dst_needed) -- called by all threads after the pair.
template <typename Src, typename Dst, typename Sink>
__device__ void large_loop(LargeSmem &sm, uint32_t count, int op, Src src, Dst dst_of, Sink sink) {
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < LSTAGES; s++) rsb::mbar_init(&sm.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s, uint32_t i) {
    const uint8_t *pa, *pb;
    uint32_t na, nb;
    src(i, pa, na, pb, nb);
    sm.meta[s][0] = na;
    sm.meta[s][1] = nb;
    sm.meta[s][2] = i;
    const uint32_t ba = (uint32_t)rs_pad16(2ull * na), bb = (uint32_t)rs_pad16(2ull * nb);
    rsb::mbar_expect_tx(&sm.bar[s], ba + bb);
    rsb::bulk_g2s(sm.a[s], pa, ba, &sm.bar[s]);
    rsb::bulk_g2s(sm.b[s], pb, bb, &sm.bar[s]);
  };
  if (t == 0)
    for (int s = 0; s < LSTAGES; s++) {
      uint32_t i = blockIdx.x + s * gridDim.x;
      if (i < count) issue(s, i);
    }
  for (uint32_t k = 0;; k++) {
    const uint32_t i = blockIdx.x + k * gridDim.x;
    if (i >= count) break;
    const int s = k % LSTAGES;
    rsb::mbar_wait(&sm.bar[s], (k / LSTAGES) & 1);
    const uint32_t na = sm.meta[s][0], nb = sm.meta[s][1];
    uint8_t type;
    uint32_t n;
    // registers hold this thread's values after large_pair's first barrier,
    // so stage s is free once that barrier has passed
    uint32_t card = large_pair(sm, op, sm.a[s], na, sm.b[s], nb, dst_of(i), k & 1, type, n, sm.a[s]);
    if (t == 0) {
      uint32_t nx = i + LSTAGES * gridDim.x;
      if (nx < count) issue(s, nx);
    }
    sink(i, card, type, n);
    __syncthreads();  // X / out / meta reuse
  }
}

}  // namespace rsl
