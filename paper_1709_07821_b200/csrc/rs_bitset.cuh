// rs_bitset.cuh -- bitset x bitset pairs, persistent and TMA-fed.
//
// bitset_op_with_count + _container_from_words (kernels/scalar.py:39-49,
// containers.py:250-253, 463-465): per pair, 2 x 8 KB in, word op, popcount,
// result kept as a bitset if it holds > 4096 values, else extracted to a
// sorted array.  Each CTA is persistent over its share of the work list; one
// elected thread streams the next pairs' 8 KB operands into a STAGES-deep
// shared-memory ring with cp.async.bulk (UBLKCP) completing on mbarriers, so
// HBM reads for pairs k+1..k+STAGES-1 overlap the compute/stores of pair k.
#pragma once
#include <cub/cub.cuh>
#include "rs_internal.cuh"

namespace rsb {

constexpr int BT = 256;  // threads; thread t owns words t, t+256, t+512, t+768
// (strided: a warp's 64-bit shared loads and global stores touch 256
// consecutive bytes -- conflict-free, fully coalesced)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 8 KB global -> shared bulk copy completing on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void st_stream(void *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int STAGES>
struct BBSmem {
  uint64_t a[STAGES][RS_WORDS];
  uint64_t b[STAGES][RS_WORDS];
  uint16_t out[RS_ARRAY_MAX];
  uint64_t bar[STAGES];
  // per-warp totals, double-buffered (no trailing barrier per item): [0] the
  // popcounts of words t and t+256 packed in 16-bit fields, [1] of t+512/t+768
  uint32_t red[2][2][BT / 32];
};

// Block totals of two packed vectors (four 16-bit row counts, each <= 16384):
// per-warp totals land in red[0..1][warp]; returns the sum of all four rows.
__device__ __forceinline__ uint32_t block_sum_packed(uint32_t v0, uint32_t v1, uint32_t (*red)[BT / 32]) {
  for (int o = 16; o; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = v0;
    red[1][threadIdx.x >> 5] = v1;
  }
  __syncthreads();
  uint32_t s0 = 0, s1 = 0;
#pragma unroll
  for (int w = 0; w < BT / 32; w++) {
    s0 += red[0][w];
    s1 += red[1][w];
  }
  return (s0 & 0xFFFFu) + (s0 >> 16) + (s1 & 0xFFFFu) + (s1 >> 16);
}

// Issue the two operand copies of one work item into stage `s`.
template <int STAGES>
__device__ __forceinline__ void issue(BBSmem<STAGES> &sm, int s, const uint8_t *pa, const uint8_t *pb) {
  mbar_expect_tx(&sm.bar[s], 2 * 8192);
  bulk_g2s(sm.a[s], pa, 8192, &sm.bar[s]);
  bulk_g2s(sm.b[s], pb, 8192, &sm.bar[s]);
}

// Persistent loop.  src(i, pa, pb) gives the operand pointers of item i;
// sink(meta, r[4], pk0, pk1, card, red) consumes the result words of this
// thread (words t + 256q; pk0/pk1 their packed popcounts) after a block-wide
// reduction made `card` uniform.  Items i = blockIdx.x + k*gridDim.x.
// Thread 0 is the producer: it refills stage s right after the reduction
// barrier of item k proves every thread has read it, with the pointers of the
// item STAGES ahead fetched one iteration early (their loads are off the
// critical path).
template <int STAGES, typename Src, typename Pre, typename Sink>
__device__ __forceinline__ void bb_loop(BBSmem<STAGES> &sm, uint32_t count, int op, Src src, Pre pre, Sink sink) {
  const int t = threadIdx.x;
  if (blockIdx.x >= count) return;  // no item for this CTA (the list may be empty)
  // per-item sink metadata (output slot, pair, ...) is loaded one item ahead
  auto meta = pre(blockIdx.x);
  if (t == 0) {
    for (int s = 0; s < STAGES; s++) mbar_init(&sm.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t *npa = nullptr, *npb = nullptr;
  uint32_t nxt = blockIdx.x + STAGES * gridDim.x;
  if (t == 0) {
    for (int s = 0; s < STAGES; s++) {
      uint32_t i = blockIdx.x + s * gridDim.x;
      if (i < count) {
        const uint8_t *pa, *pb;
        src(i, pa, pb);
        issue<STAGES>(sm, s, pa, pb);
      }
    }
    if (nxt < count) src(nxt, npa, npb);
  }
  for (uint32_t k = 0;; k++) {
    const uint32_t i = blockIdx.x + k * gridDim.x;
    if (i >= count) break;
    const int s = k % STAGES;
    mbar_wait(&sm.bar[s], (k / STAGES) & 1);
    const uint64_t *xa = sm.a[s] + t, *xb = sm.b[s] + t;
    uint64_t r[4];
    uint32_t pq[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      r[q] = rs_word_op(op, xa[BT * q], xb[BT * q]);
      pq[q] = __popcll(r[q]);
    }
    const uint32_t pk0 = pq[0] | (pq[1] << 16), pk1 = pq[2] | (pq[3] << 16);
    const auto cur = meta;
    if (i + gridDim.x < count) meta = pre(i + gridDim.x);
    const uint32_t card = block_sum_packed(pk0, pk1, sm.red[k & 1]);  // barrier: stage s is now free
    if (t == 0 && nxt < count) {
      issue<STAGES>(sm, s, npa, npb);
      nxt += gridDim.x;
      if (nxt < count) src(nxt, npa, npb);
    }
    sink(cur, r, pk0, pk1, card, sm.red[k & 1]);
  }
}

// Encode a result set held as words t + 256q (q < 4) per thread into dst:
// bitset (> 4096 values) or sorted array via the smem staging buffer.  The
// array positions come from a scan of the packed row counts that reuses the
// per-warp totals block_sum_packed() left in red (no extra barrier); each
// word is then peeled from its top bit down (FLO) into its slot range.
// Returns n.
template <int STAGES>
__device__ __forceinline__ uint32_t bb_encode(BBSmem<STAGES> &sm, const uint64_t r[4], uint32_t pk0, uint32_t pk1,
                                              uint32_t card, uint8_t *dst, const uint32_t (*red)[BT / 32]) {
  const int t = threadIdx.x;
  if (card > RS_ARRAY_MAX) {
    uint64_t *p = (uint64_t *)dst + t;
#pragma unroll
    for (int q = 0; q < 4; q++) asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p + BT * q), "l"(r[q]) : "memory");
    return RS_WORDS;
  }
  if (card == 0) return 0;
  const int lane = t & 31, w = t >> 5;
  uint32_t x0 = pk0, x1 = pk1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
    if (lane >= o) { x0 += y0; x1 += y1; }
  }
  uint32_t e0 = x0 - pk0, e1 = x1 - pk1, T0 = 0, T1 = 0;  // exclusive prefix / block totals
#pragma unroll
  for (int k = 0; k < BT / 32; k++) {
    const uint32_t a = red[0][k], b = red[1][k];
    T0 += a; T1 += b;
    if (k < w) { e0 += a; e1 += b; }
  }
  // word t + 256q starts after rows 0..q-1 and this row's words before t
  const uint32_t r0 = T0 & 0xFFFFu, r1 = T0 >> 16, r2 = T1 & 0xFFFFu;
  uint32_t end[4] = {(e0 & 0xFFFFu) + (pk0 & 0xFFFFu), r0 + (e0 >> 16) + (pk0 >> 16),
                     r0 + r1 + (e1 & 0xFFFFu) + (pk1 & 0xFFFFu), r0 + r1 + r2 + (e1 >> 16) + (pk1 >> 16)};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t pos = (uint32_t)(t + BT * q) * 64;
    uint32_t b = end[q], hi = (uint32_t)(r[q] >> 32), lo = (uint32_t)r[q];
    while (hi) {
      const uint32_t p = 31 - __clz(hi);
      sm.out[--b] = (uint16_t)(pos + 32 + p);
      hi ^= 1u << p;
    }
    while (lo) {
      const uint32_t p = 31 - __clz(lo);
      sm.out[--b] = (uint16_t)(pos + p);
      lo ^= 1u << p;
    }
  }
  const uint32_t nvec = (2 * card + 15) >> 4;
  if (t < 8 && card + t < nvec * 8) sm.out[card + t] = 0;  // pad slots are disjoint from [0, card)
  __syncthreads();
  for (uint32_t v = t; v < nvec; v += BT) ((uint4 *)dst)[v] = ((const uint4 *)sm.out)[v];
  return card;
}

}  // namespace rsb
