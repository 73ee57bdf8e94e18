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

constexpr int BT = 256;  // threads; thread t owns words [4t, 4t+4)

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
  typename cub::BlockScan<uint32_t, BT>::TempStorage scan;
  uint32_t red[2][BT / 32];  // double-buffered: no trailing barrier per item
};

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int w = 0; w < BT / 32; w++) s += red[w];
  return s;
}

// Issue the two operand copies of one work item into stage `s`.
template <int STAGES>
__device__ __forceinline__ void issue(BBSmem<STAGES> &sm, int s, const uint8_t *pa, const uint8_t *pb) {
  mbar_expect_tx(&sm.bar[s], 2 * 8192);
  bulk_g2s(sm.a[s], pa, 8192, &sm.bar[s]);
  bulk_g2s(sm.b[s], pb, 8192, &sm.bar[s]);
}

// Persistent loop.  src(i, pa, pb) gives the operand pointers of item i;
// sink(i, r[4], pc, card) consumes the result words of this thread (after a
// block-wide reduction made `card` uniform).  Items i = blockIdx.x + k*gridDim.x.
// Thread 0 is the producer: it refills stage s right after the reduction
// barrier of item k proves every thread has read it, with the pointers of the
// item STAGES ahead fetched one iteration early (their loads are off the
// critical path).
template <int STAGES, typename Src, typename Pre, typename Sink>
__device__ __forceinline__ void bb_loop(BBSmem<STAGES> &sm, uint32_t count, int op, Src src, Pre pre, Sink sink) {
  const int t = threadIdx.x;
  // per-item sink metadata (output slot, pair, ...) is loaded one item ahead
  auto meta = pre(blockIdx.x < count ? blockIdx.x : 0);
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
    const uint4 *xa = (const uint4 *)sm.a[s] + 2 * t, *xb = (const uint4 *)sm.b[s] + 2 * t;
    uint4 a0 = xa[0], a1 = xa[1], b0 = xb[0], b1 = xb[1];
    uint64_t ra[4] = {((uint64_t)a0.y << 32) | a0.x, ((uint64_t)a0.w << 32) | a0.z, ((uint64_t)a1.y << 32) | a1.x,
                      ((uint64_t)a1.w << 32) | a1.z};
    uint64_t rb[4] = {((uint64_t)b0.y << 32) | b0.x, ((uint64_t)b0.w << 32) | b0.z, ((uint64_t)b1.y << 32) | b1.x,
                      ((uint64_t)b1.w << 32) | b1.z};
    uint64_t r[4];
    uint32_t pc = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      r[q] = rs_word_op(op, ra[q], rb[q]);
      pc += __popcll(r[q]);
    }
    const auto cur = meta;
    if (i + gridDim.x < count) meta = pre(i + gridDim.x);
    const uint32_t card = block_sum(pc, sm.red[k & 1]);  // barrier: stage s is now free
    if (t == 0 && nxt < count) {
      issue<STAGES>(sm, s, npa, npb);
      nxt += gridDim.x;
      if (nxt < count) src(nxt, npa, npb);
    }
    sink(cur, r, pc, card, sm.red[k & 1]);
  }
}

// Exclusive prefix of v over the CTA, reusing the per-warp totals that
// block_sum() already left in red[] (no extra barrier): warp shuffle scan +
// the totals of the warps before this one.
__device__ __forceinline__ uint32_t block_excl_from_red(uint32_t v, const uint32_t *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  uint32_t pre = 0;
#pragma unroll
  for (int k = 0; k < BT / 32; k++) pre += k < w ? red[k] : 0;
  return pre + x - v;
}

// Encode a result set held as 4 words per thread into dst: bitset (> 4096
// values) or sorted array via the smem staging buffer.  `red` holds the
// per-warp popcount totals of this item (from block_sum).  Returns n.
template <int STAGES>
__device__ __forceinline__ uint32_t bb_encode(BBSmem<STAGES> &sm, const uint64_t r[4], uint32_t pc, uint32_t card,
                                              uint8_t *dst, const uint32_t *red) {
  const int t = threadIdx.x;
  if (card > RS_ARRAY_MAX) {
    uint4 *p = (uint4 *)dst + 2 * t;
    st_stream(p, make_uint4((uint32_t)r[0], (uint32_t)(r[0] >> 32), (uint32_t)r[1], (uint32_t)(r[1] >> 32)));
    st_stream(p + 1, make_uint4((uint32_t)r[2], (uint32_t)(r[2] >> 32), (uint32_t)r[3], (uint32_t)(r[3] >> 32)));
    return RS_WORDS;
  }
  if (card == 0) return 0;
  uint32_t base = block_excl_from_red(pc, red);
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint64_t w = r[q];
    while (w) {
      sm.out[base++] = (uint16_t)((4 * t + q) * 64 + __ffsll((long long)w) - 1);
      w &= w - 1;
    }
  }
  const uint32_t nvec = (2 * card + 15) >> 4;
  if (t < 8 && card + t < nvec * 8) sm.out[card + t] = 0;  // pad slots are disjoint from [0, card)
  __syncthreads();
  for (uint32_t v = t; v < nvec; v += BT) ((uint4 *)dst)[v] = ((const uint4 *)sm.out)[v];
  return card;
}

}  // namespace rsb
