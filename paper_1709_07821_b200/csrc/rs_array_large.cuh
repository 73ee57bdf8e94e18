// rs_array_large.cuh -- large array x array pairs (na + nb > 256) through an
// 8 KB shared-memory bitset instead of a merge path.
//
// Same results as the two-pointer kernels (kernels/scalar.py:122-267) and
// _container_from_values (containers.py:244-247):
//   and     build X from A, keep the B values whose bit is set   (sorted: B order)
//   andnot  build X from B, keep the A values whose bit is clear (sorted: A order)
//   or/xor  build X from A, OR / XOR in B's bits (B values are distinct, so XOR
//           flips each bit at most once), then popcount -> bitset if > 4096
//           values, else extract the set bits in order.
//
// CTA layout (warp-specialized): warps 0-7 are consumers (256 threads, one
// pair at a time, synchronizing only among themselves with named barrier 1);
// warp 8 is the producer.  The producer walks the CTA's items, loads each
// item's metadata (operand offsets, sizes, output slot, pair) and streams both
// arrays (variable sizes, 16-byte padded) into a 2-stage shared-memory ring
// with cp.async.bulk completing on `full` mbarriers; consumers release a stage
// through its `empty` mbarrier.  No consumer ever waits on a dependent global
// load, and no consumer barrier waits on producer work (the stall profile of
// the single-role version: 44 % of stalls at CTA barriers behind thread 0).
#pragma once
#include "rs_internal.cuh"
#include "rs_bitset.cuh"

namespace rsl {

constexpr int LT = 256;               // consumer threads
constexpr int LTHREADS = LT + 32;     // + one producer warp
constexpr int LSTAGES = 2;

struct LargeMeta {
  uint32_t na, nb, e, pair;
  uint64_t dst;
};

struct LargeSmem {
  uint16_t a[LSTAGES][RS_ARRAY_MAX];
  uint16_t b[LSTAGES][RS_ARRAY_MAX];
  uint64_t X[RS_WORDS];
  uint64_t full[LSTAGES];
  uint64_t empty[LSTAGES];
  LargeMeta meta[LSTAGES];
  uint32_t red[2][LT / 32];
};

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(LT) : "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rsb::smem_u32(bar)) : "memory");
}

// consumer-only exclusive scan with total (one named barrier); the scratch is
// double-buffered by item parity so no trailing barrier is needed
__device__ __forceinline__ uint32_t cscan(uint32_t v, uint32_t *red, uint32_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[w] = x;
  cbar();
  uint32_t pre = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < LT / 32; k++) {
    const uint32_t s = red[k];
    pre += k < w ? s : 0;
    tot += s;
  }
  total = tot;
  return pre + x - v;
}

// OR / XOR into X with one native 32-bit shared atomic per touched word
// (64-bit shared atomics lower to ATOMS.CAST.SPIN.64 CAS loops)
template <bool XOR>
__device__ __forceinline__ void flush_word(uint32_t *X32, uint32_t w, uint32_t m) {
  if (!m) return;
  if (XOR) atomicXor(&X32[w], m);
  else atomicOr(&X32[w], m);
}

// Thread t owns values [16t, 16t+16) of an array (n <= 4096 = 256 x 16): two
// 128-bit shared loads put them in registers as 8 packed words, so the probes
// below are independent loads (ILP) instead of a dependent smem walk.
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

// Copy `total` staged u16 values to dst with 128-bit stores (16-byte zero pad).
__device__ __forceinline__ void flush_stage(uint16_t *stage, uint32_t total, uint8_t *dst) {
  const int t = threadIdx.x;
  const uint32_t nvec = (2 * total + 15) >> 4;
  if (t < 8 && total + t < nvec * 8) stage[total + t] = 0;
  cbar();
  for (uint32_t v = t; v < nvec; v += LT) ((uint4 *)dst)[v] = ((const uint4 *)stage)[v];
}

// One pair (consumers only).  `stage` (the ring slot's A buffer) is free once
// the values are in registers and doubles as the output staging buffer; the
// slot goes back to the producer only after the next pair's first barrier.
__device__ uint32_t large_pair(LargeSmem &sm, int op, const uint16_t *A, uint32_t na, const uint16_t *B,
                               uint32_t nb, uint8_t *dst, int parity, uint8_t &type, uint32_t &nout,
                               uint16_t *stage, uint64_t *release) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; k++) sm.X[4 * t + k] = 0;
  uint32_t xa[8], xb[8];
  const uint32_t ca = load16(A, na, xa), cb = load16(B, nb, xb);
  cbar();
  // every consumer has finished the previous pair: its ring slot may refill
  if (t == 0 && release) mbar_arrive(release);
  if (op == RS_OP_ANDNOT) set_bits16<false>(xb, cb, sm.X);
  else set_bits16<false>(xa, ca, sm.X);
  cbar();
  const uint32_t *X32 = (const uint32_t *)sm.X;
  if (op == RS_OP_AND || op == RS_OP_ANDNOT) {
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
    uint32_t total;
    uint32_t base = cscan((uint32_t)__popc(keep), sm.red[parity], total);
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
  if (op == RS_OP_OR) set_bits16<false>(xb, cb, sm.X);
  else set_bits16<true>(xb, cb, sm.X);
  cbar();
  uint64_t r[4];
  uint32_t pc = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    r[k] = sm.X[4 * t + k];
    pc += __popcll(r[k]);
  }
  uint32_t card;
  uint32_t base = cscan(pc, sm.red[parity], card);
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

// Persistent, warp-specialized ring over items i = blockIdx.x + k*gridDim.x.
// meta_of(i, aoff, boff) -> LargeMeta (runs on the producer lane only);
// sink(meta, card, type, n) runs on every consumer thread after the pair.
template <typename MetaOf, typename Sink>
__device__ void large_loop(LargeSmem &sm, uint32_t count, int op, const uint8_t *poolA, const uint8_t *poolB,
                           uint8_t *opool, MetaOf meta_of, Sink sink) {
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < LSTAGES; s++) {
      rsb::mbar_init(&sm.full[s], 1);
      rsb::mbar_init(&sm.empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t >= LT) {  // ---------------- producer warp (one elected lane)
    if (t == LT) {
      uint64_t ao, bo;
      LargeMeta m;
      if (blockIdx.x < count) m = meta_of(blockIdx.x, ao, bo);
      for (uint32_t j = 0;; j++) {
        const uint32_t i = blockIdx.x + j * gridDim.x;
        if (i >= count) break;
        const int s = j % LSTAGES;
        // metadata of the next item is fetched before waiting for a free slot
        uint64_t nao = 0, nbo = 0;
        LargeMeta nm = m;
        if (i + gridDim.x < count) nm = meta_of(i + gridDim.x, nao, nbo);
        if (j >= LSTAGES) rsb::mbar_wait(&sm.empty[s], ((j / LSTAGES) - 1) & 1);
        sm.meta[s] = m;
        const uint32_t ba = (uint32_t)rs_pad16(2ull * m.na), bb = (uint32_t)rs_pad16(2ull * m.nb);
        rsb::mbar_expect_tx(&sm.full[s], ba + bb);
        rsb::bulk_g2s(sm.a[s], poolA + ao, ba, &sm.full[s]);
        rsb::bulk_g2s(sm.b[s], poolB + bo, bb, &sm.full[s]);
        m = nm;
        ao = nao;
        bo = nbo;
      }
    }
    return;
  }
  for (uint32_t k = 0;; k++) {  // ---------------- consumers
    const uint32_t i = blockIdx.x + k * gridDim.x;
    if (i >= count) break;
    const int s = k % LSTAGES;
    rsb::mbar_wait(&sm.full[s], (k / LSTAGES) & 1);
    const LargeMeta m = sm.meta[s];
    uint8_t type;
    uint32_t n;
    uint64_t *release = k ? &sm.empty[(k - 1) % LSTAGES] : nullptr;
    const uint32_t card = large_pair(sm, op, sm.a[s], m.na, sm.b[s], m.nb, opool ? opool + m.dst : nullptr, k & 1,
                                     type, n, sm.a[s], release);
    sink(m, card, type, n);
  }
}

}  // namespace rsl
