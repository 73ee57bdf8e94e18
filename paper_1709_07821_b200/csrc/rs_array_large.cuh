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
  uint64_t X[2][RS_WORDS];  // by pair parity: each pair clears its words after its last read
  uint64_t full[LSTAGES];
  uint64_t empty[LSTAGES];
  LargeMeta meta[LSTAGES];
  uint32_t red[2][2][LT / 32];
};

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(LT) : "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rsb::smem_u32(bar)) : "memory");
}

// The producer lane waits for a free slot suspended in the barrier (time hint
// 1 ms; the hardware resumes it when the phase completes), so its wait does
// not take issue slots from the consumer warps -- a polling loop with
// __nanosleep measured 200 M spin iterations (a quarter of all instructions).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "WB_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WB_%=;\n}\n" ::"r"(rsb::smem_u32(bar)),
      "r"(phase), "r"(1000000)
      : "memory");
}

// consumer-only exclusive scan with total (one named barrier); the scratch is
// double-buffered by item parity so no trailing barrier is needed
__device__ __forceinline__ uint32_t cscan(uint32_t v, uint32_t (*red2)[LT / 32], uint32_t &total) {
  uint32_t *red = red2[0];
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

// cscan over two packed vectors (16-bit fields): exclusive prefix and totals
__device__ __forceinline__ void cscan2(uint32_t v0, uint32_t v1, uint32_t (*red)[LT / 32], uint32_t &e0,
                                       uint32_t &e1, uint32_t &T0, uint32_t &T1) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x0 = v0, x1 = v1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
    if (lane >= o) { x0 += y0; x1 += y1; }
  }
  if (lane == 31) { red[0][w] = x0; red[1][w] = x1; }
  cbar();
  e0 = x0 - v0; e1 = x1 - v1; T0 = 0; T1 = 0;
#pragma unroll
  for (int k = 0; k < LT / 32; k++) {
    const uint32_t a = red[0][k], b = red[1][k];
    T0 += a; T1 += b;
    if (k < w) { e0 += a; e1 += b; }
  }
}

// OR / XOR into X with one native 32-bit shared atomic per touched word
// (64-bit shared atomics lower to ATOMS.CAST.SPIN.64 CAS loops)
template <bool XOR>
__device__ __forceinline__ void flush_word(uint32_t *X32, uint32_t w, uint32_t m) {
  if (!m) return;
  if (XOR) atomicXor(&X32[w], m);
  else atomicOr(&X32[w], m);
}

// Thread t owns the contiguous values [c*t, c*t + c) of an array, c =
// ceil(n / 256) <= 16, so every consumer gets an equal share whatever the
// array's size (the busiest thread sets each pair's critical path).  The
// values land in registers as 8 packed words: two 128-bit shared loads for a
// full 16-value share, single loads otherwise.
__device__ __forceinline__ uint32_t load16(const uint16_t *v, uint32_t n, uint32_t w[8]) {
  const uint32_t c = (n + LT - 1) / LT, base = c * threadIdx.x;
  if (base >= n) return 0;
  const uint32_t cnt = min(c, n - base);
  if (c == 16) {
    const uint4 *p = (const uint4 *)(v + base);
    const uint4 q0 = p[0], q1 = p[1];
    w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
    w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
    return cnt;
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const uint32_t lo = 2 * k < (int)cnt ? v[base + 2 * k] : 0, hi = 2 * k + 1 < (int)cnt ? v[base + 2 * k + 1] : 0;
    w[k] = lo | (hi << 16);
  }
  return cnt;
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

// Sorted-array membership: is x in v[0, n)?  (n <= 4096: 12 probes)
__device__ __forceinline__ bool bsearch16(const uint16_t *v, uint32_t n, uint32_t x) {
  uint32_t lo = 0, len = n;
  while (len > 1) {
    const uint32_t half = len >> 1;
    if (v[lo + half] <= x) lo += half;
    len -= half;
  }
  return n && v[lo] == x;
}

// One pair (consumers only).  `stage` (the ring slot's A buffer) is free once
// the values are in registers and doubles as the output staging buffer; the
// slot goes back to the producer only after the next pair's first barrier.
//
// AND (and ANDNOT with a small A) on very unequal sizes -- the smaller side
// at most 1/16 of the larger, so at most 256 values -- skips the bitset: one
// thread per small-side value binary-searches the larger array in shared
// memory (array_intersect_galloping's case, kernels/scalar.py:149-176).
// Otherwise AND builds X from the smaller side and probes the larger one (the
// probed side's order is the output order).
__device__ uint32_t large_pair(LargeSmem &sm, int op, const uint16_t *A, uint32_t na, const uint16_t *B,
                               uint32_t nb, uint8_t *dst, int parity, uint8_t &type, uint32_t &nout,
                               uint16_t *stage, uint64_t *release) {
  const int t = threadIdx.x;
  if (op == RS_OP_AND || op == RS_OP_ANDNOT) {
    const bool is_and = op == RS_OP_AND;
    const bool a_small = is_and ? na <= nb : true;
    const uint32_t ns = a_small ? na : nb, nl = a_small ? nb : na;
    if (16 * ns <= nl) {
      const uint16_t *S = a_small ? A : B, *L = a_small ? B : A;
      uint32_t v = 0, keep = 0;
      if ((uint32_t)t < ns) {
        v = S[t];
        keep = bsearch16(L, nl, v) == is_and;
      }
      uint32_t total;
      const uint32_t base = cscan(keep, sm.red[parity], total);
      if (t == 0 && release) mbar_arrive(release);
      type = RS_TAG_ARRAY;
      nout = total;
      if (dst && total) {
        if (keep) stage[base] = (uint16_t)v;
        flush_stage(stage, total, dst);
      }
      return total;
    }
  }
  // X (this pair's parity) is all zero on entry: zeroed at kernel start, and
  // every pair clears the words it owns after its last read of them; the
  // other parity's buffer separates that clear from the next pair's scatter.
  uint64_t *X = sm.X[parity];
  uint32_t *X32 = (uint32_t *)X;
  uint32_t xa[8], xb[8];
  const uint32_t ca = load16(A, na, xa), cb = load16(B, nb, xb);
  if (op == RS_OP_AND || op == RS_OP_ANDNOT) {
    const bool build_b = op == RS_OP_ANDNOT || (op == RS_OP_AND && nb < na);
    if (build_b) set_bits16<false>(xb, cb, X);
    else set_bits16<false>(xa, ca, X);
    cbar();
    // every consumer has finished the previous pair: its ring slot may refill
    if (t == 0 && release) mbar_arrive(release);
    const bool probe_b = !build_b;
    uint32_t P[8];
#pragma unroll
    for (int k = 0; k < 8; k++) P[k] = probe_b ? xb[k] : xa[k];
    const uint32_t cp = probe_b ? cb : ca;
    const uint32_t want = op == RS_OP_AND ? 1u : 0u;
    uint32_t keep = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const uint32_t x = val16(P, k);
      if ((uint32_t)k < cp && ((X32[x >> 5] >> (x & 31)) & 1u) == want) keep |= 1u << k;
    }
    uint32_t total;
    uint32_t base = cscan((uint32_t)__popc(keep), sm.red[parity], total);
#pragma unroll
    for (int q = 0; q < 4; q++) X[t + LT * q] = 0;  // every probe of this pair is done
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
  // OR / XOR: both arrays in one scatter phase (the updates commute; each
  // side's values are distinct, so XOR flips a bit once per side)
  if (op == RS_OP_OR) {
    set_bits16<false>(xa, ca, X);
    set_bits16<false>(xb, cb, X);
  } else {
    set_bits16<true>(xa, ca, X);
    set_bits16<true>(xb, cb, X);
  }
  cbar();
  if (t == 0 && release) mbar_arrive(release);
  // result words t + 256q (conflict-free), positions by a packed row scan
  uint64_t r[4];
  uint32_t pq[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    r[q] = X[t + LT * q];
    X[t + LT * q] = 0;
    pq[q] = __popcll(r[q]);
  }
  const uint32_t pk0 = pq[0] | (pq[1] << 16), pk1 = pq[2] | (pq[3] << 16);
  uint32_t e0, e1, T0, T1;
  cscan2(pk0, pk1, sm.red[parity], e0, e1, T0, T1);
  const uint32_t r0 = T0 & 0xFFFFu, r1 = T0 >> 16, r2 = T1 & 0xFFFFu;
  const uint32_t card = r0 + r1 + r2 + (T1 >> 16);
  if (!dst || card == 0) {
    type = RS_TAG_ARRAY;
    nout = card;
    return card;
  }
  if (card > RS_ARRAY_MAX) {
    uint64_t *p = (uint64_t *)dst + t;
#pragma unroll
    for (int q = 0; q < 4; q++) asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p + LT * q), "l"(r[q]) : "memory");
    type = RS_TAG_BITSET;
    nout = RS_WORDS;
    return card;
  }
  const uint32_t end[4] = {(e0 & 0xFFFFu) + pq[0], r0 + (e0 >> 16) + pq[1], r0 + r1 + (e1 & 0xFFFFu) + pq[2],
                           r0 + r1 + r2 + (e1 >> 16) + pq[3]};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t pos = (uint32_t)(t + LT * q) * 64;
    uint32_t b = end[q], hi = (uint32_t)(r[q] >> 32), lo = (uint32_t)r[q];
    while (hi) {
      const uint32_t p = 31 - __clz(hi);
      stage[--b] = (uint16_t)(pos + 32 + p);
      hi ^= 1u << p;
    }
    while (lo) {
      const uint32_t p = 31 - __clz(lo);
      stage[--b] = (uint16_t)(pos + p);
      lo ^= 1u << p;
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
  for (int w = t; w < 2 * RS_WORDS; w += LTHREADS) (&sm.X[0][0])[w] = 0;
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
        if (j >= LSTAGES) mbar_wait_backoff(&sm.empty[s], ((j / LSTAGES) - 1) & 1);
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
