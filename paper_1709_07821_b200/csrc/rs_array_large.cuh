// rs_array_large.cuh -- large array x array pairs (na + nb > 256) through
// shared-memory bitsets instead of a merge path.
//
// Same results as the two-pointer kernels (kernels/scalar.py:122-267) and
// _container_from_values (containers.py:244-247):
//   and / andnot  one bitset X built from the smaller side (and) or from B
//                 (andnot); the other side is filtered through it with warp
//                 ballots, so the result comes out sorted;
//   or / xor      both sides scattered into XA (shared OR, resp. XOR); the
//                 result words with a popcount scan give the cardinality, and the result is the
//                 words themselves (> 4096 values: a bitset container) or
//                 their set bits in order (<= 4096: an array container).
// AND / ANDNOT with one side at most 1/16 of the other skip the bitset and
// binary-search the larger array (array_intersect_galloping's case,
// kernels/scalar.py:149-176).
//
// CTA layout (warp-specialized): warps 0-7 are consumers (256 threads, one
// pair at a time, synchronizing only among themselves with named barrier 1);
// warp 8 is the producer.  The producer walks the CTA's items, loads each
// item's metadata (operand offsets, sizes, output slot, pair) and streams both
// arrays (variable sizes, 16-byte padded) into a byte ring in shared memory
// with cp.async.bulk completing on the item slot's `full` mbarrier.  Items
// take only the bytes they need (a ~12 KB average item leaves room for two
// more in flight behind it), and consumers hand an item's bytes back through
// the slot's `empty` mbarrier as soon as its last value has been read.
#pragma once
#include "rs_internal.cuh"
#include "rs_bitset.cuh"

namespace rsl {

constexpr int LT = 256;               // consumer threads
constexpr int LTHREADS = LT + 32;     // + one producer warp
constexpr int NSLOT = 8;              // items in flight (metadata + barrier slots)

struct LargeMeta {
  uint32_t na, nb, e, pair;
  uint64_t dst;
  uint32_t aoff, boff;  // ring offsets of the staged arrays
};

// Shared-memory layout (dynamic; carved at run time by large_layout):
//   header | pad to 8 KB | XA (8 KB) | XB (8 KB) | byte ring (rest)
// XA / XB sit on 8 KB boundaries of the shared window so a value's word
// address is base | offset (see scatter).
struct LargeHdr {
  uint64_t full[NSLOT];
  uint64_t empty[NSLOT];
  LargeMeta meta[NSLOT];
  uint32_t span[NSLOT];  // producer only: ring bytes each item holds (incl. the wrap skip)
  uint32_t red[2][2][LT / 32];
};

struct LargeSmem {
  LargeHdr *h;
  uint8_t *X;     // XA, XB, then the ring
  uint32_t ring;  // ring bytes
  __device__ __forceinline__ uint32_t *XA() const { return (uint32_t *)X; }
  __device__ __forceinline__ uint32_t *XB() const { return (uint32_t *)(X + 8192); }
  __device__ __forceinline__ uint8_t *R() const { return X + 16384; }
};

// 44 KB: five CTAs per SM (5 x (44 + 1 reserved) KB <= 228 KB; the kernels
// are capped at 5 x 288 threads' worth of registers).  The header and the pad
// to the first 8 KB boundary take at most ~8.5 KB, XA / XB 16 KB, and the
// ring the rest (>= 19 KB); large_loop traps if it is ever under 16 KB, the
// largest item (an item that does not fit before the end of the ring waits
// for the ring to drain and starts at 0).  Four CTAs of 56 KB with a 33 KB
// ring measured slower: the kernel is issue / barrier bound, so a fifth CTA's
// warps hide more of the per-pair barriers than the deeper ring hid latency.
#ifndef RS_AAL_SMEM_KB
#define RS_AAL_SMEM_KB 56
#endif
#ifndef RS_AAL_MINB
#define RS_AAL_MINB 4
#endif
constexpr size_t LARGE_SMEM_BYTES = RS_AAL_SMEM_KB * 1024;

__device__ __forceinline__ LargeSmem large_layout(uint8_t *raw) {
  LargeSmem sm;
  sm.h = (LargeHdr *)raw;
  const uint32_t b = rsb::smem_u32(raw);
  const uint32_t x = (b + (uint32_t)sizeof(LargeHdr) + 8191u) & ~8191u;
  sm.X = raw + (x - b);
  const uint32_t used = (x - b) + 16384u;
  sm.ring = used < LARGE_SMEM_BYTES ? ((uint32_t)LARGE_SMEM_BYTES - used) & ~15u : 0u;
  return sm;
}

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

// Set bit v of X (32-bit words) for every value of a staged array: two
// values per 32-bit shared load, one native shared OR per touched word (two
// values in the same word share one).  Lanes read consecutive value pairs, so
// the ORs of one warp instruction mostly hit distinct banks.  X is 8 KB
// aligned in the shared window, so a value's word address is one LOP3:
// X | ((v >> 3) & ~3); its bit is a wrapping funnel shift by v.
__device__ __forceinline__ void red_or(uint32_t addr, uint32_t bit) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(bit) : "memory");
}
__device__ __forceinline__ void red_xor(uint32_t addr, uint32_t bit) {
  asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(addr), "r"(bit) : "memory");
}
template <bool XOR>
__device__ __forceinline__ void red_set(uint32_t addr, uint32_t bit) {
  if constexpr (XOR) red_xor(addr, bit);
  else red_or(addr, bit);
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// XOR: the bits go in with shared XORs instead of ORs, so scattering both
// arrays of a pair into one bitset leaves exactly the symmetric difference
// (a value of both sides toggles twice; two values of one side sharing a word
// have distinct bits, so their combined mask is the same either way).
template <bool XOR = false>
__device__ __forceinline__ void scatter(const uint16_t *v, uint32_t n, uint32_t X) {
  const uint32_t *w = (const uint32_t *)v;
  const uint32_t nw = n >> 1;
#pragma unroll 4
  for (uint32_t i = threadIdx.x; i < nw; i += LT) {
    const uint32_t x = w[i];
    const uint32_t alo = X | ((x >> 3) & 0x1FFCu), ahi = X | ((x >> 19) & 0x1FFCu);
    const uint32_t blo = __funnelshift_l(0u, 1u, x), bhi = __funnelshift_l(0u, 1u, x >> 16);
    const bool same = alo == ahi;
    red_set<XOR>(alo, same ? blo | bhi : blo);
    if (!same) red_set<XOR>(ahi, bhi);
  }
  if ((n & 1) && threadIdx.x == LT - 1) {
    const uint32_t x = v[n - 1];
    red_set<XOR>(X | ((x >> 3) & 0x1FFCu), __funnelshift_l(0u, 1u, x));
  }
}

// Keep the values of P (np, sorted) whose bit in X equals WANT, in order:
// warp w probes a contiguous run of P (NR rounds of 32 value pairs), the kept
// flags become ballots, a CTA scan of the warp totals places each run, and
// the kept values go straight to dst with 16-bit stores (consecutive lanes
// write consecutive values).  Returns the kept count on every consumer.  NR
// (<= 8) is a template parameter -- probe_filter dispatches on it once per
// pair -- so the rounds are straight-line code (guarded rounds cost ~90
// instructions per warp per pair in branches alone); the reads are clamped
// into P, so lanes past the end only drop out of the ballots.
template <uint32_t WANT, int NR>
__device__ __forceinline__ uint32_t probe_filter_n(const uint16_t *P, uint32_t np, uint32_t X, uint16_t *dst,
                                                   uint32_t (*red2)[LT / 32], uint64_t *release) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t *P32 = (const uint32_t *)P;
  const uint32_t np2 = (np + 1) >> 1;
  const uint32_t beg = w * NR * 32u + lane, last = np2 - 1;
  uint32_t BL[NR], BH[NR], XV[NR], tot = 0;
#pragma unroll
  for (int r = 0; r < NR; r++) {
    const uint32_t i = beg + 32u * r;
    const uint32_t x = P32[min(i, last)];
    XV[r] = x;
    const uint32_t wl = lds32(X | ((x >> 3) & 0x1FFCu)), wh = lds32(X | ((x >> 19) & 0x1FFCu));
    const uint32_t bl = __funnelshift_r(wl, 0u, x) & 1u, bh = __funnelshift_r(wh, 0u, x >> 16) & 1u;
    BL[r] = __ballot_sync(0xffffffffu, (bl == WANT) & (i < np2));
    BH[r] = __ballot_sync(0xffffffffu, (bh == WANT) & (2 * i + 1 < np));
    tot += __popc(BL[r]) + __popc(BH[r]);
  }
  uint32_t *red = red2[0];
  if (lane == 0) red[w] = tot;
  cbar();
  if (threadIdx.x == 0) mbar_arrive(release);  // P's values are in registers
  uint32_t base = 0, total = 0;
#pragma unroll
  for (int k = 0; k < LT / 32; k++) {
    const uint32_t s = red[k];
    base += k < w ? s : 0;
    total += s;
  }
  if (dst && total) {
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < NR; r++) {
      const uint32_t bl = BL[r], bh = BH[r];
      const uint32_t klo = (bl >> lane) & 1u, khi = (bh >> lane) & 1u;
      const uint32_t x = XV[r];
      const uint32_t pos = base + __popc(bl & lt) + __popc(bh & lt);
      if (klo) dst[pos] = (uint16_t)x;
      if (khi) dst[pos + klo] = (uint16_t)(x >> 16);
      base += __popc(bl) + __popc(bh);
    }
    const uint32_t padded = (total + 7u) & ~7u;
    if (threadIdx.x < 8 && total + threadIdx.x < padded) dst[total + threadIdx.x] = 0;
  }
  return total;
}

template <uint32_t WANT>
__device__ __forceinline__ uint32_t probe_filter(const uint16_t *P, uint32_t np, uint32_t X, uint16_t *dst,
                                                 uint32_t (*red2)[LT / 32], uint64_t *release) {
  switch ((((np + 1) >> 1) + 255) >> 8) {  // rounds of 32 value pairs per warp (np >= 1)
    case 1: return probe_filter_n<WANT, 1>(P, np, X, dst, red2, release);
    case 2: return probe_filter_n<WANT, 2>(P, np, X, dst, red2, release);
    case 3: return probe_filter_n<WANT, 3>(P, np, X, dst, red2, release);
    case 4: return probe_filter_n<WANT, 4>(P, np, X, dst, red2, release);
    case 5: return probe_filter_n<WANT, 5>(P, np, X, dst, red2, release);
    case 6: return probe_filter_n<WANT, 6>(P, np, X, dst, red2, release);
    case 7: return probe_filter_n<WANT, 7>(P, np, X, dst, red2, release);
    default: return probe_filter_n<WANT, 8>(P, np, X, dst, red2, release);
  }
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

// One pair (consumers only).  `release` (the item's ring slot) is arrived on
// exactly once, after the barrier that follows the last read of the staged
// values.
//   and / andnot: X (XA / XB alternate by pair parity) is cleared after the
//     scan barrier; the next pair uses the other one.
//   or / xor: XA only; each thread reads and clears the words it owns
//     (t + 256q) before the scan barrier, which every consumer passes before
//     the next pair's scatter; array results are staged in XA (re-zeroed
//     behind a barrier).
template <int op>
__device__ __forceinline__ uint32_t large_pair(const LargeSmem &sm, const uint16_t *A, uint32_t na, const uint16_t *B,
                               uint32_t nb, uint8_t *dst, int parity, uint8_t &type, uint32_t &nout,
                               uint64_t *release) {
  const int t = threadIdx.x;
  uint32_t *XA = sm.XA(), *XB = sm.XB();
  type = RS_TAG_ARRAY;
  if constexpr (op == RS_OP_AND || op == RS_OP_ANDNOT) {
    constexpr bool is_and = op == RS_OP_AND;
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
      const uint32_t base = cscan(keep, sm.h->red[parity], total);
      if (t == 0) mbar_arrive(release);
      nout = total;
      if (dst && total) {
        uint16_t *d = (uint16_t *)dst;
        if (keep) d[base] = (uint16_t)v;
        const uint32_t padded = (total + 7u) & ~7u;
        if (t < 8 && total + t < padded) d[total + t] = 0;
      }
      return total;
    }
    // and: build the smaller side, filter the larger; andnot: build B, filter A
    const bool build_a = is_and && na <= nb;
    uint32_t *X = parity ? XB : XA;
    const uint32_t xs = rsb::smem_u32(X);
    scatter(build_a ? A : B, build_a ? na : nb, xs);
    cbar();
    const uint32_t total = probe_filter<is_and ? 1u : 0u>(build_a ? B : A, build_a ? nb : na, xs, (uint16_t *)dst,
                                                           sm.h->red[parity], release);
    // every probe of X is done (scan barrier above): clear it for pair + 2
    ((uint4 *)X)[t] = make_uint4(0, 0, 0, 0);
    ((uint4 *)X)[t + LT] = make_uint4(0, 0, 0, 0);
    nout = total;
    return total;
  }
  // or / xor: both arrays into one bitset (shared OR / XOR), so the result
  // words are read (and cleared) once
  constexpr bool is_xor = op == RS_OP_XOR;
  scatter<is_xor>(A, na, rsb::smem_u32(XA));
  scatter<is_xor>(B, nb, rsb::smem_u32(XA));
  cbar();
  if (t == 0) mbar_arrive(release);
  // result words t + 256q (conflict-free), positions by a packed row scan
  uint64_t *XA64 = (uint64_t *)XA;
  uint64_t r[4];
  uint32_t pq[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    r[q] = XA64[t + LT * q];
    XA64[t + LT * q] = 0;
    pq[q] = __popcll(r[q]);
  }
  // cardinality first (one warp reduction); the position scan only for an
  // array result
  uint32_t *red = sm.h->red[parity][0];
  const int lane = t & 31, w = t >> 5;
  const uint32_t wsum = __reduce_add_sync(0xffffffffu, pq[0] + pq[1] + pq[2] + pq[3]);
  if (lane == 0) red[w] = wsum;
  cbar();
  uint32_t card = 0;
#pragma unroll
  for (int k = 0; k < LT / 32; k++) card += red[k];
  if (!dst || card == 0) {
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
  const uint32_t pk0 = pq[0] | (pq[1] << 16), pk1 = pq[2] | (pq[3] << 16);
  uint32_t e0, e1, T0, T1;
  cscan2(pk0, pk1, sm.h->red[parity ^ 1], e0, e1, T0, T1);
  const uint32_t r0 = T0 & 0xFFFFu, r1 = T0 >> 16, r2 = T1 & 0xFFFFu;
  uint16_t *stage = (uint16_t *)XA;
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
  const uint32_t nvec = (2 * card + 15) >> 4;
  for (uint32_t v = t; v < nvec; v += LT) ((uint4 *)stage)[v] = make_uint4(0, 0, 0, 0);
  cbar();  // XA is zero again before any consumer's next scatter
  nout = card;
  return card;
}

// Persistent, warp-specialized byte ring over items i = blockIdx.x + k*gridDim.x.
// meta_of(i, aoff, boff) -> LargeMeta (runs on the producer lane only);
// sink(meta, card, type, n) runs on every consumer thread after the pair.
template <int op, typename MetaOf, typename Sink>
__device__ void large_loop(uint8_t *raw, uint32_t count, const uint8_t *poolA, const uint8_t *poolB,
                           uint8_t *opool, MetaOf meta_of, Sink sink) {
  const int t = threadIdx.x;
  const LargeSmem sm = large_layout(raw);
  if (sm.ring < 2u * 8192u) __trap();  // the largest item (2 x 4096 values) must fit
  if (t == 0) {
    for (int s = 0; s < NSLOT; s++) {
      rsb::mbar_init(&sm.h->full[s], 1);
      rsb::mbar_init(&sm.h->empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int w = t; w < 4 * RS_WORDS; w += LTHREADS) sm.XA()[w] = 0;  // XA and XB
  __syncthreads();
  if (t >= LT) {  // ---------------- producer warp (one elected lane)
    if (t == LT) {
      uint64_t ao, bo;
      LargeMeta m;
      if (blockIdx.x < count) m = meta_of(blockIdx.x, ao, bo);
      uint32_t phys = 0, occ = 0, oldest = 0;  // next free ring byte, bytes held, oldest unreleased item
      for (uint32_t j = 0;; j++) {
        const uint32_t i = blockIdx.x + j * gridDim.x;
        if (i >= count) break;
        const int s = j % NSLOT;
        // metadata of the next item is fetched before waiting for ring space
        uint64_t nao = 0, nbo = 0;
        LargeMeta nm = m;
        if (i + gridDim.x < count) nm = meta_of(i + gridDim.x, nao, nbo);
        const uint32_t ba = (uint32_t)rs_pad16(2ull * m.na), bb = (uint32_t)rs_pad16(2ull * m.nb);
        const uint32_t need = ba + bb;
        uint32_t pos = phys, skip = 0;
        if (phys + need > sm.ring) {  // wrap: the item starts at 0, the tail bytes go with it
          skip = sm.ring - phys;
          pos = 0;
        }
        uint32_t span = need + skip;
        if (span > sm.ring) {
          // a large item right after the middle of the ring: wait for the
          // ring to drain, then it starts at 0 with nothing to skip
          while (oldest < j) {
            mbar_wait_backoff(&sm.h->empty[oldest % NSLOT], (oldest / NSLOT) & 1);
            occ -= sm.h->span[oldest % NSLOT];
            oldest++;
          }
          span = need;
          occ = 0;
        }
        while (j - oldest >= (uint32_t)NSLOT || occ + span > sm.ring) {
          mbar_wait_backoff(&sm.h->empty[oldest % NSLOT], (oldest / NSLOT) & 1);
          occ -= sm.h->span[oldest % NSLOT];
          oldest++;
        }
        sm.h->span[s] = span;
        occ += span;
        phys = pos + need;
        m.aoff = pos;
        m.boff = pos + ba;
        sm.h->meta[s] = m;
        rsb::mbar_expect_tx(&sm.h->full[s], need);
        if (ba) rsb::bulk_g2s(sm.R() + pos, poolA + ao, ba, &sm.h->full[s]);
        if (bb) rsb::bulk_g2s(sm.R() + pos + ba, poolB + bo, bb, &sm.h->full[s]);
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
    const int s = k % NSLOT;
    rsb::mbar_wait(&sm.h->full[s], (k / NSLOT) & 1);
    const LargeMeta m = sm.h->meta[s];
    uint8_t type;
    uint32_t n;
    const uint32_t card = large_pair<op>(sm, (const uint16_t *)(sm.R() + m.aoff), m.na,
                                     (const uint16_t *)(sm.R() + m.boff), m.nb, opool ? opool + m.dst : nullptr,
                                     k & 1, type, n, &sm.h->empty[s]);
    sink(m, card, type, n);
  }
}

}  // namespace rsl
