// rs_array_large.cuh -- large array x array pairs (na + nb > 256) through
// shared-memory bitsets instead of a merge path.
//
// Same results as the two-pointer kernels (kernels/scalar.py:122-267) and
// _container_from_values (containers.py:244-247):
//   and / andnot  one bitset X built from the smaller side (and) or from B
//                 (andnot); the other side is filtered through it with warp
//                 ballots, so the result comes out sorted;
//   or / xor      both sides scattered into X (shared OR, resp. XOR); the
//                 result words with a popcount scan give the cardinality, and
//                 the result is the words themselves (> 4096 values: a bitset
//                 container) or their set bits in order (<= 4096: an array
//                 container).
// AND / ANDNOT pairs with one side at most 1/16 of the other never get here:
// the classifier sends them to the galloping kernel (gallop_pair).
//
// CTA layout (warp-specialized): warps 0-7 are consumers, split into NGRP
// groups of 256 / NGRP threads; each group works on its own pair with its own
// bitset (XA / XB) and synchronizes only among itself with named barrier
// 1 + group.  Warp 8 is the producer.  The producer walks the CTA's items,
// loads each item's metadata (operand offsets, sizes, output slot, pair) and
// streams both arrays (variable sizes, 16-byte padded) into a byte ring in
// shared memory with cp.async.bulk completing on the item slot's `full`
// mbarrier; group g consumes items g, g + NGRP, ...  Items take only the bytes
// they need, and a group hands an item's bytes back through the slot's
// `empty` mbarrier as soon as its last value has been read.
//
// Two groups of four warps (the default) against one group of eight: a pair's
// fixed work -- metadata, barriers, loop set-up, scan -- is per warp, and most
// large pairs hold a few hundred values, so eight warps per pair left most
// lanes idle; two pairs in flight per CTA halve that overhead per pair.
#pragma once
#include "rs_internal.cuh"
#include "rs_bitset.cuh"

namespace rsl {

#ifndef RS_AAL_GROUPS
#define RS_AAL_GROUPS 2
#endif
constexpr int NGRP = RS_AAL_GROUPS;     // consumer groups (1 or 2)
constexpr int NCONS = 256;              // consumer threads
constexpr int LT = NCONS / NGRP;        // threads per group (one pair at a time)
constexpr int WG = LT / 32;             // warps per group
constexpr int QW = RS_WORDS / LT;       // 64-bit result words per thread (or / xor)
constexpr int NROW = QW / 2;            // packed 16-bit scan rows (two words each)
constexpr int LTHREADS = NCONS + 32;    // + one producer warp
#ifndef RS_AAL_MAXR
#define RS_AAL_MAXR 8
#endif
#ifndef RS_AAL_NSLOT
#define RS_AAL_NSLOT 8
#endif
constexpr int NSLOT = RS_AAL_NSLOT;     // items in flight (metadata + barrier slots)
static_assert(NGRP == 1 || NGRP == 2, "one or two consumer groups");

struct LargeMeta {
  uint32_t na, nb, e, pair;
  uint64_t dst;
  uint32_t aoff, boff;  // ring offsets of the staged arrays
};

// Shared-memory layout (dynamic; carved at run time by large_layout):
//   header | byte ring | (pad) | XA (8 KB) | XB (8 KB)
// XA / XB sit on 8 KB boundaries of the shared window so a value's word
// address is base | offset (see scatter); they take the highest aligned 16 KB
// of the allocation, so the alignment pad (< 8 KB) comes out of the ring's
// tail rather than sitting between the header and the bitsets.
struct LargeHdr {
  uint64_t full[NSLOT];
  uint64_t empty[NSLOT];
  LargeMeta meta[NSLOT];
  uint32_t span[NSLOT];  // producer only: ring bytes each item holds (incl. the wrap skip)
  uint32_t red[NGRP][2][NROW][WG];  // per group, double-buffered scan scratch
};

struct LargeSmem {
  LargeHdr *h;
  uint8_t *X;     // XA, XB
  uint8_t *ring_base;
  uint32_t ring;  // ring bytes
  __device__ __forceinline__ uint32_t *XA() const { return (uint32_t *)X; }
  __device__ __forceinline__ uint32_t *XB() const { return (uint32_t *)(X + 8192); }
  __device__ __forceinline__ uint32_t *Xn(int i) const { return (uint32_t *)(X + 8192 * i); }
  __device__ __forceinline__ uint8_t *R() const { return ring_base; }
};

// Register budget: the AND / ANDNOT op kernels (probe rounds whose kept
// values are written out) run three CTAs per SM with up to 72 registers --
// at four CTAs' 56 they spill ~120 bytes per thread, and measured 1.65 /
// 2.14 ms against 1.39 / 1.97 ms on config 3; OR / XOR and the counts keep
// four CTAs (1.74 / 1.10 ms against 1.85 / 1.15 ms at three).
// RS_AAL_MINB overrides both (tuning).
constexpr int large_min_blocks(int op) {
#ifdef RS_AAL_MINB
  return RS_AAL_MINB + 0 * op;
#else
  return op == RS_OP_AND || op == RS_OP_ANDNOT ? 3 : 4;
#endif
}

// Shared memory per CTA: 56 KB, four CTAs per SM (228 KB less 1 KB reserved
// per CTA); the ring gets ~38 KB.  72 KB for the three-CTA AND / ANDNOT
// kernels (a 54 KB ring) measured no better on config 3 (AND 1.32 -> 1.44 ms,
// ANDNOT 1.90 -> 1.79 ms), nor did 16 item slots.  large_loop traps if the ring is ever under 16 KB, the largest item
// (an item that does not fit before the end of the ring waits for the ring to
// drain and starts at 0).  RS_AAL_SMEM_KB overrides (tuning).
// The AND op kernel holds two more bitsets (the dual-bitset pairs below):
// 72 KB, which its three CTAs per SM (register-bound) fit.
constexpr int large_nbits(int op, bool count) { return op == RS_OP_AND && !count ? 4 : 2; }
constexpr size_t large_smem_bytes(int op, bool count) {
#ifdef RS_AAL_SMEM_KB
  return (size_t)RS_AAL_SMEM_KB * 1024 + 8192 * (large_nbits(op, count) - 2);
#else
  return (size_t)56 * 1024 + 8192 * (large_nbits(op, count) - 2);
#endif
}

__device__ __forceinline__ LargeSmem large_layout(uint8_t *raw, uint32_t bytes, int nbits) {
  LargeSmem sm;
  sm.h = (LargeHdr *)raw;
  const uint32_t b = rsb::smem_u32(raw);
  const uint32_t r0 = (b + (uint32_t)sizeof(LargeHdr) + 127u) & ~127u;
  const uint32_t x = (b + bytes - 8192u * nbits) & ~8191u;
  sm.X = raw + (x - b);
  sm.ring_base = raw + (r0 - b);
  sm.ring = x > r0 ? (x - r0) & ~15u : 0u;
  return sm;
}

// group barrier (named barrier 1 + g, the group's threads only)
// (immediate ids: a register id makes ptxas reserve all 16 barriers)
__device__ __forceinline__ void gbar(int g) {
  if (NGRP == 1 || g == 0) asm volatile("bar.sync 1, %0;" ::"n"(LT) : "memory");
  else asm volatile("bar.sync 2, %0;" ::"n"(LT) : "memory");
}

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

// Group-wide exclusive scan of N packed vectors (16-bit fields): exclusive
// prefixes e[] and totals T[] (one group barrier).
template <int N>
__device__ __forceinline__ void gscan(const uint32_t (&v)[N], uint32_t (*red)[WG], int g, int t, uint32_t (&e)[N],
                                      uint32_t (&T)[N]) {
  const int lane = t & 31, w = t >> 5;
  uint32_t x[N];
#pragma unroll
  for (int j = 0; j < N; j++) x[j] = v[j];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < N; j++) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x[j], o);
      if (lane >= o) x[j] += y;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int j = 0; j < N; j++) red[j][w] = x[j];
  }
  gbar(g);
#pragma unroll
  for (int j = 0; j < N; j++) {
    e[j] = x[j] - v[j];
    T[j] = 0;
  }
#pragma unroll
  for (int k = 0; k < WG; k++) {
#pragma unroll
    for (int j = 0; j < N; j++) {
      const uint32_t a = red[j][k];
      T[j] += a;
      if (k < w) e[j] += a;
    }
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
__device__ __forceinline__ void scatter(const uint16_t *v, uint32_t n, uint32_t X, int t) {
  const uint32_t *w = (const uint32_t *)v;
  const uint32_t nw = n >> 1;
#pragma unroll 4
  for (uint32_t i = t; i < nw; i += LT) {
    const uint32_t x = w[i];
    const uint32_t alo = X | ((x >> 3) & 0x1FFCu), ahi = X | ((x >> 19) & 0x1FFCu);
    const uint32_t blo = __funnelshift_l(0u, 1u, x), bhi = __funnelshift_l(0u, 1u, x >> 16);
    const bool same = alo == ahi;
    red_set<XOR>(alo, same ? blo | bhi : blo);
    if (!same) red_set<XOR>(ahi, bhi);
  }
  if ((n & 1) && t == LT - 1) {
    const uint32_t x = v[n - 1];
    red_set<XOR>(X | ((x >> 3) & 0x1FFCu), __funnelshift_l(0u, 1u, x));
  }
}

// 16-byte forms of scatter / membership: a thread takes whole 8-value
// vectors (t, t + LT, ...), so one LDS.128 feeds eight values and every value
// costs its address (SHF + LOP3), its bit and one shared RED -- no pairing
// test, no divergent second RED, no loop bookkeeping per value pair (the
// 32-bit forms measured ~8 instructions per value on dense 4096-value pairs).
// Staged arrays start 16-byte aligned in the ring; the last n % 8 values go
// one per thread.
template <bool XOR>
__device__ __forceinline__ void set_pair(uint32_t x, uint32_t X) {
  red_set<XOR>(X | ((x >> 3) & 0x1FFCu), __funnelshift_l(0u, 1u, x));
  red_set<XOR>(X | ((x >> 19) & 0x1FFCu), __funnelshift_l(0u, 1u, x >> 16));
}

// Vector width of the scatter / membership loads (bytes per lane: 4, 8 or
// 16).  Wider loads cost fewer instructions per value; narrower ones keep a
// warp's lanes closer to consecutive 32-bit words of a dense array: on a
// 1/16-dense array a lane's 2 / 4 / 8 values span ~1 / 2 / 4 words, so at
// every step lanes l and l + 32 / 16 / 8 land in one bank -- none, 2-way and
// 4-way conflicts for the REDs and probes.  C3: 9.66 ms at 16 bytes, 9.19 at
// 8, 9.21 at 4.  (Rotating each lane's word order by its bank group measured
// no better.)
#ifndef RS_AAL_VEC
#define RS_AAL_VEC 8
#endif
template <int VB> struct LaneVec;
template <> struct LaneVec<4> { using T = uint32_t; };
template <> struct LaneVec<8> { using T = uint2; };
template <> struct LaneVec<16> { using T = uint4; };
__device__ __forceinline__ uint32_t vword(uint32_t v, int) { return v; }
__device__ __forceinline__ uint32_t vword(uint2 v, int k) { return k ? v.y : v.x; }
__device__ __forceinline__ uint32_t vword(uint4 v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
// A lane's four values (sorted, one 8-byte vector) with the bits of values
// that share a 32-bit word merged in registers, so each touched word takes
// one shared RED: the kernel is bound by the shared-memory pipe, not by issue
// (ncu on C3 AND: 157 M shared wavefronts = 76 % of the pipe's peak against
// 67 % issue; 73 M of them for 26.5 M RED instructions, ~2.75 per
// instruction in bank and same-word conflicts).  On C3's dense arrays
// (4,096 values: 57 % of adjacent values share a word) a lane's four values
// touch ~2.3 words, so the three predicated REDs run with ~43 % of their
// lanes; the cost is a compare and a predicated OR per adjacent pair.
#ifndef RS_AAL_MERGE
#define RS_AAL_MERGE 0
#endif
template <bool XOR>
__device__ __forceinline__ void set_vec4_merged(uint32_t x, uint32_t y, uint32_t X) {
  const uint32_t a0 = X | ((x >> 3) & 0x1FFCu), a1 = X | ((x >> 19) & 0x1FFCu);
  const uint32_t a2 = X | ((y >> 3) & 0x1FFCu), a3 = X | ((y >> 19) & 0x1FFCu);
  const uint32_t b0 = __funnelshift_l(0u, 1u, x);
  uint32_t b1 = __funnelshift_l(0u, 1u, x >> 16), b2 = __funnelshift_l(0u, 1u, y), b3 = __funnelshift_l(0u, 1u, y >> 16);
  if (a1 == a0) b1 |= b0;
  else red_set<XOR>(a0, b0);
  if (a2 == a1) b2 |= b1;
  else red_set<XOR>(a1, b1);
  if (a3 == a2) b3 |= b2;
  else red_set<XOR>(a2, b2);
  red_set<XOR>(a3, b3);
}

template <bool XOR = false>
__device__ __forceinline__ void scatter16(const uint16_t *v, uint32_t n, uint32_t X, int t) {
  constexpr int VB = RS_AAL_VEC, NV = VB / 2;  // values per lane vector
  using V = typename LaneVec<VB>::T;
  const V *vp = (const V *)v;
  const uint32_t nfull = n / NV;
#pragma unroll 2
  for (uint32_t i = t; i < nfull; i += LT) {
    const V q = vp[i];
    if constexpr (VB == 8 && RS_AAL_MERGE) set_vec4_merged<XOR>(vword(q, 0), vword(q, 1), X);
    else {
#pragma unroll
      for (int k = 0; k < VB / 4; k++) set_pair<XOR>(vword(q, k), X);
    }
  }
  if ((uint32_t)t < n - nfull * NV) {
    const uint32_t x = v[nfull * NV + t];
    red_set<XOR>(X | ((x >> 3) & 0x1FFCu), __funnelshift_l(0u, 1u, x));
  }
}

__device__ __forceinline__ uint32_t member_pair(uint32_t x, uint32_t X) {
  const uint32_t wl = lds32(X | ((x >> 3) & 0x1FFCu)), wh = lds32(X | ((x >> 19) & 0x1FFCu));
  return (__funnelshift_r(wl, 0u, x) & 1u) + (__funnelshift_r(wh, 0u, x >> 16) & 1u);
}

// |P intersect X| over the group (counts only: no positions, no ballots).
// Each thread arrives on `release` after its last read of P.
__device__ __forceinline__ uint32_t probe_count16(const uint16_t *P, uint32_t np, uint32_t X, uint32_t *red, int g,
                                                  int t, uint64_t *release) {
  constexpr int VB = RS_AAL_VEC, NV = VB / 2;
  using V = typename LaneVec<VB>::T;
  const V *vp = (const V *)P;
  const uint32_t nfull = np / NV;
  uint32_t c = 0;
#pragma unroll 2
  for (uint32_t i = t; i < nfull; i += LT) {
    const V q = vp[i];
#pragma unroll
    for (int k = 0; k < VB / 4; k++) c += member_pair(vword(q, k), X);
  }
  if ((uint32_t)t < np - nfull * NV) {
    const uint32_t x = P[nfull * NV + t];
    c += __funnelshift_r(lds32(X | ((x >> 3) & 0x1FFCu)), 0u, x) & 1u;
  }
  mbar_arrive(release);
  const int lane = t & 31, w = t >> 5;
  const uint32_t ws = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) red[w] = ws;
  gbar(g);
  uint32_t total = 0;
#pragma unroll
  for (int k = 0; k < WG; k++) total += red[k];
  return total;
}

// One chunk of probe_filter: value pairs [c2, c2 + WG * NR * 32) of P, warp w
// a contiguous run of NR rounds of 32 value pairs.  The kept flags become
// ballots, a group scan of the warp totals places each run after the `out`
// values kept by earlier chunks, and the kept values go straight to dst with
// 16-bit stores (consecutive lanes write consecutive values).  NR is a
// template parameter so the rounds are straight-line code (guarded rounds
// cost ~90 instructions per warp per pair in branches alone); the reads are
// clamped into P, so lanes past the end only drop out of the ballots.
template <uint32_t WANT, int NR>
__device__ __forceinline__ uint32_t probe_chunk(const uint32_t *P32, uint32_t np, uint32_t c2, uint32_t X,
                                                uint16_t *dst, uint32_t out, uint32_t *red, int g, int t,
                                                uint64_t *release) {
  const int lane = t & 31, w = t >> 5;
  const uint32_t np2 = (np + 1) >> 1;
  const uint32_t beg = c2 + w * NR * 32u + lane, last = np2 ? np2 - 1 : 0;
  uint32_t BL[NR], BH[NR], tot = 0;
#pragma unroll
  for (int r = 0; r < NR; r++) {
    const uint32_t i = beg + 32u * r;
    const uint32_t x = P32[min(i, last)];
    const uint32_t wl = lds32(X | ((x >> 3) & 0x1FFCu)), wh = lds32(X | ((x >> 19) & 0x1FFCu));
    const uint32_t bl = __funnelshift_r(wl, 0u, x) & 1u, bh = __funnelshift_r(wh, 0u, x >> 16) & 1u;
    BL[r] = __ballot_sync(0xffffffffu, (bl == WANT) & (i < np2));
    BH[r] = __ballot_sync(0xffffffffu, (bh == WANT) & (2 * i + 1 < np));
    tot += __popc(BL[r]) + __popc(BH[r]);
  }
  if (lane == 0) red[w] = tot;
  gbar(g);
  uint32_t base = out, total = 0;
#pragma unroll
  for (int k = 0; k < WG; k++) {
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
      const uint32_t x = P32[min(beg + 32u * r, last)];  // re-read: fewer live registers
      const uint32_t pos = base + __popc(bl & lt) + __popc(bh & lt);
      if (klo) dst[pos] = (uint16_t)x;
      if (khi) dst[pos + klo] = (uint16_t)(x >> 16);
      base += __popc(bl) + __popc(bh);
    }
  }
  if (release) mbar_arrive(release);  // this thread's last read of P (the slot counts LT arrivals)
  return total;
}

// Keep the values of P (np >= 1, sorted) whose bit in X equals WANT, in order,
// in chunks of at most 8 rounds per warp (one chunk with eight warps per
// group; two for np > 2048 with four).  Chunks alternate the two scratch rows
// starting at `parity`, so a chunk never overwrites a total another thread of
// the group may still be reading.  Each thread arrives on `release` after its
// last read of P (in the last chunk).  Returns the kept count on every thread of the group.
template <uint32_t WANT>
__device__ __forceinline__ uint32_t probe_filter(const uint16_t *P, uint32_t np, uint32_t X, uint16_t *dst,
                                                 uint32_t (*red2)[NROW][WG], int parity, int g, int t,
                                                 uint64_t *release) {
  const uint32_t *P32 = (const uint32_t *)P;
  constexpr uint32_t PER_ROUND = WG * 32u;  // value pairs per round over the group
  constexpr uint32_t MAXR = RS_AAL_MAXR;
  uint32_t rounds = (((np + 1) >> 1) + PER_ROUND - 1) / PER_ROUND;
  if (rounds == 0) rounds = 1;
  uint32_t out = 0, c2 = 0;
  int buf = parity;
  for (;;) {
    const bool lastc = rounds <= MAXR;
    uint32_t *red = red2[buf][0];
    uint64_t *rel = lastc ? release : nullptr;
    uint32_t got;
    switch (lastc ? rounds : (uint32_t)MAXR) {
      case 1: got = probe_chunk<WANT, 1>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      case 2: got = probe_chunk<WANT, 2>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      case 3: got = probe_chunk<WANT, 3>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      case 4: got = probe_chunk<WANT, 4>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      case 5: got = probe_chunk<WANT, 5>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      case 6: got = probe_chunk<WANT, 6>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      case 7: got = probe_chunk<WANT, 7>(P32, np, c2, X, dst, out, red, g, t, rel); break;
      default: got = probe_chunk<WANT, 8>(P32, np, c2, X, dst, out, red, g, t, rel); break;
    }
    out += got;
    if (lastc) break;
    rounds -= MAXR;
    c2 += MAXR * PER_ROUND;
    buf ^= 1;
  }
  if (dst && out) {
    const uint32_t padded = (out + 7u) & ~7u;
    if (t < 8 && out + t < padded) dst[out + t] = 0;
  }
  return out;
}

// Copy `total` staged u16 values to dst with 128-bit stores (16-byte zero pad).
__device__ __forceinline__ void flush_stage(uint16_t *stage, uint32_t total, uint8_t *dst, int g, int t) {
  const uint32_t nvec = (2 * total + 15) >> 4;
  if (t < 8 && total + t < nvec * 8) stage[total + t] = 0;
  gbar(g);
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

// The result words of a group's bitset X -- or of X AND X2 (DUAL) -- read
// and cleared (each thread its words t + LT q), the cardinality, and the
// result at dst: the words (> 4096 values) or their values in order, staged
// in X.  Ends with X (and X2) zero behind a group barrier.
template <bool DUAL>
__device__ __forceinline__ uint32_t sweep_encode(uint32_t *X, uint32_t *X2, uint8_t *dst,
                                                 uint32_t (*red2)[NROW][WG], int parity, int g, int t, uint8_t &type,
                                                 uint32_t &nout) {
  // result words t + LT q (conflict-free), positions by a packed row scan
  uint64_t *X64 = (uint64_t *)X, *Y64 = (uint64_t *)X2;
  uint64_t r[QW];
  uint32_t psum = 0;
#pragma unroll
  for (int q = 0; q < QW; q++) {
    r[q] = X64[t + LT * q];
    X64[t + LT * q] = 0;
    if constexpr (DUAL) {
      r[q] &= Y64[t + LT * q];
      Y64[t + LT * q] = 0;
    }
    psum += __popcll(r[q]);
  }
  // cardinality first (one warp reduction); the position scan only for an
  // array result
  uint32_t *red = red2[parity][0];
  const int lane = t & 31, w = t >> 5;
  const uint32_t wsum = __reduce_add_sync(0xffffffffu, psum);
  if (lane == 0) red[w] = wsum;
  gbar(g);
  uint32_t card = 0;
#pragma unroll
  for (int k = 0; k < WG; k++) card += red[k];
  if (!dst || card == 0) {
    nout = card;
    return card;
  }
  if (card > RS_ARRAY_MAX) {
    uint64_t *p = (uint64_t *)dst + t;
#pragma unroll
    for (int q = 0; q < QW; q++) asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p + LT * q), "l"(r[q]) : "memory");
    type = RS_TAG_BITSET;
    nout = RS_WORDS;
    return card;
  }
  // word t + LT q's values end at (values of rows < q) + (row q's prefix
  // before t) + its own count; rows are scanned two per packed vector
  uint32_t pk[NROW], e[NROW], T[NROW];
#pragma unroll
  for (int j = 0; j < NROW; j++) pk[j] = __popcll(r[2 * j]) | (__popcll(r[2 * j + 1]) << 16);
  gscan<NROW>(pk, red2[parity ^ 1], g, t, e, T);
  uint16_t *stage = (uint16_t *)X;
  uint32_t rowbase = 0;
#pragma unroll
  for (int q = 0; q < QW; q++) {
    const int j = q >> 1;
    const uint32_t ex = (q & 1) ? e[j] >> 16 : e[j] & 0xFFFFu;
    const uint32_t tot = (q & 1) ? T[j] >> 16 : T[j] & 0xFFFFu;
    const uint32_t pos = (uint32_t)(t + LT * q) * 64;
    uint32_t b = rowbase + ex + (uint32_t)__popcll(r[q]), hi = (uint32_t)(r[q] >> 32), lo = (uint32_t)r[q];
    rowbase += tot;
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
  flush_stage(stage, card, dst, g, t);
  const uint32_t nvec = (2 * card + 15) >> 4;
  for (uint32_t v = t; v < nvec; v += LT) ((uint4 *)stage)[v] = make_uint4(0, 0, 0, 0);
  gbar(g);  // X is zero again before the group's next scatter
  nout = card;
  return card;
}

// One pair (the group's threads only; t = thread within the group).
// `release` (the item's ring slot) is arrived on once by every thread of the
// group, after that thread's last read of the staged values (a slot's items
// always go to the same group: k % NSLOT fixes k % NGRP).
//   and / andnot: two groups: the group's own bitset, cleared after the probe
//     and fenced by a barrier at the start of the group's next pair; one
//     group: XA / XB alternate by pair parity, so no fence is needed.
//   or / xor: the group's bitset (XA with one group); each thread reads and
//     clears the words it owns (t + LT q) before the cardinality barrier,
//     which every thread of the group passes before its next scatter; array
//     results are staged in the same bitset (re-zeroed behind a barrier).
template <int op, bool COUNT>
__device__ __forceinline__ uint32_t large_pair(const LargeSmem &sm, int g, int t, const uint16_t *A, uint32_t na,
                                               const uint16_t *B, uint32_t nb, uint8_t *dst, int parity,
                                               uint8_t &type, uint32_t &nout, uint64_t *release) {
  uint32_t *XA = sm.XA(), *XB = sm.XB();
  uint32_t(*red2)[NROW][WG] = sm.h->red[g];
  type = RS_TAG_ARRAY;
  if constexpr (op == RS_OP_AND || op == RS_OP_ANDNOT) {
    constexpr bool is_and = op == RS_OP_AND;
    // and: build the smaller side, filter the larger; andnot: build B, filter A
    const bool build_a = is_and && na <= nb;
    uint32_t *X = (NGRP == 2 ? g : parity) ? XB : XA;
    {  // galloping pairs (gallop_pair): the small side's values binary-searched in the staged large side
      const bool a_small = is_and ? na <= nb : true;
      const uint32_t ns = a_small ? na : nb, nl = a_small ? nb : na;
#ifndef RS_AAL_GALLOP_WARP
#define RS_AAL_GALLOP_WARP 64
#endif
      if (is_and && 16 * ns <= nl && ns <= RS_AAL_GALLOP_WARP) {  // (andnot: 4 bytes of spill with it, and no such pairs routed here)
        // at most 64 searches: the group's first warp does them alone (two
        // per lane, advancing together), places the kept values by ballot
        // and takes no group barrier; the other warps only hand the item's
        // bytes back.  (The 128-thread form below spent ~950 warp
        // instructions on such a pair, most of them the idle warps' share
        // of the scan and barriers.)
        const uint16_t *Sv = a_small ? A : B, *Lv = a_small ? B : A;
        uint32_t total = 0;
        if (t < 32) {
          const uint32_t v0 = (uint32_t)t < ns ? Sv[t] : 0u, v1 = (uint32_t)t + 32u < ns ? Sv[t + 32] : 0u;
          uint32_t lo0 = 0, lo1 = 0, len = nl;
          while (len > 1) {  // nl >= 16 here
            const uint32_t half = len >> 1;
            const uint32_t m0 = Lv[lo0 + half], m1 = Lv[lo1 + half];
            if (m0 <= v0) lo0 += half;
            if (m1 <= v1) lo1 += half;
            len -= half;
          }
          const bool k0 = (uint32_t)t < ns && (Lv[lo0] == v0) == is_and;
          const bool k1 = (uint32_t)t + 32u < ns && (Lv[lo1] == v1) == is_and;
          const uint32_t b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
          const uint32_t n0 = __popc(b0);
          total = n0 + __popc(b1);
          if (!COUNT && dst && total) {
            uint16_t *d = (uint16_t *)dst;
            const uint32_t lt = (1u << t) - 1u;
            if (k0) d[__popc(b0 & lt)] = (uint16_t)v0;
            if (k1) d[n0 + __popc(b1 & lt)] = (uint16_t)v1;
            const uint32_t padded = (total + 7u) & ~7u;
            if (t < 8 && total + t < padded) d[total + t] = 0;
          }
        }
        mbar_arrive(release);  // this thread's last read of the staged values
        if constexpr (NGRP == 1) gbar(g);  // one group: X alternates by parity and relies on a barrier per pair
        nout = total;
        return total;  // valid on the group's first warp (the sink runs on its lane 0)
      }
    }
    if constexpr (NGRP == 2) gbar(g);  // the previous pair's clear of X is complete
    {
      const bool a_small = is_and ? na <= nb : true;
      const uint32_t ns = a_small ? na : nb, nl = a_small ? nb : na;
      if (16 * ns <= nl) {
        const uint16_t *Sv = a_small ? A : B, *Lv = a_small ? B : A;
        uint32_t v[2], k[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const uint32_t i = t + LT * h;  // ns <= 4096 / 16 = 256 = 2 LT
          v[h] = i < ns ? Sv[i] : 0u;
          k[h] = i < ns && bsearch16(Lv, nl, v[h]) == is_and;
        }
        mbar_arrive(release);  // this thread's last read of the staged values
        const uint32_t pk[1] = {k[0] | (k[1] << 16)};
        uint32_t e[1], T[1];
        gscan<1>(pk, red2[parity], g, t, e, T);
        const uint32_t n0 = T[0] & 0xFFFFu, total = n0 + (T[0] >> 16);
        if (!COUNT && dst && total) {
          uint16_t *d = (uint16_t *)dst;
          if (k[0]) d[e[0] & 0xFFFFu] = (uint16_t)v[0];
          if (k[1]) d[n0 + (e[0] >> 16)] = (uint16_t)v[1];
          const uint32_t padded = (total + 7u) & ~7u;
          if (t < 8 && total + t < padded) d[total + t] = 0;
        }
        nout = total;
        return total;
      }
    }
// (threshold swept on C3 AND with the one-warp galloping path in: 1024 /
// 2048 / 4096 / 8192 / off = 1.173 / 1.151 / 1.136 / 1.14-1.18 / 1.167 ms)
#ifndef RS_AAL_DUAL_MIN
#define RS_AAL_DUAL_MIN 4096
#endif
    if constexpr (is_and && !COUNT && NGRP == 2) {
      // large AND pairs: both sides scattered (a shared OR per value) into
      // the group's two bitsets, then one sweep of their AND -- for ~4096 +
      // 4096 values cheaper than probing one side value by value (address,
      // load, bit test, ballot, kept-value stores: ~3x a scatter's
      // instructions per value); the result is at most min(na, nb) values
      if (na + nb >= RS_AAL_DUAL_MIN) {
        uint32_t *X2 = sm.Xn(g + 2);
        scatter16(A, na, rsb::smem_u32(X), t);
        scatter16(B, nb, rsb::smem_u32(X2), t);
        gbar(g);
        mbar_arrive(release);  // this thread's last read of the staged values
        return sweep_encode<true>(X, X2, dst, red2, parity, g, t, type, nout);
      }
    }
    const uint32_t xs = rsb::smem_u32(X);
    scatter16(build_a ? A : B, build_a ? na : nb, xs, t);
    gbar(g);
    uint32_t total;
    if constexpr (COUNT && is_and)
      total = probe_count16(build_a ? B : A, build_a ? nb : na, xs, red2[parity][0], g, t, release);
    else
      total = probe_filter<is_and ? 1u : 0u>(build_a ? B : A, build_a ? nb : na, xs, (uint16_t *)dst, red2, parity,
                                             g, t, release);
    // every probe of X is done (the last chunk's barrier above): clear it
#pragma unroll
    for (int q = 0; q < 512 / LT; q++) ((uint4 *)X)[t + LT * q] = make_uint4(0, 0, 0, 0);
    nout = total;
    return total;
  }
  // or / xor: both arrays into one bitset (shared OR / XOR), so the result
  // words are read (and cleared) once
  constexpr bool is_xor = op == RS_OP_XOR;
  uint32_t *X = (NGRP == 2 && g) ? XB : XA;
  const uint32_t xs = rsb::smem_u32(X);
  scatter16<is_xor>(A, na, xs, t);
  scatter16<is_xor>(B, nb, xs, t);
  gbar(g);
  mbar_arrive(release);
  return sweep_encode<false>(X, nullptr, dst, red2, parity, g, t, type, nout);
}

// Persistent, warp-specialized byte ring over items [0, count), taken
// dynamically: the producer draws the next item index from *ctr (zero at
// launch).  A static split (item blockIdx.x + k gridDim.x) left the kernel
// as slow as its latest-starting CTA: run beside the other classes' kernels
// on side streams, some CTAs found no free SM slot until those finished and
// then did a full share -- C3 AND measured 1.15 or 1.55 ms from call to
// call.  The producer ends each consumer group's sequence with a sentinel
// item (na = LARGE_END).
// meta_of(i, aoff, boff) -> LargeMeta (runs on the producer lane only);
// sink(meta, card, type, n) runs on thread 0 of the group that did the pair.
constexpr uint32_t LARGE_END = 0xFFFFFFFFu;
constexpr uint32_t LARGE_CHUNK = 4;
template <int op, bool COUNT, typename MetaOf, typename Sink>
__device__ void large_loop(uint8_t *raw, uint32_t count, uint32_t *ctr, const uint8_t *poolA, const uint8_t *poolB,
                           uint8_t *opool, MetaOf meta_of, Sink sink) {
  const int t = threadIdx.x;
  constexpr uint32_t SMEM = (uint32_t)large_smem_bytes(op, COUNT);
  constexpr int NB = large_nbits(op, COUNT);
  const LargeSmem sm = large_layout(raw, SMEM, NB);
  if (sm.ring < 2u * 8192u) __trap();  // the largest item (2 x 4096 values) must fit
  if (t == 0) {
    for (int s = 0; s < NSLOT; s++) {
      rsb::mbar_init(&sm.h->full[s], 1);
      rsb::mbar_init(&sm.h->empty[s], LT);  // every thread of the consuming group arrives
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int w = t; w < 2 * NB * RS_WORDS; w += LTHREADS) sm.XA()[w] = 0;  // every bitset
  __syncthreads();
  if (t >= NCONS) {  // ---------------- producer warp (one elected lane)
    if (t == NCONS) {
      uint64_t ao = 0, bo = 0;
      LargeMeta m;
      // items are drawn LARGE_CHUNK at a time (one atomic per item on one
      // counter cost C3's counts 4 %)
      uint32_t taken = 0, chunk_end = 0;
      auto take = [&]() -> uint32_t {
        if (taken == chunk_end) {
          taken = atomicAdd(ctr, (uint32_t)LARGE_CHUNK);
          chunk_end = taken + LARGE_CHUNK;
        }
        return taken++;
      };
      uint32_t i = take();
      if (i < count) m = meta_of(i, ao, bo);
      uint32_t phys = 0, occ = 0, oldest = 0;  // next free ring byte, bytes held, oldest unreleased item
      for (uint32_t j = 0;; j++) {
        if (i >= count) {  // no work left: a sentinel for each consumer group
          for (int q = 0; q < NGRP; q++, j++) {
            while (j - oldest >= (uint32_t)NSLOT) {
              mbar_wait_backoff(&sm.h->empty[oldest % NSLOT], (oldest / NSLOT) & 1);
              oldest++;
            }
            sm.h->meta[j % NSLOT].na = LARGE_END;
            rsb::mbar_expect_tx(&sm.h->full[j % NSLOT], 0);
          }
          break;
        }
        const int s = j % NSLOT;
        // the next item's index and metadata are fetched before waiting for
        // ring space
        const uint32_t ni = take();
        uint64_t nao = 0, nbo = 0;
        LargeMeta nm = m;
        if (ni < count) nm = meta_of(ni, nao, nbo);
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
        // Items are released out of order across groups; the producer waits
        // in item order, which only ever delays a slot's reuse.
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
        i = ni;
      }
    }
    return;
  }
  const int g = t / LT, tg = t % LT;
  for (uint32_t k = g;; k += NGRP) {  // ---------------- consumer group g
    const int s = k % NSLOT;
#ifdef RS_AAL_SPIN
    rsb::mbar_wait(&sm.h->full[s], (k / NSLOT) & 1);
#else
    // suspended in the barrier, not polling: a starved group's spin loop took
    // 10% of the kernel's issue slots from the group that has data
    mbar_wait_backoff(&sm.h->full[s], (k / NSLOT) & 1);
#endif
    const LargeMeta m = sm.h->meta[s];
    if (m.na == LARGE_END) break;
    uint8_t type;
    uint32_t n;
    const uint32_t card = large_pair<op, COUNT>(sm, g, tg, (const uint16_t *)(sm.R() + m.aoff), m.na,
                                         (const uint16_t *)(sm.R() + m.boff), m.nb, opool ? opool + m.dst : nullptr,
                                         (k / NGRP) & 1, type, n, &sm.h->empty[s]);
    if (tg == 0) sink(m, card, type, n);
  }
}

}  // namespace rsl
