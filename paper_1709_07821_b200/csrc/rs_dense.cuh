// rs_dense.cuh -- device helpers shared by every kernel that materializes a
// container through an 8 KB shared-memory bitset (one CTA of 256 threads;
// thread t owns words [4t, 4t+4)).
#pragma once
#include <cub/cub.cuh>
#include "rs_internal.cuh"

namespace rsd {

constexpr int DT = 256;  // threads; thread t owns words [4t, 4t+4)

static __device__ __forceinline__ void ld_words(const uint8_t *pool, uint64_t off, int t, uint64_t r[4]) {
  const uint4 *p = (const uint4 *)(pool + off) + 2 * t;
  uint4 x = __ldg(p), y = __ldg(p + 1);
  r[0] = ((uint64_t)x.y << 32) | x.x;
  r[1] = ((uint64_t)x.w << 32) | x.z;
  r[2] = ((uint64_t)y.y << 32) | y.x;
  r[3] = ((uint64_t)y.w << 32) | y.z;
}

static __device__ __forceinline__ void st_words(uint8_t *pool, uint64_t off, int t, const uint64_t r[4]) {
  uint4 *p = (uint4 *)(pool + off) + 2 * t;
  p[0] = make_uint4((uint32_t)r[0], (uint32_t)(r[0] >> 32), (uint32_t)r[1], (uint32_t)(r[1] >> 32));
  p[1] = make_uint4((uint32_t)r[2], (uint32_t)(r[2] >> 32), (uint32_t)r[3], (uint32_t)(r[3] >> 32));
}

// Set the bits of an array or run container into a zeroed smem bitset
// (bitset_from_positions containers.py:113-119, _words_from_runs :122-135).
static __device__ void scatter_container(const DevBatch &S, uint32_t c, uint8_t type, uint64_t *X) {
  const uint16_t *v = (const uint16_t *)(S.pool + S.off[c]);
  uint32_t n = S.n[c];
  uint32_t *X32 = (uint32_t *)X;
  if (type == RS_TAG_ARRAY) {
    // 16-byte vectors (payloads are 16-byte aligned and padded), a thread's
    // two loads issued before its ORs: one DRAM round trip for <= 4096
    // values instead of one per loop iteration
    const uint4 *v4 = (const uint4 *)v;
    const uint32_t nv = (n + 7) >> 3;
    for (uint32_t k0 = threadIdx.x; k0 < nv; k0 += 2 * DT) {
      const uint4 x[2] = {__ldg(v4 + k0), k0 + DT < nv ? __ldg(v4 + k0 + DT) : make_uint4(0, 0, 0, 0)};
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const uint32_t k = k0 + DT * j;
        if (k >= nv) break;
        const uint32_t w[4] = {x[j].x, x[j].y, x[j].z, x[j].w}, left = n - 8 * k;
#pragma unroll
        for (int h = 0; h < 8; h++)
          if ((uint32_t)h < left) {
            const uint32_t val = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
            atomicOr(&X32[val >> 5], 1u << (val & 31));
          }
      }
    }
    return;
  }
  // one thread per run: the (start, length) loads of all runs are independent
  // (a warp walking runs would chain one global load per run); edge words take
  // native 32-bit shared atomics (other runs may share them), interior words
  // belong to this run alone and are plain all-ones stores
  const uint32_t *r32 = (const uint32_t *)v;
  for (uint32_t r = threadIdx.x; r < n; r += DT) {
    const uint32_t sl = r32[r];
    const uint32_t s = sl & 0xFFFF, e = s + (sl >> 16);
    const uint32_t ws = s >> 5, we = e >> 5;  // 32-bit word indices
    const uint32_t first = ~0u << (s & 31), last = ~0u >> (31 - (e & 31));
    if (ws == we) {
      atomicOr(&X32[ws], first & last);
    } else {
      atomicOr(&X32[ws], first);
      atomicOr(&X32[we], last);
      for (uint32_t w = ws + 1; w < we; w++) X32[w] = ~0u;
    }
  }
}

struct DenseSmem {
  uint64_t X[RS_WORDS];
  uint64_t Y[RS_WORDS];
  typename cub::BlockScan<uint32_t, DT>::TempStorage scan;
  uint32_t red[DT / 32][2];
};

static __device__ __forceinline__ void block_sum2(uint32_t &a, uint32_t &b, uint32_t (*red)[2]) {
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[warp][0] = a; red[warp][1] = b; }
  __syncthreads();
  a = 0; b = 0;
#pragma unroll
  for (int w = 0; w < DT / 32; w++) { a += red[w][0]; b += red[w][1]; }
}

// The set bits of word w (bit positions pos + 0..63) written in ascending
// order to out[end - popc(w), end), peeled from the top bit down (FLO on each
// 32-bit half): ~11 instructions per value, half the __ffsll loop's.
static __device__ __forceinline__ void peel_down(uint64_t w, uint32_t pos, uint32_t end, uint16_t *out) {
  uint32_t b = end, hi = (uint32_t)(w >> 32), lo = (uint32_t)w;
  while (hi) {
    const uint32_t p = 31 - __clz(hi);
    out[--b] = (uint16_t)(pos + 32 + p);
    hi ^= 1u << p;
  }
  while (lo) {
    const uint32_t p = 31 - __clz(lo);
    out[--b] = (uint16_t)(pos + p);
    lo ^= 1u << p;
  }
}

// Encode the result set held in r[4] (thread t's words) into the chosen
// container type at dst: bitset words, sorted array (extract_set_bits,
// scalar.py:61-76) or runs (_runs_from_positions, containers.py:138-147).
// Returns the container's n.  X must already hold all words when `is_run`.
static __device__ uint32_t encode_result(DenseSmem &sm, const uint64_t r[4], uint32_t pc, uint32_t card, uint8_t type,
                                  uint8_t *dst) {
  const int t = threadIdx.x;
  if (type == RS_TAG_BITSET) {
    uint4 *p = (uint4 *)dst + 2 * t;
    p[0] = make_uint4((uint32_t)r[0], (uint32_t)(r[0] >> 32), (uint32_t)r[1], (uint32_t)(r[1] >> 32));
    p[1] = make_uint4((uint32_t)r[2], (uint32_t)(r[2] >> 32), (uint32_t)r[3], (uint32_t)(r[3] >> 32));
    return RS_WORDS;
  }
  uint16_t *Y16 = (uint16_t *)sm.Y;
  if (type == RS_TAG_ARRAY) {
    uint32_t base;
    cub::BlockScan<uint32_t, DT>(sm.scan).ExclusiveSum(pc, base);
#pragma unroll
    for (int k = 0; k < 4; k++) {  // each word peeled from its top bit into its slot range
      base += (uint32_t)__popcll(r[k]);
      peel_down(r[k], (uint32_t)(4 * t + k) * 64, base, Y16);
    }
    __syncthreads();
    uint32_t nvec = (uint32_t)(rs_pad16(2ull * card) >> 4);
    if (t < 8 && card + t < nvec * 8) Y16[card + t] = 0;  // zero the 16-byte pad tail
    __syncthreads();
    for (uint32_t i = t; i < nvec; i += DT) ((uint4 *)dst)[i] = ((const uint4 *)Y16)[i];
    return card;
  }
  // runs: starts/ends from the neighbours' boundary bits (X holds all words)
  uint64_t prev = t ? sm.X[4 * t - 1] : 0, next = t < DT - 1 ? sm.X[4 * t + 4] : 0;
  uint64_t S[4], E[4];
  uint32_t ns = 0, ne = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    uint64_t cin = (k ? r[k - 1] : prev) >> 63;
    uint64_t nin = (k < 3 ? r[k + 1] : next) & 1;
    S[k] = r[k] & ~((r[k] << 1) | cin);
    E[k] = r[k] & ~((r[k] >> 1) | (nin << 63));
    ns += __popcll(S[k]);
    ne += __popcll(E[k]);
  }
  uint32_t packed = ns | (ne << 16), base, total;
  cub::BlockScan<uint32_t, DT>(sm.scan).ExclusiveSum(packed, base, total);
  uint32_t bs = base & 0xFFFF, be = base >> 16, nruns = total & 0xFFFF;
  uint16_t *Ys = Y16, *Ye = Y16 + 2048;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    bs += (uint32_t)__popcll(S[k]);
    be += (uint32_t)__popcll(E[k]);
    peel_down(S[k], (uint32_t)(4 * t + k) * 64, bs, Ys);
    peel_down(E[k], (uint32_t)(4 * t + k) * 64, be, Ye);
  }
  __syncthreads();
  uint32_t *d32 = (uint32_t *)dst;
  uint32_t padded = (uint32_t)(rs_pad16(4ull * nruns) >> 2);
  for (uint32_t i = t; i < padded; i += DT)
    d32[i] = i < nruns ? ((uint32_t)Ys[i] | ((uint32_t)(Ye[i] - Ys[i]) << 16)) : 0u;
  return nruns;
}

// The two operands' words, thread t's four: bitset sides straight from the
// pool, array / run sides densified into sm.X (a) / sm.Y (b) first.  GEN =
// false: both sides are known bitsets (no shared memory, no barrier).
template <bool GEN>
static __device__ __forceinline__ void operand_words(const DevBatch &A, uint32_t ca, uint8_t ta, const DevBatch &B,
                                                     uint32_t cb, uint8_t tb, uint64_t *X, uint64_t *Y,
                                                     uint64_t ra[4], uint64_t rb[4]) {
  const int t = threadIdx.x;
  if (!GEN) {
    ld_words(A.pool, A.off[ca], t, ra);
    ld_words(B.pool, B.off[cb], t, rb);
    return;
  }
  const bool da = ta != RS_TAG_BITSET, db = tb != RS_TAG_BITSET;
  // a bitset side's words are requested first: they arrive while the other
  // side is densified
  if (!da) ld_words(A.pool, A.off[ca], t, ra);
  if (!db) ld_words(B.pool, B.off[cb], t, rb);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (da) X[4 * t + k] = 0;
    if (db) Y[4 * t + k] = 0;
  }
  __syncthreads();
  if (da) scatter_container(A, ca, ta, X);
  if (db) scatter_container(B, cb, tb, Y);
  __syncthreads();
  if (da) for (int k = 0; k < 4; k++) ra[k] = X[4 * t + k];
  if (db) for (int k = 0; k < 4; k++) rb[k] = Y[4 * t + k];
}

// container_pairwise(op, a, b) of one matched pair by the whole CTA
// (containers.py:450-529): word op, popcount and run count, the exact
// result-type choice, and the encoded result at dst.
// Returns the cardinality (0: nothing written); type and n of the result.
// Ends with the CTA's shared memory free for reuse.
template <bool GEN>
static __device__ uint32_t dense_pair(int op, const DevBatch &A, uint32_t ca, uint8_t ta, const DevBatch &B,
                                      uint32_t cb, uint8_t tb, DenseSmem &sm, uint8_t *dst, uint8_t &type,
                                      uint32_t &n) {
  const int t = threadIdx.x;
  uint64_t ra[4], rb[4], r[4];
  operand_words<GEN>(A, ca, ta, B, cb, tb, sm.X, sm.Y, ra, rb);
  uint32_t pc = 0, nr = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    r[k] = rs_word_op(op, ra[k], rb[k]);
    pc += __popcll(r[k]);
  }
  const bool consider = GEN && rs_consider_run(ta, tb, op);
  if (consider) {
#pragma unroll
    for (int k = 0; k < 4; k++) sm.X[4 * t + k] = r[k];
    __syncthreads();
    uint64_t prev = t ? sm.X[4 * t - 1] : 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint64_t cin = (k ? r[k - 1] : prev) >> 63;
      nr += __popcll(r[k] & ~((r[k] << 1) | cin));  // _run_count_of_words, containers.py:173-178
    }
  }
  uint32_t card = pc, nruns = nr;
  block_sum2(card, nruns, sm.red);
  if (card == 0) type = RS_TAG_ARRAY;
  else if (consider && rs_run_admissible(card, nruns)) type = RS_TAG_RUN;  // container_normalize
  else type = card <= RS_ARRAY_MAX ? RS_TAG_ARRAY : RS_TAG_BITSET;       // from_words / from_values
  n = 0;
  if (card) {
    __syncthreads();  // smem Y may still be read by the densify phase
    n = encode_result(sm, r, pc, card, type, dst);
  }
  __syncthreads();  // smem reuse by the caller's next pair
  return card;
}

// |a AND b| of one matched pair by the whole CTA (the count path); the
// block total is returned on every thread.
template <bool GEN>
static __device__ uint32_t dense_and_count(const DevBatch &A, uint32_t ca, uint8_t ta, const DevBatch &B,
                                           uint32_t cb, uint8_t tb, uint64_t *X, uint64_t *Y, uint32_t (*red)[2]) {
  uint64_t ra[4], rb[4];
  operand_words<GEN>(A, ca, ta, B, cb, tb, X, Y, ra, rb);
  uint32_t pc = 0, z = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) pc += __popcll(ra[k] & rb[k]);
  block_sum2(pc, z, red);
  __syncthreads();  // smem reuse
  return pc;
}


}  // namespace rsd
