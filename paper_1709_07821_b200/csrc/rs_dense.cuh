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
    for (uint32_t i = threadIdx.x; i < n; i += DT) atomicOr(&X32[v[i] >> 5], 1u << (v[i] & 31));
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
    for (int k = 0; k < 4; k++) {
      uint64_t w = r[k];
      while (w) {
        Y16[base++] = (uint16_t)((4 * t + k) * 64 + __ffsll((long long)w) - 1);
        w &= w - 1;
      }
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
    uint64_t w = S[k];
    while (w) { Ys[bs++] = (uint16_t)((4 * t + k) * 64 + __ffsll((long long)w) - 1); w &= w - 1; }
    w = E[k];
    while (w) { Ye[be++] = (uint16_t)((4 * t + k) * 64 + __ffsll((long long)w) - 1); w &= w - 1; }
  }
  __syncthreads();
  uint32_t *d32 = (uint32_t *)dst;
  uint32_t padded = (uint32_t)(rs_pad16(4ull * nruns) >> 2);
  for (uint32_t i = t; i < padded; i += DT)
    d32[i] = i < nruns ? ((uint32_t)Ys[i] | ((uint32_t)(Ye[i] - Ys[i]) << 16)) : 0u;
  return nruns;
}


}  // namespace rsd
