// rs_pairwise.cu -- the hot path: batched RoaringBitmap.op / op_cardinality
// (bitmap.py:169-241) and container_pairwise[_cardinality]
// (containers.py:450-570) over flattened device batches.
//
// Pipeline of one materialized batched op:
//   k_pair_msize + scan      merged key-space size per bitmap pair
//   k_merge                  merge-path join of the sorted u16 key arrays: one
//                            thread per key, a binary search in the other side
//                            gives its merged position and its match
//   scans (keep, ub)         entry slot and upper-bound payload slot per output
//   k_emit                   entry records + per-type-pair work lists
//   per-class kernels        bitset x bitset (k_pair_dense<false>),
//                            array x array (k_aa_merge),
//                            everything else (k_pair_dense<true>: densify to
//                            8 KB in smem, word op, popcount + run count,
//                            exact result-type choice, encode), copies (k_copy)
//   compaction               drop empty results, per-bitmap container ranges
#include <cub/cub.cuh>
#include <algorithm>
#include <mutex>
#include "rs_internal.cuh"
#include "rs_dense.cuh"
#include "rs_array.cuh"
#include "rs_bitset.cuh"
#include "rs_array_large.cuh"
#include "rs_single.h"

using namespace rs;

namespace {

enum { CLS_COPY = 0, CLS_BB = 1, CLS_AAS = 2, CLS_AAM = 3, CLS_AAL = 4, CLS_GEN = 5, CLS_PRB = 6, CLS_AAG = 7, NCLS = 8 };
// counters after the class sizes: [NCLS, NCLS + 1] fused-scan arrivals,
// [CNT_LARGE], [CNT_GEN] the large-pair and generic-pair kernels' dynamic
// item counters (all zeroed per op)
constexpr int CNT_LARGE = NCLS + 2, CNT_GEN = NCLS + 3;

struct Entries {
  uint16_t *key;
  uint32_t *ca, *cb, *pair;
  uint64_t *off;
};

struct OutDesc {
  uint8_t *type;
  uint32_t *card, *n;
};

struct Lists {
  uint32_t *list[NCLS];
  uint32_t *cnt;           // device counters [NCLS]
  uint64_t *aoff, *boff;   // TMA-fed classes (bitset x bitset, large array x array): operand payload offsets
  uint32_t *nab;           // large array x array: na | nb << 16
  uint64_t cap;
};

__device__ __forceinline__ bool tma_class(int c) { return c == 1 /*CLS_BB*/ || c == 4 /*CLS_AAL*/; }

__device__ __forceinline__ uint32_t pair_a(const uint32_t *ia, uint64_t p) { return ia ? ia[p] : (uint32_t)p; }

// array x array size classes: <= 256 merged items -> small-pair kernel; up to
// the op's medium bound -> a warp merge path per pair (16 items per lane);
// above -> smem-bitset kernel.  Measured on C3: for AND / ANDNOT (and the
// counts) the bitset kernel -- its filter needs no result sweep, and very
// unequal AND pairs binary-search -- wins for everything above 256
// (RS_AA_LARGE_MIN); for OR / XOR the warp merge path wins up to 512 items
// (RS_AA_UNION_MEDIUM; OR 2.07 -> 1.93 ms, XOR 2.07 -> 1.99 ms).
__constant__ uint32_t c_aa_large_min = 256;
__constant__ uint32_t c_aa_union_medium = 512;
// Galloping pairs of the COUNT path go to the large-pair kernel, which
// binary-searches the small side's values in the staged large side (shared
// memory; the bytes stream in with the TMA) instead of the warp-per-pair
// in-place search over HBM: C3 counts 0.84 -> 0.79 ms.  The op path does the
// same for AND pairs of at most 64 searches, which one warp of the large-pair
// kernel's group handles without a group barrier (rs_array_large.cuh): run
// as its own kernel, the galloping class waited for the persistent
// large-pair CTAs to leave the SMs, so C3 AND paid its 0.24 ms in full after
// them.  Longer small sides keep the warp kernel (the 128-thread form costs
// ~950 warp instructions per pair).  RS_GALLOP_TMA: bit 0 = counts, bit 1 =
// ops (both on by default).
__constant__ uint32_t c_gallop_tma = 3;

// `op` is the materialized op, or AND for the intersection counts.  An
// array against a bitset or runs under AND (either side), or an array minus a
// bitset or runs, keeps a subset of the array: bit / interval probes of its
// values (CLS_PRB) instead of densifying both sides.
// Array x array pairs past the small class whose AND (or ANDNOT, small A)
// keeps a subset of a side at most 1/16 of the other's size go to the
// galloping class: a warp per pair binary-searches the large side in place
// (array_intersect_galloping's case, kernels/scalar.py:149-176,
// _shared.py:14) -- a CTA-per-pair bitset kernel spent ~900 warp
// instructions per such pair on staging and barriers for <= 256 searches.
__device__ __forceinline__ bool gallop_pair(uint32_t na, uint32_t nb, int op) {
  if (na + nb <= 256) return false;
  if (op == RS_OP_AND) return 16 * min(na, nb) <= max(na, nb);
  return op == RS_OP_ANDNOT && 16 * na <= nb;
}

__device__ __forceinline__ int classify(uint8_t ta, uint32_t na, uint8_t tb, uint32_t nb, int op, bool count = false) {
  if (ta == RS_TAG_BITSET && tb == RS_TAG_BITSET) return CLS_BB;
  if (ta == RS_TAG_ARRAY && tb == RS_TAG_ARRAY && gallop_pair(na, nb, op))
    return (count ? c_gallop_tma & 1u : (c_gallop_tma & 2u) && op == RS_OP_AND && min(na, nb) <= 64u) ? CLS_AAL : CLS_AAG;
  if (ta == RS_TAG_ARRAY && tb == RS_TAG_ARRAY)
    return na + nb <= 256 ? CLS_AAS
           : na + nb <= (op == RS_OP_OR || op == RS_OP_XOR ? c_aa_union_medium : c_aa_large_min) ? CLS_AAM
                                                                                                : CLS_AAL;
  if (op == RS_OP_AND && (ta == RS_TAG_ARRAY || tb == RS_TAG_ARRAY)) return CLS_PRB;
  if (op == RS_OP_ANDNOT && ta == RS_TAG_ARRAY) return CLS_PRB;
  return CLS_GEN;
}

// warp-aggregated append of `item` to list[cls] (returns the slot); bitset x
// bitset items also record their operand payload offsets
__device__ __forceinline__ uint32_t list_append(Lists L, int cls, bool active, uint32_t item, uint64_t aoff = 0,
                                                uint64_t boff = 0, uint32_t nab = 0) {
  unsigned lane = threadIdx.x & 31;
  uint32_t slot = 0;
#pragma unroll
  for (int c = 0; c < NCLS; c++) {
    unsigned m = __ballot_sync(0xffffffffu, active && cls == c);
    if (!m) continue;
    int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)lane == leader) base = atomicAdd(&L.cnt[c], (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (active && cls == c) {
      slot = base + __popc(m & ((1u << lane) - 1));
      L.list[c][slot] = item;
      if (c == CLS_BB) {
        L.aoff[slot] = aoff;
        L.boff[slot] = boff;
      } else if (c == CLS_AAL) {
        L.aoff[L.cap + slot] = aoff;
        L.boff[L.cap + slot] = boff;
        L.nab[slot] = nab;
      }
    }
  }
  return slot;
}

// CTA-aggregated list_append for the one-item-per-thread kernels: every
// thread of the block calls it exactly once.  Warps reserve their slots in
// shared counters and one thread per class takes the CTA's range from the
// global counter -- per-warp global atomics on the eight list counters
// serialized at L2 (k_cont_list: 70 us for 1 M container pairs, issue 13 %,
// all long-scoreboard).
__device__ __forceinline__ uint32_t list_append_cta(Lists L, int cls, bool active, uint32_t item, uint64_t aoff = 0,
                                                    uint64_t boff = 0, uint32_t nab = 0) {
  __shared__ uint32_t s_cnt[NCLS], s_base[NCLS];
  const unsigned lane = threadIdx.x & 31;
  if (threadIdx.x < NCLS) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  uint32_t wslot = 0;
#pragma unroll
  for (int c = 0; c < NCLS; c++) {
    const unsigned m = __ballot_sync(0xffffffffu, active && cls == c);
    if (!m) continue;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)lane == leader) base = atomicAdd(&s_cnt[c], (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (active && cls == c) wslot = base + __popc(m & ((1u << lane) - 1));
  }
  __syncthreads();
  if (threadIdx.x < NCLS) {
    const uint32_t n = s_cnt[threadIdx.x];
    s_base[threadIdx.x] = n ? atomicAdd(&L.cnt[threadIdx.x], n) : 0;
  }
  __syncthreads();
  uint32_t slot = 0;
  if (active) {
    slot = s_base[cls] + wslot;
    L.list[cls][slot] = item;
    if (cls == CLS_BB) {
      L.aoff[slot] = aoff;
      L.boff[slot] = boff;
    } else if (cls == CLS_AAL) {
      L.aoff[L.cap + slot] = aoff;
      L.boff[L.cap + slot] = boff;
      L.nab[slot] = nab;
    }
  }
  return slot;
}

__global__ void k_pair_msize(uint64_t npairs, DevBatch A, DevBatch B, const uint32_t *ia, const uint32_t *ib,
                             int count_mode, uint64_t *__restrict__ msz) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (p > npairs) return;
  if (p == npairs) { msz[p] = 0; return; }
  uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
  uint64_t na = A.bm_start[a + 1] - A.bm_start[a];
  uint64_t nb = B.bm_start[b + 1] - B.bm_start[b];
  msz[p] = count_mode ? na : na + nb;
}

__device__ __forceinline__ uint64_t find_pair(const uint64_t *__restrict__ mbase, uint64_t npairs, uint64_t t) {
  uint64_t lo = 0, hi = npairs;  // largest p with mbase[p] <= t
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (mbase[m] <= t) lo = m; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ uint32_t lower_bound16(const uint16_t *__restrict__ k, uint32_t n, uint16_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t m = (lo + hi) >> 1;
    if (k[m] < x) lo = m + 1; else hi = m;
  }
  return lo;
}
__device__ __forceinline__ uint32_t upper_bound16(const uint16_t *__restrict__ k, uint32_t n, uint16_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t m = (lo + hi) >> 1;
    if (k[m] <= x) lo = m + 1; else hi = m;
  }
  return lo;
}

// Merge-path join (bitmap.py:181-209 two-pointer walk, parallel form): thread
// t owns one key of one side of one pair.  A keys land at i + #(B < key), B
// keys at j + #(A <= key), so a matched B key sits right after its A partner
// and is marked as a duplicate.  keep/ub are written at the merged position.
// One merged position t of pair p (local index l): A's key l, or B's key
// l - na; keys come from kA / kB (global memory or a CTA's smem copy).
__device__ __forceinline__ void merge_position(uint64_t base, uint32_t l, uint32_t p, uint64_t a0, uint64_t b0,
                                               uint32_t na, uint32_t nb, const uint16_t *kA, const uint16_t *kB,
                                               const DevBatch &A, const DevBatch &B, int op, uint16_t *mkey,
                                               uint32_t *mca, uint32_t *mcb, uint32_t *mpair, uint32_t *keep,
                                               uint64_t *ub) {
  const bool keep_a = op != RS_OP_AND;                        // _KEEP_A, bitmap.py:21
  const bool keep_b = op == RS_OP_OR || op == RS_OP_XOR;      // _KEEP_B, bitmap.py:22
  if (l < na) {
    uint16_t key = kA[l];
    uint32_t j = lower_bound16(kB, nb, key);
    bool matched = j < nb && kB[j] == key;
    uint64_t pos = base + l + j;
    uint64_t ca = a0 + l;
    mkey[pos] = key;
    mca[pos] = (uint32_t)ca;
    mcb[pos] = matched ? (uint32_t)(b0 + j) : RS_NONE;
    mpair[pos] = p;
    bool k = matched || keep_a;
    keep[pos] = k;
    uint32_t u = 0;
    if (matched) u = rs_result_ub(A.type[ca], A.card[ca], B.type[b0 + j], B.card[b0 + j], op);
    else if (k) u = rs_payload_bytes(A.type[ca], A.n[ca]);
    ub[pos] = rs_pad16(u);
  } else {
    uint32_t j = l - na;
    uint16_t key = kB[j];
    uint32_t i = upper_bound16(kA, na, key);
    bool matched = i > 0 && kA[i - 1] == key;
    uint64_t pos = base + i + j;
    bool k = !matched && keep_b;
    keep[pos] = k;
    ub[pos] = k ? rs_pad16(rs_payload_bytes(B.type[b0 + j], B.n[b0 + j])) : 0;
    if (k) {
      mkey[pos] = key;
      mca[pos] = RS_NONE;
      mcb[pos] = (uint32_t)(b0 + j);
      mpair[pos] = p;
    }
  }
}

// thread per merged position, keys searched in global memory (any sizes)
__global__ void k_merge(uint64_t M, uint64_t npairs, const uint64_t *__restrict__ mbase, DevBatch A, DevBatch B,
                        const uint32_t *ia, const uint32_t *ib, int op, uint16_t *__restrict__ mkey,
                        uint32_t *__restrict__ mca, uint32_t *__restrict__ mcb, uint32_t *__restrict__ mpair,
                        uint32_t *__restrict__ keep, uint64_t *__restrict__ ub) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t == 0) {  // scan sentinels (the exclusive scans run over M + 1)
    keep[M] = 0;
    ub[M] = 0;
  }
  if (t >= M) return;
  uint64_t p = find_pair(mbase, npairs, t);
  uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
  uint64_t a0 = A.bm_start[a], b0 = B.bm_start[b];
  uint32_t na = (uint32_t)(A.bm_start[a + 1] - a0), nb = (uint32_t)(B.bm_start[b + 1] - b0);
  merge_position(mbase[p], (uint32_t)(t - mbase[p]), (uint32_t)p, a0, b0, na, nb, A.key + a0, B.key + b0, A, B, op,
                 mkey, mca, mcb, mpair, keep, ub);
}

// CTA per pair when every bitmap has at most MERGE_SMEM_KEYS containers: both
// key lists staged in shared memory, so the binary searches of the join hit
// smem instead of chaining global loads (and no search for the pair index)
constexpr uint32_t MERGE_SMEM_KEYS = 2048;
// Scans over pairs fused into the kernel that produces their inputs ("last
// block" pattern): every CTA publishes its per-pair value, fences, and bumps a
// zeroed counter; the CTA that arrives last scans all of them.  Used when the
// pairs fit one CTA's serial chunks (npairs <= FUSED_SCAN_MAX); it removes a
// launch per scan, which is most of a small batch's host time (config 1:
// ~3 us per launch, 10 launches per op).
constexpr uint64_t FUSED_SCAN_MAX = 4096;

__device__ __forceinline__ bool last_block_arrives(uint32_t *done, uint64_t nblocks) {
  __shared__ bool last;
  __syncthreads();  // every thread's writes of this CTA precede the fence below
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == (uint32_t)(nblocks - 1);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// exclusive scan of in[0, n) into out (in[n-1] is the zero sentinel, so
// out[n-1] is the total); one CTA of 256 threads, 256 values per round
template <typename T>
__device__ void block_exclusive_scan(const T *in, T *out, uint64_t n) {
  using BS = cub::BlockScan<T, 256>;
  __shared__ typename BS::TempStorage ts;
  T carry = 0;
  for (uint64_t b0 = 0; b0 < n; b0 += 256) {
    const uint64_t i = b0 + threadIdx.x;
    const T v = i < n ? __ldcg(in + i) : (T)0;  // other CTAs' writes: read through L2
    T ex, agg;
    BS(ts).ExclusiveSum(v, ex, agg);
    if (i < n) out[i] = carry + ex;
    carry += agg;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_merge_pair(uint64_t M, uint64_t npairs, const uint64_t *__restrict__ mbase,
                                                    DevBatch A, DevBatch B, const uint32_t *ia, const uint32_t *ib,
                                                    int op, uint16_t *__restrict__ mkey, uint32_t *__restrict__ mca,
                                                    uint32_t *__restrict__ mcb, uint32_t *__restrict__ mpair,
                                                    uint32_t *__restrict__ keep, uint64_t *__restrict__ ub,
                                                    uint32_t *__restrict__ pk, uint64_t *__restrict__ pu,
                                                    uint32_t *done, uint32_t *pke, uint64_t *pue) {
  __shared__ uint16_t kA[MERGE_SMEM_KEYS], kB[MERGE_SMEM_KEYS];
  __shared__ uint64_t red[8];
  const uint32_t p = blockIdx.x;
  if (p == 0 && threadIdx.x == 0) {
    keep[M] = 0;
    ub[M] = 0;
    pk[npairs] = 0;  // sentinels of the scans over pairs
    pu[npairs] = 0;
  }
  const uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
  const uint64_t a0 = A.bm_start[a], b0 = B.bm_start[b];
  const uint32_t na = (uint32_t)(A.bm_start[a + 1] - a0), nb = (uint32_t)(B.bm_start[b + 1] - b0);
  for (uint32_t i = threadIdx.x; i < na; i += blockDim.x) kA[i] = A.key[a0 + i];
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) kB[i] = B.key[b0 + i];
  __syncthreads();
  const uint64_t base = mbase[p];
  for (uint32_t l = threadIdx.x; l < na + nb; l += blockDim.x)
    merge_position(base, l, p, a0, b0, na, nb, kA, kB, A, B, op, mkey, mca, mcb, mpair, keep, ub);
  // per-pair totals of keep and ub (packed: keep count << 40 | ub bytes)
  __syncthreads();
  uint64_t v = 0;
  for (uint32_t l = threadIdx.x; l < na + nb; l += blockDim.x) v += ((uint64_t)keep[base + l] << 40) + ub[base + l];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int w = 0; w < 8; w++) s += red[w];
    pk[p] = (uint32_t)(s >> 40);
    pu[p] = s & ((1ull << 40) - 1);
  }
  if (done && last_block_arrives(done, npairs)) {  // fused scans over pairs
    block_exclusive_scan<uint32_t>(pk, pke, npairs + 1);
    block_exclusive_scan<uint64_t>(pu, pue, npairs + 1);
  }
}

// The single-pair op (the RoaringBitmap API's a & b, config 1): join and
// emit in ONE CTA -- with one pair its entry and slot bases are 0, so the
// scans over pairs vanish and the join's outputs feed the emit in place.
// pke[0..1] / pue[0..1] get the pair's entry / slot totals for the
// compaction.  (Two launches and a memset fewer per call: host-bound calls
// pay ~3 us per launch.)
template <bool CTA = false>
__device__ __forceinline__ void emit_entry(bool active, uint32_t e, uint64_t off, uint64_t t,
                                           const uint16_t *__restrict__ mkey, const uint32_t *__restrict__ mca,
                                           const uint32_t *__restrict__ mcb, const uint32_t *__restrict__ mpair,
                                           const DevBatch &A, const DevBatch &B, Entries E, Lists L, int op);

__global__ void __launch_bounds__(256) k_merge_emit1(DevBatch A, DevBatch B, const uint32_t *ia, const uint32_t *ib,
                                                     int op, uint16_t *__restrict__ mkey, uint32_t *__restrict__ mca,
                                                     uint32_t *__restrict__ mcb, uint32_t *__restrict__ mpair,
                                                     uint32_t *__restrict__ keep, uint64_t *__restrict__ ub,
                                                     uint32_t *__restrict__ pke, uint64_t *__restrict__ pue,
                                                     Entries E, Lists L) {
  __shared__ uint16_t kA[2048], kB[2048];
  using BS = cub::BlockScan<uint64_t, 256>;
  __shared__ typename BS::TempStorage ts;
  const uint32_t a = pair_a(ia, 0), b = pair_a(ib, 0);
  const uint64_t a0 = A.bm_start[a], b0 = B.bm_start[b];
  const uint32_t na = (uint32_t)(A.bm_start[a + 1] - a0), nb = (uint32_t)(B.bm_start[b + 1] - b0);
  for (uint32_t i = threadIdx.x; i < na; i += blockDim.x) kA[i] = A.key[a0 + i];
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) kB[i] = B.key[b0 + i];
  __syncthreads();
  for (uint32_t l = threadIdx.x; l < na + nb; l += blockDim.x)
    merge_position(0, l, 0, a0, b0, na, nb, kA, kB, A, B, op, mkey, mca, mcb, mpair, keep, ub);
  __syncthreads();  // the join's writes are visible to the whole CTA
  uint32_t ck = 0;
  uint64_t cu = 0;
  for (uint32_t t0 = 0; t0 < na + nb; t0 += blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    const bool in = t < na + nb;
    const uint32_t k = in ? keep[t] : 0;
    const uint64_t v = in ? (((uint64_t)k << 32) | ub[t]) : 0;
    uint64_t ex, tot;
    BS(ts).ExclusiveSum(v, ex, tot);
    emit_entry(in && k, ck + (uint32_t)(ex >> 32), cu + (ex & 0xFFFFFFFFull), t, mkey, mca, mcb, mpair, A, B, E, L,
               op);
    ck += (uint32_t)(tot >> 32);
    cu += tot & 0xFFFFFFFFull;
    __syncthreads();  // ts reuse
  }
  if (threadIdx.x == 0) {
    pke[0] = 0;
    pke[1] = ck;
    pue[0] = 0;
    pue[1] = cu;
  }
}

// One kept merged position becomes entry e with result slot `off`: the
// entry record and its per-type-pair work list (whole warps must call this:
// list_append aggregates with ballots).
template <bool CTA>
__device__ __forceinline__ void emit_entry(bool active, uint32_t e, uint64_t off, uint64_t t,
                                           const uint16_t *__restrict__ mkey, const uint32_t *__restrict__ mca,
                                           const uint32_t *__restrict__ mcb, const uint32_t *__restrict__ mpair,
                                           const DevBatch &A, const DevBatch &B, Entries E, Lists L, int op) {
  int cls = CLS_COPY;
  uint32_t nab = 0;
  uint64_t ao = 0, bo = 0;
  if (active) {
    uint32_t ca = mca[t], cb = mcb[t];
    E.key[e] = mkey[t];
    E.ca[e] = ca;
    E.cb[e] = cb;
    E.pair[e] = mpair[t];
    E.off[e] = off;
    cls = (ca == RS_NONE || cb == RS_NONE) ? CLS_COPY : classify(A.type[ca], A.card[ca], B.type[cb], B.card[cb], op);
    if (tma_class(cls)) {
      ao = A.off[ca];
      bo = B.off[cb];
      nab = A.card[ca] | (B.card[cb] << 16);
    }
  }
  if constexpr (CTA) list_append_cta(L, cls, active, e, ao, bo, nab);
  else list_append(L, cls, active, e, ao, bo, nab);
}

__global__ void k_emit(uint64_t M, const uint32_t *__restrict__ keep, const uint32_t *__restrict__ epos,
                       const uint64_t *__restrict__ uoff, const uint16_t *__restrict__ mkey,
                       const uint32_t *__restrict__ mca, const uint32_t *__restrict__ mcb,
                       const uint32_t *__restrict__ mpair, DevBatch A, DevBatch B, Entries E, Lists L, int op) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const bool active = t < M && keep[t];
  emit_entry<true>(active, active ? epos[t] : 0, active ? uoff[t] : 0, t, mkey, mca, mcb, mpair, A, B, E, L, op);
}

// CTA per pair (the per-pair join path): entry indices and result slots from
// the pair's bases (a scan over pairs) plus a block scan of the pair's own
// positions -- no scan over every merged position.  keep (<= 256 per tile)
// and ub (< 2^23 per tile) share one packed 64-bit block scan.
__global__ void __launch_bounds__(256) k_emit_pair(const uint64_t *__restrict__ mbase, const uint32_t *__restrict__ keep,
                                                   const uint64_t *__restrict__ ub, const uint32_t *__restrict__ pke,
                                                   const uint64_t *__restrict__ pue, const uint16_t *__restrict__ mkey,
                                                   const uint32_t *__restrict__ mca, const uint32_t *__restrict__ mcb,
                                                   const uint32_t *__restrict__ mpair, DevBatch A, DevBatch B, Entries E,
                                                   Lists L, int op) {
  using BS = cub::BlockScan<uint64_t, 256>;
  __shared__ typename BS::TempStorage ts;
  const uint32_t p = blockIdx.x;
  const uint64_t base = mbase[p], end = mbase[p + 1];
  uint32_t ck = pke[p];
  uint64_t cu = pue[p];
  for (uint64_t t0 = base; t0 < end; t0 += blockDim.x) {
    const uint64_t t = t0 + threadIdx.x;
    const bool in = t < end;
    const uint32_t k = in ? keep[t] : 0;
    const uint64_t v = in ? (((uint64_t)k << 32) | ub[t]) : 0;
    uint64_t ex, tot;
    BS(ts).ExclusiveSum(v, ex, tot);
    emit_entry(in && k, ck + (uint32_t)(ex >> 32), cu + (ex & 0xFFFFFFFFull), t, mkey, mca, mcb, mpair, A, B, E, L,
               op);
    ck += (uint32_t)(tot >> 32);
    cu += tot & 0xFFFFFFFFull;
    __syncthreads();  // ts reuse
  }
}



// ----------------------------------------------------------------- copies

// Unmatched containers kept by OR / XOR / ANDNOT are deep-copied
// (Container.copy, bitmap.py:191-209).  One warp per container, persistent
// over the list; the next item's metadata chain (list -> entry -> container)
// is loaded while the current payload streams, and each lane keeps four
// 16-byte loads in flight.
__global__ void k_copy(const uint32_t *__restrict__ list, const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B,
                       Entries E, OutDesc O, uint8_t *__restrict__ opool, uint64_t *__restrict__ res_card) {
  const int lane = threadIdx.x & 31;
  const uint32_t total = *cnt, nw = (gridDim.x * blockDim.x) >> 5;
  struct Item {
    uint32_t e, c;
    bool from_a;
  };
  auto fetch = [&](uint32_t w) {
    Item it;
    it.e = list[w];
    const uint32_t ca = E.ca[it.e];
    it.from_a = ca != RS_NONE;
    it.c = it.from_a ? ca : E.cb[it.e];
    return it;
  };
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= total) return;
  Item cur = fetch(w);
  for (; w < total; w += nw) {
    if (cur.c == RS_NONE) {  // container-level op with an empty result (nothing kept)
      if (lane == 0) {
        O.type[cur.e] = RS_TAG_ARRAY;
        O.card[cur.e] = 0;
        O.n[cur.e] = 0;
      }
      if (w + nw < total) cur = fetch(w + nw);
      continue;
    }
    const DevBatch &S = cur.from_a ? A : B;
    const uint8_t t = S.type[cur.c];
    const uint32_t n = S.n[cur.c], card = S.card[cur.c];
    const uint4 *src = (const uint4 *)(S.pool + S.off[cur.c]);
    uint4 *dst = (uint4 *)(opool + E.off[cur.e]);
    const uint32_t e = cur.e;
    if (w + nw < total) cur = fetch(w + nw);
    const uint32_t nv = (uint32_t)(rs_pad16(rs_payload_bytes(t, n)) >> 4);
    // rounds of 8 predicated 16-byte loads per lane (4 KB per warp), all
    // issued before any store: a typical container is one round trip (a
    // remainder loop of one load -> store per step made it two or three)
    for (uint32_t i0 = 0; i0 < nv; i0 += 256) {
      uint4 x[8];
#pragma unroll
      for (int k = 0; k < 8; k++)
        if (i0 + lane + 32 * k < nv) x[k] = __ldcs(src + i0 + lane + 32 * k);
#pragma unroll
      for (int k = 0; k < 8; k++)
        if (i0 + lane + 32 * k < nv) __stcs(dst + i0 + lane + 32 * k, x[k]);
    }
    if (lane == 0) {
      O.type[e] = t;
      O.card[e] = card;
      O.n[e] = n;
      atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)card);
    }
  }
}

// ------------------------------------------------- dense (8 KB) pair kernel

using namespace rsd;

// Materialized pair op over a work list.  GEN=false: bitset x bitset only
// (bitset_op_with_count + _container_from_words, containers.py:463-465).
// GEN=true: any matched pair; array/run sides are densified in smem first.
// ctr (zero at launch; nullptr: static stride) hands out items dynamically:
// this kernel runs beside the other classes' kernels, and a CTA that found
// no free SM slot until they finished took a full static share late.
template <bool GEN>
__global__ void __launch_bounds__(DT, 4) k_pair_dense(int op, const uint32_t *__restrict__ list,
                                                   const uint32_t *__restrict__ cnt, uint32_t *ctr, DevBatch A,
                                                   DevBatch B, Entries E, OutDesc O, uint8_t *__restrict__ opool,
                                                   uint64_t *__restrict__ res_card) {
  __shared__ __align__(16) DenseSmem sm;
  __shared__ uint32_t s_init[2], s_take[2];
  const int t = threadIdx.x;
  const uint32_t total = *cnt;
  // the next item's metadata chain (list -> entry -> containers) is loaded
  // while the current item is processed: it is off the critical path
  struct Item {
    uint32_t e, ca, cb;
    uint8_t ta, tb;
  };
  auto fetch = [&](uint32_t item) {
    Item m;
    m.e = list[item];
    m.ca = E.ca[m.e];
    m.cb = E.cb[m.e];
    m.ta = GEN ? A.type[m.ca] : (uint8_t)RS_TAG_BITSET;
    m.tb = GEN ? B.type[m.cb] : (uint8_t)RS_TAG_BITSET;
    return m;
  };
  uint32_t item = blockIdx.x, next = blockIdx.x + gridDim.x;
  if (ctr) {
    if (t == 0) {
      s_init[0] = atomicAdd(ctr, 1u);
      s_init[1] = atomicAdd(ctr, 1u);
    }
    __syncthreads();
    item = s_init[0];
    next = s_init[1];
  }
  Item nxt;
  if (item < total) nxt = fetch(item);
  for (int par = 0; item < total; par ^= 1) {
    const Item cur = nxt;
    if (next < total) nxt = fetch(next);
    if (ctr && t == 0) s_take[par] = atomicAdd(ctr, 1u);  // the item after next (read behind dense_pair's barriers)
    const uint32_t e = cur.e;
    uint8_t type;
    uint32_t n;
    const uint32_t card = dense_pair<GEN>(op, A, cur.ca, cur.ta, B, cur.cb, cur.tb, sm, opool + E.off[e], type, n);
    if (t == 0) {
      O.type[e] = type;
      O.card[e] = card;
      O.n[e] = n;
      if (card) atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)card);
    }
    item = next;
    next = ctr ? s_take[par] : next + gridDim.x;
  }
}

// Count-only: |a AND b| accumulated per bitmap pair (container_pairwise_cardinality
// "and", bitmap.py:225-234).  Persistent over the device-sized work list.
template <bool GEN>
__global__ void __launch_bounds__(DT) k_pair_count(int op, const uint32_t *__restrict__ lca, const uint32_t *__restrict__ lcb,
                                                   const uint32_t *__restrict__ lpair, const uint32_t *__restrict__ cnt,
                                                   DevBatch A, DevBatch B, uint64_t *__restrict__ acc) {
  __shared__ __align__(16) uint64_t X[RS_WORDS];
  __shared__ __align__(16) uint64_t Y[RS_WORDS];
  __shared__ uint32_t red[DT / 32][2];
  const int t = threadIdx.x;
  const uint32_t total = *cnt;
  for (uint32_t i = blockIdx.x; i < total; i += gridDim.x) {
    const uint32_t ca = lca[i], cb = lcb[i];
    const uint8_t ta = GEN ? A.type[ca] : (uint8_t)RS_TAG_BITSET, tb = GEN ? B.type[cb] : (uint8_t)RS_TAG_BITSET;
    const uint32_t pc = dense_and_count<GEN>(A, ca, ta, B, cb, tb, X, Y, red);
    if (t == 0 && pc) atomicAdd((unsigned long long *)&acc[lpair[i]], (unsigned long long)pc);
  }
}

// ------------------------------------- bitset x bitset, persistent + TMA ring

template <int STAGES>
__global__ void __launch_bounds__(rsb::BT) k_bb_op(int op, const uint32_t *__restrict__ list,
                                                    const uint64_t *__restrict__ laoff, const uint64_t *__restrict__ lboff,
                                                    const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B, Entries E, OutDesc O,
                                                    uint8_t *__restrict__ opool, uint64_t *__restrict__ res_card) {
  extern __shared__ __align__(128) uint8_t smraw[];
  auto &sm = *reinterpret_cast<rsb::BBSmem<STAGES> *>(smraw);
  auto src = [&](uint32_t i, const uint8_t *&pa, const uint8_t *&pb) {
    pa = A.pool + laoff[i];
    pb = B.pool + lboff[i];
  };
  struct Meta {
    uint32_t e, pair;
    uint64_t off;
  };
  auto pre = [&](uint32_t i) {
    Meta m;
    m.e = list[i];
    m.off = E.off[m.e];
    m.pair = E.pair[m.e];
    return m;
  };
  auto sink = [&](const Meta &m, const uint64_t *r, uint32_t pk0, uint32_t pk1, uint32_t card,
                  const uint32_t (*red)[rsb::BT / 32]) {
    const uint32_t n = rsb::bb_encode<STAGES>(sm, r, pk0, pk1, card, opool + m.off, red);
    if (threadIdx.x == 0) {
      O.type[m.e] = card > RS_ARRAY_MAX ? RS_TAG_BITSET : RS_TAG_ARRAY;
      O.card[m.e] = card;
      O.n[m.e] = n;
      if (card) atomicAdd((unsigned long long *)&res_card[m.pair], (unsigned long long)card);
    }
  };
  rsb::bb_loop<STAGES>(sm, *cnt, op, src, pre, sink);
}

template <int STAGES>
__global__ void __launch_bounds__(rsb::BT) k_bb_count(int op, const uint64_t *__restrict__ laoff,
                                                       const uint64_t *__restrict__ lboff, const uint32_t *__restrict__ lpair,
                                                       const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B,
                                                       uint64_t *__restrict__ acc) {
  extern __shared__ __align__(128) uint8_t smraw[];
  auto &sm = *reinterpret_cast<rsb::BBSmem<STAGES> *>(smraw);
  auto src = [&](uint32_t i, const uint8_t *&pa, const uint8_t *&pb) {
    pa = A.pool + laoff[i];
    pb = B.pool + lboff[i];
  };
  auto pre = [&](uint32_t i) { return lpair[i]; };
  auto sink = [&](uint32_t pair, const uint64_t *, uint32_t, uint32_t, uint32_t card, const uint32_t (*)[rsb::BT / 32]) {
    if (threadIdx.x == 0 && card) atomicAdd((unsigned long long *)&acc[pair], (unsigned long long)card);
  };
  rsb::bb_loop<STAGES>(sm, *cnt, op, src, pre, sink);
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// RS_BB_KERNEL=dense selects the register-fed kernels (A/B testing);
// RS_BB_STAGES picks the TMA ring depth (2, 3 or 4).
int bb_kernel_choice() {
  static int choice = -1;
  if (choice < 0) {
    const char *v = getenv("RS_BB_KERNEL");
    choice = (v && std::string(v) == "dense") ? 0 : 1;
  }
  return choice;
}

int bb_stages() {
  static int s = -1;
  if (s < 0) {
    s = env_int("RS_BB_STAGES", 2);
    if (s < 2 || s > 4) s = 2;
  }
  return s;
}

inline int env_int_(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
template <typename K>
unsigned persistent_grid(K kernel, size_t smem, uint64_t count, int want_per_sm = 4) {
  int sms = 148;
  int per = occupancy_per_sm((const void *)kernel, rsb::BT, smem, &sms);
  // 4 CTAs per SM (of the 5 that fit) measured best for the streaming bitset
  // kernels (OR/ANDNOT/XOR and the counts: C2 step 7.18 -> 6.96 ms, op kernel
  // 5.95 -> 6.21 TB/s, count 6.99 -> 7.08 TB/s -- fewer concurrent 8 KB
  // streams per SM); AND, whose array extraction is instruction-heavy, keeps
  // 5.  RS_BB_CTAS overrides both.
  static const int env_cap = env_int_("RS_BB_CTAS", 0);
  const int cap = env_cap > 0 ? env_cap : want_per_sm;
  if (cap > 0 && cap < per) per = cap;
  uint64_t g = (uint64_t)sms * (per > 0 ? per : 1);
  return (unsigned)(count < g ? count : g);
}

template <int S>
int launch_bb_op(int op, const Lists &L, uint64_t count, DevBatch dA, DevBatch dB, Entries En, OutDesc O,
                 uint8_t *pool, uint64_t *res_card) {
  const size_t smem = sizeof(rsb::BBSmem<S>);
  static bool attr = false;
  if (!attr) {
    RS_CK(cudaFuncSetAttribute(k_bb_op<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  RS_LAUNCH_PROF("bitset_pair", 0, k_bb_op<S>, persistent_grid(k_bb_op<S>, smem, count, op == RS_OP_AND ? 5 : 4), rsb::BT, smem, op,
                 L.list[CLS_BB], L.aoff, L.boff, L.cnt + CLS_BB, dA, dB, En, O, pool, res_card);
  return RS_OK;
}

template <int S>
int launch_bb_count(int op, const Lists &L, uint32_t *lpair, DevBatch dA, DevBatch dB, uint64_t *inter) {
  const size_t smem = sizeof(rsb::BBSmem<S>);
  static bool attr = false;
  if (!attr) {
    RS_CK(cudaFuncSetAttribute(k_bb_count<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  RS_LAUNCH_PROF("bitset_count", 0, k_bb_count<S>, persistent_grid(k_bb_count<S>, smem, L.cap), rsb::BT, smem, op,
                 L.aoff, L.boff, lpair, L.cnt + CLS_BB, dA, dB, inter);
  return RS_OK;
}

// ------------------------------------ large array x array (smem bitset + TMA)

template <int OP>
__global__ void __launch_bounds__(rsl::LTHREADS, rsl::large_min_blocks(OP)) k_aa_large_op(const uint32_t *__restrict__ list,
                                                               const uint64_t *__restrict__ laoff,
                                                               const uint64_t *__restrict__ lboff,
                                                               const uint32_t *__restrict__ lnab,
                                                               const uint32_t *__restrict__ cnt, uint32_t *ctr,
                                                               DevBatch A, DevBatch B, Entries E, OutDesc O,
                                                               uint8_t *__restrict__ opool,
                                                               uint64_t *__restrict__ res_card) {
  extern __shared__ __align__(128) uint8_t smraw[];
  auto meta_of = [&](uint32_t i, uint64_t &ao, uint64_t &bo) {
    rsl::LargeMeta m;
    ao = laoff[i];
    bo = lboff[i];
    const uint32_t x = lnab[i];
    m.na = x & 0xFFFF;
    m.nb = x >> 16;
    m.e = list[i];
    m.dst = E.off[m.e];
    m.pair = E.pair[m.e];
    return m;
  };
  auto sink = [&](const rsl::LargeMeta &m, uint32_t card, uint8_t type, uint32_t n) {  // one thread per pair
    O.type[m.e] = type;
    O.card[m.e] = card;
    O.n[m.e] = n;
    if (card) atomicAdd((unsigned long long *)&res_card[m.pair], (unsigned long long)card);
  };
  rsl::large_loop<OP, false>(smraw, *cnt, ctr, A.pool, B.pool, opool, meta_of, sink);
}

__global__ void __launch_bounds__(rsl::LTHREADS, rsl::large_min_blocks(-1)) k_aa_large_count(const uint64_t *__restrict__ laoff,
                                                                  const uint64_t *__restrict__ lboff,
                                                                  const uint32_t *__restrict__ lnab,
                                                                  const uint32_t *__restrict__ lpair,
                                                                  const uint32_t *__restrict__ cnt, uint32_t *ctr,
                                                                  DevBatch A, DevBatch B, uint64_t *__restrict__ acc) {
  extern __shared__ __align__(128) uint8_t smraw[];
  auto meta_of = [&](uint32_t i, uint64_t &ao, uint64_t &bo) {
    rsl::LargeMeta m;
    ao = laoff[i];
    bo = lboff[i];
    const uint32_t x = lnab[i];
    m.na = x & 0xFFFF;
    m.nb = x >> 16;
    m.e = i;
    m.dst = 0;
    m.pair = lpair[i];
    return m;
  };
  auto sink = [&](const rsl::LargeMeta &m, uint32_t card, uint8_t, uint32_t) {
    if (card) atomicAdd((unsigned long long *)&acc[m.pair], (unsigned long long)card);  // one thread per pair
  };
  rsl::large_loop<RS_OP_AND, true>(smraw, *cnt, ctr, A.pool, B.pool, nullptr, meta_of, sink);
}

template <typename K>
unsigned persistent_grid_t(K kernel, int threads, size_t smem, uint64_t count) {
  int sms = 148;
  int per = occupancy_per_sm((const void *)kernel, threads, smem, &sms);
  static const int cap = env_int_("RS_AAL_CTAS", 0);  // CTAs per SM cap (tuning)
  if (cap > 0 && cap < per) per = cap;
  uint64_t g = (uint64_t)sms * (per > 0 ? per : 1);
  return (unsigned)(count < g ? count : g);
}

template <int OP>
int launch_aa_large_op_t(const Lists &L, uint64_t n, DevBatch dA, DevBatch dB, Entries En, OutDesc O, uint8_t *pool,
                         uint64_t *res_card, bool exact) {
  const size_t smem = rsl::large_smem_bytes(OP, false);
  static bool attr = false;
  if (!attr) {
    RS_CK(cudaFuncSetAttribute(k_aa_large_op<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  RS_LAUNCH_PROF("array_pair_l", exact ? n : 0, k_aa_large_op<OP>,
                 persistent_grid_t(k_aa_large_op<OP>, rsl::LTHREADS, smem, n), rsl::LTHREADS, smem, L.list[CLS_AAL],
                 L.aoff + L.cap, L.boff + L.cap, L.nab, L.cnt + CLS_AAL, L.cnt + CNT_LARGE, dA, dB, En, O, pool,
                 res_card);
  return RS_OK;
}

int launch_aa_large_op(int op, const Lists &L, uint64_t n, DevBatch dA, DevBatch dB, Entries En, OutDesc O,
                       uint8_t *pool, uint64_t *res_card, bool exact) {
  switch (op) {  // one instantiation per op: no per-value op tests in the kernel
    case RS_OP_AND: return launch_aa_large_op_t<RS_OP_AND>(L, n, dA, dB, En, O, pool, res_card, exact);
    case RS_OP_OR: return launch_aa_large_op_t<RS_OP_OR>(L, n, dA, dB, En, O, pool, res_card, exact);
    case RS_OP_ANDNOT: return launch_aa_large_op_t<RS_OP_ANDNOT>(L, n, dA, dB, En, O, pool, res_card, exact);
    default: return launch_aa_large_op_t<RS_OP_XOR>(L, n, dA, dB, En, O, pool, res_card, exact);
  }
}

int launch_aa_large_count(const Lists &L, uint32_t *lpair, DevBatch dA, DevBatch dB, uint64_t *inter) {
  const size_t smem = rsl::large_smem_bytes(RS_OP_AND, true);
  static bool attr = false;
  if (!attr) {
    RS_CK(cudaFuncSetAttribute(k_aa_large_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  RS_LAUNCH_PROF("array_count_l", 0, k_aa_large_count,
                 persistent_grid_t(k_aa_large_count, rsl::LTHREADS, smem, L.cap), rsl::LTHREADS, smem,
                 L.aoff + L.cap, L.boff + L.cap, L.nab, lpair, L.cnt + CLS_AAL, L.cnt + CNT_LARGE, dA, dB, inter);
  return RS_OK;
}

// ---------------------------------------- array x {bitset, runs}: probes
//
// array AND {bitset, runs} (either side) and array ANDNOT {bitset, runs}: the
// result is the subset of the array's values that are (not) members of the
// other container -- already sorted, always an array (App. A) -- so only the
// other side is materialized: one warp per pair copies the bitset (or sets the
// runs' bits) into a warp-private 8 KB shared-memory bitset, then its lanes
// bit-test 32 array values at a time (_bitset_probe containers.py:181-186,
// _values_in_runs :189-197) and a ballot compacts the kept ones into
// consecutive output slots.  No extraction, no block barriers.
constexpr int PRB_WARPS = 4;

__device__ __forceinline__ void warp_load_member_set(uint64_t *W, uint8_t type, const uint8_t *payload, uint32_t n,
                                                      int lane) {
  if (type == RS_TAG_BITSET) {
    const uint4 *src = (const uint4 *)payload;
    uint4 *dst = (uint4 *)W;
#pragma unroll 4
    for (int k = lane; k < RS_WORDS / 2; k += 32) dst[k] = src[k];
  } else {
    for (int k = lane; k < RS_WORDS; k += 32) W[k] = 0;
    __syncwarp();
    uint32_t *W32 = (uint32_t *)W;
    const uint32_t *r32 = (const uint32_t *)payload;
    for (uint32_t r = lane; r < n; r += 32) {
      const uint32_t sl = r32[r];
      const uint32_t s = sl & 0xFFFF, e = s + (sl >> 16);
      const uint32_t ws = s >> 5, we = e >> 5;
      const uint32_t first = ~0u << (s & 31), last = ~0u >> (31 - (e & 31));
      if (ws == we) {
        atomicOr(&W32[ws], first & last);
      } else {
        atomicOr(&W32[ws], first);
        atomicOr(&W32[we], last);
        for (uint32_t w = ws + 1; w < we; w++) W32[w] = ~0u;
      }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * PRB_WARPS) k_probe(int op, const uint32_t *__restrict__ list,
                                                          const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B,
                                                          Entries E, OutDesc O, uint8_t *__restrict__ opool,
                                                          uint64_t *__restrict__ res_card) {
  __shared__ __align__(16) uint64_t Xs[PRB_WARPS][RS_WORDS];
  const int lane = threadIdx.x & 31;
  uint64_t *W = Xs[threadIdx.x >> 5];
  const uint32_t total = *cnt, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nw) {
    const uint32_t e = list[i], ca = E.ca[e], cb = E.cb[e];
    const bool from_a = op != RS_OP_AND || A.type[ca] == RS_TAG_ARRAY;  // the array side
    const DevBatch &V = from_a ? A : B, &X = from_a ? B : A;
    const uint32_t cv = from_a ? ca : cb, cx = from_a ? cb : ca;
    const uint16_t *vals = (const uint16_t *)(V.pool + V.off[cv]);
    const uint32_t n = V.n[cv];
    // a bitset is probed where it lies (independent 64-bit loads, mostly L2
    // hits); runs are first set into the warp's smem bitset
    const uint8_t xt = X.type[cx];
    const uint64_t *M = xt == RS_TAG_BITSET ? (const uint64_t *)(X.pool + X.off[cx]) : W;
    if (xt != RS_TAG_BITSET) warp_load_member_set(W, xt, X.pool + X.off[cx], X.n[cx], lane);
    const uint32_t want = op == RS_OP_AND ? 1u : 0u;
    uint16_t *out = (uint16_t *)(opool + E.off[e]);
    // 512 values per round: lane l takes [512c + 8l, +8) and [512c + 256 +
    // 8l, +8) with two 16-byte loads (payloads are 16-byte aligned and
    // zero-padded), the next round's loads issued before this round's 16
    // probes, so a round costs one probe round trip (4096 values: 8, against
    // 32 dependent round trips at 256 values with in-round value loads).  A
    // warp scan of the packed per-lane kept counts (first half | second half
    // << 16) keeps the output in value order.
    uint32_t base = 0;
    auto ld = [&](uint32_t j) { return j < n ? *(const uint4 *)(vals + j) : make_uint4(0, 0, 0, 0); };
    uint4 n0 = ld(8 * lane), n1 = ld(256 + 8 * lane);
    for (uint32_t c0 = 0; c0 < n; c0 += 512) {
      const uint32_t j0 = c0 + 8 * lane, j1 = j0 + 256;
      const uint32_t w[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
      n0 = ld(j0 + 512);
      n1 = ld(j1 + 512);
      uint32_t keepm = 0;
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const uint32_t v = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFF;
        if ((k < 8 ? j0 + k : j1 + k - 8) < n && ((M[v >> 6] >> (v & 63)) & 1) == want) keepm |= 1u << k;
      }
      const uint32_t c = __popc(keepm & 0xFFu) | (__popc(keepm >> 8) << 16);
      uint32_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, x, 31), ex = x - c;
      uint32_t p0 = base + (ex & 0xFFFFu), p1 = base + (tot & 0xFFFFu) + (ex >> 16);
#pragma unroll
      for (int k = 0; k < 16; k++)
        if (keepm >> k & 1) out[k < 8 ? p0++ : p1++] = (uint16_t)((w[k >> 1] >> (16 * (k & 1))) & 0xFFFF);
      base += (tot & 0xFFFFu) + (tot >> 16);
    }
    const uint32_t padded = (uint32_t)(rs_pad16(2ull * base) >> 1);
    for (uint32_t k = base + lane; k < padded; k += 32) out[k] = 0;
    if (lane == 0) {
      O.type[e] = RS_TAG_ARRAY;
      O.card[e] = base;
      O.n[e] = base;
      if (base) atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)base);
    }
    __syncwarp();  // W is rebuilt for the next pair
  }
}

// |array AND {bitset, runs}| for the counts: the same probes, counted
__global__ void __launch_bounds__(32 * PRB_WARPS) k_probe_count(const uint32_t *__restrict__ lca,
                                                                const uint32_t *__restrict__ lcb,
                                                                const uint32_t *__restrict__ lpair,
                                                                const uint32_t *__restrict__ cnt, DevBatch A,
                                                                DevBatch B, uint64_t *__restrict__ acc) {
  __shared__ __align__(16) uint64_t Xs[PRB_WARPS][RS_WORDS];
  const int lane = threadIdx.x & 31;
  uint64_t *W = Xs[threadIdx.x >> 5];
  const uint32_t total = *cnt, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nw) {
    const uint32_t ca = lca[i], cb = lcb[i];
    const bool from_a = A.type[ca] == RS_TAG_ARRAY;
    const DevBatch &V = from_a ? A : B, &X = from_a ? B : A;
    const uint32_t cv = from_a ? ca : cb, cx = from_a ? cb : ca;
    const uint16_t *vals = (const uint16_t *)(V.pool + V.off[cv]);
    const uint32_t n = V.n[cv];
    const uint8_t xt = X.type[cx];
    const uint64_t *M = xt == RS_TAG_BITSET ? (const uint64_t *)(X.pool + X.off[cx]) : W;
    if (xt != RS_TAG_BITSET) warp_load_member_set(W, xt, X.pool + X.off[cx], X.n[cx], lane);
    uint32_t c = 0;
    // (the rounds of k_probe: 512 values, the next round's loads in flight)
    auto ld = [&](uint32_t j) { return j < n ? *(const uint4 *)(vals + j) : make_uint4(0, 0, 0, 0); };
    uint4 n0 = ld(8 * lane), n1 = ld(256 + 8 * lane);
    for (uint32_t j0 = 8 * lane; j0 - 8 * lane < n; j0 += 512) {
      const uint32_t w[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
      n0 = ld(j0 + 512);
      n1 = ld(j0 + 768);
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const uint32_t v = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFF;
        c += (k < 8 ? j0 + k : j0 + 248 + k) < n ? (uint32_t)((M[v >> 6] >> (v & 63)) & 1) : 0u;
      }
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0 && c) atomicAdd((unsigned long long *)&acc[lpair[i]], (unsigned long long)c);
    __syncwarp();
  }
}

// ------------------------------------------------- array x array (merge path)

// Materialized array x array pairs: one group of GT threads per pair
// (array_intersect/union/difference/xor + _container_from_values).
// Small array x array pairs (na + nb <= 256), 32 list items per warp at a
// time: a lane takes item (batch + lane) alone when it is tiny (na + nb <=
// c_aa_tiny: a scalar two-pointer merge, ~10 thread instructions per value,
// 32 pairs per warp instruction), and the warp then runs the merge path on
// the batch's remaining items one by one.  Config 3's Zipf sizes make ~85 %
// of the small pairs tiny; the warp-per-pair kernel spent ~350 warp
// instructions on each of them whatever its size.
__constant__ uint32_t c_aa_tiny = 64;

template <int op>
__global__ void __launch_bounds__(256) k_aa_small(const uint32_t *__restrict__ list,
                                                  const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B, Entries E,
                                                  OutDesc O, uint8_t *__restrict__ opool,
                                                  uint64_t *__restrict__ res_card) {
  __shared__ __align__(16) rsa::AASmem<32, 8> sm[8];
  const int gid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t total = *cnt, tiny = c_aa_tiny;
  // A long list is cut into 32 consecutive items per warp (coalesced list /
  // entry loads); a short one (fewer than 32 per warp) is strided so that it
  // still spreads over every warp: warp w owns w, w + W, w + 2W, ...
  const uint32_t W = gridDim.x * 8, gw = blockIdx.x * 8 + gid;
  const bool wide = total >= 32u * W;
  const uint32_t first = wide ? 32 * gw : gw, lstep = wide ? 1u : W;
  for (uint32_t b0 = first; b0 < total; b0 += 32 * W) {
    const uint32_t it = b0 + lane * lstep;
    const bool valid = it < total;
    uint32_t e = 0, ca = 0, cb = 0, na = 0, nb = 0;
    if (valid) {
      e = list[it];
      ca = E.ca[e];
      cb = E.cb[e];
      na = A.card[ca];
      nb = B.card[cb];
    }
    const bool is_tiny = valid && na + nb <= tiny;
    if (is_tiny) {
      const uint32_t card = rsa::aa_pair_thread(op, (const uint16_t *)(A.pool + A.off[ca]), na,
                                                (const uint16_t *)(B.pool + B.off[cb]), nb,
                                                (uint16_t *)(opool + E.off[e]));
      O.type[e] = RS_TAG_ARRAY;
      O.card[e] = card;
      O.n[e] = card;
      if (card) atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)card);
    }
    uint32_t rest = __ballot_sync(0xffffffffu, valid && !is_tiny);
    while (rest) {  // the batch's larger items through the warp merge path
      const int src = __ffs(rest) - 1;
      rest &= rest - 1;
      const uint32_t e1 = __shfl_sync(0xffffffffu, e, src), ca1 = __shfl_sync(0xffffffffu, ca, src),
                     cb1 = __shfl_sync(0xffffffffu, cb, src), na1 = __shfl_sync(0xffffffffu, na, src),
                     nb1 = __shfl_sync(0xffffffffu, nb, src);
      uint8_t type;
      uint32_t n;
      const uint32_t card = rsa::aa_pair<32, 8, op>(op, false, A.pool + A.off[ca1], (int)na1, B.pool + B.off[cb1],
                                                (int)nb1, sm[gid], gid, opool + E.off[e1], type, n);
      if (lane == 0) {
        O.type[e1] = type;
        O.card[e1] = card;
        O.n[e1] = n;
        if (card) atomicAdd((unsigned long long *)&res_card[E.pair[e1]], (unsigned long long)card);
      }
      __syncwarp();
    }
  }
}

template <int GT, int VT, int OPC = -1>
__global__ void __launch_bounds__(256) k_aa_pair(int op, const uint32_t *__restrict__ list, const uint32_t *__restrict__ cnt,
                                                 DevBatch A, DevBatch B, Entries E, OutDesc O,
                                                 uint8_t *__restrict__ opool, uint64_t *__restrict__ res_card) {
  constexpr int G = 256 / GT;
  __shared__ __align__(16) rsa::AASmem<GT, VT> sm[G];
  const int gid = threadIdx.x / GT, lt = threadIdx.x % GT;
  const uint32_t total = *cnt;
  for (uint32_t i = blockIdx.x * G + gid; i < total; i += gridDim.x * G) {
    const uint32_t e = list[i], ca = E.ca[e], cb = E.cb[e];
    uint8_t type;
    uint32_t n;
    uint32_t card = rsa::aa_pair<GT, VT, OPC>(op, false, A.pool + A.off[ca], (int)A.card[ca], B.pool + B.off[cb],
                                         (int)B.card[cb], sm[gid], gid, opool + E.off[e], type, n);
    if (lt == 0) {
      O.type[e] = type;
      O.card[e] = card;
      O.n[e] = n;
      if (card) atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)card);
    }
    rsa::group_sync<GT>(gid);
  }
}

// |a ∩ b| of array x array pairs (array_intersect count_only).
// Galloping pairs (gallop_pair): a warp per pair, persistent over the list.
// Lane l takes small-side values l, l+32, ... (at most NV per lane) and
// binary-searches each in the large side, all NV searches of a lane advancing
// together (NV independent loads per step; the top levels of the large
// array are shared by every search and stay in L1).  Kept values are
// compacted in order with warp ballots; the small side is sorted, so the
// result is.  With `out` (materialized) the result array goes to the entry's
// slot; the count path adds to acc[pair].
// 8-ary search (nl <= 4096 = 8^4): four levels of seven independent probes,
// so a lookup is five dependent global loads instead of thirteen (the search
// runs in place in HBM / L1, latency-bound).
__device__ __forceinline__ uint32_t gallop_search(const uint16_t *__restrict__ L, uint32_t nl, uint32_t x) {
  uint32_t lo = 0;
#pragma unroll
  for (uint32_t step = 512; step; step >>= 3) {
    uint32_t c = 0;
#pragma unroll
    for (uint32_t k = 1; k < 8; k++) {
      const uint32_t i = lo + k * step;
      c += i < nl && __ldg(L + i) <= x;
    }
    lo += c * step;
  }
  return nl && __ldg(L + lo) == x;
}

template <int NV>
__device__ __forceinline__ uint32_t gallop_warp(const uint16_t *__restrict__ S, uint32_t ns, const uint16_t *__restrict__ L,
                                                uint32_t nl, bool keep_found, uint16_t *dst, int lane) {
  uint32_t x[NV], k[NV];
#pragma unroll
  for (int j = 0; j < NV; j++) {
    const uint32_t i = lane + 32 * j;
    x[j] = i < ns ? __ldg(S + i) : 0;
  }
#pragma unroll
  for (int j = 0; j < NV; j++) {
    const uint32_t i = lane + 32 * j;
    k[j] = i < ns && gallop_search(L, nl, x[j]) == keep_found;
  }
  uint32_t base = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < NV; j++) {
    const uint32_t m = __ballot_sync(0xffffffffu, k[j]);
    if (dst && k[j]) dst[base + __popc(m & lt)] = (uint16_t)x[j];
    base += __popc(m);
  }
  if (dst && lane < 8 && ((base + lane) & 7) != 0 && ((base + 7) & ~7u) > base + lane) dst[base + lane] = 0;  // pad
  return base;
}

__device__ __forceinline__ uint32_t gallop_dispatch(const uint16_t *S, uint32_t ns, const uint16_t *L, uint32_t nl,
                                                    bool keep_found, uint16_t *dst, int lane) {
  if (ns <= 32) return gallop_warp<1>(S, ns, L, nl, keep_found, dst, lane);
  if (ns <= 64) return gallop_warp<2>(S, ns, L, nl, keep_found, dst, lane);
  if (ns <= 128) return gallop_warp<4>(S, ns, L, nl, keep_found, dst, lane);
  return gallop_warp<8>(S, ns, L, nl, keep_found, dst, lane);  // ns <= 4096 / 16
}

__global__ void __launch_bounds__(256) k_aa_gallop(int op, const uint32_t *__restrict__ list,
                                                   const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B, Entries E,
                                                   OutDesc O, uint8_t *__restrict__ opool,
                                                   uint64_t *__restrict__ res_card) {
  const int lane = threadIdx.x & 31;
  const uint32_t total = *cnt, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < total; it += nw) {
    const uint32_t e = list[it], ca = E.ca[e], cb = E.cb[e];
    const uint32_t na = A.card[ca], nb = B.card[cb];
    const uint16_t *pa = (const uint16_t *)(A.pool + A.off[ca]), *pb = (const uint16_t *)(B.pool + B.off[cb]);
    const bool a_small = op == RS_OP_ANDNOT || na <= nb;  // and: search the smaller side's values
    const uint32_t card = gallop_dispatch(a_small ? pa : pb, a_small ? na : nb, a_small ? pb : pa,
                                          a_small ? nb : na, op == RS_OP_AND, (uint16_t *)(opool + E.off[e]), lane);
    if (lane == 0) {
      O.type[e] = RS_TAG_ARRAY;
      O.card[e] = card;
      O.n[e] = card;
      if (card) atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)card);
    }
  }
}

// The galloping pairs staged: a warp per pair copies the large side into its
// own 8 KB of shared memory with one bulk copy (cp.async.bulk, lane 0,
// completing on the warp's mbarrier) while its lanes load the small side's
// values, then every value is binary-searched in shared memory -- the NV
// searches of a lane advance level by level together.  The in-place 8-ary
// search (k_aa_gallop) waited on ~5 dependent L2/HBM round trips per pair
// and touched most sectors of the large side anyway (C3 AND: 0.93 GB at
// 24 % issue); here a pair costs one bulk copy round trip and its bytes
// stream at the copy rate.
constexpr int GS_WARPS = 4;  // 4 x 8 KB per CTA: 7 CTAs per SM
template <int NV>
__device__ __forceinline__ uint32_t gallop_warp_smem(const uint16_t *__restrict__ S, uint32_t ns, const uint16_t *Ls,
                                                     uint32_t nl, bool keep_found, uint16_t *dst, int lane,
                                                     uint64_t *bar, uint32_t phase) {
  uint32_t x[NV], lo[NV];
#pragma unroll
  for (int j = 0; j < NV; j++) {
    const uint32_t i = lane + 32 * j;
    x[j] = i < ns ? __ldg(S + i) : 0;
    lo[j] = 0;
  }
  rsb::mbar_wait(bar, phase);
  for (uint32_t len = nl; len > 1;) {
    const uint32_t half = len >> 1;
#pragma unroll
    for (int j = 0; j < NV; j++)
      if (Ls[lo[j] + half] <= x[j]) lo[j] += half;
    len -= half;
  }
  uint32_t base = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < NV; j++) {
    const bool k = lane + 32 * j < ns && (nl && Ls[lo[j]] == x[j]) == keep_found;
    const uint32_t m = __ballot_sync(0xffffffffu, k);
    if (dst && k) dst[base + __popc(m & lt)] = (uint16_t)x[j];
    base += __popc(m);
  }
  if (dst && lane < 8 && ((base + lane) & 7) != 0 && ((base + 7) & ~7u) > base + lane) dst[base + lane] = 0;  // pad
  return base;
}

__global__ void __launch_bounds__(32 * GS_WARPS) k_aa_gallop_smem(int op, const uint32_t *__restrict__ list,
                                                                  const uint32_t *__restrict__ cnt, DevBatch A,
                                                                  DevBatch B, Entries E, OutDesc O,
                                                                  uint8_t *__restrict__ opool,
                                                                  uint64_t *__restrict__ res_card) {
  __shared__ __align__(128) uint16_t Ls[GS_WARPS][RS_ARRAY_MAX];
  __shared__ __align__(8) uint64_t bar[GS_WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    rsb::mbar_init(&bar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint32_t total = *cnt, nw = gridDim.x * GS_WARPS;
  uint32_t phase = 0;
  for (uint32_t it = blockIdx.x * GS_WARPS + w; it < total; it += nw, phase ^= 1) {
    const uint32_t e = list[it], ca = E.ca[e], cb = E.cb[e];
    const uint32_t na = A.card[ca], nb = B.card[cb];
    const uint16_t *pa = (const uint16_t *)(A.pool + A.off[ca]), *pb = (const uint16_t *)(B.pool + B.off[cb]);
    const bool a_small = op == RS_OP_ANDNOT || na <= nb;  // and: search the smaller side's values
    const uint16_t *S = a_small ? pa : pb, *L = a_small ? pb : pa;
    const uint32_t ns = a_small ? na : nb, nl = a_small ? nb : na;
    if (lane == 0) {  // the large side into this warp's buffer (the previous pair's reads are done: __syncwarp)
      const uint32_t bytes = (uint32_t)rs_pad16(2ull * nl);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      rsb::mbar_expect_tx(&bar[w], bytes);
      if (bytes) rsb::bulk_g2s(Ls[w], L, bytes, &bar[w]);
    }
    uint16_t *dst = (uint16_t *)(opool + E.off[e]);
    uint32_t card;
    if (ns <= 32) card = gallop_warp_smem<1>(S, ns, Ls[w], nl, op == RS_OP_AND, dst, lane, &bar[w], phase);
    else if (ns <= 64) card = gallop_warp_smem<2>(S, ns, Ls[w], nl, op == RS_OP_AND, dst, lane, &bar[w], phase);
    else if (ns <= 128) card = gallop_warp_smem<4>(S, ns, Ls[w], nl, op == RS_OP_AND, dst, lane, &bar[w], phase);
    else card = gallop_warp_smem<8>(S, ns, Ls[w], nl, op == RS_OP_AND, dst, lane, &bar[w], phase);
    if (lane == 0) {
      O.type[e] = RS_TAG_ARRAY;
      O.card[e] = card;
      O.n[e] = card;
      if (card) atomicAdd((unsigned long long *)&res_card[E.pair[e]], (unsigned long long)card);
    }
    __syncwarp();  // every lane's searches are done before the buffer is refilled
  }
}

__global__ void __launch_bounds__(256) k_aa_gallop_count(const uint32_t *__restrict__ lca,
                                                         const uint32_t *__restrict__ lcb,
                                                         const uint32_t *__restrict__ lpair,
                                                         const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B,
                                                         uint64_t *__restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const uint32_t total = *cnt, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < total; it += nw) {
    const uint32_t ca = lca[it], cb = lcb[it];
    const uint32_t na = A.card[ca], nb = B.card[cb];
    const uint16_t *pa = (const uint16_t *)(A.pool + A.off[ca]), *pb = (const uint16_t *)(B.pool + B.off[cb]);
    const bool a_small = na <= nb;
    const uint32_t c = gallop_dispatch(a_small ? pa : pb, a_small ? na : nb, a_small ? pb : pa, a_small ? nb : na,
                                       true, nullptr, lane);
    if (lane == 0 && c) atomicAdd((unsigned long long *)&acc[lpair[it]], (unsigned long long)c);
  }
}

// |A n B| of small pairs, laid out like k_aa_small: tiny pairs one per lane
// (scalar intersection count), the rest through the warp merge path.
__global__ void __launch_bounds__(256) k_aa_count_small(const uint32_t *__restrict__ lca,
                                                        const uint32_t *__restrict__ lcb,
                                                        const uint32_t *__restrict__ lpair,
                                                        const uint32_t *__restrict__ cnt, DevBatch A, DevBatch B,
                                                        uint64_t *__restrict__ acc) {
  __shared__ __align__(16) rsa::AASmem<32, 8> sm[8];
  const int gid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t total = *cnt, tiny = c_aa_tiny;
  const uint32_t W = gridDim.x * 8, gw = blockIdx.x * 8 + gid;  // item layout as in k_aa_small
  const bool wide = total >= 32u * W;
  const uint32_t first = wide ? 32 * gw : gw, lstep = wide ? 1u : W;
  for (uint32_t b0 = first; b0 < total; b0 += 32 * W) {
    const uint32_t it = b0 + lane * lstep;
    const bool valid = it < total;
    uint32_t ca = 0, cb = 0, na = 0, nb = 0;
    if (valid) {
      ca = lca[it];
      cb = lcb[it];
      na = A.card[ca];
      nb = B.card[cb];
    }
    const bool is_tiny = valid && na + nb <= tiny;
    if (is_tiny) {
      const uint32_t c = rsa::aa_pair_thread(RS_OP_AND, (const uint16_t *)(A.pool + A.off[ca]), na,
                                             (const uint16_t *)(B.pool + B.off[cb]), nb, nullptr);
      if (c) atomicAdd((unsigned long long *)&acc[lpair[it]], (unsigned long long)c);
    }
    uint32_t rest = __ballot_sync(0xffffffffu, valid && !is_tiny);
    while (rest) {
      const int src = __ffs(rest) - 1;
      rest &= rest - 1;
      const uint32_t ca1 = __shfl_sync(0xffffffffu, ca, src), cb1 = __shfl_sync(0xffffffffu, cb, src),
                     na1 = __shfl_sync(0xffffffffu, na, src), nb1 = __shfl_sync(0xffffffffu, nb, src);
      uint8_t type;
      uint32_t n;
      const uint32_t c = rsa::aa_pair<32, 8>(RS_OP_AND, true, A.pool + A.off[ca1], (int)na1, B.pool + B.off[cb1],
                                             (int)nb1, sm[gid], gid, nullptr, type, n);
      if (lane == 0 && c) atomicAdd((unsigned long long *)&acc[lpair[b0 + src * lstep]], (unsigned long long)c);
      __syncwarp();
    }
  }
}

template <int GT, int VT>
__global__ void __launch_bounds__(256) k_aa_count(const uint32_t *__restrict__ lca, const uint32_t *__restrict__ lcb,
                                                  const uint32_t *__restrict__ lpair, const uint32_t *__restrict__ cnt,
                                                  DevBatch A, DevBatch B, uint64_t *__restrict__ acc) {
  constexpr int G = 256 / GT;
  __shared__ __align__(16) rsa::AASmem<GT, VT> sm[G];
  const int gid = threadIdx.x / GT, lt = threadIdx.x % GT;
  const uint32_t total = *cnt;
  for (uint32_t i = blockIdx.x * G + gid; i < total; i += gridDim.x * G) {
    const uint32_t ca = lca[i], cb = lcb[i];
    uint8_t type;
    uint32_t n;
    uint32_t c = rsa::aa_pair<GT, VT>(RS_OP_AND, true, A.pool + A.off[ca], (int)A.card[ca], B.pool + B.off[cb],
                                      (int)B.card[cb], sm[gid], gid, nullptr, type, n);
    if (lt == 0 && c) atomicAdd((unsigned long long *)&acc[lpair[i]], (unsigned long long)c);
    rsa::group_sync<GT>(gid);
  }
}

// ------------------------------------------------------------ compaction

__global__ void k_keep_nonempty(uint64_t E, const uint32_t *__restrict__ dE, const uint32_t *__restrict__ card,
                                uint32_t *__restrict__ keep) {
  uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t lim = dE ? *dE : E;
  if (e <= E) keep[e] = e < lim && card[e] > 0;
}

__global__ void k_compact(uint64_t E, const uint32_t *__restrict__ dE, const uint32_t *__restrict__ keep, const uint32_t *__restrict__ fpos, Entries En,
                          OutDesc O, uint16_t *key, uint8_t *type, uint32_t *card, uint32_t *nn, uint64_t *off) {
  uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= E || !keep[e]) return;
  uint32_t f = fpos[e];
  key[f] = En.key[e];
  type[f] = O.type[e];
  card[f] = O.card[e];
  nn[f] = O.n[e];
  off[f] = En.off[e];
}

// result bitmap p starts at the compacted position of its first entry:
// entry epos[mbase[p]] for a key join, entry p for container-level ops
__global__ void k_bm_start(uint64_t npairs, const uint64_t *__restrict__ mbase, const uint32_t *__restrict__ epos,
                           const uint32_t *__restrict__ fpos, uint64_t *__restrict__ bm_start) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  // first entry of pair p: epos[mbase[p]] (key join), epos[p] (per-pair
  // entry bases: mbase == nullptr, epos != nullptr), p (container ops)
  if (p <= npairs) bm_start[p] = fpos[mbase ? epos[mbase[p]] : epos ? epos[p] : p];
}

// Per-pair compaction (entries of pair p are [pbase[p], pbase[p+1])): the
// non-empty results per pair, then CTA per pair writes them at the pair's base
// (a scan over pairs) plus an in-CTA scan -- no scan over every entry.
__global__ void __launch_bounds__(256) k_pair_nonempty(uint64_t npairs, const uint32_t *__restrict__ pbase,
                                                       const uint32_t *__restrict__ card, uint32_t *__restrict__ nz,
                                                       uint32_t *done, uint32_t *fb) {
  __shared__ uint32_t red[8];
  const uint32_t p = blockIdx.x;
  if (p == 0 && threadIdx.x == 0) nz[npairs] = 0;
  uint32_t c = 0;
  for (uint32_t e = pbase[p] + threadIdx.x; e < pbase[p + 1]; e += blockDim.x) c += card[e] > 0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < 8; w++) s += red[w];
    nz[p] = s;
  }
  if (done && last_block_arrives(done, npairs)) block_exclusive_scan<uint32_t>(nz, fb, npairs + 1);
}

// fbase == nullptr: the single-pair op (one CTA): the pair's kept count is
// this loop's own total, and the bitmap's cardinality is summed here (the
// class kernels' atomic sums went to a scratch word, so no memset was needed)
// (NT threads: 1024 when pairs hold thousands of entries, each CTA's chunks
// being serial)
template <int NT>
__global__ void __launch_bounds__(NT) k_compact_pair(uint64_t npairs, const uint32_t *__restrict__ pbase,
                                                     const uint32_t *__restrict__ fbase, Entries En, OutDesc O,
                                                     uint16_t *key, uint8_t *type, uint32_t *card, uint32_t *nn,
                                                     uint64_t *off, uint64_t *bm_start, uint64_t *bm_card) {
  using BS = cub::BlockScan<uint32_t, NT>;
  __shared__ typename BS::TempStorage ts;
  __shared__ unsigned long long csum;
  const uint32_t p = blockIdx.x;
  uint32_t f = fbase ? fbase[p] : 0;
  if (threadIdx.x == 0) {
    bm_start[p] = f;
    if (p == 0 && fbase) bm_start[npairs] = fbase[npairs];
    csum = 0;
  }
  uint64_t my = 0;
  const uint32_t e1 = pbase[p + 1];
  for (uint32_t e0 = pbase[p]; e0 < e1; e0 += blockDim.x) {
    const uint32_t e = e0 + threadIdx.x;
    const uint32_t k = e < e1 && O.card[e] > 0;
    uint32_t ex, tot;
    BS(ts).ExclusiveSum(k, ex, tot);
    if (k) {
      const uint32_t d = f + ex;
      key[d] = En.key[e];
      type[d] = O.type[e];
      card[d] = O.card[e];
      nn[d] = O.n[e];
      off[d] = En.off[e];
      my += O.card[e];
    }
    f += tot;
    __syncthreads();
  }
  if (!fbase) {
    atomicAdd(&csum, (unsigned long long)my);
    __syncthreads();
    if (threadIdx.x == 0) {
      bm_start[1] = f;
      bm_card[0] = csum;
    }
  }
}

// ---------------------------------------------- A-indexed join (and / andnot)

// AND and ANDNOT keep a subset of A's keys, in A's order (bitmap.py:169-210,
// _KEEP_A / _KEEP_B), so a result entry can sit at its A container's
// position: entry e = abase[p] + i for container i of pair p's A bitmap,
// with an 8 KB slot at 8192 e.  A CTA per chunk of a pair's A containers
// finds each key in B's keys (staged in shared memory), writes the entry and
// appends it to its class list (or marks an AND miss empty); the
// merged-position join's two scans over both sides' keys and its emit pass
// are not needed, and the per-pair compaction drops the empty entries.
// A CTA takes JA_CHUNK of one pair's A containers (grid: npairs x chunks of
// the largest A bitmap), with B's keys staged in shared memory when they fit.
constexpr uint32_t JA_CHUNK = 512, JA_SMEM_KEYS = 4096;
__global__ void __launch_bounds__(256) k_join_a(uint32_t chunks, const uint64_t *__restrict__ abase, DevBatch A,
                                                DevBatch B, const uint32_t *ia, const uint32_t *ib, int op, Entries E,
                                                OutDesc O, Lists L) {
  __shared__ uint16_t kB[JA_SMEM_KEYS];
  const uint32_t p = blockIdx.x / chunks, c = blockIdx.x % chunks;
  const uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
  const uint64_t a0 = A.bm_start[a], b0 = B.bm_start[b];
  const uint32_t na = (uint32_t)(A.bm_start[a + 1] - a0), nb = (uint32_t)(B.bm_start[b + 1] - b0);
  if (c * JA_CHUNK >= na) return;  // (the whole CTA)
  const bool staged = nb <= JA_SMEM_KEYS;
  if (staged) {
    for (uint32_t u = threadIdx.x; u < nb; u += blockDim.x) kB[u] = B.key[b0 + u];
    __syncthreads();
  }
  const uint16_t *keys = staged ? kB : B.key + b0;
  const uint64_t ebase = abase[p];
  for (uint32_t r = 0; r < JA_CHUNK; r += 256) {
    const uint32_t i = c * JA_CHUNK + r + threadIdx.x;
    if (c * JA_CHUNK + r >= na) break;  // (uniform over the CTA)
    bool active = false;
    int cls = CLS_COPY;
    uint32_t nab = 0;
    uint64_t ao = 0, bo = 0;
    const uint64_t e = ebase + i;
    if (i < na) {
      const uint32_t ca = (uint32_t)(a0 + i);
      const uint16_t key = A.key[ca];
      const uint32_t j = lower_bound16(keys, nb, key);
      const bool matched = j < nb && keys[j] == key;
      active = matched || op == RS_OP_ANDNOT;
      if (active) {
        const uint32_t cb = matched ? (uint32_t)(b0 + j) : RS_NONE;
        E.key[e] = key;
        E.ca[e] = ca;
        E.cb[e] = cb;
        E.pair[e] = p;
        E.off[e] = 8192ull * e;
        if (matched) {
          cls = classify(A.type[ca], A.card[ca], B.type[cb], B.card[cb], op);
          if (tma_class(cls)) {
            ao = A.off[ca];
            bo = B.off[cb];
            nab = A.card[ca] | (B.card[cb] << 16);
          }
        }
      } else {
        O.card[e] = 0;  // an AND miss: nothing kept
      }
    }
    list_append_cta(L, cls, active, (uint32_t)e, ao, bo, nab);
  }
}

// -------------------------------------------------- count-only join + formula

// count-path append: ca into the class list, cb / pair into parallel arrays
// at the same slot (and the operand offsets for bitset x bitset items)
template <bool CTA = false>
__device__ __forceinline__ void count_append(Lists L, int cls, bool active, uint32_t ca, uint32_t cb, uint32_t pair,
                                             uint32_t *lcb_base, uint32_t *lpair_base, const DevBatch &A,
                                             const DevBatch &B) {
  uint64_t ao = 0, bo = 0;
  uint32_t nab = 0;
  if (active && tma_class(cls)) {
    ao = A.off[ca];
    bo = B.off[cb];
    nab = A.card[ca] | (B.card[cb] << 16);
  }
  uint32_t slot;
  if constexpr (CTA) slot = list_append_cta(L, cls, active, ca, ao, bo, nab);
  else slot = list_append(L, cls, active, ca, ao, bo, nab);
  if (active) {
    lcb_base[cls * L.cap + slot] = cb;
    lpair_base[cls * L.cap + slot] = pair;
  }
}

__global__ void k_match(uint64_t Ma, uint64_t npairs, const uint64_t *__restrict__ mbase, DevBatch A, DevBatch B,
                        const uint32_t *ia, const uint32_t *ib, Lists L, uint32_t *__restrict__ lcb_base,
                        uint32_t *__restrict__ lpair_base) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  bool active = false;
  int cls = CLS_GEN;
  uint32_t ca = 0, cb = 0, p32 = 0;
  if (t < Ma) {
    uint64_t p = find_pair(mbase, npairs, t);
    uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
    uint64_t a0 = A.bm_start[a], b0 = B.bm_start[b];
    uint32_t nb = (uint32_t)(B.bm_start[b + 1] - b0);
    uint32_t l = (uint32_t)(t - mbase[p]);
    uint16_t key = A.key[a0 + l];
    uint32_t j = lower_bound16(B.key + b0, nb, key);
    if (j < nb && B.key[b0 + j] == key) {
      active = true;
      ca = (uint32_t)(a0 + l);
      cb = (uint32_t)(b0 + j);
      p32 = (uint32_t)p;
      cls = classify(A.type[ca], A.card[ca], B.type[cb], B.card[cb], RS_OP_AND, true);
    }
  }
  count_append<true>(L, cls, active, ca, cb, p32, lcb_base, lpair_base, A, B);
}

// CTA per pair with B's keys in shared memory (every bitmap at most
// MERGE_SMEM_KEYS containers); the warp-aggregated list appends need whole
// warps, so each warp walks A's keys in steps of 32
__global__ void __launch_bounds__(256) k_match_pair(const uint64_t *__restrict__ mbase, DevBatch A, DevBatch B,
                                                    const uint32_t *ia, const uint32_t *ib, Lists L,
                                                    uint32_t *__restrict__ lcb_base, uint32_t *__restrict__ lpair_base) {
  __shared__ uint16_t kB[MERGE_SMEM_KEYS];
  const uint32_t p = blockIdx.x;
  const uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
  const uint64_t a0 = A.bm_start[a], b0 = B.bm_start[b];
  const uint32_t na = (uint32_t)(A.bm_start[a + 1] - a0), nb = (uint32_t)(B.bm_start[b + 1] - b0);
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) kB[i] = B.key[b0 + i];
  __syncthreads();
  for (uint32_t l0 = threadIdx.x & ~31u; l0 < na; l0 += blockDim.x) {
    const uint32_t l = l0 + (threadIdx.x & 31);
    bool active = false;
    int cls = CLS_GEN;
    uint32_t ca = 0, cb = 0;
    if (l < na) {
      const uint16_t key = A.key[a0 + l];
      const uint32_t j = lower_bound16(kB, nb, key);
      if (j < nb && kB[j] == key) {
        active = true;
        ca = (uint32_t)(a0 + l);
        cb = (uint32_t)(b0 + j);
        cls = classify(A.type[ca], A.card[ca], B.type[cb], B.card[cb], RS_OP_AND, true);
      }
    }
    count_append(L, cls, active, ca, cb, p, lcb_base, lpair_base, A, B);
  }
}

// bitmap.py:235-241: every count from |A ∩ B|
__global__ void k_formula(uint64_t npairs, int op, const uint64_t *__restrict__ cardA, const uint64_t *__restrict__ cardB,
                          const uint32_t *ia, const uint32_t *ib, const uint64_t *__restrict__ inter,
                          uint64_t *__restrict__ out) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  uint64_t x = cardA[pair_a(ia, p)], y = cardB[pair_a(ib, p)], i = inter[p];
  out[p] = op == RS_OP_AND ? i : op == RS_OP_OR ? x + y - i : op == RS_OP_ANDNOT ? x - i : x + y - 2 * i;
}

// container_pairwise_cardinality (containers.py:554-570) formula from ∩
__global__ void k_formula_containers(uint64_t npairs, int op, DevBatch A, DevBatch B, const uint32_t *ia,
                                     const uint32_t *ib, const uint64_t *__restrict__ inter, uint64_t *__restrict__ out) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  const uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
  // an image without containers is the empty container (len 0)
  uint64_t x = A.bm_start[a + 1] > A.bm_start[a] ? A.card[A.bm_start[a]] : 0;
  uint64_t y = B.bm_start[b + 1] > B.bm_start[b] ? B.card[B.bm_start[b]] : 0, i = inter[p];
  out[p] = op == RS_OP_AND ? i : op == RS_OP_OR ? x + y - i : op == RS_OP_ANDNOT ? x - i : x + y - 2 * i;
}

// container-level entries: pair p -> the single containers of A[ia[p]], B[ib[p]]
__global__ void k_cont_entries(uint64_t npairs, DevBatch A, DevBatch B, const uint32_t *ia, const uint32_t *ib, int op,
                               Entries E, uint64_t *__restrict__ ub, Lists L) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  bool active = p < npairs;
  int cls = CLS_GEN;
  uint64_t ao = 0, bo = 0;
  uint32_t nab = 0;
  if (active) {
    const uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
    uint32_t ca = (uint32_t)A.bm_start[a], cb = (uint32_t)B.bm_start[b];
    const bool ea = A.bm_start[a + 1] == ca, eb = B.bm_start[b + 1] == cb;
    E.pair[p] = (uint32_t)p;
    if (ea || eb) {
      // an empty image is the empty container: op(empty, x) is x for OR/XOR,
      // op(x, empty) is x for OR/XOR/ANDNOT -- a deep copy of x, whose type is
      // already the one container_pairwise picks (an empty array side keeps
      // the other side's canonical type, App. A); anything else is empty.
      // Both sides RS_NONE = nothing to copy (k_copy writes an empty result).
      const bool keep_b = ea && !eb && (op == RS_OP_OR || op == RS_OP_XOR);
      const bool keep_a = eb && !ea && op != RS_OP_AND;
      ca = keep_a ? ca : RS_NONE;
      cb = keep_b ? cb : RS_NONE;
      E.key[p] = keep_a ? A.key[ca] : keep_b ? B.key[cb] : 0;
      E.ca[p] = ca;
      E.cb[p] = cb;
      ub[p] = keep_a ? rs_pad16(rs_payload_bytes(A.type[ca], A.n[ca]))
            : keep_b ? rs_pad16(rs_payload_bytes(B.type[cb], B.n[cb])) : 0;
      cls = CLS_COPY;
    } else {
    E.key[p] = A.key[ca];
    E.ca[p] = ca;
    E.cb[p] = cb;
    ub[p] = rs_pad16(rs_result_ub(A.type[ca], A.card[ca], B.type[cb], B.card[cb], op));
    cls = classify(A.type[ca], A.card[ca], B.type[cb], B.card[cb], op);
    }
    if (tma_class(cls)) {
      ao = A.off[ca];
      bo = B.off[cb];
      nab = A.card[ca] | (B.card[cb] << 16);
    }
  } else if (p == npairs) {
    ub[p] = 0;
  }
  list_append_cta(L, cls, active, (uint32_t)p, ao, bo, nab);
}

__global__ void k_cont_list(uint64_t npairs, DevBatch A, DevBatch B, const uint32_t *ia, const uint32_t *ib, Lists L,
                            uint32_t *__restrict__ lcb_base, uint32_t *__restrict__ lpair_base) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  bool active = p < npairs;
  int cls = CLS_GEN;
  uint32_t ca = 0, cb = 0;
  if (active) {
    const uint32_t a = pair_a(ia, p), b = pair_a(ib, p);
    ca = (uint32_t)A.bm_start[a];
    cb = (uint32_t)B.bm_start[b];
    // an empty side: |empty ∩ x| = 0, no work item
    active = A.bm_start[a + 1] > ca && B.bm_start[b + 1] > cb;
    if (active) cls = classify(A.type[ca], A.card[ca], B.type[cb], B.card[cb], RS_OP_AND, true);
  }
  count_append<true>(L, cls, active, ca, cb, (uint32_t)p, lcb_base, lpair_base, A, B);
}

// ------------------------------------------------------------- host side

// Per-op scratch: a bump allocator over one cached device block, so an op's
// ~25 scratch arrays cost a pointer bump each instead of a trip through the
// caching allocator (host time is what a small op like config 1 spends).  The
// block is reused by the next op in stream order; scopes nest LIFO; an op
// that outgrows it spills to dalloc and the block grows before a later op.
struct Scratch {
  static uint8_t *arena;
  static size_t cap, top, want;
  static cudaStream_t stream;
  static std::recursive_mutex mu;  // the arena is shared: ops from several host threads serialize
  std::lock_guard<std::recursive_mutex> lock{mu};
  size_t base, need;
  bool failed = false;
  std::vector<void *> spill;
  Scratch() {
    if (top == 0) {
      if (stream != g_stream) {  // reused blocks are ordered on the old stream
        if (arena) cudaStreamSynchronize(stream);
        stream = g_stream;
      }
      if (want > cap) {
        dfree(arena);
        arena = (uint8_t *)dalloc(want);
        cap = arena ? want : 0;
      }
    }
    base = need = top;
  }
  void *get(size_t bytes) {
    const size_t b = (bytes + 255) & ~(size_t)255;
    need += b;
    if (arena && top + b <= cap) {
      void *p = arena + top;
      top += b;
      return p;
    }
    void *p = dalloc(bytes);
    if (!p) failed = true;
    spill.push_back(p);
    return p;
  }
  bool ok() const { return !failed; }
  ~Scratch() {
    top = base;
    for (void *p : spill) dfree(p);
    if (need > cap) want = std::max(want, need + need / 4);
  }
};
uint8_t *Scratch::arena = nullptr;
size_t Scratch::cap = 0, Scratch::top = 0, Scratch::want = 1 << 20;
cudaStream_t Scratch::stream = nullptr;
std::recursive_mutex Scratch::mu;

unsigned grid_for(uint64_t n, unsigned block) { return (unsigned)((n + block - 1) / block); }

uint32_t g_aa_large_min = 256, g_aa_union_medium = 512;
// medium bound of the op's array x array pairs (host mirror of classify())
uint32_t aa_medium_max(int op) { return op == RS_OP_OR || op == RS_OP_XOR ? g_aa_union_medium : g_aa_large_min; }
bool aa_medium_possible(int op = RS_OP_AND) { return aa_medium_max(op) > 256; }

int check_op(int op) {
  if (op < 0 || op > 3) {
    set_error("unknown op " + std::to_string(op));
    return RS_EOP;
  }
  static int tuned = 0;  // one-time device tuning constants
  if (!tuned) {
    RS_TRY(ensure_device());
    // medium bounds are capped at 2048 merged items: the capacity of the
    // largest merge-path kernel they select (k_aa_pair/k_aa_count<128,16>)
    uint32_t v = (uint32_t)std::min(std::max(env_int("RS_AA_LARGE_MIN", 256), 0), 2048);
    g_aa_large_min = v;
    RS_CK(cudaMemcpyToSymbol(c_aa_large_min, &v, sizeof v));
    const uint32_t um = (uint32_t)std::min(std::max(env_int("RS_AA_UNION_MEDIUM", 512), 0), 2048);
    g_aa_union_medium = um;
    RS_CK(cudaMemcpyToSymbol(c_aa_union_medium, &um, sizeof um));
    const uint32_t tiny = (uint32_t)env_int("RS_AA_TINY", 64);  // tuning: largest pair merged by one thread
    RS_CK(cudaMemcpyToSymbol(c_aa_tiny, &tiny, sizeof tiny));
    const uint32_t gt = (uint32_t)env_int("RS_GALLOP_TMA", 3);
    RS_CK(cudaMemcpyToSymbol(c_gallop_tma, &gt, sizeof gt));
    tuned = 1;
  }
  return RS_OK;
}

int check_pairs(const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib, uint64_t npairs) {
  if (!ia && npairs > A->nb) { set_error("identity pairing needs npairs <= len(A)"); return RS_EARG; }
  if (!ib && npairs > B->nb) { set_error("identity pairing needs npairs <= len(B)"); return RS_EARG; }
  for (uint64_t p = 0; ia && p < npairs; p++)
    if (ia[p] >= A->nb) { set_error("pair index out of range (A)"); return RS_EARG; }
  for (uint64_t p = 0; ib && p < npairs; p++)
    if (ib[p] >= B->nb) { set_error("pair index out of range (B)"); return RS_EARG; }
  return RS_OK;
}

// An op's small host-side inputs (pair indices, per-pair merge bases, zeroed
// counters) gathered into one block and sent up as ONE copy, instead of a
// copy and a memset each.
struct Upload {
  static constexpr size_t NONE = ~(size_t)0;
  std::vector<uint8_t> h;
  uint8_t *d = nullptr;
  size_t add(const void *src, size_t bytes) {  // src == nullptr: zeros
    const size_t o = h.size();
    h.resize(o + ((bytes + 15) & ~(size_t)15), 0);
    if (src && bytes) memcpy(h.data() + o, src, bytes);
    return o;
  }
  int commit(Scratch &S) {
    if (h.empty()) return RS_OK;
    d = (uint8_t *)S.get(h.size());
    if (!d) { set_error("device allocation failed (upload)"); return RS_ENOMEM; }
    return h2d_small(d, h.data(), h.size());
  }
  template <typename T> T *at(size_t o) const { return o == NONE ? nullptr : (T *)(d + o); }
};

// mbase[p] = exclusive prefix of the per-pair merged key counts (na + nb, or
// na for the count path), summed on the host (which holds bm_start) for small
// pair lists; false = use the device size kernel + scan instead.
bool pair_bases_host(const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib, uint64_t npairs,
                     int count_mode, std::vector<uint64_t> &h) {
  if (npairs > 16384) return false;
  h.resize(npairs + 1);
  uint64_t acc = 0;
  for (uint64_t p = 0; p < npairs; p++) {
    h[p] = acc;
    uint32_t a = ia ? ia[p] : (uint32_t)p, b = ib ? ib[p] : (uint32_t)p;
    acc += (A->h_bm_start[a + 1] - A->h_bm_start[a]) + (count_mode ? 0 : (B->h_bm_start[b + 1] - B->h_bm_start[b]));
  }
  h[npairs] = acc;
  return true;
}

// Which work classes can occur between batches with these container-type
// masks (bit t = type t present)?  Impossible classes are never launched.
struct ClassMask {
  bool bb, aa, gen, prb;
};
// which type-pair classes can occur (op: the materialized op, or AND for counts)
ClassMask class_mask(uint8_t ma, uint8_t mb, int op) {
  const uint8_t AR = 1 << RS_TAG_ARRAY, BS = 1 << RS_TAG_BITSET, RN = 1 << RS_TAG_RUN;
  ClassMask m;
  m.bb = (ma & BS) && (mb & BS);
  m.aa = (ma & AR) && (mb & AR);
  const bool a_x = (ma & AR) && (mb & (BS | RN)), x_a = (ma & (BS | RN)) && (mb & AR);
  m.prb = op == RS_OP_AND ? (a_x || x_a) : op == RS_OP_ANDNOT ? a_x : false;
  const bool gen_all = ((ma | mb) & RN) || a_x || x_a;
  m.gen = op == RS_OP_AND ? (ma & (BS | RN)) && (mb & (BS | RN)) && ((ma | mb) & RN)
        : op == RS_OP_ANDNOT ? x_a || ((ma & (BS | RN)) && (mb & (BS | RN)) && ((ma | mb) & RN))
        : gen_all;
  return m;
}

// container types an op result may hold (run results need a run input)
// single-pair calls with at most this many result slots take the one-launch
// path (its last CTA compacts the slots alone); RS_SINGLE=0 turns it off
constexpr uint32_t SINGLE_MAX_SLOTS = 4096;
bool single_path_on() {
  static const bool on = env_int("RS_SINGLE", 1) != 0;
  return on;
}

uint8_t result_mask(uint8_t ma, uint8_t mb) {
  const uint8_t AR = 1 << RS_TAG_ARRAY, BS = 1 << RS_TAG_BITSET, RN = 1 << RS_TAG_RUN;
  return (uint8_t)(AR | BS | ((ma | mb) & RN));
}

unsigned sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return (unsigned)sms;
}

// Run the per-class kernels over prepared entries, then compact into `out`.
// Exact mode: hcnt holds the class sizes (host) and E/P are exact.  Upper-
// bound mode (hcnt == nullptr): E/P are capacities, the real entry count is
// *dE on the device, and every class kernel is persistent over its device
// counter -- the op then runs without any host synchronization.
int run_classes_and_compact(int op, const rs_batch *A, const rs_batch *B, Scratch &S, Entries En, Lists L,
                            uint64_t E, uint64_t P, const uint32_t *hcnt, const uint32_t *dE,
                            const uint64_t *mbase, const uint32_t *epos, uint64_t npairs, rs_batch **out,
                            const OutDesc *pre = nullptr) {
  OutDesc O;
  if (pre) {
    O = *pre;
  } else {
    O.type = (uint8_t *)S.get(E + 1);
    O.card = (uint32_t *)S.get((E + 1) * 4);
    O.n = (uint32_t *)S.get((E + 1) * 4);
  }
  uint32_t *keep2 = (uint32_t *)S.get((E + 1) * 4), *fpos = (uint32_t *)S.get((E + 1) * 4);
  if (!S.ok()) { set_error("device allocation failed (op scratch)"); return RS_ENOMEM; }
  host_mark(5);
  RS_TRY(ub_reserve(P));
  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, npairs, E, P);
  if (rc) { rs_batch_free(b); return rc; }
  ub_register(b);
  b->type_mask = result_mask(A->type_mask, B->type_mask);
  host_mark(6);
  // one pair (per-pair entry bases): the compaction sums the bitmap's
  // cardinality itself, so the class kernels' atomic sums go to scratch and
  // there is nothing to zero first
  const bool single = npairs == 1 && !mbase && epos;
  uint64_t *res_card = b->d_bm_card;
  if (single) {
    res_card = (uint64_t *)S.get(16);
    if (!S.ok()) { set_error("device allocation failed (op scratch)"); return RS_ENOMEM; }
  } else {
    RS_CK(cudaMemsetAsync(b->d_bm_card, 0, (npairs + 1) * 8, g_stream));
  }
  host_mark(7);
  DevBatch dA = A->dev(), dB = B->dev();
  const ClassMask cm = class_mask(A->type_mask, B->type_mask, op);
  const unsigned sms = sm_count();
  auto want = [&](int c, bool possible) -> uint64_t {  // 0 = skip, else capacity for the grid
    if (hcnt) return hcnt[c];
    return possible ? L.cap : 0;
  };
  // the class kernels are independent (disjoint lists and output slots): with
  // more than one of them they run concurrently on side streams
  const uint64_t n_copy = want(CLS_COPY, op != RS_OP_AND), n_bb = want(CLS_BB, cm.bb),
                 n_aas = want(CLS_AAS, cm.aa), n_aam = want(CLS_AAM, cm.aa && aa_medium_possible(op)),
                 n_aal = want(CLS_AAL, cm.aa), n_gen = want(CLS_GEN, cm.gen), n_prb = want(CLS_PRB, cm.prb),
                 n_aag = want(CLS_AAG, cm.aa && (op == RS_OP_AND || op == RS_OP_ANDNOT));
  const int nk = (n_copy > 0) + (n_bb > 0) + (n_aas > 0) + (n_aam > 0) + (n_aal > 0) + (n_gen > 0) + (n_prb > 0) +
                 (n_aag > 0);
  Fork F;  // (tiny ops are host-bound: the fork's event calls would cost more than they overlap)
  static const int nofork = env_int_("RS_NO_FORK", 0);
  if (nk > 1 && E >= 16384 && !nofork) RS_TRY(F.begin(nk));
  // copies: persistent warps over the list (8 warps per CTA)
  if (uint64_t n = n_copy) {
    F.next();
    static const int copy_cta = env_int_("RS_COPY_CTAS", 16);  // CTAs per SM (tuning)
    unsigned g = std::min<uint64_t>(grid_for(n, 8), sms * copy_cta);
    RS_LAUNCH_PROF("copy", hcnt ? n : 0, k_copy, g, 256, 0, L.list[CLS_COPY], L.cnt + CLS_COPY, dA, dB, En, O,
                   b->d_pool, res_card);
  }
  if (uint64_t n = n_bb) {
    F.next();
    if (bb_kernel_choice() == 0) {
      RS_LAUNCH_PROF("bitset_pair", hcnt ? n : 0, k_pair_dense<false>, std::min<uint64_t>(n, sms * 6), DT, 0, op,
                     L.list[CLS_BB], L.cnt + CLS_BB, (uint32_t *)nullptr, dA, dB, En, O, b->d_pool, res_card);
    } else {
      switch (bb_stages()) {
        case 3: RS_TRY(launch_bb_op<3>(op, L, n, dA, dB, En, O, b->d_pool, res_card)); break;
        case 4: RS_TRY(launch_bb_op<4>(op, L, n, dA, dB, En, O, b->d_pool, res_card)); break;
        default: RS_TRY(launch_bb_op<2>(op, L, n, dA, dB, En, O, b->d_pool, res_card)); break;
      }
    }
  }
  if (uint64_t n = n_aas) {
    F.next();
    if (env_int_("RS_AA_SMALL_PLAIN", 0))  // the warp-per-pair kernel (A/B only)
      RS_LAUNCH_PROF("array_pair_s", hcnt ? n : 0, (k_aa_pair<32, 8>), std::min<uint64_t>(grid_for(n, 8), sms * 8),
                     256, 0, op, L.list[CLS_AAS], L.cnt + CLS_AAS, dA, dB, En, O, b->d_pool, res_card);
    else
      switch (op) {  // one instantiation per op: the keep rules are constants
#define RS_AAS(OP) RS_LAUNCH_PROF("array_pair_s", hcnt ? n : 0, k_aa_small<OP>, std::min<uint64_t>(grid_for(n, 8), sms * 8), \
                                  256, 0, L.list[CLS_AAS], L.cnt + CLS_AAS, dA, dB, En, O, b->d_pool, res_card)
        case RS_OP_AND: RS_AAS(RS_OP_AND); break;
        case RS_OP_OR: RS_AAS(RS_OP_OR); break;
        case RS_OP_ANDNOT: RS_AAS(RS_OP_ANDNOT); break;
        default: RS_AAS(RS_OP_XOR); break;
#undef RS_AAS
      }
  }
  if (uint64_t n = n_aam) {
    F.next();
    // medium pairs: a warp per pair (16 items per lane) up to 512 items, else
    // the 128-thread groups
    if (aa_medium_max(op) <= 512) {
      switch (op) {  // per-op instantiations (constant keep rules)
#define RS_AAM(OP) RS_LAUNCH_PROF("array_pair_m", hcnt ? n : 0, (k_aa_pair<32, 16, OP>), \
                                  std::min<uint64_t>(grid_for(n, 8), sms * 8), 256, 0, op, L.list[CLS_AAM], \
                                  L.cnt + CLS_AAM, dA, dB, En, O, b->d_pool, res_card)
        case RS_OP_AND: RS_AAM(RS_OP_AND); break;
        case RS_OP_OR: RS_AAM(RS_OP_OR); break;
        case RS_OP_ANDNOT: RS_AAM(RS_OP_ANDNOT); break;
        default: RS_AAM(RS_OP_XOR); break;
#undef RS_AAM
      }
    } else
      RS_LAUNCH_PROF("array_pair_m", hcnt ? n : 0, (k_aa_pair<128, 16>), std::min<uint64_t>(grid_for(n, 2), sms * 8),
                     256, 0, op, L.list[CLS_AAM], L.cnt + CLS_AAM, dA, dB, En, O, b->d_pool, res_card);
  }
  if (uint64_t n = n_aal) {
    F.next();
    if (env_int("RS_AA_LARGE_MERGE", 0))
      RS_LAUNCH_PROF("array_pair_l", hcnt ? n : 0, (k_aa_pair<256, 32>), std::min<uint64_t>(n, sms * 8), 256, 0, op,
                     L.list[CLS_AAL], L.cnt + CLS_AAL, dA, dB, En, O, b->d_pool, res_card);
    else
      RS_TRY(launch_aa_large_op(op, L, n, dA, dB, En, O, b->d_pool, res_card, hcnt != nullptr));
  }
  if (uint64_t n = n_aag) {
    F.next();
    static const int staged = env_int("RS_GALLOP_SMEM", 1);  // 0: the in-place search (A/B)
    if (staged)
      RS_LAUNCH_PROF("array_pair_g", hcnt ? n : 0, k_aa_gallop_smem,
                     std::min<uint64_t>(grid_for(n, GS_WARPS), sms * 7), 32 * GS_WARPS, 0, op, L.list[CLS_AAG],
                     L.cnt + CLS_AAG, dA, dB, En, O, b->d_pool, res_card);
    else
      RS_LAUNCH_PROF("array_pair_g", hcnt ? n : 0, k_aa_gallop, std::min<uint64_t>(grid_for(n, 8), sms * 8), 256, 0,
                     op, L.list[CLS_AAG], L.cnt + CLS_AAG, dA, dB, En, O, b->d_pool, res_card);
  }
  if (uint64_t n = n_gen) {
    F.next();
    RS_LAUNCH_PROF("generic_pair", hcnt ? n : 0, k_pair_dense<true>, std::min<uint64_t>(n, sms * 8), DT, 0, op,
                   L.list[CLS_GEN], L.cnt + CLS_GEN, L.cnt + CNT_GEN, dA, dB, En, O, b->d_pool, res_card);
  }
  if (uint64_t n = n_prb) {
    F.next();
    RS_LAUNCH_PROF("probe_pair", hcnt ? n : 0, k_probe, std::min<uint64_t>(grid_for(n, PRB_WARPS), sms * 12),
                   32 * PRB_WARPS, 0, op,
                   L.list[CLS_PRB], L.cnt + CLS_PRB, dA, dB, En, O, b->d_pool, res_card);
  }
  RS_TRY(F.end());
  host_mark(8);
  // compaction: drop empty results (bitmap.py:185-188)
  if (single) {  // one CTA: kept count and cardinality computed in place
    RS_LAUNCH(k_compact_pair<256>, 1u, 256, 0, npairs, epos, (const uint32_t *)nullptr, En, O, b->d_key, b->d_type,
              b->d_card, b->d_n, b->d_off, b->d_bm_start, b->d_bm_card);
    b->h_valid = false;
    *out = b;
    host_mark(9);
    return RS_OK;
  }
  if (!mbase && epos && npairs) {  // per-pair entry bases: per-pair compaction
    uint32_t *nz = (uint32_t *)S.get((npairs + 1) * 4), *fb = (uint32_t *)S.get((npairs + 1) * 4);
    if (!S.ok()) { set_error("device allocation failed (compaction)"); return RS_ENOMEM; }
    const bool fuse = npairs <= FUSED_SCAN_MAX;
    RS_LAUNCH(k_pair_nonempty, (unsigned)npairs, 256, 0, npairs, epos, O.card, nz, fuse ? L.cnt + NCLS + 1 : nullptr,
              fb);
    if (!fuse) RS_TRY(scan_exclusive<uint32_t>(nz, fb, npairs + 1));
if (E > 1024 * npairs)
      RS_LAUNCH(k_compact_pair<1024>, (unsigned)npairs, 1024, 0, npairs, epos, fb, En, O, b->d_key, b->d_type,
                b->d_card, b->d_n, b->d_off, b->d_bm_start, b->d_bm_card);
    else
      RS_LAUNCH(k_compact_pair<256>, (unsigned)npairs, 256, 0, npairs, epos, fb, En, O, b->d_key, b->d_type,
                b->d_card, b->d_n, b->d_off, b->d_bm_start, b->d_bm_card);
    b->h_valid = false;
    *out = b;
    host_mark(9);
    return RS_OK;
  }
  RS_LAUNCH(k_keep_nonempty, grid_for(E + 1, 256), 256, 0, E, dE, O.card, keep2);
  RS_TRY(scan_exclusive<uint32_t>(keep2, fpos, E + 1));
  RS_LAUNCH(k_compact, grid_for(E, 256), 256, 0, E, dE, keep2, fpos, En, O, b->d_key, b->d_type, b->d_card, b->d_n,
            b->d_off);
  RS_LAUNCH(k_bm_start, grid_for(npairs + 1, 256), 256, 0, npairs, mbase, epos, fpos, b->d_bm_start);
  b->h_valid = false;
  *out = b;
  return RS_OK;
}

// device path of the merge bases for large pair lists: size kernel + scan
int pair_bases_device(uint64_t npairs, DevBatch dA, DevBatch dB, const uint32_t *dia, const uint32_t *dib,
                      int count_mode, uint64_t *msz, uint64_t *mbase) {
  RS_LAUNCH(k_pair_msize, grid_for(npairs + 1, 256), 256, 0, npairs, dA, dB, dia, dib, count_mode, msz);
  return scan_exclusive<uint64_t>(msz, mbase, npairs + 1);
}



// container_pairwise needs exactly one container per image (checked once per
// batch and cached, then per pair only when some image is not single)
int check_single_containers(const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib,
                            uint64_t npairs) {
  for (const rs_batch *X : {A, B}) {
    rs_batch *x = const_cast<rs_batch *>(X);
    if (x->single < 0) {  // 1: one container each; 2: at most one (some empty); 0: other
      x->single = 1;
      for (uint64_t i = 0; i < x->nb && x->single; i++) {
        const uint64_t k = x->h_bm_start[i + 1] - x->h_bm_start[i];
        if (k > 1) x->single = 0;
        else if (k == 0) x->single = 2;
      }
    }
  }
  if (A->single && B->single) return RS_OK;
  for (uint64_t p = 0; p < npairs; p++) {
    uint32_t a = ia ? ia[p] : (uint32_t)p, b = ib ? ib[p] : (uint32_t)p;
    if (a < A->nb && b < B->nb &&
        (A->h_bm_start[a + 1] - A->h_bm_start[a] > 1 || B->h_bm_start[b + 1] - B->h_bm_start[b] > 1)) {
      set_error("container_pairwise needs at most one container per image");
      return RS_ESHAPE;
    }
  }
  return RS_OK;
}

Lists make_lists(Scratch &S, uint64_t cap) {
  Lists L;
  L.cap = cap ? cap : 1;
  for (int c = 0; c < NCLS; c++) L.list[c] = (uint32_t *)S.get(L.cap * 4);
  L.cnt = (uint32_t *)S.get((NCLS + 4) * 4);  // + the fused-scan arrival counters, the large-pair item counter
  L.aoff = (uint64_t *)S.get(2 * L.cap * 8);  // [0,cap): bitset class, [cap,2cap): large-array class
  L.boff = (uint64_t *)S.get(2 * L.cap * 8);
  L.nab = (uint32_t *)S.get(L.cap * 4);
  return L;
}

}  // namespace

namespace {
// AND / ANDNOT through the A-indexed join (k_join_a): entries at A's
// container positions, 8 KB slots, per-pair compaction.  Ea = sum of the
// pairs' A container counts; npairs <= 16384 (host-computed bases).
int a_join_op(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib, uint64_t npairs,
              uint64_t Ea, rs_batch **out) {
  Scratch S;
  Upload U;
  const size_t o_ia = ia ? U.add(ia, npairs * 4) : Upload::NONE, o_ib = ib ? U.add(ib, npairs * 4) : Upload::NONE;
  std::vector<uint64_t> hb;
  pair_bases_host(A, B, ia, ib, npairs, 1, hb);  // A-side counts only
  std::vector<uint32_t> hb32(hb.begin(), hb.end());
  const size_t o_ab = U.add(hb.data(), (npairs + 1) * 8), o_ab32 = U.add(hb32.data(), (npairs + 1) * 4);
  const size_t o_cnt = U.add(nullptr, (NCLS + 4) * 4);
  Entries En;
  En.key = (uint16_t *)S.get((Ea + 1) * 2);
  En.ca = (uint32_t *)S.get((Ea + 1) * 4);
  En.cb = (uint32_t *)S.get((Ea + 1) * 4);
  En.pair = (uint32_t *)S.get((Ea + 1) * 4);
  En.off = (uint64_t *)S.get((Ea + 1) * 8);
  OutDesc O;
  O.type = (uint8_t *)S.get(Ea + 1);
  O.card = (uint32_t *)S.get((Ea + 1) * 4);
  O.n = (uint32_t *)S.get((Ea + 1) * 4);
  Lists L = make_lists(S, Ea);
  if (!S.ok()) { set_error("device allocation failed (op)"); return RS_ENOMEM; }
  RS_TRY(U.commit(S));
  L.cnt = U.at<uint32_t>(o_cnt);
  const uint64_t *abase = U.at<uint64_t>(o_ab);
  uint64_t maxa = 0;
  for (uint64_t p = 0; p < npairs; p++) maxa = std::max(maxa, hb[p + 1] - hb[p]);
  const uint32_t chunks = (uint32_t)std::max<uint64_t>((maxa + JA_CHUNK - 1) / JA_CHUNK, 1);
  RS_LAUNCH(k_join_a, (unsigned)(npairs * chunks), 256, 0, chunks, abase, A->dev(), B->dev(), U.at<uint32_t>(o_ia),
            U.at<uint32_t>(o_ib), op, En, O, L);
  host_mark(4);
  return run_classes_and_compact(op, A, B, S, En, L, Ea, 8192 * std::max<uint64_t>(Ea, 1), nullptr, nullptr,
                                 nullptr, U.at<uint32_t>(o_ab32), npairs, out, &O);
}
}  // namespace

extern "C" int rs_pairwise(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib,
                           uint64_t npairs, rs_batch **out) {
  host_mark(0);
  RS_TRY(check_op(op));
  RS_TRY(ensure_device());
  *out = nullptr;
  RS_TRY(fetch_host_meta(A));
  RS_TRY(fetch_host_meta(B));
  RS_TRY(check_pairs(A, B, ia, ib, npairs));
  host_mark(1);
  Scratch S;
  uint64_t M = 0, Ecap = 0, maxk = 0, Ea = 0;
  for (uint64_t p = 0; p < npairs; p++) {
    uint32_t a = ia ? ia[p] : (uint32_t)p, b = ib ? ib[p] : (uint32_t)p;
    uint64_t na = A->h_bm_start[a + 1] - A->h_bm_start[a], nb = B->h_bm_start[b + 1] - B->h_bm_start[b];
    M += na + nb;
    Ea += na;
    Ecap += op == RS_OP_AND ? std::min(na, nb) : op == RS_OP_ANDNOT ? na : na + nb;
    maxk = std::max(maxk, std::max(na, nb));
  }
  // Upper-bound mode (no host sync) when an 8 KB slot per possible output
  // container costs at most ~2x the inputs' pools; else size exactly.
  static const int ub_force = env_int("RS_UB_FORCE", 0);  // diagnostics: upper-bound slots whatever they cost
  auto ub_affordable = [&](uint64_t slots) {
    return ub_force || 8192.0 * (double)slots <= 2.0 * (double)(A->pool_bytes + B->pool_bytes) + 64e6;
  };
  if (npairs == 1 && single_path_on()) {  // one pair of small bitmaps: one launch (rs_single.cu)
    const uint32_t a = ia ? ia[0] : 0, b = ib ? ib[0] : 0;
    const uint32_t E = single_pair_slots(op, (uint32_t)(A->h_bm_start[a + 1] - A->h_bm_start[a]),
                                         (uint32_t)(B->h_bm_start[b + 1] - B->h_bm_start[b]));
    if (E <= SINGLE_MAX_SLOTS && ub_affordable(E) && env_int("RS_EXACT_ALLOC", 0) == 0) {
      const uint64_t P = 8192ull * std::max<uint32_t>(E, 1);
      RS_TRY(ub_reserve(P));
      rs_batch *r = new rs_batch();
      int rc = batch_alloc(r, 1, E, P);
      if (!rc) {
        ub_register(r);
        r->type_mask = result_mask(A->type_mask, B->type_mask);
        rc = single_pair_op(op, A, B, a, b, r);
      }
      if (rc) { rs_batch_free(r); return rc; }
      r->h_valid = false;
      *out = r;
      return RS_OK;
    }
  }
  const bool ub_mode = env_int("RS_EXACT_ALLOC", 0) == 0 && ub_affordable(Ecap);
  // per-pair path (CTA per pair, keys in smem, scans over pairs): when the
  // bitmaps are small enough for smem and there are enough pairs to fill the
  // GPU (or few positions per pair); a handful of pairs with thousands of keys
  // each (config 4) keep a thread-per-position join
  static const int force_pp = env_int("RS_PER_PAIR", -1);  // A/B: 1 forces, 0 disables the per-pair join
  const bool per_pair = M && maxk <= MERGE_SMEM_KEYS &&
                        (force_pp >= 0 ? force_pp == 1 : (npairs >= 2 * sm_count() || M <= 1024 * npairs));
  // AND / ANDNOT otherwise join on A's positions (no scans, no emit pass)
  // -- and, since one k_join_a launch replaces the per-pair path's merge /
  // match / emit passes, also for per-pair batches of at least
  // RS_AJOIN_MIN_SLOTS A containers (default 32,768) averaging 8 or more per
  // pair (config 2: AND 1.19 -> 1.11 ms, ANDNOT 1.045 -> 1.016; 4,096 pairs
  // x 16 keys: AND 0.137 -> 0.117 ms, ANDNOT 0.205 -> 0.195; 16,384 pairs x
  // 4 keys and 256 pairs x 32 keys measured 3 and 10 % slower and keep the
  // per-pair join; tools/probe_join.py); RS_AJOIN=0 keeps the
  // merged-position join
  static const int ajoin = env_int("RS_AJOIN", 1);
  static const int ajoin_min_slots = env_int("RS_AJOIN_MIN_SLOTS", 32768);
  const bool ajoin_over_pp = force_pp < 0 && Ea >= (uint64_t)ajoin_min_slots && Ea >= 8 * npairs;
  if (ajoin && (op == RS_OP_AND || op == RS_OP_ANDNOT) && (!per_pair || ajoin_over_pp) && npairs <= 16384 &&
      env_int("RS_EXACT_ALLOC", 0) == 0 && ub_affordable(Ea))
    return a_join_op(op, A, B, ia, ib, npairs, Ea, out);
  Upload U;
  const size_t o_ia = ia ? U.add(ia, npairs * 4) : Upload::NONE, o_ib = ib ? U.add(ib, npairs * 4) : Upload::NONE;
  std::vector<uint64_t> hb;
  const bool hbases = pair_bases_host(A, B, ia, ib, npairs, 0, hb);
  const size_t o_mb = hbases ? U.add(hb.data(), (npairs + 1) * 8) : Upload::NONE;
  const size_t o_cnt = U.add(nullptr, (NCLS + 4) * 4);
  uint64_t *msz = hbases ? nullptr : (uint64_t *)S.get((npairs + 1) * 8);
  uint64_t *mbase = hbases ? nullptr : (uint64_t *)S.get((npairs + 1) * 8);
  uint16_t *mkey = (uint16_t *)S.get((M + 1) * 2);
  uint32_t *mca = (uint32_t *)S.get((M + 1) * 4), *mcb = (uint32_t *)S.get((M + 1) * 4),
           *mpair = (uint32_t *)S.get((M + 1) * 4), *keep = (uint32_t *)S.get((M + 1) * 4),
           *epos = (uint32_t *)S.get((M + 1) * 4);
  uint64_t *ub = (uint64_t *)S.get((M + 1) * 8), *uoff = (uint64_t *)S.get((M + 1) * 8);
  Entries En;
  En.key = (uint16_t *)S.get((M + 1) * 2);
  En.ca = (uint32_t *)S.get((M + 1) * 4);
  En.cb = (uint32_t *)S.get((M + 1) * 4);
  En.pair = (uint32_t *)S.get((M + 1) * 4);
  En.off = (uint64_t *)S.get((M + 1) * 8);
  Lists L = make_lists(S, M);
  if (!S.ok()) { set_error("device allocation failed (op)"); return RS_ENOMEM; }
  host_mark(2);
  RS_TRY(U.commit(S));
  host_mark(3);
  const uint32_t *dia = U.at<uint32_t>(o_ia), *dib = U.at<uint32_t>(o_ib);
  L.cnt = U.at<uint32_t>(o_cnt);
  DevBatch dA = A->dev(), dB = B->dev();
  if (hbases) mbase = U.at<uint64_t>(o_mb);
  else RS_TRY(pair_bases_device(npairs, dA, dB, dia, dib, 0, msz, mbase));
  if (M == 0) {  // k_merge writes these sentinels otherwise
    RS_CK(cudaMemsetAsync(keep, 0, 4, g_stream));
    RS_CK(cudaMemsetAsync(ub, 0, 8, g_stream));
  }
  if (per_pair) {
    // the join, then entry / slot bases from scans over pairs
    uint32_t *pk = (uint32_t *)S.get((npairs + 1) * 4), *pke = (uint32_t *)S.get((npairs + 1) * 4);
    uint64_t *pu = (uint64_t *)S.get((npairs + 1) * 8), *pue = (uint64_t *)S.get((npairs + 1) * 8);
    if (!S.ok()) { set_error("device allocation failed (op)"); return RS_ENOMEM; }
    const bool fuse = npairs <= FUSED_SCAN_MAX;
    if (npairs == 1 && ub_mode) {  // join + emit in one CTA (no scans over pairs)
      RS_LAUNCH(k_merge_emit1, 1u, 256, 0, dA, dB, dia, dib, op, mkey, mca, mcb, mpair, keep, ub, pke, pue, En, L);
    } else {
      RS_LAUNCH(k_merge_pair, (unsigned)npairs, 256, 0, M, npairs, mbase, dA, dB, dia, dib, op, mkey, mca, mcb, mpair,
                keep, ub, pk, pu, fuse ? L.cnt + NCLS : nullptr, pke, pue);
      if (!fuse) {
        RS_TRY(scan_exclusive<uint32_t>(pk, pke, npairs + 1));
        RS_TRY(scan_exclusive<uint64_t>(pu, pue, npairs + 1));
      }
      RS_LAUNCH(k_emit_pair, (unsigned)npairs, 256, 0, mbase, keep, ub, pke, pue, mkey, mca, mcb, mpair, dA, dB, En,
                L, op);
    }
    host_mark(4);
    if (ub_mode)
      return run_classes_and_compact(op, A, B, S, En, L, M, 8192 * std::max<uint64_t>(Ecap, 1), nullptr,
                                     pke + npairs, nullptr, pke, npairs, out);
    struct { uint32_t E; uint32_t pad; uint64_t P; uint32_t cnt[NCLS]; } h;
    RS_CK(cudaMemcpyAsync(&h.E, pke + npairs, 4, cudaMemcpyDeviceToHost, g_stream));
    RS_CK(cudaMemcpyAsync(&h.P, pue + npairs, 8, cudaMemcpyDeviceToHost, g_stream));
    RS_CK(cudaMemcpyAsync(h.cnt, L.cnt, NCLS * 4, cudaMemcpyDeviceToHost, g_stream));
    RS_CK(cudaStreamSynchronize(g_stream));
    return run_classes_and_compact(op, A, B, S, En, L, h.E, h.P, h.cnt, nullptr, nullptr, pke, npairs, out);
  }
  if (M)
    RS_LAUNCH(k_merge, grid_for(M, 256), 256, 0, M, npairs, mbase, dA, dB, dia, dib, op, mkey, mca, mcb, mpair, keep,
              ub);
  host_mark(10);
  RS_TRY(scan_exclusive<uint32_t>(keep, epos, M + 1));
  RS_TRY(scan_exclusive<uint64_t>(ub, uoff, M + 1));
  host_mark(11);
  RS_LAUNCH(k_emit, grid_for(M, 256), 256, 0, M, keep, epos, uoff, mkey, mca, mcb, mpair, dA, dB, En, L, op);
  host_mark(12);
  if (ub_mode)
    return run_classes_and_compact(op, A, B, S, En, L, M, 8192 * std::max<uint64_t>(Ecap, 1), nullptr, epos + M,
                                   mbase, epos, npairs, out);
  // exact mode: one host sync for the totals, then exact grids
  struct { uint32_t E; uint32_t pad; uint64_t P; uint32_t cnt[NCLS]; } h;
  RS_CK(cudaMemcpyAsync(&h.E, epos + M, 4, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaMemcpyAsync(&h.P, uoff + M, 8, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaMemcpyAsync(h.cnt, L.cnt, NCLS * 4, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaStreamSynchronize(g_stream));
  return run_classes_and_compact(op, A, B, S, En, L, h.E, h.P, h.cnt, nullptr, mbase, epos, npairs, out);
}

extern "C" int rs_container_pairwise(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia,
                                     const uint32_t *ib, uint64_t npairs, rs_batch **out) {
  RS_TRY(check_op(op));
  RS_TRY(ensure_device());
  *out = nullptr;
  RS_TRY(fetch_host_meta(A));
  RS_TRY(fetch_host_meta(B));
  RS_TRY(check_single_containers(A, B, ia, ib, npairs));
  RS_TRY(check_pairs(A, B, ia, ib, npairs));
  Scratch S;
  Upload U;
  const size_t o_ia = ia ? U.add(ia, npairs * 4) : Upload::NONE, o_ib = ib ? U.add(ib, npairs * 4) : Upload::NONE;
  const size_t o_cnt = U.add(nullptr, (NCLS + 4) * 4);
  Entries En;
  En.key = (uint16_t *)S.get((npairs + 1) * 2);
  En.ca = (uint32_t *)S.get((npairs + 1) * 4);
  En.cb = (uint32_t *)S.get((npairs + 1) * 4);
  En.pair = (uint32_t *)S.get((npairs + 1) * 4);
  En.off = (uint64_t *)S.get((npairs + 1) * 8);
  uint64_t *ub = (uint64_t *)S.get((npairs + 1) * 8);
  Lists L = make_lists(S, npairs);
  if (!S.ok()) { set_error("device allocation failed (container op)"); return RS_ENOMEM; }
  RS_TRY(U.commit(S));
  const uint32_t *dia = U.at<uint32_t>(o_ia), *dib = U.at<uint32_t>(o_ib);
  L.cnt = U.at<uint32_t>(o_cnt);
  DevBatch dA = A->dev(), dB = B->dev();
  RS_LAUNCH(k_cont_entries, grid_for(npairs + 1, 256), 256, 0, npairs, dA, dB, dia, dib, op, En, ub, L);
  RS_TRY(scan_exclusive<uint64_t>(ub, En.off, npairs + 1));
  // Array-only inputs with the identity pairing: every result slot is at most
  // 2(na + nb) bytes (+16 pad), so the input pools bound the result pool and
  // the op needs no host synchronization.
  const uint8_t AR = 1 << RS_TAG_ARRAY;
  // (empty images need the exact class counts: their entries go through k_copy)
  if (!ia && !ib && A->type_mask == AR && B->type_mask == AR && A->single == 1 && B->single == 1 &&
      env_int("RS_EXACT_ALLOC", 0) == 0) {
    const uint64_t Pub = A->pool_bytes + B->pool_bytes + 16 * npairs;
    return run_classes_and_compact(op, A, B, S, En, L, npairs, Pub, nullptr, nullptr, nullptr, nullptr, npairs,
                                   out);
  }
  uint64_t P = 0;
  uint32_t cnt[NCLS];
  RS_CK(cudaMemcpyAsync(&P, En.off + npairs, 8, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaMemcpyAsync(cnt, L.cnt, NCLS * 4, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaStreamSynchronize(g_stream));
  return run_classes_and_compact(op, A, B, S, En, L, npairs, P, cnt, nullptr, nullptr, nullptr, npairs, out);
}

namespace {
int launch_counts(int op_kernel, const rs_batch *A, const rs_batch *B, Lists L, uint32_t *lcb, uint32_t *lpair,
                  uint64_t *inter) {
  DevBatch dA = A->dev(), dB = B->dev();
  const ClassMask cm = class_mask(A->type_mask, B->type_mask, RS_OP_AND);
  // Persistent grids, but never more CTAs than the list can fill (one item
  // per warp / per CTA): a one-pair call of a few thousand container pairs
  // would otherwise launch 1184 mostly idle CTAs per class kernel.
  const unsigned pg = std::min<uint64_t>(sm_count() * 8, grid_for(L.cap, 8));
  const unsigned pg_cta = std::min<uint64_t>(sm_count() * 8, std::max<uint64_t>(L.cap, 1));
  const int nk = cm.bb + cm.aa + cm.gen + cm.prb;  // independent: concurrent on side streams
  Fork F;
  if (nk > 1 && L.cap >= 16384) RS_TRY(F.begin(nk));
  if (cm.bb) {
    F.next();
    if (bb_kernel_choice() == 0) {
      RS_LAUNCH_PROF("bitset_count", 0, k_pair_count<false>, pg_cta, DT, 0, op_kernel, L.list[CLS_BB],
                     lcb + CLS_BB * L.cap, lpair + CLS_BB * L.cap, L.cnt + CLS_BB, dA, dB, inter);
    } else {
      uint32_t *lp = lpair + CLS_BB * L.cap;
      switch (bb_stages()) {
        case 3: RS_TRY(launch_bb_count<3>(op_kernel, L, lp, dA, dB, inter)); break;
        case 4: RS_TRY(launch_bb_count<4>(op_kernel, L, lp, dA, dB, inter)); break;
        default: RS_TRY(launch_bb_count<2>(op_kernel, L, lp, dA, dB, inter)); break;
      }
    }
  }
  if (cm.aa) {
    F.next();
    if (env_int_("RS_AA_SMALL_PLAIN", 0))  // the warp-per-pair kernel (A/B only)
      RS_LAUNCH_PROF("array_count_s", 0, (k_aa_count<32, 8>), pg, 256, 0, L.list[CLS_AAS], lcb + CLS_AAS * L.cap,
                     lpair + CLS_AAS * L.cap, L.cnt + CLS_AAS, dA, dB, inter);
    else
      RS_LAUNCH_PROF("array_count_s", 0, k_aa_count_small, pg, 256, 0, L.list[CLS_AAS], lcb + CLS_AAS * L.cap,
                     lpair + CLS_AAS * L.cap, L.cnt + CLS_AAS, dA, dB, inter);
    if (aa_medium_possible())
    {
      if (g_aa_large_min <= 512)
        RS_LAUNCH_PROF("array_count_m", 0, (k_aa_count<32, 16>), pg, 256, 0, L.list[CLS_AAM], lcb + CLS_AAM * L.cap,
                       lpair + CLS_AAM * L.cap, L.cnt + CLS_AAM, dA, dB, inter);
      else
        RS_LAUNCH_PROF("array_count_m", 0, (k_aa_count<128, 16>), pg, 256, 0, L.list[CLS_AAM], lcb + CLS_AAM * L.cap,
                       lpair + CLS_AAM * L.cap, L.cnt + CLS_AAM, dA, dB, inter);
    }
    if (env_int("RS_AA_LARGE_MERGE", 0))
      RS_LAUNCH_PROF("array_count_l", 0, (k_aa_count<256, 32>), pg, 256, 0, L.list[CLS_AAL], lcb + CLS_AAL * L.cap,
                     lpair + CLS_AAL * L.cap, L.cnt + CLS_AAL, dA, dB, inter);
    else
      RS_TRY(launch_aa_large_count(L, lpair + CLS_AAL * L.cap, dA, dB, inter));
    RS_LAUNCH_PROF("array_count_g", 0, k_aa_gallop_count, pg, 256, 0, L.list[CLS_AAG], lcb + CLS_AAG * L.cap,
                   lpair + CLS_AAG * L.cap, L.cnt + CLS_AAG, dA, dB, inter);
  }
  if (cm.gen) {
    F.next();
    RS_LAUNCH_PROF("generic_count", 0, k_pair_count<true>, pg_cta, DT, 0, op_kernel, L.list[CLS_GEN],
                   lcb + CLS_GEN * L.cap, lpair + CLS_GEN * L.cap, L.cnt + CLS_GEN, dA, dB, inter);
  }
  if (cm.prb) {
    F.next();
    RS_LAUNCH_PROF("probe_count", 0, k_probe_count, std::min<uint64_t>(sm_count() * 12, grid_for(L.cap, PRB_WARPS)),
                   32 * PRB_WARPS, 0, L.list[CLS_PRB],
                   lcb + CLS_PRB * L.cap,
                   lpair + CLS_PRB * L.cap, L.cnt + CLS_PRB, dA, dB, inter);
  }
  return F.end();
}
}  // namespace

// ---------------------------------------------- small count calls: graphs
//
// A few-pair count (config 1: one pair, ~10 launches of tiny grids, then a
// synchronizing read-back) is host- and launch-latency-bound.  Its launch
// sequence is captured once into a CUDA graph and replayed: everything the
// kernels see -- the batches' device arrays, the scratch addresses (the bump
// arena is deterministic for an identical call), the grid sizes (derived from
// the container counts and type masks) -- is in the key, and the per-call
// inputs (pair indices, bases) go through a page-locked upload block that the
// graph's first node copies to the device; the counts come back through a
// page-locked block the last node fills.  RS_NO_GRAPH=1 disables it.
struct CountGraphKey {
  DevBatch a, b;
  uint64_t amask, bmask, op, on_dev, npairs, Ma, maxk, up_bytes, top;
  const void *arena, *counts, *stream;
};
struct CountGraph {
  CountGraphKey key;
  cudaGraphExec_t exec = nullptr;
  void *h_up = nullptr, *h_out = nullptr;
  uint64_t launches = 0, last_use = 0;
};
std::vector<CountGraph> g_count_graphs;
uint64_t g_count_graph_clock = 0;
constexpr size_t COUNT_GRAPHS_MAX = 16;
// A key is captured on its third sighting (capture + instantiation cost
// ~1 ms: a stream of distinct one-off calls must never pay it); keys whose
// capture failed are not retried.
struct SeenKey {
  CountGraphKey key;
  uint32_t hits;
};
std::vector<SeenKey> g_count_seen;  // small ring of recent keys
size_t g_count_seen_next = 0;
constexpr size_t COUNT_SEEN_MAX = 64;
constexpr uint32_t COUNT_CAPTURE_AFTER = 3, COUNT_CAPTURE_FAILED = ~0u;

uint32_t count_key_sighting(const CountGraphKey &k) {
  for (auto &e : g_count_seen)
    if (!memcmp(&e.key, &k, sizeof k)) return e.hits == COUNT_CAPTURE_FAILED ? e.hits : ++e.hits;
  if (g_count_seen.size() < COUNT_SEEN_MAX) g_count_seen.push_back({k, 1});
  else g_count_seen[g_count_seen_next++ % COUNT_SEEN_MAX] = {k, 1};
  return 1;
}
void count_key_failed(const CountGraphKey &k) {
  for (auto &e : g_count_seen)
    if (!memcmp(&e.key, &k, sizeof k)) e.hits = COUNT_CAPTURE_FAILED;
}

void count_graph_free(CountGraph &g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.h_up) cudaFreeHost(g.h_up);
  if (g.h_out) cudaFreeHost(g.h_out);
  g.exec = nullptr;
  g.h_up = g.h_out = nullptr;
}

CountGraph *count_graph_find(const CountGraphKey &k) {
  for (auto &g : g_count_graphs)
    if (!memcmp(&g.key, &k, sizeof k)) {
      g.last_use = ++g_count_graph_clock;
      return &g;
    }
  return nullptr;
}

extern "C" int rs_pairwise_cardinality(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia,
                                       const uint32_t *ib, uint64_t npairs, uint64_t *counts, int counts_on_device) {
  RS_TRY(check_op(op));
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(A));
  RS_TRY(fetch_host_meta(B));
  if (!counts_on_device) {  // host readback: surface deferred decode errors
    RS_TRY(resolve_pending(A));
    RS_TRY(resolve_pending(B));
  }
  RS_TRY(check_pairs(A, B, ia, ib, npairs));
  if (npairs == 1 && single_path_on()) {  // one pair of small bitmaps: one launch (rs_single.cu)
    const uint32_t a = ia ? ia[0] : 0, b = ib ? ib[0] : 0;
    if (A->h_bm_start[a + 1] - A->h_bm_start[a] <= SINGLE_MAX_SLOTS) {
      if (counts_on_device) return single_pair_count(op, A, B, a, b, counts);
      thread_local uint64_t *h = nullptr;  // page-locked: the kernel writes the count there
      if (!h) RS_CK(cudaMallocHost(&h, 64));
      RS_TRY(single_pair_count(op, A, B, a, b, h));
      RS_CK(cudaStreamSynchronize(g_stream));
      *counts = *(volatile uint64_t *)h;
      return RS_OK;
    }
  }
  Scratch S;
  uint64_t Ma = 0, maxk = 0;
  for (uint64_t p = 0; p < npairs; p++) {
    uint32_t a = ia ? ia[p] : (uint32_t)p, b = ib ? ib[p] : (uint32_t)p;
    const uint64_t na = A->h_bm_start[a + 1] - A->h_bm_start[a];
    Ma += na;
    maxk = std::max(maxk, std::max(na, B->h_bm_start[b + 1] - B->h_bm_start[b]));
  }
  Upload U;
  const size_t o_ia = ia ? U.add(ia, npairs * 4) : Upload::NONE, o_ib = ib ? U.add(ib, npairs * 4) : Upload::NONE;
  std::vector<uint64_t> hb;
  const bool hbases = pair_bases_host(A, B, ia, ib, npairs, 1, hb);
  const size_t o_mb = hbases ? U.add(hb.data(), (npairs + 1) * 8) : Upload::NONE;
  const size_t o_cnt = U.add(nullptr, (NCLS + 4) * 4);
  const size_t o_inter = npairs <= 16384 ? U.add(nullptr, (npairs + 1) * 8) : Upload::NONE;
  const size_t top0 = Scratch::top;
  uint64_t *msz = hbases ? nullptr : (uint64_t *)S.get((npairs + 1) * 8);
  uint64_t *mbase = hbases ? nullptr : (uint64_t *)S.get((npairs + 1) * 8);
  Lists L = make_lists(S, Ma);
  uint32_t *lcb = (uint32_t *)S.get(NCLS * L.cap * 4), *lpair = (uint32_t *)S.get(NCLS * L.cap * 4);
  uint64_t *inter = o_inter == Upload::NONE ? (uint64_t *)S.get((npairs + 1) * 8) : nullptr;
  uint64_t *dout = counts_on_device ? counts : (uint64_t *)S.get((npairs + 1) * 8);
  U.d = U.h.empty() ? nullptr : (uint8_t *)S.get(U.h.size());
  if (!S.ok() || (!U.h.empty() && !U.d)) { set_error("device allocation failed (count)"); return RS_ENOMEM; }
  const uint32_t *dia = U.at<uint32_t>(o_ia), *dib = U.at<uint32_t>(o_ib);
  L.cnt = U.at<uint32_t>(o_cnt);
  DevBatch dA = A->dev(), dB = B->dev();
  if (hbases) mbase = U.at<uint64_t>(o_mb);
  if (!inter) inter = U.at<uint64_t>(o_inter);

  // the whole device side of the call; `up` is the host block to upload from
  static const bool gdbg = env_int("RS_GRAPH_DEBUG", 0) != 0;
  auto stage = [&](const char *what) {
    if (!gdbg) return;
    cudaStreamCaptureStatus st;
    if (cudaStreamIsCapturing(g_stream, &st) == cudaSuccess && st == cudaStreamCaptureStatusInvalidated)  // (g_stream = the capture stream here)
      fprintf(stderr, "[rs graph] capture invalidated by: %s\n", what);
  };
  auto enqueue = [&](const void *up, uint64_t *hout) -> int {
    RS_TRY(h2d_small(U.d, up, U.h.size()));
    stage("upload");
    if (o_inter == Upload::NONE) RS_CK(cudaMemsetAsync(inter, 0, (npairs + 1) * 8, g_stream));
    if (!hbases) RS_TRY(pair_bases_device(npairs, dA, dB, dia, dib, 1, msz, mbase));
    if (Ma && maxk <= MERGE_SMEM_KEYS && (npairs >= 2 * sm_count() || Ma <= 512 * npairs))
      RS_LAUNCH(k_match_pair, (unsigned)npairs, 256, 0, mbase, dA, dB, dia, dib, L, lcb, lpair);
    else
      RS_LAUNCH(k_match, grid_for(Ma, 256), 256, 0, Ma, npairs, mbase, dA, dB, dia, dib, L, lcb, lpair);
    stage("match");
    RS_TRY(launch_counts(RS_OP_AND, A, B, L, lcb, lpair, inter));
    stage("counts");
    RS_LAUNCH(k_formula, grid_for(npairs, 256), 256, 0, npairs, op, A->d_bm_card, B->d_bm_card, dia, dib, inter,
              dout);
    if (hout) RS_CK(cudaMemcpyAsync(hout, dout, npairs * 8, cudaMemcpyDeviceToHost, g_stream));
    return RS_OK;
  };

  static const bool graphs_on = env_int("RS_NO_GRAPH", 0) == 0;
  // (host read-back calls only: their synchronization is what makes the
  // page-locked upload block free for the next call)
  if (graphs_on && !counts_on_device && npairs <= 64 && hbases && o_inter != Upload::NONE && S.spill.empty() &&
      !g_prof_on) {
    CountGraphKey k;
    memset(&k, 0, sizeof k);
    k.a = dA;
    k.b = dB;
    k.amask = A->type_mask;
    k.bmask = B->type_mask;
    k.op = (uint64_t)op;
    k.on_dev = (uint64_t)counts_on_device;
    k.npairs = npairs;
    k.Ma = Ma;
    k.maxk = maxk;
    k.up_bytes = U.h.size();
    k.top = top0;
    k.arena = Scratch::arena;
    k.counts = counts_on_device ? counts : nullptr;
    k.stream = g_stream;
    CountGraph *g = count_graph_find(k);
    static const bool dbg = env_int("RS_GRAPH_DEBUG", 0) != 0;
    const uint32_t seen = g ? 0 : count_key_sighting(k);
    if (!g && seen >= COUNT_CAPTURE_AFTER && seen != COUNT_CAPTURE_FAILED) {
      CountGraph ng;
      ng.key = k;
      if (cudaMallocHost(&ng.h_up, std::max<size_t>(U.h.size(), 16)) == cudaSuccess &&
          cudaMallocHost(&ng.h_out, std::max<uint64_t>(npairs * 8, 16)) == cudaSuccess) {
        const uint64_t l0 = g_launches;
        cudaGraph_t graph = nullptr;
        // captured on a private stream (the library stream may be the legacy
        // default stream, which cannot be captured); the graph is launched
        // on the library stream
        static cudaStream_t cap = nullptr;
        static int cap_dev = -1;
        int dev = 0;
        cudaGetDevice(&dev);
        if (cap && cap_dev != dev) cap = nullptr;  // (leaked per device switch; rare)
        if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess) cap_dev = dev;
        cudaError_t e = cap ? cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) : cudaErrorNotReady;
        bool ok = e == cudaSuccess;
        if (ok) {
          const cudaStream_t saved = g_stream;
          g_stream = cap;
          const int rc = enqueue(ng.h_up, counts_on_device ? nullptr : (uint64_t *)ng.h_out);
          g_stream = saved;
          e = cudaStreamEndCapture(cap, &graph);
          ok = e == cudaSuccess && rc == RS_OK && graph;
          if (dbg && rc != RS_OK) fprintf(stderr, "[rs graph] capture enqueue failed: %s\n", rs_last_error());
        }
        if (ok) ok = (e = cudaGraphInstantiate(&ng.exec, graph, 0)) == cudaSuccess;
        if (dbg) fprintf(stderr, "[rs graph] capture npairs=%llu Ma=%llu: %s\n", (unsigned long long)npairs,
                         (unsigned long long)Ma, ok ? "ok" : cudaGetErrorString(e));
        if (!ok) count_key_failed(k);
        if (graph) cudaGraphDestroy(graph);
        ng.launches = g_launches - l0;
        g_launches = l0;
        cudaGetLastError();  // a failed capture falls back to plain launches
        if (ok) {
          if (g_count_graphs.size() >= COUNT_GRAPHS_MAX) {  // evict the least recently used
            auto lru = std::min_element(g_count_graphs.begin(), g_count_graphs.end(),
                                        [](const CountGraph &x, const CountGraph &y) { return x.last_use < y.last_use; });
            count_graph_free(*lru);
            g_count_graphs.erase(lru);
          }
          ng.last_use = ++g_count_graph_clock;
          g_count_graphs.push_back(ng);
          g = &g_count_graphs.back();
        }
      }
      if (!g) count_graph_free(ng);
    }
    if (g) {
      memcpy(g->h_up, U.h.data(), U.h.size());
      RS_CK(cudaGraphLaunch(g->exec, g_stream));
      g_launches += g->launches;
      if (!counts_on_device) {
        RS_CK(cudaStreamSynchronize(g_stream));
        memcpy(counts, g->h_out, npairs * 8);
      }
      return RS_OK;
    }
  }
  RS_TRY(enqueue(U.h.data(), nullptr));
  if (!counts_on_device) RS_TRY(d2h(counts, dout, npairs * 8));
  return RS_OK;
}

extern "C" int rs_container_pairwise_cardinality(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia,
                                                 const uint32_t *ib, uint64_t npairs, uint64_t *counts,
                                                 int counts_on_device) {
  RS_TRY(check_op(op));
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(A));
  RS_TRY(fetch_host_meta(B));
  if (!counts_on_device) {  // host readback: surface deferred decode errors
    RS_TRY(resolve_pending(A));
    RS_TRY(resolve_pending(B));
  }
  RS_TRY(check_single_containers(A, B, ia, ib, npairs));
  RS_TRY(check_pairs(A, B, ia, ib, npairs));
  Scratch S;
  Upload U;
  const size_t o_ia = ia ? U.add(ia, npairs * 4) : Upload::NONE, o_ib = ib ? U.add(ib, npairs * 4) : Upload::NONE;
  const size_t o_cnt = U.add(nullptr, (NCLS + 4) * 4);
  const size_t o_inter = npairs <= 16384 ? U.add(nullptr, (npairs + 1) * 8) : Upload::NONE;
  Lists L = make_lists(S, npairs);
  uint32_t *lcb = (uint32_t *)S.get(NCLS * L.cap * 4), *lpair = (uint32_t *)S.get(NCLS * L.cap * 4);
  uint64_t *inter = o_inter == Upload::NONE ? (uint64_t *)S.get((npairs + 1) * 8) : nullptr;
  uint64_t *dout = counts_on_device ? counts : (uint64_t *)S.get((npairs + 1) * 8);
  if (!S.ok()) { set_error("device allocation failed (count)"); return RS_ENOMEM; }
  RS_TRY(U.commit(S));
  const uint32_t *dia = U.at<uint32_t>(o_ia), *dib = U.at<uint32_t>(o_ib);
  L.cnt = U.at<uint32_t>(o_cnt);
  if (inter) RS_CK(cudaMemsetAsync(inter, 0, (npairs + 1) * 8, g_stream));
  else inter = U.at<uint64_t>(o_inter);
  DevBatch dA = A->dev(), dB = B->dev();
  RS_LAUNCH(k_cont_list, grid_for(npairs, 256), 256, 0, npairs, dA, dB, dia, dib, L, lcb, lpair);
  RS_TRY(launch_counts(RS_OP_AND, A, B, L, lcb, lpair, inter));
  RS_LAUNCH(k_formula_containers, grid_for(npairs, 256), 256, 0, npairs, op, dA, dB, dia, dib, inter, dout);
  if (!counts_on_device) RS_TRY(d2h(counts, dout, npairs * 8));
  return RS_OK;
}
