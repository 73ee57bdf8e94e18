// rs_single.cu -- one bitmap pair in ONE launch: RoaringBitmap.op and
// op_cardinality of a single pair (bitmap.py:169-241), the call a user of the
// reference's class makes (`a & b`, `a.and_cardinality(b)`).
//
// The batched pipeline (rs_pairwise.cu) spends 5-7 launches on a call --
// join, emit, one kernel per container-type class, compaction -- which for a
// pair of a few dozen containers is launch and host bound (~25 us per call
// against ~5 us of device work).  Here a CTA takes one container of either
// side and does everything for its key:
//   join      the key's rank in the other side's sorted keys (two rounds of
//             a CTA-wide sampled search: no serial binary-search chain);
//   result    a matched key: container_pairwise through the 8 KB shared
//             bitsets (rsd::dense_pair: every type pair, the exact result-type
//             choice); an unmatched key kept by the op: a copy
//             (bitmap.py:191-209); dropped otherwise;
//   slot      the key's position in the merged key order, whose 8 KB slot of
//             the result pool it writes (upper-bound layout, packed later by
//             repack_pool like every op result);
//   compact   the last CTA to finish (a self-resetting ticket) drops empty
//             results in place and writes the bitmap's range and cardinality
//             (bitmap.py:185-188).
// The count kernel sums |a AND b| over matched keys and applies the
// cardinality formulas (bitmap.py:225-241) in its last CTA, writing the count
// straight to its destination (device memory, or page-locked host memory).
#include <cub/cub.cuh>
#include <atomic>
#include <mutex>
#include "rs_internal.cuh"
#include "rs_dense.cuh"
#include "rs_single.h"

using namespace rs;
using namespace rsd;

namespace {

// Self-resetting completion tickets (zero at module load; each call's last
// CTA puts its ticket back to zero), rotated per call so back-to-back calls
// on different streams do not share one.
constexpr int NTICKET = 256;
__device__ uint32_t g_ticket[NTICKET];
__device__ unsigned long long g_acc[NTICKET];

// Rank of x in the sorted keys k[0, n): #{keys < x}, by the whole CTA in two
// dependent rounds of loads (a sample every `step` keys, then the step's
// keys), n <= 256 * 256.
__device__ __forceinline__ uint32_t cta_rank(const uint16_t *__restrict__ k, uint32_t n, uint32_t x) {
  if (n == 0) return 0;
  const uint32_t step = (n + DT - 1) / DT, t = threadIdx.x;
  const uint32_t p = t * step;
  const uint32_t c1 = (uint32_t)__syncthreads_count(p < n && k[p] < x);
  if (c1 == 0) return 0;
  const uint32_t base = (c1 - 1) * step + 1;  // keys [.., base) are < x; keys from base + step - 1 on are not
  const uint32_t q = base + t;
  const uint32_t c2 = (uint32_t)__syncthreads_count(t + 1 < step && q < n && k[q] < x);
  return base + c2;
}

// Rank of x in the other side's keys: staged in shared memory when they fit
// (one coalesced load instead of two dependent rounds from L2).
constexpr uint32_t SMEM_KEYS = 2048;
__device__ __forceinline__ uint32_t side_rank(const uint16_t *__restrict__ k, uint32_t n, uint32_t x,
                                              uint16_t *kbuf) {
  if (n > SMEM_KEYS) return cta_rank(k, n, x);
  for (uint32_t u = threadIdx.x; u < n; u += DT) kbuf[u] = k[u];
  __syncthreads();
  return cta_rank(kbuf, n, x);
}

__device__ __forceinline__ bool last_cta(uint32_t *ticket) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// CTA-wide copy of a container's payload (16-byte units, padded).
__device__ __forceinline__ void copy_payload(const DevBatch &S, uint32_t c, uint8_t *dst) {
  const uint32_t nv = (uint32_t)(rs_pad16(rs_payload_bytes(S.type[c], S.n[c])) >> 4);
  const uint4 *src = (const uint4 *)(S.pool + S.off[c]);
  for (uint32_t i = threadIdx.x; i < nv; i += DT) ((uint4 *)dst)[i] = __ldg(src + i);
}

// Grid: AND / ANDNOT one CTA per container of a (slot = its index: the result
// keeps a's key order); OR / XOR one per container of a, then one per
// container of b (slot = the key's rank in a plus its rank in b -- every key
// of the union gets a distinct slot, and a matched key leaves the slot after
// it empty, which its a-side CTA marks).  E slots in all; gridDim.x >= 1.
template <int OP>
__global__ void __launch_bounds__(DT) k_single_op(DevBatch A, DevBatch B, uint32_t a0, uint32_t na, uint32_t b0,
                                                  uint32_t nb, uint32_t E,
                                                  uint16_t *__restrict__ key, uint8_t *__restrict__ type,
                                                  uint32_t *__restrict__ card, uint32_t *__restrict__ nn,
                                                  uint64_t *__restrict__ off, uint8_t *__restrict__ opool,
                                                  uint64_t *__restrict__ bm_start, uint64_t *__restrict__ bm_card,
                                                  uint32_t *ticket) {
  __shared__ __align__(16) DenseSmem sm;
  __shared__ uint16_t kbuf[SMEM_KEYS];
  constexpr bool KEEP_B = OP == RS_OP_OR || OP == RS_OP_XOR;
  const int t = threadIdx.x;
  const uint32_t i = blockIdx.x;
  if (i < na) {  // ------------------------------------------------ a's container
    const uint32_t ca = a0 + i;
    const uint16_t k = A.key[ca];
    const uint32_t j = side_rank(B.key + b0, nb, k, kbuf);
    const bool matched = j < nb && B.key[b0 + j] == k;
    const uint32_t s = KEEP_B ? i + j : i;
    uint8_t ty = RS_TAG_ARRAY;
    uint32_t c = 0, n = 0;
    if (matched) {
      const uint32_t cb = b0 + j;
      c = dense_pair<true>(OP, A, ca, A.type[ca], B, cb, B.type[cb], sm, opool + 8192ull * s, ty, n);
    } else if (OP != RS_OP_AND) {
      copy_payload(A, ca, opool + 8192ull * s);
      ty = A.type[ca];
      c = A.card[ca];
      n = A.n[ca];
    }
    if (t == 0) {
      key[s] = k;
      type[s] = ty;
      card[s] = c;
      nn[s] = n;
      if (KEEP_B && matched) card[s + 1] = 0;  // the matched key's empty slot
    }
  } else if (KEEP_B && i < na + nb) {  // ------------ b's container, kept when unmatched
    const uint32_t cb = b0 + (i - na);
    const uint16_t k = B.key[cb];
    const uint32_t j = side_rank(A.key + a0, na, k, kbuf);
    if (!(j < na && A.key[a0 + j] == k)) {
      const uint32_t s = (i - na) + j;
      copy_payload(B, cb, opool + 8192ull * s);
      if (t == 0) {
        key[s] = k;
        type[s] = B.type[cb];
        card[s] = B.card[cb];
        nn[s] = B.n[cb];
      }
    }
  }
  if (!last_cta(ticket)) return;
  // ---------------------------------------------- compaction (last CTA only)
  // in place: a chunk's records are read before any is written, and a kept
  // record only moves down
  using BS = cub::BlockScan<uint32_t, DT>;
  uint32_t f = 0;
  unsigned long long sum = 0;
  for (uint32_t e0 = 0; e0 < E; e0 += DT) {
    const uint32_t e = e0 + t;
    const uint32_t c = e < E ? __ldcg(card + e) : 0u;
    const uint32_t kp = c > 0;
    uint16_t k = 0;
    uint8_t ty = 0;
    uint32_t n = 0;
    if (kp) {
      k = __ldcg(key + e);
      ty = __ldcg(type + e);
      n = __ldcg(nn + e);
    }
    uint32_t ex, tot;
    BS(sm.scan).ExclusiveSum(kp, ex, tot);  // (its barrier orders this chunk's reads before the writes)
    if (kp) {
      const uint32_t d = f + ex;
      key[d] = k;
      type[d] = ty;
      card[d] = c;
      nn[d] = n;
      off[d] = 8192ull * e;
      sum += c;
    }
    f += tot;
    __syncthreads();  // scan storage reuse
  }
  __shared__ unsigned long long wsum[DT / 32];
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((t & 31) == 0) wsum[t >> 5] = sum;
  __syncthreads();
  if (t == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < DT / 32; w++) s += wsum[w];
    bm_start[0] = 0;
    bm_start[1] = f;
    bm_card[0] = s;
    *ticket = 0;
  }
}

// |a op b| of one pair: a CTA per container of a sums |a_c AND b_c| over the
// matched keys; the last CTA applies op_cardinality's formula
// (bitmap.py:225-241) to the bitmaps' cardinalities.
__global__ void __launch_bounds__(DT) k_single_count(int op, DevBatch A, DevBatch B, uint32_t a, uint32_t b,
                                                     uint32_t a0, uint32_t na, uint32_t b0, uint32_t nb,
                                                     uint64_t *out, uint32_t *ticket, unsigned long long *acc) {
  __shared__ __align__(16) uint64_t X[RS_WORDS];
  __shared__ __align__(16) uint64_t Y[RS_WORDS];
  __shared__ uint32_t red[DT / 32][2];
  __shared__ uint16_t kbuf[SMEM_KEYS];
  const uint32_t i = blockIdx.x;
  if (i < na) {
    const uint32_t ca = a0 + i;
    const uint16_t k = A.key[ca];
    const uint32_t j = side_rank(B.key + b0, nb, k, kbuf);
    if (j < nb && B.key[b0 + j] == k) {
      const uint32_t cb = b0 + j;
      const uint32_t c = dense_and_count<true>(A, ca, A.type[ca], B, cb, B.type[cb], X, Y, red);
      if (threadIdx.x == 0 && c) atomicAdd(acc, (unsigned long long)c);
    }
  }
  if (!last_cta(ticket)) return;
  if (threadIdx.x == 0) {
    const unsigned long long inter = atomicExch(acc, 0ull);
    const uint64_t ca = A.bm_card[a], cb = B.bm_card[b];
    const uint64_t r = op == RS_OP_AND ? inter : op == RS_OP_OR ? ca + cb - inter
                       : op == RS_OP_XOR ? ca + cb - 2 * inter : ca - inter;
    *out = r;  // (page-locked host memory: visible to the host once the kernel completes)
    *ticket = 0;
  }
}

uint32_t next_ticket() {  // (calls from several host threads take distinct tickets)
  static std::atomic<uint32_t> k{0};
  return k.fetch_add(1, std::memory_order_relaxed) % NTICKET;
}

// the device addresses of the ticket / accumulator arrays, per device
constexpr int MAX_DEV = 64;
struct Symbols {
  uint32_t *tickets = nullptr;
  unsigned long long *accs = nullptr;
};
int symbols(Symbols &out) {
  static Symbols cache[MAX_DEV];
  static std::mutex mu;
  int dev = 0;
  RS_CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= MAX_DEV) { set_error("device index out of range"); return RS_ECUDA; }
  std::lock_guard<std::mutex> g(mu);
  Symbols &c = cache[dev];
  if (!c.tickets) {
    void *p = nullptr, *q = nullptr;
    RS_CK(cudaGetSymbolAddress(&p, g_ticket));
    RS_CK(cudaGetSymbolAddress(&q, g_acc));
    c.tickets = (uint32_t *)p;
    c.accs = (unsigned long long *)q;
  }
  out = c;
  return RS_OK;
}

}  // namespace

namespace rs {

int single_pair_op(int op, const rs_batch *A, const rs_batch *B, uint32_t a, uint32_t b, rs_batch *out) {
  const uint32_t a0 = (uint32_t)A->h_bm_start[a], na = (uint32_t)(A->h_bm_start[a + 1] - a0);
  const uint32_t b0 = (uint32_t)B->h_bm_start[b], nb = (uint32_t)(B->h_bm_start[b + 1] - b0);
  const bool keep_b = op == RS_OP_OR || op == RS_OP_XOR;
  const uint32_t E = keep_b ? na + nb : na;
  Symbols sy;
  RS_TRY(symbols(sy));
  uint32_t *tk = sy.tickets + next_ticket();
  const DevBatch dA = A->dev(), dB = B->dev();
  const unsigned grid = std::max<uint32_t>(E, 1u);
  rs_batch *r = out;
#define RS_SINGLE(OP)                                                                                          \
  RS_LAUNCH(k_single_op<OP>, grid, DT, 0, dA, dB, a0, na, b0, nb, E, r->d_key, r->d_type, r->d_card, r->d_n, r->d_off, \
            r->d_pool, r->d_bm_start, r->d_bm_card, tk)
  switch (op) {
    case RS_OP_AND: RS_SINGLE(RS_OP_AND); break;
    case RS_OP_OR: RS_SINGLE(RS_OP_OR); break;
    case RS_OP_ANDNOT: RS_SINGLE(RS_OP_ANDNOT); break;
    default: RS_SINGLE(RS_OP_XOR); break;
  }
#undef RS_SINGLE
  return RS_OK;
}

uint32_t single_pair_slots(int op, uint32_t na, uint32_t nb) {
  return op == RS_OP_OR || op == RS_OP_XOR ? na + nb : na;
}

int single_pair_count(int op, const rs_batch *A, const rs_batch *B, uint32_t a, uint32_t b, uint64_t *out) {
  const uint32_t a0 = (uint32_t)A->h_bm_start[a], na = (uint32_t)(A->h_bm_start[a + 1] - a0);
  const uint32_t b0 = (uint32_t)B->h_bm_start[b], nb = (uint32_t)(B->h_bm_start[b + 1] - b0);
  Symbols sy;
  RS_TRY(symbols(sy));
  const uint32_t k = next_ticket();
  RS_LAUNCH(k_single_count, std::max<uint32_t>(na, 1u), DT, 0, op, A->dev(), B->dev(), a, b, a0, na, b0, nb, out,
            sy.tickets + k, sy.accs + k);
  return RS_OK;
}

}  // namespace rs
