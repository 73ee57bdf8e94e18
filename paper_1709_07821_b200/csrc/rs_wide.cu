// rs_wide.cu -- operations over many bitmaps at once:
//   rs_union_many            RoaringBitmap.union_many (bitmap.py:257-304)
//   rs_all_pairs_cardinality |A∩B|, |A∪B| for all pairs (op_cardinality, bitmap.py:212-241)
//   rs_batch_run_optimize    RoaringBitmap.run_optimize (bitmap.py:308-316)
// All three group containers by chunk key with one radix sort of
// (key << 40 | container index) so contributors stay in input order.
#include <cub/cub.cuh>
#include <algorithm>
#include "rs_internal.cuh"
#include "rs_dense.cuh"
#include "rs_umma.cuh"
#include <cudaTypedefs.h>

using namespace rs;
using namespace rsd;

namespace {

unsigned grid_for(uint64_t n, unsigned block) { return (unsigned)((n + block - 1) / block); }

unsigned sm_count_() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return (unsigned)sms;
}

bool env_flag_(const char *name) {
  const char *v = getenv(name);
  return v && *v == '1';
}

// item t of the ordered selection -> container index; sort key = key << 40 | t
__global__ void k_group_keys(uint64_t T, uint64_t nsel, const uint64_t *__restrict__ qbase,
                             const uint64_t *__restrict__ qsrc, DevBatch S, uint64_t *__restrict__ keys,
                             uint32_t *__restrict__ item_c) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  uint64_t lo = 0, hi = nsel;
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (qbase[m] <= t) lo = m; else hi = m;
  }
  uint64_t c = qsrc[lo] + (t - qbase[lo]);
  item_c[t] = (uint32_t)c;
  keys[t] = ((uint64_t)S.key[c] << 40) | t;
}

__global__ void k_seg_flags(uint64_t T, const uint64_t *__restrict__ keys, uint32_t *__restrict__ flag) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i <= T) flag[i] = i < T && (i == 0 || (keys[i] >> 40) != (keys[i - 1] >> 40));
}

__global__ void k_seg_starts(uint64_t T, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ pos,
                             uint32_t *__restrict__ seg_start) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < T && flag[i]) seg_start[pos[i]] = (uint32_t)i;
  if (i == T) seg_start[pos[T]] = (uint32_t)T;
}

// OR container c of S into the smem bitset X (no zeroing; bitsets OR word-wise)
__device__ void or_into(const DevBatch &S, uint32_t c, uint8_t t, uint64_t *X) {
  if (t == RS_TAG_BITSET) {
    uint64_t w[4];
    ld_words(S.pool, S.off[c], threadIdx.x, w);
#pragma unroll
    for (int k = 0; k < 4; k++) X[4 * threadIdx.x + k] |= w[k];
  } else {
    scatter_container(S, c, t, X);
  }
}

__device__ __forceinline__ void block_card_runs(const uint64_t *X, uint32_t &card, uint32_t &nruns,
                                                uint32_t (*red)[2], bool want_runs) {
  const int t = threadIdx.x;
  uint32_t pc = 0, nr = 0;
  uint64_t prev = t ? X[4 * t - 1] : 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    uint64_t w = X[4 * t + k];
    pc += __popcll(w);
    if (want_runs) {
      uint64_t cin = (k ? X[4 * t + k - 1] : prev) >> 63;
      nr += __popcll(w & ~((w << 1) | cin));
    }
  }
  block_sum2(pc, nr, red);
  card = pc;
  nruns = nr;
}

// One CTA per chunk key replays the sequential fold of union_many
// (SURVEY App. B): acc = copy(c0); per next contributor ci:
//   acc bitset            -> acc |= ci, stays bitset          (bitmap.py:278-287)
//   ci bitset             -> acc becomes bitset(ci | acc)      (:288-296)
//   both array/run        -> container_pairwise("or")         (:297-298)
//                            = array/bitset by card, or norm(run) if a run is involved
// Runs over the keys in list[0..*cnt) (the keys without a bitset
// contributor: their type can depend on the order, App. B), persistent.
// Scatter one 16-byte unit u of an array (8 values) or run (4 runs)
// payload holding nv values / runs into the shared bitset X32.
__device__ __forceinline__ void scatter_unit(const uint4 q, uint32_t u, uint32_t nv, bool is_array, uint32_t *X32) {
  const uint32_t x[4] = {q.x, q.y, q.z, q.w};
  if (is_array) {
    const uint32_t v0 = 8 * u;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint32_t lo16 = x[j] & 0xFFFF, hi16 = x[j] >> 16;
      const bool a = v0 + 2 * j < nv, b = v0 + 2 * j + 1 < nv;
      const uint32_t wl = lo16 >> 5, wh = hi16 >> 5;
      const uint32_t bl = 1u << (lo16 & 31), bh = 1u << (hi16 & 31);
      if (a && b && wl == wh) {
        atomicOr(&X32[wl], bl | bh);
      } else {
        if (a) atomicOr(&X32[wl], bl);
        if (b) atomicOr(&X32[wh], bh);
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; j++) {
    if (4 * u + j >= nv) break;
    const uint32_t st = x[j] & 0xFFFF, en = st + (x[j] >> 16);
    const uint32_t ws = st >> 5, we = en >> 5;
    const uint32_t first = ~0u << (st & 31), last = ~0u >> (31 - (en & 31));
    if (ws == we) {
      atomicOr(&X32[ws], first & last);
    } else {
      atomicOr(&X32[ws], first);
      atomicOr(&X32[we], last);
      for (uint32_t w = ws + 1; w < we; w++) X32[w] = ~0u;  // all-ones commutes with the ORs
    }
  }
}

__device__ __forceinline__ uint32_t units_of(uint8_t type, uint32_t n) {
  return type == RS_TAG_ARRAY ? (n + 7) >> 3 : type == RS_TAG_RUN ? (n + 3) >> 2 : 512u;
}

// One CTA per key (persistent over the keys in list[0..*cnt), fetched
// dynamically): the keys without a bitset contributor, whose result type can
// depend on the order (App. B).  The fold replays the sequence:
//   acc = copy(c0); per next ci: container_pairwise("or", acc, ci), i.e.
//   array / bitset by card, or norm(run) when a run is involved
//   (containers.py:459-527); once a bitset, the rest ORs in order-free
//   (bitmap.py:278-287).
// The contributors' metadata comes in one round of loads; each step's payload
// (at most 8 KB: 512 16-byte units, two per thread) is loaded into registers
// one step ahead, so a step is scatter + two barriers, with no global load on
// its critical path.
__global__ void __launch_bounds__(DT) k_union_fold(const uint32_t *__restrict__ list, const uint32_t *__restrict__ cnt,
                                                   const uint32_t *__restrict__ seg_start,
                                                   const uint32_t *__restrict__ item_c, const uint64_t *__restrict__ keys,
                                                   DevBatch S, uint16_t *okey, uint8_t *otype, uint32_t *ocard,
                                                   uint32_t *on, uint64_t *ooff, uint8_t *__restrict__ opool) {
  __shared__ __align__(16) DenseSmem sm;
  __shared__ uint64_t mo[DT];   // contributor payload offset
  __shared__ uint32_t mn[DT];   // contributor n
  __shared__ uint8_t mt[DT];    // contributor type
  __shared__ uint32_t mc[DT];   // contributor cardinality
  __shared__ uint32_t next_li;
  const int t = threadIdx.x;
  uint32_t *X32 = (uint32_t *)sm.X;
  const uint32_t total = cnt[0];
  for (;;) {
    __syncthreads();  // the previous key's smem reads are done
    if (t == 0) next_li = atomicAdd(const_cast<uint32_t *>(cnt) + 2, 1u);  // dynamic: keys differ in cost
    __syncthreads();
    const uint32_t li = next_li;
    if (li >= total) break;
    const uint64_t g = list[li];
    const uint32_t s = seg_start[g], e = seg_start[g + 1];
    // metadata of the first DT contributors in one parallel round of loads
    if (s + t < e) {
      const uint32_t c = item_c[s + t];
      mt[t] = S.type[c];
      mo[t] = S.off[c];
      mn[t] = S.n[c];
      mc[t] = S.card[c];
    }
#pragma unroll
    for (int k = 0; k < 4; k++) sm.X[4 * t + k] = 0;
    __syncthreads();
    auto meta = [&](uint32_t i, uint8_t &ty, uint64_t &of, uint32_t &n, uint32_t &cd) {
      if (i - s < DT) { ty = mt[i - s]; of = mo[i - s]; n = mn[i - s]; cd = mc[i - s]; }
      else { const uint32_t c = item_c[i]; ty = S.type[c]; of = S.off[c]; n = S.n[c]; cd = S.card[c]; }
    };
    auto load = [&](uint64_t of, uint32_t nu, uint4 &q0, uint4 &q1) {
      const uint4 *p = (const uint4 *)(S.pool + of);
      if ((uint32_t)t < nu) q0 = __ldg(p + t);
      if ((uint32_t)t + DT < nu) q1 = __ldg(p + t + DT);
    };
    uint8_t ty;
    uint64_t of;
    uint32_t n, cd;
    meta(s, ty, of, n, cd);
    uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0;
    load(of, units_of(ty, n), q0, q1);
    // The type decisions of the sequence need the running union's card and
    // run count only where bounds cannot settle them: card lies in
    // [max of the contributors' cards, sum of them], the run count is at most
    // the contributors' runs (an array value is a run).  A step the bounds
    // decide takes no barrier -- the shared ORs of consecutive steps commute
    // -- and only an undecided one synchronizes and sweeps the words.
    uint8_t acc = ty;  // acc = copy(c0); arrays / runs only in this list
    uint32_t card_lo = cd, card_hi = cd, runs_hi = ty == RS_TAG_RUN ? n : cd;
    for (uint32_t i = s; i < e; i++) {
      const uint8_t cty = ty;
      const uint32_t cn = n, cu = units_of(cty, cn), ccd = cd;
      const uint4 c0q = q0, c1q = q1;
      if (i + 1 < e) {  // the next contributor's payload, in flight during this step
        meta(i + 1, ty, of, n, cd);
        load(of, units_of(ty, n), q0, q1);
      }
      if ((uint32_t)t < cu) scatter_unit(c0q, t, cn, cty == RS_TAG_ARRAY, X32);
      if ((uint32_t)t + DT < cu) scatter_unit(c1q, t + DT, cn, cty == RS_TAG_ARRAY, X32);
      if (i == s || acc == RS_TAG_BITSET) continue;  // nothing to decide
      const bool run_rule = acc == RS_TAG_RUN || cty == RS_TAG_RUN;
      card_lo = max(card_lo, ccd);
      card_hi = min(card_hi + ccd, 65536u);
      runs_hi = min(runs_hi + (cty == RS_TAG_RUN ? cn : ccd), 65536u);
      if (run_rule) {  // a run iff admissible (containers.py:202-205) for every card in the bounds
        const bool sure = card_lo > RS_ARRAY_MAX
                              ? runs_hi <= RS_RUN_MAX_RUNS
                              : 2 * runs_hi < card_lo && (card_hi <= RS_ARRAY_MAX || runs_hi <= RS_RUN_MAX_RUNS);
        if (sure) { acc = RS_TAG_RUN; continue; }
      } else {  // array / bitset by card
        if (card_hi <= RS_ARRAY_MAX) { acc = RS_TAG_ARRAY; continue; }
        if (card_lo > RS_ARRAY_MAX) { acc = RS_TAG_BITSET; continue; }
      }
      __syncthreads();  // every step's ORs are in
      uint32_t cexact, nruns;
      block_card_runs(sm.X, cexact, nruns, sm.red, run_rule);
      if (run_rule && rs_run_admissible(cexact, nruns)) acc = RS_TAG_RUN;
      else acc = cexact <= RS_ARRAY_MAX ? RS_TAG_ARRAY : RS_TAG_BITSET;
      card_lo = card_hi = cexact;
      if (run_rule) runs_hi = nruns;
      __syncthreads();
    }
    __syncthreads();  // the last steps' ORs are in
    uint64_t r[4];
    uint32_t pc = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) { r[k] = sm.X[4 * t + k]; pc += __popcll(r[k]); }
    uint32_t card = pc, z = 0;
    block_sum2(card, z, sm.red);
    __syncthreads();
    const uint32_t nout = encode_result(sm, r, pc, card, acc, opool + g * 8192);
    if (t == 0) {
      okey[g] = (uint16_t)(keys[s] >> 40);
      otype[g] = acc;
      ocard[g] = card;
      on[g] = nout;
      ooff[g] = g * 8192;
    }
  }
}

// Keys of union_many by result rule: a key with at least one bitset
// contributor ends as a bitset holding the OR of all its contributors,
// whatever their order (App. B: once a bitset, always a bitset, and a
// bitset contributor turns the accumulator into one; its cardinality is
// >= 4097 from then on) -> list 0, an order-free streaming OR.  The other
// keys replay the fold (list 1).
__global__ void k_union_classify(uint64_t G, const uint32_t *__restrict__ seg_start,
                                 const uint32_t *__restrict__ item_c, DevBatch S, uint32_t *__restrict__ list0,
                                 uint32_t *__restrict__ list1, uint32_t *__restrict__ cnt) {
  const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  bool bs = false;
  if (g < G)
    for (uint32_t i = seg_start[g]; i < seg_start[g + 1] && !bs; i++) bs = S.type[item_c[i]] == RS_TAG_BITSET;
  const bool active = g < G;
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const unsigned m = __ballot_sync(0xffffffffu, active && bs == (c == 0));
    if (!m) continue;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)lane == leader) base = atomicAdd(&cnt[c], (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (active && bs == (c == 0)) (c == 0 ? list0 : list1)[base + __popc(m & ((1u << lane) - 1))] = (uint32_t)g;
  }
}

// The order-free keys: OR of every contributor, written as a bitset.
// Persistent CTAs over list[0..*cnt); thread t owns words [4t, 4t+4).  The
// key's contributors are handled in windows of up to DT: one round of
// metadata loads (container, type, offset, size) into shared memory, then
// every payload load of the window is independent of the others -- bitset
// words go into registers (four contributors in flight per thread), array
// values and runs are flattened over the window (thread f takes element f of
// the concatenation) and scattered into a shared bitset with native shared
// ORs, which is folded into the registers at the end and re-zeroed by its
// owners.  A CTA-per-contributor-chain kernel spent most of its time in
// dependent load chains (metadata -> payload per contributor).
// k_union_or threads: thread t owns words [4(t + UT h), 4(t + UT h) + 4), h < UH.
// Small CTAs keep more keys in flight per SM (the kernel waits on dependent
// metadata -> payload chains): 64 threads give ~2x the keys of 128.
constexpr int UT = 64, UH = RS_WORDS / (4 * UT);
__global__ void __launch_bounds__(UT) k_union_or(const uint32_t *__restrict__ list, const uint32_t *__restrict__ cnt,
                                                 const uint32_t *__restrict__ seg_start,
                                                 const uint32_t *__restrict__ item_c, const uint64_t *__restrict__ keys,
                                                 DevBatch S, uint16_t *okey, uint8_t *otype, uint32_t *ocard,
                                                 uint32_t *on, uint64_t *ooff, uint8_t *__restrict__ opool) {
  __shared__ __align__(16) uint64_t X[RS_WORDS];
  __shared__ uint64_t moff[UT];          // bitset contributors' payload offsets (compacted)
  __shared__ uint64_t eoff[UT];          // array / run contributors' payload offsets (compacted)
  __shared__ uint32_t ebase[UT + 1];     // their 16-byte unit prefix; [UT] = slot counter
  __shared__ uint8_t etype[UT];
  __shared__ uint32_t eunits_n[UT];      // their value / run counts
  __shared__ uint32_t nbits, nelem, next_li;
  __shared__ uint32_t red[UT / 32];
  const int t = threadIdx.x, lane = t & 31;
  uint32_t *X32 = (uint32_t *)X;
#pragma unroll
  for (int k = 0; k < RS_WORDS / UT; k++) X[t + UT * k] = 0;
  if (t == 0) {
    ebase[UT] = 0;
    next_li = atomicAdd(const_cast<uint32_t *>(cnt) + 2, 1u);  // dynamic: keys differ in cost
  }
  const uint32_t total = cnt[0];
  __syncthreads();
  for (;;) {
    const uint32_t li = next_li;
    if (li >= total) break;
    const uint32_t g = list[li];
    const uint32_t s = seg_start[g], e = seg_start[g + 1];
    uint64_t r[4 * UH];
#pragma unroll
    for (int k = 0; k < 4 * UH; k++) r[k] = 0;
    for (uint32_t w0 = s; w0 < e; w0 += UT) {
      // window metadata: thread t = contributor w0 + t
      const bool have = w0 + t < e;
      uint8_t ty = 0;
      uint64_t of = 0;
      uint32_t nn = 0;
      if (have) {
        const uint32_t c = item_c[w0 + t];
        ty = S.type[c];
        of = S.off[c];
        nn = S.n[c];
      }
      if (t == 0) { nbits = 0; nelem = 0; }
      __syncthreads();  // (every thread has read next_li)
      if (t == 0 && w0 == s) next_li = atomicAdd(const_cast<uint32_t *>(cnt) + 2, 1u);  // the next key, early
      // compact: bitset offsets to moff, array/run ones to eoff (an OR commutes:
      // the order inside the window does not matter)
      const bool isb = have && ty == RS_TAG_BITSET, ise = have && !isb;
      {
        const unsigned mb = __ballot_sync(0xffffffffu, isb);
        uint32_t base = 0;
        if (lane == 0 && mb) base = atomicAdd(&nbits, (uint32_t)__popc(mb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (isb) moff[base + __popc(mb & ((1u << lane) - 1))] = of;
      }
      {
        const unsigned me = __ballot_sync(0xffffffffu, ise);
        uint32_t base = 0;
        if (lane == 0 && me) base = atomicAdd(&ebase[UT], (uint32_t)__popc(me));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (ise) {
          const uint32_t slot = base + __popc(me & ((1u << lane) - 1));
          eoff[slot] = of;
          etype[slot] = ty;
          eunits_n[slot] = nn;
          ebase[slot] = ty == RS_TAG_ARRAY ? (nn + 7) >> 3 : (nn + 3) >> 2;  // 16-byte units
        }
      }
      __syncthreads();
      const uint32_t nb = nbits, ne = ebase[UT];
      if (t < 32) {  // exclusive prefix of the unit counts (one warp)
        uint32_t carry = 0;
        for (uint32_t k0 = 0; k0 < ne; k0 += 32) {
          const uint32_t k = k0 + lane;
          const uint32_t v = k < ne ? ebase[k] : 0;
          uint32_t x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          if (k < ne) ebase[k] = carry + x - v;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) nelem = carry;
      }
      // bitset contributors: words straight into registers, 2 contributors
      // (4 x 16-byte loads per thread) in flight
      for (uint32_t k = 0; k < nb; k++) {  // each contributor: UH independent 32-byte loads per thread
        uint64_t w[UH][4];
#pragma unroll
        for (int h = 0; h < UH; h++) ld_words(S.pool, moff[k], t + UT * h, w[h]);
#pragma unroll
        for (int h = 0; h < UH; h++)
#pragma unroll
          for (int q = 0; q < 4; q++) r[4 * h + q] |= w[h][q];
      }
      __syncthreads();  // prefix and nelem visible
      // array / run payloads, flattened over the window in 16-byte units
      // (8 array values or 4 runs per load; every unit's load is independent)
      const uint32_t tot = nelem;
      uint32_t lo = 0;  // contributor lo with ebase[lo] <= f < ebase[lo+1]
      if ((uint32_t)t < tot) {  // binary search for the thread's first unit ...
        uint32_t hi = ne;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (ebase[mid] <= (uint32_t)t) lo = mid; else hi = mid;
        }
      }
      // two units per step, both loads issued before either is scattered
      // (a load per step waited out a round trip between the scatters)
      for (uint32_t f = t; f < tot; f += 2 * UT) {
        while (lo + 1 < ne && ebase[lo + 1] <= f) lo++;  // ... then forward (units ascend)
        const uint32_t l0 = lo, u0 = f - ebase[l0];
        const uint4 q0 = __ldg((const uint4 *)(S.pool + eoff[l0]) + u0);
        const bool two = f + UT < tot;
        uint32_t l1 = l0, u1 = 0;
        uint4 q1 = make_uint4(0, 0, 0, 0);
        if (two) {
          while (lo + 1 < ne && ebase[lo + 1] <= f + UT) lo++;
          l1 = lo;
          u1 = f + UT - ebase[l1];
          q1 = __ldg((const uint4 *)(S.pool + eoff[l1]) + u1);
        }
        scatter_unit(q0, u0, eunits_n[l0], etype[l0] == RS_TAG_ARRAY, X32);
        if (two) scatter_unit(q1, u1, eunits_n[l1], etype[l1] == RS_TAG_ARRAY, X32);
      }
      if (t == 0) ebase[UT] = 0;
      __syncthreads();  // window done: its smem may be reused
    }
    uint32_t pc = 0;
#pragma unroll
    for (int h = 0; h < UH; h++)
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int wd = 4 * (t + UT * h) + q;
        r[4 * h + q] |= X[wd];
        X[wd] = 0;
        pc += __popcll(r[4 * h + q]);
      }
#pragma unroll
    for (int h = 0; h < UH; h++) st_words(opool, (uint64_t)g * 8192, t + UT * h, r + 4 * h);
    pc = __reduce_add_sync(0xffffffffu, pc);
    if (lane == 0) red[t >> 5] = pc;
    __syncthreads();  // also orders the X clears before the next key's scatter
    if (t == 0) {
      uint32_t card = 0;
#pragma unroll
      for (int w = 0; w < UT / 32; w++) card += red[w];
      okey[g] = (uint16_t)(keys[s] >> 40);
      otype[g] = RS_TAG_BITSET;
      ocard[g] = card;
      on[g] = RS_WORDS;
      ooff[g] = (uint64_t)g * 8192;
    }
  }
}

// D (T densified 8 KB rows) as a 2D uint8 tensor for TMA: boxes of 32 rows x
// 128 bytes, SWIZZLE_128B, rows past T read as zero.  The encoder comes from
// the driver through the runtime (no libcuda link).
static int rows_tensor_map(CUtensorMap *tm, const void *D, uint64_t T) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode) {
      encode = nullptr;
      set_error("cuTensorMapEncodeTiled unavailable");
      return RS_ECUDA;
    }
  }
  const cuuint64_t dims[2] = {8192, T ? T : 1}, strides[1] = {8192};
  const cuuint32_t box[2] = {(cuuint32_t)rsu::UBOXB, (cuuint32_t)rsu::UBOXR}, es[2] = {1, 1};  // 128 B x 32 rows
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(D), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return RS_ECUDA;
  }
  return RS_OK;
}

// ------------------------------------------------------------ all pairs

// densify every grouped container into its own 8 KB slot.  Thread t owns
// words t + 256q (conflict-free smem, coalesced 64-bit stores); the slots are
// written with streaming stores (read back once by the all-pairs tiles).
__global__ void __launch_bounds__(DT) k_densify(uint64_t T, const uint32_t *__restrict__ item_c, DevBatch S,
                                                uint64_t *__restrict__ D) {
  __shared__ __align__(16) uint64_t X[RS_WORDS];
  uint64_t i = blockIdx.x;
  if (i >= T) return;
  const int t = threadIdx.x;
  uint32_t c = item_c[i];
  uint8_t type = S.type[c];
  uint64_t *dst = D + i * RS_WORDS;
  if (type == RS_TAG_BITSET) {
    const uint64_t *src = (const uint64_t *)(S.pool + S.off[c]);
#pragma unroll
    for (int q = 0; q < 4; q++) __stcs(dst + t + DT * q, __ldcs(src + t + DT * q));
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; q++) X[t + DT * q] = 0;
  __syncthreads();
  scatter_container(S, c, type, X);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; q++) __stcs(dst + t + DT * q, X[t + DT * q]);
}

// The same rows, one WARP per container (persistent over the items, with the
// next item's metadata loaded before the current row is built).  k_densify's
// CTA per 8 KB row was latency-bound (125 k CTAs of dependent metadata loads,
// two block barriers each: 2.9 TB/s of row writes on config 5).  Here a
// bitset row is 16 independent 16-byte loads per lane then 16 streaming
// stores; an array / run row is built in the warp's own 8 KB of shared
// memory (16-byte zeroing, 16-byte value loads masked to n, native shared
// ORs) and streamed out with 16-byte stores.  No block barriers.
constexpr int DW_WARPS = 4;  // 4 x 8 KB rows of shared memory per CTA; 6 CTAs per SM (80 registers)
constexpr int DW_PF = 8;     // 16-byte array vectors in flight per lane
// `list` (optional): densify only items list[0..T) (the rows the CUDA-core
// tiles read when the tensor-core tiles build their own rows).
__global__ void __launch_bounds__(32 * DW_WARPS) k_densify_warp(uint64_t T, const uint32_t *__restrict__ item_c,
                                                                DevBatch S, uint64_t *__restrict__ D,
                                                                const uint32_t *__restrict__ list) {
  __shared__ __align__(16) uint4 Xs[DW_WARPS][RS_WORDS / 2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint4 *X = Xs[wib];
  uint32_t *X32 = (uint32_t *)X;
  const uint64_t step = (uint64_t)gridDim.x * DW_WARPS;
  uint64_t li = (uint64_t)blockIdx.x * DW_WARPS + wib;
  if (li >= T) return;
  uint64_t i = list ? list[li] : li;
  uint32_t c = item_c[i];
  uint8_t type = S.type[c];
  uint64_t off = S.off[c];
  uint32_t n = S.n[c];
  for (;;) {
    // next item's metadata first: its dependent loads overlap this row
    const uint64_t nli = li + step;
    const uint64_t ni = nli < T ? (list ? list[nli] : nli) : ~0ull;
    uint32_t nc = 0, nn = 0;
    uint8_t ntype = 0;
    uint64_t noff = 0;
    if (nli < T) {
      nc = item_c[ni];
      ntype = S.type[nc];
      noff = S.off[nc];
      nn = S.n[nc];
    }
    uint4 *dst = (uint4 *)(D + i * RS_WORDS);
    if (type == RS_TAG_BITSET) {
      const uint4 *src = (const uint4 *)(S.pool + off);
      uint4 r[16];
#pragma unroll
      for (int q = 0; q < 16; q++) r[q] = __ldcs(src + lane + 32 * q);
#pragma unroll
      for (int q = 0; q < 16; q++) __stcs(dst + lane + 32 * q, r[q]);
    } else {
#pragma unroll
      for (int q = 0; q < 16; q++) X[lane + 32 * q] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      if (type == RS_TAG_ARRAY) {
        // all of a lane's 16-byte vectors are loaded before any is scattered
        // (DW_PF per round: <= 2 rounds for 4096 values): a load per loop
        // iteration put a DRAM round trip between every 8 shared ORs
        // (62 % of the kernel's stall samples sat on the first OR)
        const uint4 *v = (const uint4 *)(S.pool + off);
        const uint32_t nv = (n + 7) >> 3;
        for (uint32_t k0 = 0; k0 < nv; k0 += 32 * DW_PF) {
          uint4 xs[DW_PF];
#pragma unroll
          for (int j = 0; j < DW_PF; j++) {
            const uint32_t k = k0 + lane + 32 * j;
            xs[j] = k < nv ? __ldg(v + k) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int j = 0; j < DW_PF; j++) {
            const uint32_t k = k0 + lane + 32 * j;
            if (k >= nv) break;
            const uint32_t w[4] = {xs[j].x, xs[j].y, xs[j].z, xs[j].w};
            const uint32_t left = n - 8 * k;  // values of this vector inside the array
#pragma unroll
            for (int h = 0; h < 8; h++) {
              if ((uint32_t)h < left) {
                const uint32_t val = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
                atomicOr(&X32[val >> 5], 1u << (val & 31));
              }
            }
          }
        }
      } else {  // runs (_words_from_runs, containers.py:122-135): edge words by atomics, interior by stores
        const uint32_t *r32 = (const uint32_t *)(S.pool + off);
        for (uint32_t r = lane; r < n; r += 32) {
          const uint32_t sl = r32[r];
          const uint32_t s = sl & 0xFFFF, e = s + (sl >> 16);
          const uint32_t ws = s >> 5, we = e >> 5;
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
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 16; q++) __stcs(dst + lane + 32 * q, X[lane + 32 * q]);
      __syncwarp();  // the row is read out before the next item zeroes it
    }
    if (nli >= T) break;
    li = nli;
    i = ni;
    c = nc;
    type = ntype;
    off = noff;
    n = nn;
  }
}

#ifdef RS_UMMA_TRACE  // timeline of CTA 0 (tools only): 6 events x 256 chunks
__device__ long long g_umma_trace[6][256];
#define UTR(e, i) \
  if (blockIdx.x == 0) g_umma_trace[e][i] = clock64()
#else
#define UTR(e, i)
#endif

// One CTA per tensor-core tile (see rs_umma.cuh): A = rows [r0, r0+128),
// B = rows [c0, c0+nb) of one key segment; counts of pairs u < v go into the
// same N x N matrix as the CUDA-core tiles.  tmD maps D as a 2D tensor
// (8192 bytes x T rows).
__global__ void __launch_bounds__(rsu::UTHREADS, 1)
    k_allpairs_umma(const uint32_t *__restrict__ tp_seg, const uint16_t *__restrict__ tp_r0,
                    const uint16_t *__restrict__ tp_c0, const uint16_t *__restrict__ tp_nb,
                    const uint32_t *__restrict__ seg_start, const __grid_constant__ CUtensorMap tmD,
                    const uint32_t *__restrict__ item_bm, uint64_t N, unsigned long long *__restrict__ Mx) {
  using namespace rsu;
  extern __shared__ __align__(1024) uint8_t usm_raw[];
  // 1024-byte alignment for the swizzled TMA boxes and operand atoms
  uint8_t *usm = (uint8_t *)(((uintptr_t)usm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(usm + URING), *empty = full + UNST, *rfull = empty + UNST,
           *rempty = rfull + URAWMAX, *done = rempty + URAWMAX;
  uint32_t *tslot = (uint32_t *)(done + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t seg = tp_seg[blockIdx.x];
  const uint32_t s0 = seg_start[seg], m = seg_start[seg + 1] - s0;
  const uint32_t r0 = tp_r0[blockIdx.x], c0 = tp_c0[blockIdx.x], nb = tp_nb[blockIdx.x];
  const bool shared_a = r0 == c0;  // A = the first 128 rows of the B operand
  // raw stage: the B rows in 32-row boxes, then a separate A's 128 rows
  // (128 bytes per row either way, so raw row r sits at r * 128); expanded
  // stage: the B operand (rows_b rows) in shared memory -- the A operand of
  // the same stage sits in TMEM (32 columns per chunk from column UACOL)
  const uint32_t rows_b = max(nb, (uint32_t)UM), nbox = (rows_b + UBOXR - 1) / UBOXR;
  const uint32_t rbytes = nbox * UBOX + (shared_a ? 0u : (uint32_t)(UM * UBOXB));
  const uint32_t sbytes = rows_b * UROWB;
  const int nraw = min(URAWMAX, (int)((URING - UNST * sbytes) / rbytes));
  uint8_t *raw = usm, *xst = usm + nraw * rbytes;
  // expanded rows never written below (past m, past nb) must read as zero
  for (uint32_t i = t; i < UNST * sbytes / 16; i += UTHREADS) ((uint4 *)xst)[i] = make_uint4(0, 0, 0, 0);
  if (t == 0) {
    for (int i = 0; i < UNST; i++) {
      ubar_init(&full[i], 4);  // the four warps of the stage's producer group
      ubar_init(&empty[i], 1);
    }
    for (int i = 0; i < nraw; i++) {
      ubar_init(&rfull[i], 1);
      ubar_init(&rempty[i], UPROD / 32);  // every producer warp reads each box
    }
    ubar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(UTMEM)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp < 4) {  // unit block scales: 0x7F (E8M0 2^0) in columns USCOL.. of every lane
    const uint32_t one = 0x7F7F7F7Fu;
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((uint32_t)(32 * warp) << 16) + USCOL + c),
                   "r"(one)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  constexpr int NCH = RS_WORDS * 64 / UKC;   // 256-bit chunks per row
  constexpr int NRAW = 8192 / UBOXB;         // raw boxes per row (one K chunk per producer group)
  static_assert(NCH == NRAW * UNST, "one chunk per producer group and raw box");
  if (warp == UPROD / 32 + 1) {  // ------------------------------ TMA (raw rows)
    if (lane == 0) {
      uint32_t st = 0, ph = 0;
      for (int r = 0; r < NRAW; r++) {
        if (r >= nraw) ubar_wait(&rempty[st], ph ^ 1u);
        uint8_t *dst = raw + st * rbytes;
        UTR(4, r);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&rfull[st])), "r"(rbytes)
                     : "memory");
        const uint32_t nload = nbox + (shared_a ? 0u : (uint32_t)(UM / UBOXR));
        for (uint32_t bx = 0; bx < nload; bx++) {
          // B boxes, then a separate A's
          const uint32_t row = bx < nbox ? s0 + c0 + bx * UBOXR : s0 + r0 + (bx - nbox) * UBOXR;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
              "[%4];" ::"r"(su32(dst + bx * UBOX)),
              "l"((uint64_t)&tmD), "r"(r * UBOXB), "r"(row), "r"(su32(&rfull[st]))
              : "memory");
        }
        if (++st == (uint32_t)nraw) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == UPROD / 32) {  // ------------------------------ MMA issuer
    // The whole warp walks the stages with warp-uniform state (stage, phase,
    // descriptors stay in uniform registers) and one elected lane issues: a
    // single issuing thread is instruction-latency bound, so per chunk there
    // is one wait, four MMAs and one commit, and nothing else.
    const uint32_t idesc = idesc_mxf4(UM, (int)nb);
    const uint64_t db0 = sw128_desc(su32(xst));
    const uint32_t sstep = sbytes >> 4;  // descriptor address units per stage
    const uint32_t sfa = tmem + USCOL, sfb = tmem + USCOL + 16u;
    uint32_t b = 0, ph = 0;
    for (int c = 0; c < NCH; c++) {
      ubar_wait(&full[b], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t db = db0 + (uint64_t)(b * sstep);
      const uint32_t ta = tmem + UACOL + 32u * b;
      if (elect_one()) {
        UTR(2, c);
        // K = 64 nibbles per MMA: 8 TMEM columns of A, 32 bytes (2 descriptor units) of the B atom row
        umma_mxf4(tmem, ta, db, idesc, sfa, sfb, c > 0);
        umma_mxf4(tmem, ta + 8u, db + 2, idesc, sfa, sfb, true);
        umma_mxf4(tmem, ta + 16u, db + 4, idesc, sfa, sfb, true);
        umma_mxf4(tmem, ta + 24u, db + 6, idesc, sfa, sfb, true);
        umma_commit(&empty[b]);
        UTR(3, c);
        if (c == NCH - 1) umma_commit(done);
      }
      __syncwarp();
      if (++b == (uint32_t)UNST) {
        b = 0;
        ph ^= 1u;
      }
    }
  } else {  // ------------------------------------------- producers
    // UNST groups of four warps; group g expands K chunk g of every raw box
    // (chunk 4r + g) into its own stage g, so stage and phases advance by
    // one per box with no arithmetic.  Warp q of a group owns rows 32q +
    // lane (+128): it expands them from the raw box -- 128-byte rows whose
    // 16-byte units are XOR-swizzled by row % 8 -- into the B atom rows in
    // shared memory, and writes rows < 128 of A (B's own rows, or the
    // separate A rows) into the stage's TMEM columns with one tcgen05.st
    // (warp q reaches TMEM lanes 32q..32q+31 = those rows); rows past the key
    // are zeros.
    const int grp = warp >> 2, q = warp & 3;
    const uint32_t nrow_b = c0 < m ? min(nb, m - c0) : 0u, nrow_a = shared_a ? nrow_b : min((uint32_t)UM, m - r0);
    const uint32_t arow = 32 * q + lane, sw = arow & 7;
    const uint32_t aoff = (shared_a ? 0u : nbox * UBOX) + arow * UBOXB;
    const uint32_t u0 = ((2 * grp) ^ sw) << 4, u1 = ((2 * grp + 1) ^ sw) << 4;  // this chunk's two raw units
    uint8_t *sb = xst + grp * sbytes;
    const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + UACOL + 32u * grp;
    uint32_t st = 0, rph = 0, eph = 0;
    for (int r = 0; r < NRAW; r++) {
      const int c = 4 * r + grp;
      ubar_wait(&rfull[st], rph);
      UTR(5, c);
      if (r) {
        ubar_wait(&empty[grp], eph);
        eph ^= 1u;
      }
      UTR(0, c);
      const uint8_t *rs = raw + st * rbytes;
      uint32_t e[32];
      {  // A row arow (and B row arow when shared)
        uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
        if (arow < nrow_a) {
          lo = *(const uint4 *)(rs + aoff + u0);
          hi = *(const uint4 *)(rs + aoff + u1);
        }
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const uint4 v = nib32(w[u]);
          e[4 * u] = v.x; e[4 * u + 1] = v.y; e[4 * u + 2] = v.z; e[4 * u + 3] = v.w;
          if (shared_a && arow < nrow_b) *(uint4 *)(sb + sw_off((int)arow, 16 * u, (int)rows_b)) = v;
        }
      }
      tmem_st32(ta, e);
      // the other B rows: all of them for a separate A, rows >= 128 otherwise
      for (uint32_t row = shared_a ? UM + arow : arow; row < nrow_b; row += UM) {
        const uint8_t *p = rs + row * UBOXB;
        const uint32_t rsw = row & 7;
        expand_row(sb, (int)row, (int)rows_b, *(const uint4 *)(p + (((2 * grp) ^ rsw) << 4)),
                   *(const uint4 *)(p + (((2 * grp + 1) ^ rsw) << 4)));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        UTR(1, c);
        ubar_arrive(&full[grp]);
        ubar_arrive(&rempty[st]);  // this warp's reads of the raw box are done
      }
      if (++st == (uint32_t)nraw) {
        st = 0;
        rph ^= 1u;
      }
    }
  }
  ubar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {  // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3, colh = warp >> 2;  // warps 0-7; the issuer warp idles
    if (warp < 8) {
      const uint32_t u = r0 + 32 * quarter + lane;
      const uint32_t bu = u < m ? item_bm[s0 + u] : 0;
      for (uint32_t cb = 128 * colh; cb < 128 * colh + 128 && cb < nb; cb += 32) {
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * quarter) << 16) + cb;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (u < m) {
#pragma unroll
          for (int j = 0; j < 32; j++) {
            const uint32_t vc = c0 + cb + j;
            const uint32_t cnt = (uint32_t)__uint_as_float(v[j]);  // exact: an integer <= 65,536
            if (cnt && vc < m && u < vc) {
              const uint32_t bv = item_bm[s0 + vc];
              const uint32_t lo = min(bu, bv), hi = max(bu, bv);
              atomicAdd(&Mx[(uint64_t)lo * N + hi], (unsigned long long)cnt);
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(UTMEM) : "memory");
}

// ---------------------------------------------------- all pairs, direct rows
// (experimental, RS_ALLPAIRS_DIRECT=1; measured 7x slower than the TMA-fed
// tiles, see rs_all_pairs_cardinality.)
// The same tensor-core tiles without the densified copy of every row: the
// producer threads build each row's 256-bit K chunk straight from its
// container -- a bitset's 32 bytes, or the bits of the array values / runs
// that fall into the chunk -- so the 8 KB rows are never written to HBM and
// read back (config 5: 1 GB each way, the densify kernel alone was 0.33 ms).
// K order does not matter to a Gram matrix, so producer group g walks the
// contiguous quarter [16384 g, 16384 (g+1)) of every row, one chunk per stage
// visit; the MMA issuer still visits the stages round-robin.  Array / run
// rows keep a cursor (and a 16-byte value window plus the next one, loaded
// ahead) in shared memory; their starting index in the quarter comes from a
// per-item table (k_quarter_index).  Bitset rows load the next chunk's 32
// bytes one visit ahead.
namespace rsd2 {
// Two row slots per producer thread: (A row, B row) for a block tile with a
// separate A (its B side has <= 128 rows), (row arow, row arow + 128) when A
// is the first 128 rows of B.  48 bytes each: 2 x 512 x 48 = 48 KB beside
// the 4 expanded stages (<= 128 KB) in the 192 KB ring.
struct RowCur {
  uint4 win, nwin;   // array / run: elements [wpos, wpos+8) and the next 8; bitset: the next chunk's 32 bytes
  uint64_t base;     // payload address
  uint16_t idx, wpos, n;
  uint8_t type;      // 0 = no row
};
static_assert(sizeof(RowCur) == 48, "RowCur layout");
}  // namespace rsd2

// per grouped item: first array value / run index in each quarter of the chunk
__global__ void k_quarter_index(uint64_t T, const uint32_t *__restrict__ item_c, DevBatch S, ushort4 *__restrict__ Q) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= T) return;
  const uint32_t c = item_c[i];
  const uint8_t t = S.type[c];
  const uint32_t n = S.n[c];
  uint16_t q[4] = {0, 0, 0, 0};
  if (t != RS_TAG_BITSET) {
    const uint16_t *v = (const uint16_t *)(S.pool + S.off[c]);
    for (int g = 1; g < 4; g++) {
      const uint32_t lim = 16384u * g;
      uint32_t lo = 0, hi = n;  // first element whose (last) value >= lim
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t last = t == RS_TAG_ARRAY ? v[mid] : (uint32_t)v[2 * mid] + v[2 * mid + 1];
        if (last < lim) lo = mid + 1; else hi = mid;
      }
      q[g] = (uint16_t)lo;
    }
  }
  Q[i] = make_ushort4(q[0], q[1], q[2], q[3]);
}

__device__ __forceinline__ uint32_t elem_of(const uint4 w, uint32_t j) {  // u32 element j < 4 of a window
  return j == 0 ? w.x : j == 1 ? w.y : j == 2 ? w.z : w.w;
}

// set bit b (< 256) of the 8-word chunk
__device__ __forceinline__ void set_chunk_bit(uint32_t (&w)[8], uint32_t b) {
  const uint32_t word = b >> 5, bit = 1u << (b & 31);
#pragma unroll
  for (int k = 0; k < 8; k++) w[k] |= word == (uint32_t)k ? bit : 0u;
}

// bits [a, b] (inclusive, both < 256) of the 8-word chunk
__device__ __forceinline__ void set_chunk_range(uint32_t (&w)[8], uint32_t a, uint32_t b) {
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const uint32_t lo = 32u * k, hi = lo + 31;
    if (b < lo || a > hi) continue;
    const uint32_t s = a > lo ? a - lo : 0, e = b < hi ? b - lo : 31;
    w[k] |= (~0u << s) & (~0u >> (31 - e));
  }
}

// Asynchronous 16-byte global -> shared copies (LDGSTS): the row data a
// producer needs at its NEXT visit lands in its shared slot while the tile's
// other chunks are multiplied; a register prefetch would be waited for as
// soon as the cursor state is written back to shared memory.
__device__ __forceinline__ void cp_async16(void *smem, uint64_t gaddr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rsu::su32(smem)), "l"(gaddr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// every COMMITTED group done (copies issued since the last commit keep flying)
__device__ __forceinline__ void cp_async_wait_committed() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Build the 256-bit chunk k (bits [256k, 256k+256)) of one row from its
// source; r is the row's shared-memory slot (this thread's own).
__device__ __forceinline__ void row_chunk(rsd2::RowCur *r, uint32_t k, uint32_t (&w)[8]) {
#pragma unroll
  for (int j = 0; j < 8; j++) w[j] = 0;
  const uint32_t type = r->type;
  if (type == 0) return;
  if (type == RS_TAG_BITSET) {
    const uint4 a = r->win, b = r->nwin;
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    if ((k & 63) != 63) {  // the next chunk of this quarter, for the next visit
      cp_async16(&r->win, r->base + 32ull * (k + 1));
      cp_async16(&r->nwin, r->base + 32ull * (k + 1) + 16);
    }
    return;
  }
  const uint32_t lo = 256u * k, hi = lo + 256u;
  const bool arr = type == RS_TAG_ARRAY;
  const uint32_t per = arr ? 8u : 4u, esz = arr ? 2u : 4u;
  uint32_t idx = r->idx, wpos = r->wpos;
  const uint32_t n = r->n;
  uint4 win = r->win;
  while (idx < n) {
    if (idx >= wpos + per) {  // next window (prefetched); fetch the one after it
      cp_async_wait_all();  // (it may have been issued during this visit)
      win = r->nwin;
      r->win = win;
      wpos += per;
      if (wpos + per < n) cp_async16(&r->nwin, r->base + (uint64_t)esz * (wpos + per));
    }
    const uint32_t j = idx - wpos;
    if (arr) {
      const uint32_t x = elem_of(win, j >> 1), v = (j & 1) ? x >> 16 : x & 0xFFFFu;
      if (v >= hi) break;
      set_chunk_bit(w, v - lo);
      idx++;
    } else {
      const uint32_t x = elem_of(win, j), st = x & 0xFFFFu, en = st + (x >> 16);
      if (st >= hi) break;
      set_chunk_range(w, st > lo ? st - lo : 0u, (en < hi - 1 ? en : hi - 1) - lo);
      if (en >= hi) break;  // the run continues into the next chunk
      idx++;
    }
  }
  r->idx = (uint16_t)idx;
  r->wpos = (uint16_t)wpos;
}

__device__ __forceinline__ void row_init(rsd2::RowCur *r, bool have, uint32_t item, const uint32_t *item_c,
                                         const DevBatch &S, const ushort4 *Q, int grp) {
  r->type = 0;
  if (!have) return;
  const uint32_t c = item_c[item];
  const uint8_t type = S.type[c];
  const uint32_t n = S.n[c];
  const uint64_t base = (uint64_t)(S.pool + S.off[c]);
  r->type = type;
  r->n = (uint16_t)n;
  r->base = base;
  const uint32_t k0 = 64u * grp;
  if (type == RS_TAG_BITSET) {
    cp_async16(&r->win, base + 32ull * k0);
    cp_async16(&r->nwin, base + 32ull * k0 + 16);
    return;
  }
  const ushort4 q = Q[item];
  const uint32_t idx = grp == 0 ? q.x : grp == 1 ? q.y : grp == 2 ? q.z : q.w;
  const bool arr = type == RS_TAG_ARRAY;
  const uint32_t per = arr ? 8u : 4u, esz = arr ? 2u : 4u;
  const uint32_t wpos = idx & ~(per - 1);
  r->idx = (uint16_t)idx;
  r->wpos = (uint16_t)wpos;
  if (wpos < n) cp_async16(&r->win, base + (uint64_t)esz * wpos);
  if (wpos + per < n) cp_async16(&r->nwin, base + (uint64_t)esz * (wpos + per));
}

__global__ void __launch_bounds__(rsu::UTHREADS, 1)
    k_allpairs_umma_direct(const uint32_t *__restrict__ tp_seg, const uint16_t *__restrict__ tp_r0,
                           const uint16_t *__restrict__ tp_c0, const uint16_t *__restrict__ tp_nb,
                           const uint32_t *__restrict__ seg_start, const uint32_t *__restrict__ item_c, DevBatch S,
                           const ushort4 *__restrict__ Q, const uint32_t *__restrict__ item_bm, uint64_t N,
                           unsigned long long *__restrict__ Mx) {
  using namespace rsu;
  extern __shared__ __align__(1024) uint8_t usm_raw[];
  uint8_t *usm = (uint8_t *)(((uintptr_t)usm_raw + 1023) & ~(uintptr_t)1023);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t seg = tp_seg[blockIdx.x];
  const uint32_t s0 = seg_start[seg], m = seg_start[seg + 1] - s0;
  const uint32_t r0 = tp_r0[blockIdx.x], c0 = tp_c0[blockIdx.x], nb = tp_nb[blockIdx.x];
  const bool shared_a = r0 == c0;
  const uint32_t rows_b = max(nb, (uint32_t)UM);
  const uint32_t sbytes = rows_b * UROWB;
  uint8_t *xst = usm;                                  // UNST expanded B stages
  rsd2::RowCur *cur = (rsd2::RowCur *)(usm + UNST * sbytes);  // producer row cursors: [slot][thread], 2 slots
  uint64_t *full = (uint64_t *)(usm + URING), *empty = full + UNST, *done = empty + UNST;
  uint32_t *tslot = (uint32_t *)(done + 1);
  for (uint32_t i = t; i < UNST * sbytes / 16; i += UTHREADS) ((uint4 *)xst)[i] = make_uint4(0, 0, 0, 0);
  if (t == 0) {
    for (int i = 0; i < UNST; i++) {
      ubar_init(&full[i], 4);
      ubar_init(&empty[i], 1);
    }
    ubar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(UTMEM)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp < 4) {  // unit block scales
    const uint32_t one = 0x7F7F7F7Fu;
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((uint32_t)(32 * warp) << 16) + USCOL + c),
                   "r"(one)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  constexpr int NCH = RS_WORDS * 64 / UKC;  // 256-bit chunks per row
  constexpr int PER = NCH / UNST;           // chunks per producer group (a quarter of the row)
  if (warp == UPROD / 32) {  // ------------------------------ MMA issuer
    const uint32_t idesc = idesc_mxf4(UM, (int)nb);
    const uint64_t db0 = sw128_desc(su32(xst));
    const uint32_t sstep = sbytes >> 4;
    const uint32_t sfa = tmem + USCOL, sfb = tmem + USCOL + 16u;
    uint32_t b = 0, ph = 0;
    for (int c = 0; c < NCH; c++) {
      ubar_wait(&full[b], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t db = db0 + (uint64_t)(b * sstep);
      const uint32_t ta = tmem + UACOL + 32u * b;
      if (elect_one()) {
        umma_mxf4(tmem, ta, db, idesc, sfa, sfb, c > 0);
        umma_mxf4(tmem, ta + 8u, db + 2, idesc, sfa, sfb, true);
        umma_mxf4(tmem, ta + 16u, db + 4, idesc, sfa, sfb, true);
        umma_mxf4(tmem, ta + 24u, db + 6, idesc, sfa, sfb, true);
        umma_commit(&empty[b]);
        if (c == NCH - 1) umma_commit(done);
      }
      __syncwarp();
      if (++b == (uint32_t)UNST) {
        b = 0;
        ph ^= 1u;
      }
    }
  } else if (warp < UPROD / 32) {  // ----------------------- producers
    // group g = warp / 4 builds chunks 64 g .. 64 g + 63 into stage g; warp q
    // of the group owns rows 32 q + lane (A) and B rows arow, arow + 128
    const int grp = warp >> 2, q = warp & 3;
    const uint32_t nrow_b = c0 < m ? min(nb, m - c0) : 0u, nrow_a = shared_a ? nrow_b : min((uint32_t)UM, m - r0);
    const uint32_t arow = 32 * q + lane;
    const int pt = t;  // producer thread index (< UPROD)
    // slot 0: the A row (= B row arow when shared); slot 1: B row arow (separate
    // A) or B row arow + 128 (shared A)
    rsd2::RowCur *c0s = &cur[pt], *c1s = &cur[UPROD + pt];
    if (shared_a) row_init(c0s, arow < nrow_b, s0 + c0 + arow, item_c, S, Q, grp);
    else row_init(c0s, arow < nrow_a, s0 + r0 + arow, item_c, S, Q, grp);
    if (shared_a) row_init(c1s, arow + UM < nrow_b, s0 + c0 + arow + UM, item_c, S, Q, grp);
    else row_init(c1s, arow < nrow_b, s0 + c0 + arow, item_c, S, Q, grp);
    cp_async_commit();
    uint8_t *sb = xst + grp * sbytes;
    const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + UACOL + 32u * grp;
    uint32_t eph = 0;
    for (int i = 0; i < PER; i++) {
      const uint32_t k = (uint32_t)(PER * grp + i);  // this visit's chunk
      if (i) {
        ubar_wait(&empty[grp], eph);
        eph ^= 1u;
      }
      cp_async_wait_committed();  // this visit's row data (issued and committed one visit ago)
      uint32_t e[32];
      {
        uint32_t w[8];
        row_chunk(c0s, k, w);
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const uint4 v = nib32(w[u]);
          e[4 * u] = v.x; e[4 * u + 1] = v.y; e[4 * u + 2] = v.z; e[4 * u + 3] = v.w;
          if (shared_a && arow < nrow_b) *(uint4 *)(sb + sw_off((int)arow, 16 * u, (int)rows_b)) = v;
        }
      }
      tmem_st32(ta, e);
      const uint32_t brow = shared_a ? arow + UM : arow;  // slot 1's B row
      if (brow < nrow_b) {
        uint32_t w[8];
        row_chunk(c1s, k, w);
#pragma unroll
        for (int u = 0; u < 8; u++) *(uint4 *)(sb + sw_off((int)brow, 16 * u, (int)rows_b)) = nib32(w[u]);
      }
      cp_async_commit();  // the next visit's row data
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) ubar_arrive(&full[grp]);
    }
    cp_async_wait_all();
  }
  ubar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {  // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3, colh = warp >> 2;
    if (warp < 8) {
      const uint32_t u = r0 + 32 * quarter + lane;
      const uint32_t bu = u < m ? item_bm[s0 + u] : 0;
      for (uint32_t cb = 128 * colh; cb < 128 * colh + 128 && cb < nb; cb += 32) {
        uint32_t v[32];
        const uint32_t tadr = tmem + ((uint32_t)(32 * quarter) << 16) + cb;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tadr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (u < m) {
#pragma unroll
          for (int j = 0; j < 32; j++) {
            const uint32_t vc = c0 + cb + j;
            const uint32_t cnt = (uint32_t)__uint_as_float(v[j]);
            if (cnt && vc < m && u < vc) {
              const uint32_t bv = item_bm[s0 + vc];
              const uint32_t lo = min(bu, bv), hi = max(bu, bv);
              atomicAdd(&Mx[(uint64_t)lo * N + hi], (unsigned long long)cnt);
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(UTMEM) : "memory");
}

constexpr int AP_TILE = 16;   // containers per tile side
constexpr int AP_KW = 64;     // words per smem chunk

// One CTA per (segment, tile i, tile j>=i): 16x16 popcount(AND) over 1024 words,
// accumulated into the N x N intersection matrix.
__global__ void __launch_bounds__(256) k_allpairs_tiles(const uint32_t *__restrict__ tp_seg,
                                                        const uint16_t *__restrict__ tp_i, const uint16_t *__restrict__ tp_j,
                                                        const uint32_t *__restrict__ seg_start,
                                                        const uint64_t *__restrict__ D, const uint32_t *__restrict__ item_bm,
                                                        uint64_t N, unsigned long long *__restrict__ M) {
  __shared__ uint64_t Ai[AP_TILE][AP_KW + 1];
  __shared__ uint64_t Bj[AP_TILE][AP_KW + 1];
  uint32_t seg = tp_seg[blockIdx.x];
  uint32_t s = seg_start[seg], m = seg_start[seg + 1] - s;
  uint32_t ti = tp_i[blockIdx.x], tj = tp_j[blockIdx.x];
  const int t = threadIdx.x;
  const int u = t >> 4, v = t & 15;
  uint32_t gu = ti * AP_TILE + u, gv = tj * AP_TILE + v;
  uint32_t acc = 0;
  for (int k0 = 0; k0 < RS_WORDS; k0 += AP_KW) {
    for (int x = t; x < AP_TILE * AP_KW; x += 256) {
      int row = x / AP_KW, col = x % AP_KW;
      uint32_t ra = ti * AP_TILE + row, rb = tj * AP_TILE + row;
      Ai[row][col] = ra < m ? D[(uint64_t)(s + ra) * RS_WORDS + k0 + col] : 0;
      Bj[row][col] = rb < m ? D[(uint64_t)(s + rb) * RS_WORDS + k0 + col] : 0;
    }
    __syncthreads();
#pragma unroll 16
    for (int k = 0; k < AP_KW; k++) acc += __popcll(Ai[u][k] & Bj[v][k]);
    __syncthreads();
  }
  bool valid = gu < m && gv < m && (ti != tj || u < v);
  if (valid && acc) {
    uint32_t bu = item_bm[s + gu], bv = item_bm[s + gv];
    uint32_t lo = min(bu, bv), hi = max(bu, bv);
    atomicAdd(&M[(uint64_t)lo * N + hi], (unsigned long long)acc);
  }
}

// Register-tiled variant: 32 x 32 containers per CTA, thread (u0, v0) owns the
// 2 x 2 block {u0, u0+16} x {v0, v0+16}, so every 4 shared loads feed 4
// AND-popcounts.  Row stride 33 words keeps the 16 distinct v rows of a warp
// on distinct banks; the 2 u rows of a warp are broadcasts.
constexpr int AP2_TILE = 32;
constexpr int AP2_KW = 32;

__global__ void __launch_bounds__(256) k_allpairs_tiles2(const uint32_t *__restrict__ tp_seg,
                                                         const uint16_t *__restrict__ tp_i, const uint16_t *__restrict__ tp_j,
                                                         const uint32_t *__restrict__ seg_start,
                                                         const uint64_t *__restrict__ D, const uint32_t *__restrict__ item_bm,
                                                         uint64_t N, unsigned long long *__restrict__ M) {
  __shared__ uint64_t Ai[AP2_TILE][AP2_KW + 1];
  __shared__ uint64_t Bj[AP2_TILE][AP2_KW + 1];
  const uint32_t seg = tp_seg[blockIdx.x];
  const uint32_t s = seg_start[seg], m = seg_start[seg + 1] - s;
  const uint32_t ti = tp_i[blockIdx.x], tj = tp_j[blockIdx.x];
  const int t = threadIdx.x, u0 = t >> 4, v0 = t & 15;
  uint32_t acc[4] = {0, 0, 0, 0};
  for (int k0 = 0; k0 < RS_WORDS; k0 += AP2_KW) {
#pragma unroll
    for (int q = 0; q < (AP2_TILE * AP2_KW) / 256; q++) {
      const int x = t + 256 * q, row = x / AP2_KW, col = x % AP2_KW;
      const uint32_t ra = ti * AP2_TILE + row, rb = tj * AP2_TILE + row;
      Ai[row][col] = ra < m ? D[(uint64_t)(s + ra) * RS_WORDS + k0 + col] : 0;
      Bj[row][col] = rb < m ? D[(uint64_t)(s + rb) * RS_WORDS + k0 + col] : 0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < AP2_KW; k++) {
      const uint64_t a0 = Ai[u0][k], a1 = Ai[u0 + 16][k], b0 = Bj[v0][k], b1 = Bj[v0 + 16][k];
      acc[0] += __popcll(a0 & b0);
      acc[1] += __popcll(a0 & b1);
      acc[2] += __popcll(a1 & b0);
      acc[3] += __popcll(a1 & b1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t u = u0 + 16 * (q >> 1), v = v0 + 16 * (q & 1);
    const uint32_t gu = ti * AP2_TILE + u, gv = tj * AP2_TILE + v;
    const bool valid = gu < m && gv < m && (ti != tj || u < v);
    if (valid && acc[q]) {
      const uint32_t bu = item_bm[s + gu], bv = item_bm[s + gv];
      const uint32_t lo = min(bu, bv), hi = max(bu, bv);
      atomicAdd(&M[(uint64_t)lo * N + hi], (unsigned long long)acc[q]);
    }
  }
}

__global__ void k_item_bitmap(uint64_t T, const uint32_t *__restrict__ item_c, const uint64_t *__restrict__ bm_start,
                              uint64_t nb, uint32_t *__restrict__ item_bm) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= T) return;
  uint64_t c = item_c[i], lo = 0, hi = nb;
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (bm_start[m] <= c) lo = m; else hi = m;
  }
  item_bm[i] = (uint32_t)lo;
}

__global__ void k_upper_triangle(uint64_t N, const unsigned long long *__restrict__ M, const uint64_t *__restrict__ card,
                                 uint64_t *__restrict__ inter, uint64_t *__restrict__ uni) {
  uint64_t i = blockIdx.y, j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= N || j >= N || j <= i) return;
  uint64_t k = i * (2 * N - i - 1) / 2 + (j - i - 1);
  uint64_t x = M[i * N + j];
  inter[k] = x;
  if (uni) uni[k] = card[i] + card[j] - x;
}

// --------------------------------------------------------- run_optimize

// container_normalize(c, consider_run=True) (containers.py:208-241) in place:
// the run form is only taken when strictly smaller, so it fits the slot.
__global__ void __launch_bounds__(DT) k_run_optimize(uint64_t nc, DevBatch S, uint8_t *otype, uint32_t *on,
                                                     uint8_t *__restrict__ pool, uint32_t *__restrict__ changed) {
  __shared__ __align__(16) DenseSmem sm;
  uint64_t c = blockIdx.x;
  if (c >= nc) return;
  uint8_t type = S.type[c];
  if (type == RS_TAG_RUN) return;  // normalized runs stay runs
  const int t = threadIdx.x;
  uint64_t r[4];
  if (type == RS_TAG_BITSET) {
    ld_words(S.pool, S.off[c], t, r);
    for (int k = 0; k < 4; k++) sm.X[4 * t + k] = r[k];
  } else {
    for (int k = 0; k < 4; k++) sm.X[4 * t + k] = 0;
    __syncthreads();
    scatter_container(S, (uint32_t)c, type, sm.X);
    __syncthreads();
    for (int k = 0; k < 4; k++) r[k] = sm.X[4 * t + k];
  }
  __syncthreads();
  uint32_t pc = 0;
  for (int k = 0; k < 4; k++) pc += __popcll(r[k]);
  uint32_t card, nruns;
  block_card_runs(sm.X, card, nruns, sm.red, true);
  if (!rs_run_admissible(card, nruns)) return;
  __syncthreads();
  uint32_t n = encode_result(sm, r, pc, card, RS_TAG_RUN, pool + S.off[c]);
  if (t == 0) {
    otype[c] = RS_TAG_RUN;
    on[c] = n;
    uint64_t lo = 0, hi = S.nb;
    while (hi - lo > 1) {
      uint64_t m = (lo + hi) >> 1;
      if (S.bm_start[m] <= c) lo = m; else hi = m;
    }
    changed[lo] = 1;
  }
}

struct Grouped {
  uint64_t T = 0, G = 0;
  uint64_t *keys = nullptr;
  uint32_t *item_c = nullptr, *seg_start = nullptr;
  void release() { dfree(keys); dfree(item_c); dfree(seg_start); }
};

// ---- grouping by a counting sort over the 2^16 chunk keys (selections of at
// most CS_MAX_SEL bitmaps).  A bitmap holds each key at most once, so key k's
// contributors are the set bits of a presence row P[k] (one bit per selection
// position): its count is the row's popcount, a contributor's rank inside the
// key is the popcount of the bits below it -- a stable order by selection
// position with no sort.  Three kernels and a scan replace the grouping
// keys, the two radix passes, the segment flags / scan / starts and the
// reorder of the radix path.
constexpr uint64_t CS_MAX_SEL = 1024;  // presence rows <= 32 words (8 MB); rank <= 32 popcounts
constexpr uint64_t CS_KEYS = 65536;
constexpr uint64_t CS_M40 = (1ull << 40) - 1;

__device__ __forceinline__ uint64_t sel_of_item(uint64_t t, uint64_t nsel, const uint64_t *__restrict__ qbase) {
  uint64_t lo = 0, hi = nsel;
  while (hi - lo > 1) {
    const uint64_t m = (lo + hi) >> 1;
    if (qbase[m] <= t) lo = m; else hi = m;
  }
  return lo;
}

__global__ void k_cs_mark(uint64_t T, uint64_t nsel, const uint64_t *__restrict__ qbase,
                          const uint64_t *__restrict__ qsrc, DevBatch S, uint32_t W, uint32_t *__restrict__ P) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint64_t k = sel_of_item(t, nsel, qbase);
  const uint32_t key = S.key[qsrc[k] + (t - qbase[k])];
  atomicOr(&P[(uint64_t)key * W + (k >> 5)], 1u << (k & 31));
}

// per key: (nonzero << 40) | count; entry CS_KEYS = 0, so the exclusive scan
// leaves (G << 40) | T there
__global__ void k_cs_count(uint32_t W, const uint32_t *__restrict__ P, uint64_t *__restrict__ cnt) {
  const uint64_t key = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (key > CS_KEYS) return;
  uint32_t s = 0;
  if (key < CS_KEYS)
    for (uint32_t w = 0; w < W; w++) s += __popc(P[key * W + w]);
  cnt[key] = s ? ((1ull << 40) | s) : 0ull;
}

__global__ void k_cs_scatter(uint64_t T, uint64_t nsel, const uint64_t *__restrict__ qbase,
                             const uint64_t *__restrict__ qsrc, DevBatch S, uint32_t W,
                             const uint32_t *__restrict__ P, const uint64_t *__restrict__ base,
                             uint64_t *__restrict__ keys, uint32_t *__restrict__ item_c,
                             uint32_t *__restrict__ seg_start) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t == 0) {
    const uint64_t tot = base[CS_KEYS];
    seg_start[tot >> 40] = (uint32_t)(tot & CS_M40);
  }
  if (t >= T) return;
  const uint64_t k = sel_of_item(t, nsel, qbase);
  const uint32_t c = (uint32_t)(qsrc[k] + (t - qbase[k]));
  const uint32_t key = S.key[c];
  const uint32_t *row = P + (uint64_t)key * W;
  uint32_t r = __popc(row[k >> 5] & ((1u << (k & 31)) - 1u));
  for (uint32_t w = 0; w < (uint32_t)(k >> 5); w++) r += __popc(row[w]);
  const uint64_t b = base[key], pos = (b & CS_M40) + r;
  keys[pos] = ((uint64_t)key << 40) | t;
  item_c[pos] = c;
  if (r == 0) seg_start[b >> 40] = (uint32_t)pos;
}

// The counting-sort grouping: item_c comes out already in key order.
int group_by_key_counting(const rs_batch *in, const std::vector<uint64_t> &sel, Grouped &g) {
  const uint64_t n = sel.size();
  std::vector<uint64_t> qbase(n + 1, 0), qsrc(n + 1, 0);
  for (uint64_t k = 0; k < n; k++) {
    qsrc[k] = in->h_bm_start[sel[k]];
    qbase[k + 1] = qbase[k] + (in->h_bm_start[sel[k] + 1] - in->h_bm_start[sel[k]]);
  }
  const uint64_t T = g.T = qbase[n];
  const uint32_t W = (uint32_t)((n + 31) / 32);
  uint64_t *d_q = (uint64_t *)dalloc(2 * (n + 1) * 8);
  uint32_t *P = (uint32_t *)dalloc(CS_KEYS * W * 4);
  uint64_t *cnt = (uint64_t *)dalloc((CS_KEYS + 1) * 8), *base = (uint64_t *)dalloc((CS_KEYS + 1) * 8);
  g.keys = (uint64_t *)dalloc((T + 1) * 8);
  g.item_c = (uint32_t *)dalloc((T + 1) * 4);
  g.seg_start = (uint32_t *)dalloc((std::min<uint64_t>(T, CS_KEYS) + 2) * 4);
  if (!d_q || !P || !cnt || !base || !g.keys || !g.item_c || !g.seg_start) {
    set_error("device allocation failed (group)");
    return RS_ENOMEM;
  }
  qbase.insert(qbase.end(), qsrc.begin(), qsrc.end());  // one upload: qbase then qsrc
  RS_TRY(h2d(d_q, qbase.data(), 2 * (n + 1) * 8));
  const uint64_t *d_qb = d_q, *d_qs = d_q + n + 1;
  RS_CK(cudaMemsetAsync(P, 0, CS_KEYS * W * 4, g_stream));
  if (T) RS_LAUNCH(k_cs_mark, grid_for(T, 256), 256, 0, T, n, d_qb, d_qs, in->dev(), W, P);
  RS_LAUNCH(k_cs_count, grid_for(CS_KEYS + 1, 256), 256, 0, W, P, cnt);
  RS_TRY(scan_exclusive<uint64_t>(cnt, base, CS_KEYS + 1));
  RS_LAUNCH(k_cs_scatter, grid_for(T ? T : 1, 256), 256, 0, T, n, d_qb, d_qs, in->dev(), W, P, base, g.keys,
            g.item_c, g.seg_start);
  uint64_t tot = 0;
  RS_TRY(d2h(&tot, base + CS_KEYS, 8));
  g.G = tot >> 40;
  dfree(d_q); dfree(P); dfree(cnt); dfree(base);
  if ((tot & CS_M40) != T) {
    set_error("grouping lost items (a chunk key repeated inside a bitmap)");
    return RS_EARG;
  }
  return RS_OK;
}

// Group the containers of bitmaps sel[0..n) (in that order) by chunk key.
int group_by_key(const rs_batch *in, const std::vector<uint64_t> &sel, Grouped &g) {
  uint64_t n = sel.size();
  std::vector<uint64_t> qbase(n + 1, 0), qsrc(n + 1, 0);
  for (uint64_t k = 0; k < n; k++) {
    qsrc[k] = in->h_bm_start[sel[k]];
    qbase[k + 1] = qbase[k] + (in->h_bm_start[sel[k] + 1] - in->h_bm_start[sel[k]]);
  }
  g.T = qbase[n];
  uint64_t T = g.T;
  uint64_t *d_qb = (uint64_t *)dalloc((n + 1) * 8), *d_qs = (uint64_t *)dalloc((n + 1) * 8);
  g.keys = (uint64_t *)dalloc((T + 1) * 8);
  g.item_c = (uint32_t *)dalloc((T + 1) * 4);
  uint32_t *flag = (uint32_t *)dalloc((T + 1) * 4), *pos = (uint32_t *)dalloc((T + 1) * 4);
  g.seg_start = (uint32_t *)dalloc((T + 2) * 4);
  if (!d_qb || !d_qs || !g.keys || !g.item_c || !flag || !pos || !g.seg_start) {
    set_error("device allocation failed (group)");
    return RS_ENOMEM;
  }
  RS_TRY(h2d(d_qb, qbase.data(), (n + 1) * 8));
  RS_TRY(h2d(d_qs, qsrc.data(), (n + 1) * 8));
  RS_LAUNCH(k_group_keys, grid_for(T, 256), 256, 0, T, n, d_qb, d_qs, in->dev(), g.keys, g.item_c);
  // the low 40 bits (item index) are already ascending: a stable sort of the
  // 16-bit key field alone gives the full order (2 radix passes instead of 7)
  RS_TRY(sort_u64(g.keys, T, 56, 40));
  // item index after the sort comes from the low 40 bits: reorder item_c
  RS_LAUNCH(k_seg_flags, grid_for(T + 1, 256), 256, 0, T, g.keys, flag);
  RS_TRY(scan_exclusive<uint32_t>(flag, pos, T + 1));
  RS_LAUNCH(k_seg_starts, grid_for(T + 1, 256), 256, 0, T, flag, pos, g.seg_start);
  uint32_t G = 0;
  RS_TRY(d2h(&G, pos + T, 4));
  g.G = G;
  dfree(d_qb); dfree(d_qs); dfree(flag); dfree(pos);
  return RS_OK;
}

__global__ void k_reorder_items(uint64_t T, const uint64_t *__restrict__ keys, const uint32_t *__restrict__ item_in,
                                uint32_t *__restrict__ item_out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < T) item_out[i] = item_in[keys[i] & ((1ull << 40) - 1)];
}

int group_and_reorder(const rs_batch *in, const std::vector<uint64_t> &sel, Grouped &g) {
  // RS_GROUP_RADIX=1: the radix-sort grouping whatever the selection size (A/B)
  if (sel.size() <= CS_MAX_SEL && !env_flag_("RS_GROUP_RADIX")) return group_by_key_counting(in, sel, g);
  RS_TRY(group_by_key(in, sel, g));
  uint32_t *sorted_c = (uint32_t *)dalloc((g.T + 1) * 4);
  if (!sorted_c) { set_error("device allocation failed (group)"); return RS_ENOMEM; }
  RS_LAUNCH(k_reorder_items, grid_for(g.T, 256), 256, 0, g.T, g.keys, g.item_c, sorted_c);
  dfree(g.item_c);
  g.item_c = sorted_c;
  return RS_OK;
}

}  // namespace

extern "C" int rs_union_many(const rs_batch *in, const uint64_t *idx, uint64_t n, rs_batch **out) {
  RS_TRY(ensure_device());
  *out = nullptr;
  RS_TRY(fetch_host_meta(in));
  std::vector<uint64_t> sel(n);
  for (uint64_t k = 0; k < n; k++) {
    sel[k] = idx ? idx[k] : k;
    if (sel[k] >= in->nb) { set_error("bitmap index out of range"); return RS_EARG; }
  }
  Grouped g;
  RS_TRY(group_and_reorder(in, sel, g));
  RS_TRY(ub_reserve(g.G * 8192));
  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, 1, g.G, g.G * 8192);
  if (rc) { g.release(); rs_batch_free(b); return rc; }
  ub_register(b);  // one 8 KB slot per key until packed
  // keys by result rule: order-free bitset ORs and order-dependent folds,
  // the two kernels concurrently on side streams
  uint32_t *lists = (uint32_t *)dalloc((2 * g.G + 2) * 4), *cnt = (uint32_t *)dalloc(32);
  if (!lists || !cnt) { g.release(); rs_batch_free(b); set_error("device allocation failed (union lists)"); return RS_ENOMEM; }
  RS_CK(cudaMemsetAsync(cnt, 0, 32, g_stream));  // [0,1] list sizes, [2,3] work counters
  RS_LAUNCH(k_union_classify, grid_for(g.G, 256), 256, 0, g.G, g.seg_start, g.item_c, in->dev(), lists,
            lists + g.G + 1, cnt);
  {
    const unsigned sms = sm_count_();
    Fork F;
    RS_TRY(F.begin(2));
    F.next();
    int occ_or = 0, occ_fold = 0;
    RS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_or, k_union_or, UT, 0));
    RS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_fold, k_union_fold, DT, 0));
    // the two persistent kernels share the SMs: one resident wave of each
    RS_LAUNCH_PROF("union_or", g.G, k_union_or, (unsigned)std::min<uint64_t>(g.G, sms * std::max(occ_or, 1)), UT, 0,
                   lists, cnt,
                   g.seg_start, g.item_c, g.keys, in->dev(), b->d_key, b->d_type, b->d_card, b->d_n, b->d_off,
                   b->d_pool);
    F.next();
    RS_LAUNCH_PROF("union_fold", g.G, k_union_fold, (unsigned)std::min<uint64_t>(g.G, sms * std::max(occ_fold, 1)), DT, 0,
                   lists + g.G + 1, cnt + 1, g.seg_start, g.item_c, g.keys, in->dev(), b->d_key, b->d_type, b->d_card,
                   b->d_n, b->d_off, b->d_pool);
    RS_TRY(F.end());
  }
  dfree(lists);
  dfree(cnt);
  uint64_t hs[2] = {0, g.G};
  RS_TRY(h2d(b->d_bm_start, hs, 16));
  RS_TRY(finalize_batch(b));
  RS_CK(cudaStreamSynchronize(g_stream));
  g.release();
  b->h_bm_start.assign(hs, hs + 2);
  b->type_mask = (uint8_t)((1u << RS_TAG_ARRAY) | (1u << RS_TAG_BITSET) | (in->type_mask & (1u << RS_TAG_RUN)));
  b->h_valid = true;
  *out = b;
  return RS_OK;
}

extern "C" int rs_all_pairs_cardinality(const rs_batch *in, uint64_t *inter, uint64_t *uni) {
  RS_TRY(resolve_pending(in));
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(in));
  uint64_t N = in->nb;
  uint64_t npairs = N * (N - 1) / 2;
  if (N < 2) return RS_OK;
  std::vector<uint64_t> sel(N);
  for (uint64_t k = 0; k < N; k++) sel[k] = k;
  Grouped g;
  trace("allpairs: start");
  RS_TRY(group_and_reorder(in, sel, g));
  trace("allpairs: group by key");
  // Keys with enough containers to fill 128-row tiles go to the tensor cores
  // (k_allpairs_umma); the rest use the CUDA-core 16x16 POPC tiles, whose cost
  // shrinks with m^2 (RS_ALLPAIRS_UMMA=0 sends everything to POPC tiles,
  // RS_ALLPAIRS_UMMA_MIN sets the threshold).  The 32x32 register-tiled POPC
  // variant (RS_ALLPAIRS_TILES=2) measured slower (5.5 vs 4.6 ms on C5).
  const char *tv = getenv("RS_ALLPAIRS_TILES");
  const bool tiles2 = tv && *tv == '2';
  const char *uv = getenv("RS_ALLPAIRS_UMMA");
  const bool use_umma = !(uv && *uv == '0');
  const char *mv = getenv("RS_ALLPAIRS_UMMA_MIN");
  const uint32_t umma_min = mv && *mv ? (uint32_t)atoi(mv) : 48;
  // RS_ALLPAIRS_DIRECT=1: the tensor-core tiles build their rows from the
  // containers (k_allpairs_umma_direct, no densified copy).  Measured 3.3 ms
  // against 0.44 ms for the TMA-fed tiles on config 5: the producers become
  // instruction-bound (~1,360 warp instructions per visit against a ~1,300-
  // cycle budget per visit; each lane walks its row's array values one by
  // one with divergent, select-heavy bit setting), so the densify + TMA path
  // stays the default.
  const char *dv = getenv("RS_ALLPAIRS_DIRECT");
  const bool direct = use_umma && dv && *dv == '1';
  std::vector<uint32_t> dlist;  // direct: the items the CUDA-core tiles read
  // The densify needs only the grouping: it is queued right behind the
  // segment starts' copy to the host, and the host builds and uploads the
  // tile lists while it runs (the copy is waited for by its event, not by
  // draining the stream).
  uint64_t *D = (uint64_t *)dalloc((g.T ? g.T : 1) * 8192);
  uint32_t *item_bm = (uint32_t *)dalloc((g.T + 1) * 4);
  if (!D || !item_bm) { set_error("device allocation failed (all pairs)"); return RS_ENOMEM; }
  thread_local uint32_t *hseg_pin = nullptr;
  thread_local uint64_t hseg_cap = 0;
  thread_local cudaEvent_t seg_ev = nullptr;
  if (hseg_cap < g.G + 1) {
    if (hseg_pin) cudaFreeHost(hseg_pin);
    hseg_pin = nullptr;
    RS_CK(cudaMallocHost(&hseg_pin, (g.G + 1) * 4));
    hseg_cap = g.G + 1;
  }
  if (!seg_ev) RS_CK(cudaEventCreateWithFlags(&seg_ev, cudaEventDisableTiming));
  RS_CK(cudaMemcpyAsync(hseg_pin, g.seg_start, (g.G + 1) * 4, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaEventRecord(seg_ev, g_stream));
  RS_LAUNCH(k_item_bitmap, grid_for(g.T, 256), 256, 0, g.T, g.item_c, in->d_bm_start, in->nb, item_bm);
  auto densify = [&](uint64_t nd, const uint32_t *d_dlist) -> int {
    if (env_flag_("RS_DENSIFY_CTA") && !d_dlist) {  // the CTA-per-row kernel (A/B only)
      RS_LAUNCH_PROF("densify", g.T, k_densify, (unsigned)g.T, DT, 0, g.T, g.item_c, in->dev(), D);
    } else {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const uint64_t g_need = (nd + DW_WARPS - 1) / DW_WARPS;
      const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g_need, (uint64_t)sms * 6));
      RS_LAUNCH_PROF("densify", nd, k_densify_warp, grid, 32 * DW_WARPS, 0, nd, g.item_c, in->dev(), D, d_dlist);
    }
    return RS_OK;
  };
  if (!direct) RS_TRY(densify(g.T, nullptr));
  RS_CK(cudaEventSynchronize(seg_ev));
  std::vector<uint32_t> hseg(hseg_pin, hseg_pin + g.G + 1);
  std::vector<uint32_t> tseg, useg;
  std::vector<uint16_t> ti, tj, ur0, uc0, unb;
  const uint32_t tile = tiles2 ? AP2_TILE : AP_TILE;
  auto popc_tiles = [&](uint64_t s, uint32_t first, uint32_t m) {  // tiles over rows [first*tile, m)
    const uint32_t nt = (m + tile - 1) / tile;
    for (uint32_t a = first; a < nt; a++)
      for (uint32_t b2 = a; b2 < nt; b2++) { tseg.push_back((uint32_t)s); ti.push_back(a); tj.push_back(b2); }
    for (uint32_t r = first * tile; direct && r < m; r++) dlist.push_back(hseg[s] + r);
  };
  auto umma_tile = [&](uint64_t s, uint32_t r0, uint32_t c0, uint32_t nb) {
    useg.push_back((uint32_t)s); ur0.push_back(r0); uc0.push_back(c0); unb.push_back((nb + 15) & ~15u);
  };
  for (uint64_t s = 0; s < g.G; s++) {
    const uint32_t m = hseg[s + 1] - hseg[s];
    if (m < 2) continue;
    if (!use_umma || m < umma_min) {
      popc_tiles(s, 0, m);
    } else if (m <= (uint32_t)rsu::UNMAX) {
      // one tile: rows 0..127 against all m rows; the corner past row 128 on CUDA cores
      umma_tile(s, 0, 0, m);
      if (m > (uint32_t)rsu::UM) popc_tiles(s, rsu::UM / tile, m);
    } else {
      const uint32_t nt = (m + rsu::UM - 1) / rsu::UM;
      for (uint32_t a = 0; a < nt; a++)
        for (uint32_t b2 = a; b2 < nt; b2++)
          umma_tile(s, a * rsu::UM, b2 * rsu::UM, std::min<uint32_t>(rsu::UM, m - b2 * rsu::UM));
    }
  }
  uint64_t ntp = tseg.size(), nup = useg.size();
  const uint64_t nd = direct ? dlist.size() : g.T;  // rows to densify
  uint32_t *d_dlist = direct ? (uint32_t *)dalloc((nd + 1) * 4) : nullptr;
  ushort4 *d_Q = direct ? (ushort4 *)dalloc((g.T + 1) * 8) : nullptr;
  if (direct && (!d_dlist || !d_Q)) { set_error("device allocation failed (all pairs)"); return RS_ENOMEM; }
  if (direct && nd) RS_TRY(h2d(d_dlist, dlist.data(), nd * 4));
  // the seven tile lists in one page-locked block, one copy (16-byte aligned parts)
  const uint64_t lt_bytes[7] = {ntp * 4, ntp * 2, ntp * 2, nup * 4, nup * 2, nup * 2, nup * 2};
  const void *lt_src[7] = {tseg.data(), ti.data(), tj.data(), useg.data(), ur0.data(), uc0.data(), unb.data()};
  uint64_t lt_off[8] = {0};
  for (int k = 0; k < 7; k++) lt_off[k + 1] = lt_off[k] + rs_pad16(lt_bytes[k] + 16);
  thread_local uint8_t *lt_pin = nullptr;
  thread_local uint64_t lt_cap = 0;
  thread_local cudaEvent_t lt_ev = nullptr;
  if (!lt_ev) RS_CK(cudaEventCreateWithFlags(&lt_ev, cudaEventDisableTiming));
  RS_CK(cudaEventSynchronize(lt_ev));  // the previous call's copy out of the block is done
  if (lt_cap < lt_off[7]) {
    if (lt_pin) cudaFreeHost(lt_pin);
    lt_pin = nullptr;
    RS_CK(cudaMallocHost(&lt_pin, lt_off[7]));
    lt_cap = lt_off[7];
  }
  for (int k = 0; k < 7; k++)
    if (lt_bytes[k]) memcpy(lt_pin + lt_off[k], lt_src[k], lt_bytes[k]);
  uint8_t *d_lists = (uint8_t *)dalloc(lt_off[7]);
  unsigned long long *Mx = (unsigned long long *)dalloc(N * N * 8);
  uint64_t *d_inter = (uint64_t *)dalloc(npairs * 8), *d_uni = (uint64_t *)dalloc(npairs * 8);
  if (!d_lists || !Mx || !d_inter || !d_uni) {
    set_error("device allocation failed (all pairs)");
    return RS_ENOMEM;
  }
  uint32_t *d_tseg = (uint32_t *)(d_lists + lt_off[0]), *d_useg = (uint32_t *)(d_lists + lt_off[3]);
  uint16_t *d_ti = (uint16_t *)(d_lists + lt_off[1]), *d_tj = (uint16_t *)(d_lists + lt_off[2]),
           *d_ur0 = (uint16_t *)(d_lists + lt_off[4]), *d_uc0 = (uint16_t *)(d_lists + lt_off[5]),
           *d_unb = (uint16_t *)(d_lists + lt_off[6]);
  trace("allpairs: tile lists + allocs");
  RS_CK(cudaMemcpyAsync(d_lists, lt_pin, lt_off[7], cudaMemcpyHostToDevice, g_stream));
  RS_CK(cudaEventRecord(lt_ev, g_stream));
  RS_CK(cudaMemsetAsync(Mx, 0, N * N * 8, g_stream));
  trace("allpairs: uploads + memset");
  if (direct) {
    RS_LAUNCH(k_quarter_index, grid_for(g.T, 256), 256, 0, g.T, g.item_c, in->dev(), d_Q);
    RS_TRY(densify(nd, d_dlist));
  }
  trace("allpairs: densify");
  // (running the tensor-core and CUDA-core tiles concurrently on side streams
  // measured no faster: 1.078 vs 1.087 ms, the umma tiles slowing 0.44 -> 0.50)
  if (nup && direct) {
    static bool attr_d = false;
    if (!attr_d) {
      RS_CK(cudaFuncSetAttribute(k_allpairs_umma_direct, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)rsu::USMEM));
      attr_d = true;
    }
    RS_LAUNCH_PROF("allpairs_umma", nup, k_allpairs_umma_direct, (unsigned)nup, rsu::UTHREADS, rsu::USMEM, d_useg,
                   d_ur0, d_uc0, d_unb, g.seg_start, g.item_c, in->dev(), d_Q, item_bm, N, Mx);
  } else if (nup) {
    static bool attr = false;
    if (!attr) {
      RS_CK(cudaFuncSetAttribute(k_allpairs_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsu::USMEM));
      attr = true;
    }
    CUtensorMap tmD;
    RS_TRY(rows_tensor_map(&tmD, D, g.T));
    RS_LAUNCH_PROF("allpairs_umma", nup, k_allpairs_umma, (unsigned)nup, rsu::UTHREADS, rsu::USMEM, d_useg, d_ur0,
                   d_uc0, d_unb, g.seg_start, tmD, item_bm, N, Mx);
#ifdef RS_UMMA_TRACE
    {
      long long h[6][256];
      cudaStreamSynchronize(g_stream);
      cudaMemcpyFromSymbol(h, g_umma_trace, sizeof h);
      const long long t0 = h[4][0];
      for (int c = 0; c < 256; c += 1)
        fprintf(stderr, "c=%3d raw(box)=%7lld rfull=%7lld start=%7lld full=%7lld issue=%7lld commit=%7lld\n", c,
                c < 64 ? h[4][c] - t0 : 0, h[5][c] - t0, h[0][c] - t0, h[1][c] - t0, h[2][c] - t0, h[3][c] - t0);
    }
#endif
  }
  if (!ntp) {
  } else if (tiles2)
    RS_LAUNCH_PROF("allpairs", ntp, k_allpairs_tiles2, (unsigned)ntp, 256, 0, d_tseg, d_ti, d_tj, g.seg_start, D,
                   item_bm, N, Mx);
  else
    RS_LAUNCH_PROF("allpairs", ntp, k_allpairs_tiles, (unsigned)ntp, 256, 0, d_tseg, d_ti, d_tj, g.seg_start, D,
                   item_bm, N, Mx);
  trace("allpairs: tiles");
  dim3 grid(grid_for(N, 256), (unsigned)N);
  k_upper_triangle<<<grid, 256, 0, g_stream>>>(N, Mx, in->d_bm_card, d_inter, uni ? d_uni : nullptr);
  ++g_launches;
  RS_CK(cudaGetLastError());
  trace("allpairs: upper triangle");
  if (uni) RS_CK(cudaMemcpyAsync(uni, d_uni, npairs * 8, cudaMemcpyDeviceToHost, g_stream));
  RS_TRY(d2h(inter, d_inter, npairs * 8));  // one synchronization for both
  trace("allpairs: readback");
  dfree(d_dlist); dfree(d_Q);
  dfree(D); dfree(item_bm); dfree(Mx); dfree(d_inter); dfree(d_uni);
  dfree(d_lists);
  g.release();
  return RS_OK;
}

extern "C" int rs_batch_run_optimize(rs_batch *b, uint8_t *changed) {
  RS_TRY(resolve_pending(b));
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(b));
  uint32_t *d_ch = (uint32_t *)dalloc((b->nb + 1) * 4);
  if (!d_ch) { set_error("device allocation failed (run_optimize)"); return RS_ENOMEM; }
  RS_CK(cudaMemsetAsync(d_ch, 0, (b->nb + 1) * 4, g_stream));
  RS_LAUNCH(k_run_optimize, (unsigned)b->nc, DT, 0, b->nc, b->dev(), b->d_type, b->d_n, b->d_pool, d_ch);
  std::vector<uint32_t> h(b->nb + 1);
  RS_TRY(d2h(h.data(), d_ch, (b->nb + 1) * 4));
  if (changed)
    for (uint64_t i = 0; i < b->nb; i++) changed[i] = (uint8_t)(h[i] != 0);
  dfree(d_ch);
  b->type_mask |= (uint8_t)(1u << RS_TAG_RUN);
  return RS_OK;
}
