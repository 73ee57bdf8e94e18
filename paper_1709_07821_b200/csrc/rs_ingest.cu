// rs_ingest.cu -- batch construction: wire images (serde.deserialize) and
// uint32 values (RoaringBitmap.from_values), plus concat / select copies.
#include <cub/cub.cuh>
#include <algorithm>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include "rs_internal.cuh"

using namespace rs;

namespace {

// ------------------------------------------------------------- wire ingest

enum : uint8_t {
  V_OK = 0,
  V_ARRAY_ORDER = 1,
  V_BITSET_CARD = 2,
  V_BITSET_SMALL = 3,
  V_RUN_ESCAPE = 4,
  V_RUN_OVERLAP = 5,
  V_RUN_CARD = 6,
  V_RUN_ADMISSIBLE = 7
};

// 16-byte output vector from two consecutive aligned source chunks c0, c1
// shifted down by Q words and RB bits (the source's misalignment).
template <int Q>
__device__ __forceinline__ uint4 realign(const uint4 &c0, const uint4 &c1, uint32_t rb) {
  const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  uint32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; j++) o[j] = rb ? __funnelshift_r(w[j + Q], w[j + Q + 1], rb) : w[j + Q];
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// Copy nbytes (even) from a 2-byte aligned source to a 16-byte aligned
// destination in 16-byte vectors, zeroing the pad tail.  The source is read
// as aligned 16-byte chunks (from the one at or below src; a chunk past the
// last needed byte is never touched) and each output vector is funnel-shifted
// out of two of them; a lane's CPK vectors are loaded before any is stored.
// (Wire payloads sit at any even offset: the 2- and 4-byte copy loops this
// replaces took 72 % of the ingest kernel's stall samples, one load -> store
// round trip per element.)
constexpr int CPK = 4;
__device__ void warp_copy_payload(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src,
                                  uint32_t nbytes, int lane) {
  const uint32_t sh = (uint32_t)((uintptr_t)src & 15), q = sh >> 2, rb = 8 * (sh & 3);
  const uint4 *as = (const uint4 *)(src - sh);
  const uint32_t nv = (nbytes + 15) >> 4;
  for (uint32_t i0 = 0; i0 < nv; i0 += 32 * CPK) {
    uint4 c0[CPK], c1[CPK];
#pragma unroll
    for (int k = 0; k < CPK; k++) {
      const uint32_t i = i0 + lane + 32 * k;
      c0[k] = c1[k] = make_uint4(0, 0, 0, 0);
      if (i < nv) {
        c0[k] = as[i];
        if (sh && 16 * i + 16 - sh < nbytes) c1[k] = as[i + 1];
      }
    }
#pragma unroll
    for (int k = 0; k < CPK; k++) {
      const uint32_t i = i0 + lane + 32 * k;
      if (i >= nv) break;
      uint4 o;
      switch (q) {
        case 0: o = realign<0>(c0[k], c1[k], rb); break;
        case 1: o = realign<1>(c0[k], c1[k], rb); break;
        case 2: o = realign<2>(c0[k], c1[k], rb); break;
        default: o = realign<3>(c0[k], c1[k], rb); break;
      }
      const uint32_t rem = nbytes - 16 * i;  // valid bytes of this vector (even)
      if (rem < 16) {
        uint32_t *ow = (uint32_t *)&o;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int v = (int)rem - 4 * j;
          ow[j] &= v >= 4 ? ~0u : v == 2 ? 0xFFFFu : 0u;
        }
      }
      ((uint4 *)dst)[i] = o;
    }
  }
}

// One warp per container: copy the payload from the staged wire bytes into
// the aligned pool and run the payload checks of serde.deserialize
// (serde.py:122-164) in the reference's order.  With `card_fix` (deferred
// validation) a failing container is also made self-consistent -- escaping
// runs clamped to the chunk, the descriptor cardinality replaced by what the
// payload holds -- so ops issued before the checks are read back stay in
// bounds; the batch is rejected at rs_batch_wait either way.
__global__ void k_wire_gather_validate(uint64_t nc, uint64_t nvalidate, const uint8_t *__restrict__ staged,
                                       const uint64_t *__restrict__ src_off, DevBatch B,
                                       uint8_t *__restrict__ pool, uint8_t *__restrict__ vcode,
                                       uint32_t *__restrict__ vval, int *__restrict__ any_err,
                                       uint32_t *__restrict__ card_fix) {
  uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (c >= nc) return;
  uint8_t t = B.type[c];
  uint32_t n = B.n[c], card = B.card[c];
  const uint8_t *src = staged + src_off[c];
  warp_copy_payload(pool + B.off[c], src, rs_payload_bytes(t, n), lane);
  if (c >= nvalidate) return;
  const uint16_t *s16 = (const uint16_t *)src;
  uint8_t code = V_OK;
  uint32_t val = 0, fixed = card;
  if (t == RS_TAG_ARRAY) {
    // first position that breaks strict increase (n = none)
    uint32_t first_bad = n;
    for (uint32_t i = 1 + lane; i < n; i += 32)
      if (s16[i] <= s16[i - 1]) { first_bad = i; break; }
    for (int o = 16; o; o >>= 1) first_bad = min(first_bad, __shfl_xor_sync(0xffffffffu, first_bad, o));
    if (first_bad < n) {
      code = V_ARRAY_ORDER;
      // deferred mode: keep only the strictly increasing prefix, so every
      // kernel's per-pair output bound (2*min(na,nb), containers.py:471)
      // holds until the batch is rejected at rs_batch_wait
      fixed = first_bad;
      if (card_fix && lane == 0) const_cast<uint32_t *>(B.n)[c] = first_bad;
    }
  } else if (t == RS_TAG_BITSET) {
    uint32_t pc = 0;
    for (uint32_t i = lane; i < 2048; i += 32) pc += __popc((uint32_t)s16[2 * i] | ((uint32_t)s16[2 * i + 1] << 16));
    for (int o = 16; o; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
    if (pc != card) { code = V_BITSET_CARD; val = pc; }
    else if (card <= RS_ARRAY_MAX) code = V_BITSET_SMALL;
    fixed = pc;
  } else {
    bool esc = false, ovl = false;
    uint32_t sum = 0, clamped = 0;
    for (uint32_t i = lane; i < n; i += 32) {
      uint32_t st = s16[2 * i], ln = s16[2 * i + 1];
      esc |= st + ln > 0xFFFFu;
      if (i > 0) ovl |= !(st > (uint32_t)s16[2 * i - 2] + s16[2 * i - 1] + 1);
      sum += ln;
      clamped += min(ln, 0xFFFFu - st) + 1;
    }
    for (int o = 16; o; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      clamped += __shfl_xor_sync(0xffffffffu, clamped, o);
    }
    if (__any_sync(0xffffffffu, esc)) code = V_RUN_ESCAPE;
    else if (__any_sync(0xffffffffu, ovl)) code = V_RUN_OVERLAP;
    else if (sum + n != card) { code = V_RUN_CARD; val = sum + n; }
    else if (!rs_run_admissible(card, n)) code = V_RUN_ADMISSIBLE;
    fixed = clamped;
    if (card_fix && code == V_RUN_ESCAPE) {
      uint16_t *d16 = (uint16_t *)(pool + B.off[c]);
      for (uint32_t i = lane; i < n; i += 32) {
        uint32_t st = s16[2 * i], ln = s16[2 * i + 1];
        d16[2 * i + 1] = (uint16_t)min(ln, 0xFFFFu - st);
      }
    }
  }
  if (lane == 0) {
    vcode[c] = code;
    vval[c] = val;
    if (code) {
      atomicOr(any_err, 1);
      if (card_fix) card_fix[c] = fixed;
    }
  }
}

struct WireErr {
  bool set = false;
  uint64_t image = 0, container = 0;  // container: global index where payload checks stop
  bool descriptor_stage = false;
  int64_t offset = 0;
  std::string msg;
};

static inline uint16_t g16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static inline uint32_t g32(const uint8_t *p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Host walk of the descriptor sections (serde.py:87-169 structure): container
// table, payload sources and pool offsets, and the first structural error.
struct WireWalk {
  std::vector<uint64_t> bm_start;
  std::vector<uint16_t> key;
  std::vector<uint8_t> type;
  std::vector<uint32_t> card, cnt;
  std::vector<uint64_t> src, poff;  // src: absolute offset in buf
  uint64_t pool = 0, nb_built = 0, max_runs = 0;
  WireErr err;
};

void walk_wire(const uint8_t *buf, const uint64_t *offs, uint64_t n, WireWalk &W) {
  W.bm_start.assign(n + 1, 0);
  WireErr &err = W.err;
  char msg[256];
  for (uint64_t i = 0; i < n && !err.set; i++) {
    const uint8_t *d = buf + offs[i];
    uint64_t len = offs[i + 1] - offs[i], off = 0, start = 0;
    W.bm_start[i] = W.key.size();
    auto fail = [&](int64_t o, bool desc_stage) {
      err.set = true;
      err.image = i;
      err.container = W.key.size();
      err.descriptor_stage = desc_stage;
      err.offset = o;
      err.msg = msg;
    };
    auto need = [&](uint64_t nb, const char *what, bool desc_stage) -> bool {
      if (len - off < nb) {
        snprintf(msg, sizeof msg, "truncated %s: need %llu bytes, have %llu", what,
                 (unsigned long long)nb, (unsigned long long)(len - off));
        fail((int64_t)off, desc_stage);
        return false;
      }
      start = off;
      off += nb;
      return true;
    };
    if (!need(4, "magic", true)) break;
    if (memcmp(d, "ROAR", 4) != 0) { snprintf(msg, sizeof msg, "bad magic"); fail(0, true); break; }
    if (!need(4, "container count", true)) break;
    uint32_t count = g32(d + start);
    const uint64_t desc0 = off;
    int64_t prev_key = -1;
    bool ok = true;
    for (uint32_t k = 0; k < count; k++) {
      if (!need(8, "descriptor", true)) { ok = false; break; }
      uint16_t kk = g16(d + start);
      uint8_t tag = d[start + 2], pad = d[start + 3];
      if (pad != 0) { snprintf(msg, sizeof msg, "nonzero descriptor pad"); fail(start + 3, true); ok = false; break; }
      if (tag < 1 || tag > 3) { snprintf(msg, sizeof msg, "unknown container type %u", tag); fail(start + 2, true); ok = false; break; }
      if ((int64_t)kk <= prev_key) { snprintf(msg, sizeof msg, "keys not strictly increasing at %u", kk); fail(start, true); ok = false; break; }
      prev_key = kk;
    }
    if (!ok) break;
    for (uint32_t k = 0; k < count; k++) {
      const uint8_t *dd = d + desc0 + 8ull * k;
      uint16_t kk = g16(dd);
      uint8_t tag = dd[2];
      uint32_t cc = g32(dd + 4), nn;
      if (tag == RS_TAG_ARRAY) {
        if (!(cc >= 1 && cc <= RS_ARRAY_MAX)) {
          snprintf(msg, sizeof msg, "array cardinality %u out of range", cc);
          fail((int64_t)off, false); ok = false; break;
        }
        if (!need(2ull * cc, "array payload", false)) { ok = false; break; }
        nn = cc;
      } else if (tag == RS_TAG_BITSET) {
        if (!need(8192, "bitset payload", false)) { ok = false; break; }
        nn = RS_WORDS;
      } else {
        if (!need(2, "run count", false)) { ok = false; break; }
        nn = g16(d + start);
        if (nn == 0) { snprintf(msg, sizeof msg, "empty run container"); fail((int64_t)start, false); ok = false; break; }
        if (!need(4ull * nn, "run payload", false)) { ok = false; break; }
        if (nn > W.max_runs) W.max_runs = nn;
      }
      W.key.push_back(kk); W.type.push_back(tag); W.card.push_back(cc); W.cnt.push_back(nn);
      W.src.push_back(offs[i] + start);
      W.poff.push_back(W.pool);
      W.pool += rs_pad16(rs_payload_bytes(tag, nn));
    }
    if (!ok) break;
    if (off != len) {
      snprintf(msg, sizeof msg, "%llu trailing bytes", (unsigned long long)(len - off));
      fail((int64_t)off, false);
      break;
    }
  }
  uint64_t nc = W.key.size();
  W.nb_built = err.set ? err.image + 1 : n;
  for (uint64_t i = W.nb_built; i <= n; i++) W.bm_start[i] = nc;
  if (err.set) W.bm_start[err.image + 1] = nc;
}

// The reference raises the first error in image order; within an image the
// payload checks of earlier containers precede a later structural error.
// vcode/vval: device check results (null when none failed); src is relative
// to offs[0].  Sets the thread-local error; returns RS_EDECODE.
int format_wire_error(const WireErr &err, uint64_t nc, const uint8_t *vcode, const uint32_t *vval,
                      const std::vector<uint64_t> &bm_start, uint64_t nb_built, const std::vector<uint32_t> &card,
                      const std::vector<uint64_t> &src, const uint64_t *offs, std::string *out_msg,
                      int64_t *out_off, int64_t *out_idx) {
  char msg[256];
  for (uint64_t c = 0; vcode && c < nc; c++) {
    if (!vcode[c]) continue;
    uint64_t img = std::upper_bound(bm_start.begin(), bm_start.begin() + nb_built + 1, c) - bm_start.begin() - 1;
    if (err.set && img > err.image) break;
    uint64_t at = src[c] - (offs[img] - offs[0]);  // payload start inside the image
    switch (vcode[c]) {
      case V_ARRAY_ORDER: snprintf(msg, sizeof msg, "array values not strictly increasing"); break;
      case V_BITSET_CARD: snprintf(msg, sizeof msg, "cardinality mismatch: descriptor says %u, payload holds %u", card[c], vval[c]); break;
      case V_BITSET_SMALL: snprintf(msg, sizeof msg, "bitset container with only %u values", card[c]); break;
      case V_RUN_ESCAPE: snprintf(msg, sizeof msg, "run escapes the 16-bit chunk"); break;
      case V_RUN_OVERLAP: snprintf(msg, sizeof msg, "runs overlap or are adjacent"); break;
      case V_RUN_CARD: snprintf(msg, sizeof msg, "cardinality mismatch: descriptor says %u, runs hold %u", card[c], vval[c]); break;
      default: snprintf(msg, sizeof msg, "run form is not the smallest representation"); break;
    }
    *out_msg = "at byte " + std::to_string(at) + ": " + msg;
    *out_off = (int64_t)at;
    *out_idx = (int64_t)img;
    set_error(*out_msg, *out_off, *out_idx);
    return RS_EDECODE;
  }
  *out_msg = "at byte " + std::to_string(err.offset) + ": " + err.msg;
  *out_off = err.offset;
  *out_idx = (int64_t)err.image;
  set_error(*out_msg, *out_off, *out_idx);
  return RS_EDECODE;
}

uint8_t type_mask_of(const std::vector<uint8_t> &type) {
  uint8_t tm = 0;
  for (uint8_t t : type) tm |= (uint8_t)(1u << t);
  return tm;
}

}  // namespace

extern "C" int rs_batch_from_wire(const uint8_t *buf, const uint64_t *offs, uint64_t n,
                                  rs_batch **out) {
  RS_TRY(ensure_device());
  *out = nullptr;
  WireWalk W;
  walk_wire(buf, offs, n, W);
  const uint64_t nc = W.key.size();

  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, n, nc, W.pool);
  if (rc) { rs_batch_free(b); return rc; }
  uint64_t stage_bytes = offs[n] - offs[0];
  uint8_t *staged = (uint8_t *)dalloc(stage_bytes ? stage_bytes : 16);
  uint64_t *d_src = (uint64_t *)dalloc((nc ? nc : 1) * 8);
  uint8_t *d_vcode = (uint8_t *)dalloc(nc ? nc : 1);
  uint32_t *d_vval = (uint32_t *)dalloc((nc ? nc : 1) * 4);
  int *d_any = (int *)dalloc(sizeof(int));
  if (!staged || !d_src || !d_vcode || !d_vval || !d_any) {
    rs_batch_free(b);
    dfree(staged); dfree(d_src); dfree(d_vcode); dfree(d_vval); dfree(d_any);
    set_error("device allocation failed (wire ingest)");
    return RS_ENOMEM;
  }
  for (uint64_t c = 0; c < nc; c++) W.src[c] -= offs[0];
  RS_TRY(h2d(staged, buf + offs[0], stage_bytes));
  RS_TRY(h2d(b->d_bm_start, W.bm_start.data(), (n + 1) * 8));
  RS_TRY(h2d(b->d_key, W.key.data(), nc * 2));
  RS_TRY(h2d(b->d_type, W.type.data(), nc));
  RS_TRY(h2d(b->d_card, W.card.data(), nc * 4));
  RS_TRY(h2d(b->d_n, W.cnt.data(), nc * 4));
  RS_TRY(h2d(b->d_off, W.poff.data(), nc * 8));
  RS_TRY(h2d(d_src, W.src.data(), nc * 8));
  RS_CK(cudaMemsetAsync(d_any, 0, sizeof(int), g_stream));
  RS_LAUNCH(k_wire_gather_validate, (unsigned)((nc * 32 + 255) / 256), 256, 0, nc, nc, staged, d_src,
            b->dev(), b->d_pool, d_vcode, d_vval, d_any, (uint32_t *)nullptr);
  int any = 0;
  RS_TRY(d2h(&any, d_any, sizeof(int)));
  // The host walk must finish before the (pageable) host vectors go away:
  // d2h above synchronized the stream.
  int result = RS_OK;
  if (any || W.err.set) {
    std::vector<uint8_t> vcode(nc);
    std::vector<uint32_t> vval(nc);
    if (any) {
      RS_TRY(d2h(vcode.data(), d_vcode, nc));
      RS_TRY(d2h(vval.data(), d_vval, nc * 4));
    }
    std::string m;
    int64_t o, ix;
    result = format_wire_error(W.err, nc, any ? vcode.data() : nullptr, vval.data(), W.bm_start, W.nb_built,
                               W.card, W.src, offs, &m, &o, &ix);
  }
  dfree(staged); dfree(d_src); dfree(d_vcode); dfree(d_vval); dfree(d_any);
  if (result != RS_OK) { rs_batch_free(b); return result; }
  b->h_bm_start = std::move(W.bm_start);
  b->type_mask = type_mask_of(W.type);
  b->h_valid = true;
  RS_TRY(finalize_batch(b));
  *out = b;
  return RS_OK;
}

// ------------------------------------------------ asynchronous wire ingest
// The payload bytes go HBM-ward on a dedicated copy stream through a ring of
// device staging slots, so the transfer of batch k+1 overlaps the kernels of
// batch k on the library stream; payload checks are read back at
// rs_batch_wait (or implicitly by any call that returns data to the host).
namespace {

struct PinnedBlock { uint8_t *p; size_t bytes; cudaEvent_t done; };
struct StageSlot { uint8_t *d; size_t bytes; cudaEvent_t copied, consumed; bool in_use; };
std::mutex g_async_mu;
std::deque<PinnedBlock> g_pinned;  // deque: element addresses stay valid as it grows
std::deque<StageSlot> g_slots;
cudaStream_t g_copy = nullptr;
int g_copy_dev = -1;

int copy_stream(cudaStream_t *s) {
  int dev = 0;
  RS_CK(cudaGetDevice(&dev));
  if (!g_copy || g_copy_dev != dev) {
    RS_CK(cudaStreamCreateWithFlags(&g_copy, cudaStreamNonBlocking));
    g_copy_dev = dev;
  }
  *s = g_copy;
  return RS_OK;
}

int get_pinned(size_t bytes, PinnedBlock **out) {
  for (auto &b : g_pinned)
    if (b.bytes >= bytes && cudaEventQuery(b.done) == cudaSuccess) { *out = &b; return RS_OK; }
  PinnedBlock b;
  b.bytes = std::max<size_t>(bytes, 1 << 20);
  RS_CK(cudaHostAlloc((void **)&b.p, b.bytes, cudaHostAllocDefault));
  RS_CK(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
  g_pinned.push_back(b);
  *out = &g_pinned.back();
  return RS_OK;
}

int get_slot(size_t bytes, StageSlot **out) {
  for (auto &s : g_slots)
    if (!s.in_use && s.bytes >= bytes && cudaEventQuery(s.consumed) == cudaSuccess) {
      s.in_use = true;
      *out = &s;
      return RS_OK;
    }
  StageSlot s;
  s.bytes = bytes;
  s.in_use = true;
  if (cudaMalloc((void **)&s.d, bytes) != cudaSuccess) {
    cudaGetLastError();
    // out of memory: wait for the slots in flight and retry once in them
    for (auto &t : g_slots) {
      if (t.in_use || t.bytes < bytes) continue;
      RS_CK(cudaEventSynchronize(t.consumed));
      t.in_use = true;
      *out = &t;
      return RS_OK;
    }
    set_error("device allocation failed (wire staging)");
    return RS_ENOMEM;
  }
  RS_CK(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming));
  RS_CK(cudaEventCreateWithFlags(&s.consumed, cudaEventDisableTiming));
  g_slots.push_back(s);
  *out = &g_slots.back();
  return RS_OK;
}

// staged metadata section -> the batch's container table
__global__ void k_unpack_meta(uint64_t nb, uint64_t nc, const uint8_t *__restrict__ meta, uint64_t *bm_start,
                              uint64_t *off, uint64_t *src, uint32_t *card, uint32_t *n, uint16_t *key,
                              uint8_t *type) {
  const uint64_t *m_bm = (const uint64_t *)meta;
  const uint64_t *m_off = m_bm + rs_pad16((nb + 1) * 8) / 8;
  const uint64_t *m_src = m_off + nc;
  const uint32_t *m_card = (const uint32_t *)(m_src + nc);
  const uint32_t *m_n = m_card + nc;
  const uint16_t *m_key = (const uint16_t *)(m_n + nc);
  const uint8_t *m_type = (const uint8_t *)(m_key + rs_pad16(nc * 2) / 2);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nc || i <= nb;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i <= nb) bm_start[i] = m_bm[i];
    if (i < nc) {
      off[i] = m_off[i]; src[i] = m_src[i]; card[i] = m_card[i]; n[i] = m_n[i];
      key[i] = m_key[i]; type[i] = m_type[i];
    }
  }
}

}  // namespace

namespace rs {
// First use of an asynchronously ingested batch: queue its unpack + payload
// gather/check on the library stream behind the copy.  Deferring this to the
// consumer keeps kernels queued meanwhile (earlier batches' ops, exports)
// from waiting on the transfer.
int materialize(const rs_batch *cb) {
  rs_batch *b = const_cast<rs_batch *>(cb);
  rs_pending *P = b->pending;
  if (!P || !P->slot) return RS_OK;
  std::lock_guard<std::mutex> g(g_async_mu);
  StageSlot *slot = (StageSlot *)P->slot;
  const uint64_t nc = b->nc, n = b->nb;
  uint64_t *d_src = (uint64_t *)dalloc((nc ? nc : 1) * 8);
  if (!d_src) { set_error("device allocation failed (async wire ingest)"); return RS_ENOMEM; }
  RS_CK(cudaStreamWaitEvent(g_stream, slot->copied, 0));
  const uint64_t items = std::max<uint64_t>(nc, n + 1);
  RS_LAUNCH(k_unpack_meta, (unsigned)std::min<uint64_t>((items + 255) / 256, 148 * 16), 256, 0, n, nc, slot->d,
            b->d_bm_start, b->d_off, d_src, b->d_card, b->d_n, b->d_key, b->d_type);
  RS_CK(cudaMemsetAsync(P->d_any, 0, sizeof(int), g_stream));
  if (nc)
    RS_LAUNCH(k_wire_gather_validate, (unsigned)((nc * 32 + 255) / 256), 256, 0, nc, nc, slot->d + P->meta_bytes,
              d_src, b->dev(), b->d_pool, P->d_vcode, P->d_vval, P->d_any, b->d_card);
  RS_CK(cudaEventRecord(slot->consumed, g_stream));
  slot->in_use = false;
  P->slot = nullptr;
  dfree(d_src);
  return finalize_batch(b);
}

// A batch freed before first use hands its staging slot back once the copy
// into it has landed.
void drop_staged(rs_batch *b) {
  rs_pending *P = b->pending;
  if (!P || !P->slot) return;
  std::lock_guard<std::mutex> g(g_async_mu);
  StageSlot *slot = (StageSlot *)P->slot;
  cudaStreamWaitEvent(g_stream, slot->copied, 0);
  cudaEventRecord(slot->consumed, g_stream);
  slot->in_use = false;
  P->slot = nullptr;
}

int resolve_pending(const rs_batch *cb) {
  rs_batch *b = const_cast<rs_batch *>(cb);
  rs_pending *P = b->pending;
  if (!P) return RS_OK;
  RS_TRY(materialize(b));
  if (P->failed) { set_error(P->msg, P->offset, P->index); return RS_EDECODE; }
  int any = 0;
  RS_TRY(d2h(&any, P->d_any, sizeof(int)));
  if (!any) {
    dfree(P->d_any); dfree(P->d_vcode); dfree(P->d_vval);
    delete P;
    b->pending = nullptr;
    return RS_OK;
  }
  const uint64_t nc = b->nc;
  std::vector<uint8_t> vcode(nc);
  std::vector<uint32_t> vval(nc);
  RS_TRY(d2h(vcode.data(), P->d_vcode, nc));
  RS_TRY(d2h(vval.data(), P->d_vval, nc * 4));
  WireErr none;
  P->failed = true;
  return format_wire_error(none, nc, vcode.data(), vval.data(), b->h_bm_start, b->nb, P->card, P->src,
                           P->offs.data(), &P->msg, &P->offset, &P->index);
}
}  // namespace rs

extern "C" int rs_batch_from_wire_async(const uint8_t *buf, const uint64_t *offs, uint64_t n,
                                        rs_batch **out) {
  RS_TRY(ensure_device());
  *out = nullptr;
  WireWalk W;
  walk_wire(buf, offs, n, W);
  // A structural error, or a run container that can never be admissible
  // (more runs than any valid chunk holds), goes through the synchronous path,
  // which reports the reference's exact first error.
  if (W.err.set || W.max_runs > RS_RUN_MAX_RUNS) return rs_batch_from_wire(buf, offs, n, out);
  const uint64_t nc = W.key.size();
  for (uint64_t c = 0; c < nc; c++) W.src[c] -= offs[0];
  // metadata image: bm_start | off | src | card | n | key | type (16-B sections)
  const size_t s_bm = rs_pad16((n + 1) * 8), s_off = nc * 8, s_card = nc * 4, s_key = rs_pad16(nc * 2);
  const size_t meta = rs_pad16(s_bm + 2 * s_off + 2 * s_card + s_key + nc);
  const uint64_t wire_bytes = offs[n] - offs[0];
  PinnedBlock *pb;
  StageSlot *slot;
  std::unique_lock<std::mutex> lk(g_async_mu);
  cudaStream_t cs;
  RS_TRY(copy_stream(&cs));
  RS_TRY(get_pinned(meta, &pb));
  RS_TRY(get_slot(meta + rs_pad16(wire_bytes ? wire_bytes : 16), &slot));
  {
    uint8_t *h = pb->p;
    memcpy(h, W.bm_start.data(), (n + 1) * 8); h += s_bm;
    memcpy(h, W.poff.data(), s_off); h += s_off;
    memcpy(h, W.src.data(), s_off); h += s_off;
    memcpy(h, W.card.data(), s_card); h += s_card;
    memcpy(h, W.cnt.data(), s_card); h += s_card;
    memcpy(h, W.key.data(), nc * 2); h += s_key;
    memcpy(h, W.type.data(), nc);
  }
  RS_CK(cudaStreamWaitEvent(cs, slot->consumed, 0));
  RS_CK(cudaMemcpyAsync(slot->d, pb->p, meta, cudaMemcpyHostToDevice, cs));
  if (wire_bytes) RS_CK(cudaMemcpyAsync(slot->d + meta, buf + offs[0], wire_bytes, cudaMemcpyHostToDevice, cs));
  RS_CK(cudaEventRecord(pb->done, cs));
  RS_CK(cudaEventRecord(slot->copied, cs));
  lk.unlock();

  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, n, nc, W.pool);
  rs_pending *P = new rs_pending();
  b->pending = P;
  P->slot = slot;
  P->meta_bytes = meta;
  P->d_any = (int *)dalloc(sizeof(int));
  P->d_vcode = (uint8_t *)dalloc(nc ? nc : 1);
  P->d_vval = (uint32_t *)dalloc((nc ? nc : 1) * 4);
  if (rc || !P->d_any || !P->d_vcode || !P->d_vval) {
    rs_batch_free(b);  // hands the slot back behind the queued copy
    set_error("device allocation failed (async wire ingest)");
    return RS_ENOMEM;
  }
  P->card = std::move(W.card);
  P->src = std::move(W.src);
  P->offs.assign(offs, offs + n + 1);
  b->h_bm_start = std::move(W.bm_start);
  b->type_mask = type_mask_of(W.type);
  b->h_valid = true;
  *out = b;
  return RS_OK;
}

extern "C" int rs_batch_wait(const rs_batch *b) {
  if (!b) { set_error("null batch"); return RS_EARG; }
  return resolve_pending(b);
}

// --------------------------------------------------------- from_values ingest

namespace {

__global__ void k_mark_seg(uint64_t n, const uint64_t *__restrict__ offs, uint8_t *__restrict__ segstart) {
  uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b < n && offs[b] < offs[b + 1]) segstart[offs[b]] = 1;
}

__global__ void k_check_sorted(uint64_t V, const uint32_t *__restrict__ v, const uint8_t *__restrict__ segstart,
                               int *__restrict__ unsorted) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < V && i > 0 && !segstart[i] && v[i] <= v[i - 1]) atomicOr(unsorted, 1);
}

// warp per bitmap writes key = seg << 32 | value
__global__ void k_make_keys(uint64_t n, const uint64_t *__restrict__ offs, const uint32_t *__restrict__ v,
                            uint64_t *__restrict__ keys) {
  uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= n) return;
  for (uint64_t i = offs[w] + lane; i < offs[w + 1]; i += 32) keys[i] = (w << 32) | v[i];
}

__global__ void k_unique_flags(uint64_t V, const uint64_t *__restrict__ keys, uint64_t *__restrict__ flag) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < V) flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_unique_scatter(uint64_t V, const uint64_t *__restrict__ keys, const uint64_t *__restrict__ flag,
                                 const uint64_t *__restrict__ pos, uint32_t *__restrict__ v_out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < V && flag[i]) v_out[pos[i]] = (uint32_t)keys[i];
}

// new segment offsets: offs[b] = #unique keys with segment < b
__global__ void k_seg_offsets(uint64_t n, uint64_t V, const uint64_t *__restrict__ keys, const uint64_t *__restrict__ flag,
                              const uint64_t *__restrict__ pos, uint64_t U, uint64_t *__restrict__ offs) {
  uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b > n) return;
  // lower_bound over sorted keys for b << 32
  uint64_t lo = 0, hi = V, target = b << 32;
  while (lo < hi) {
    uint64_t m = (lo + hi) >> 1;
    if (keys[m] < target) lo = m + 1; else hi = m;
  }
  offs[b] = lo < V ? pos[lo] : U;
}

// chunk starts: value i starts a container if it starts its bitmap or its
// high 16 bits differ from the previous value's
__global__ void k_chunk_flags(uint64_t V, const uint32_t *__restrict__ v, const uint8_t *__restrict__ segstart,
                              uint64_t *__restrict__ flag) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < V) flag[i] = (i == 0 || segstart[i] || (v[i] >> 16) != (v[i - 1] >> 16)) ? 1 : 0;
}

__global__ void k_chunk_starts(uint64_t V, const uint64_t *__restrict__ flag, const uint64_t *__restrict__ cpos,
                               const uint32_t *__restrict__ v, uint64_t *__restrict__ cstart,
                               uint16_t *__restrict__ key) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < V && flag[i]) {
    cstart[cpos[i]] = i;
    key[cpos[i]] = (uint16_t)(v[i] >> 16);
  }
}

__global__ void k_chunk_meta(uint64_t C, uint64_t V, uint64_t *__restrict__ cstart, uint8_t *__restrict__ type,
                             uint32_t *__restrict__ card, uint32_t *__restrict__ nn, uint64_t *__restrict__ psize) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= C) return;
  uint64_t e = c + 1 < C ? cstart[c + 1] : V;
  uint32_t k = (uint32_t)(e - cstart[c]);
  card[c] = k;
  // bitmap.py:55-59: array if <= ARRAY_MAX values, else bitset_from_positions
  if (k <= RS_ARRAY_MAX) { type[c] = RS_TAG_ARRAY; nn[c] = k; psize[c] = rs_pad16(2ull * k); }
  else { type[c] = RS_TAG_BITSET; nn[c] = RS_WORDS; psize[c] = 8192; }
}

__global__ void k_bm_start_from_values(uint64_t n, uint64_t V, uint64_t C, const uint64_t *__restrict__ offs,
                                       const uint64_t *__restrict__ cpos, uint64_t *__restrict__ bm_start) {
  uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b <= n) bm_start[b] = offs[b] < V ? cpos[offs[b]] : C;
}

// one CTA per container: arrays copy low halves; bitsets build in smem
__global__ void __launch_bounds__(256) k_fill_from_values(uint64_t C, uint64_t V, const uint32_t *__restrict__ v,
                                                          const uint64_t *__restrict__ cstart, DevBatch B,
                                                          uint8_t *__restrict__ pool) {
  __shared__ uint32_t bits[2048];
  uint64_t c = blockIdx.x;
  if (c >= C) return;
  uint64_t s = cstart[c];
  uint32_t k = B.card[c];
  uint8_t *dst = pool + B.off[c];
  if (B.type[c] == RS_TAG_ARRAY) {
    uint16_t *d16 = (uint16_t *)dst;
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) d16[i] = (uint16_t)(v[s + i] & 0xFFFF);
    uint32_t padded = (uint32_t)rs_pad16(2ull * k) >> 1;
    for (uint32_t i = k + threadIdx.x; i < padded; i += blockDim.x) d16[i] = 0;
    return;
  }
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) bits[i] = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    uint32_t lo = v[s + i] & 0xFFFF;
    atomicOr(&bits[lo >> 5], 1u << (lo & 31));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) ((uint4 *)dst)[i] = ((const uint4 *)bits)[i];
}

}  // namespace

extern "C" int rs_batch_from_u32(const uint32_t *vals, const uint64_t *offs, uint64_t n, int on_device,
                                 rs_batch **out) {
  RS_TRY(ensure_device());
  *out = nullptr;
  uint64_t V;
  std::vector<uint64_t> h_offs(n + 1);
  if (on_device) RS_TRY(d2h(h_offs.data(), offs, (n + 1) * 8));
  else memcpy(h_offs.data(), offs, (n + 1) * 8);
  uint64_t base = h_offs[0];
  for (auto &o : h_offs) o -= base;
  V = h_offs[n];
  uint64_t *d_offs = (uint64_t *)dalloc((n + 1) * 8);
  uint32_t *d_v = (uint32_t *)dalloc((V ? V : 1) * 4);
  uint8_t *segstart = (uint8_t *)dalloc(V ? V : 1);
  int *d_flag = (int *)dalloc(sizeof(int));
  if (!d_offs || !d_v || !segstart || !d_flag) { set_error("device allocation failed (from_values)"); return RS_ENOMEM; }
  RS_TRY(h2d(d_offs, h_offs.data(), (n + 1) * 8));
  if (V) {
    if (on_device) RS_CK(cudaMemcpyAsync(d_v, vals + base, V * 4, cudaMemcpyDeviceToDevice, g_stream));
    else RS_TRY(h2d(d_v, vals + base, V * 4));
  }
  RS_CK(cudaMemsetAsync(segstart, 0, V ? V : 1, g_stream));
  RS_CK(cudaMemsetAsync(d_flag, 0, sizeof(int), g_stream));
  unsigned gb = (unsigned)((n + 255) / 256), gv = (unsigned)((V + 255) / 256);
  RS_LAUNCH(k_mark_seg, gb, 256, 0, n, d_offs, segstart);
  RS_LAUNCH(k_check_sorted, gv, 256, 0, V, d_v, segstart, d_flag);
  int unsorted = 0;
  RS_TRY(d2h(&unsorted, d_flag, sizeof(int)));
  if (unsorted) {
    // np.unique per bitmap: radix sort of (bitmap << 32 | value), then dedup
    uint64_t *keys = (uint64_t *)dalloc(V * 8), *flag = (uint64_t *)dalloc((V + 1) * 8),
             *pos = (uint64_t *)dalloc((V + 1) * 8);
    if (!keys || !flag || !pos) { set_error("device allocation failed (from_values sort)"); return RS_ENOMEM; }
    RS_LAUNCH(k_make_keys, (unsigned)((n * 32 + 255) / 256), 256, 0, n, d_offs, d_v, keys);
    int segbits = 1;
    while ((1ull << segbits) <= n) segbits++;
    RS_TRY(sort_u64(keys, V, 32 + segbits));
    RS_LAUNCH(k_unique_flags, gv, 256, 0, V, keys, flag);
    RS_TRY(scan_exclusive<uint64_t>(flag, pos, V));
    uint64_t last[2];
    RS_TRY(d2h(&last[0], pos + V - 1, 8));
    RS_TRY(d2h(&last[1], flag + V - 1, 8));
    uint64_t U = last[0] + last[1];
    RS_LAUNCH(k_unique_scatter, gv, 256, 0, V, keys, flag, pos, d_v);
    RS_LAUNCH(k_seg_offsets, (unsigned)((n + 1 + 255) / 256), 256, 0, n, V, keys, flag, pos, U, d_offs);
    RS_TRY(d2h(h_offs.data(), d_offs, (n + 1) * 8));
    V = U;
    dfree(keys); dfree(flag); dfree(pos);
    RS_CK(cudaMemsetAsync(segstart, 0, V ? V : 1, g_stream));
    RS_LAUNCH(k_mark_seg, gb, 256, 0, n, d_offs, segstart);
    gv = (unsigned)((V + 255) / 256);
  }
  // containers
  uint64_t *cflag = (uint64_t *)dalloc((V + 1) * 8), *cpos = (uint64_t *)dalloc((V + 1) * 8);
  if (!cflag || !cpos) { set_error("device allocation failed (from_values)"); return RS_ENOMEM; }
  RS_LAUNCH(k_chunk_flags, gv, 256, 0, V, d_v, segstart, cflag);
  RS_TRY(scan_exclusive<uint64_t>(cflag, cpos, V));
  uint64_t C = 0;
  if (V) {
    uint64_t t[2];
    RS_TRY(d2h(&t[0], cpos + V - 1, 8));
    RS_TRY(d2h(&t[1], cflag + V - 1, 8));
    C = t[0] + t[1];
  }
  rs_batch *b = new rs_batch();
  // pool size needs the container types: allocate metadata first
  uint64_t *cstart = (uint64_t *)dalloc((C ? C : 1) * 8), *psize = (uint64_t *)dalloc((C + 1) * 8);
  b->nb = n; b->nc = C; b->cap_c = C;
  b->d_bm_start = (uint64_t *)dalloc((n + 1) * 8);
  b->d_bm_card = (uint64_t *)dalloc((n + 1) * 8);
  b->d_key = (uint16_t *)dalloc((C ? C : 1) * 2);
  b->d_type = (uint8_t *)dalloc(C ? C : 1);
  b->d_card = (uint32_t *)dalloc((C ? C : 1) * 4);
  b->d_n = (uint32_t *)dalloc((C ? C : 1) * 4);
  b->d_off = (uint64_t *)dalloc((C + 1) * 8);
  if (!cstart || !psize || !b->d_bm_start || !b->d_bm_card || !b->d_key || !b->d_type || !b->d_card ||
      !b->d_n || !b->d_off) {
    rs_batch_free(b);
    set_error("device allocation failed (from_values)");
    return RS_ENOMEM;
  }
  RS_LAUNCH(k_chunk_starts, gv, 256, 0, V, cflag, cpos, d_v, cstart, b->d_key);
  RS_LAUNCH(k_chunk_meta, (unsigned)((C + 255) / 256), 256, 0, C, V, cstart, b->d_type, b->d_card, b->d_n, psize);
  RS_LAUNCH(k_bm_start_from_values, (unsigned)((n + 1 + 255) / 256), 256, 0, n, V, C, d_offs, cpos, b->d_bm_start);
  RS_TRY(scan_exclusive<uint64_t>(psize, b->d_off, C + 1));
  uint64_t P = 0;
  RS_TRY(d2h(&P, b->d_off + C, 8));
  b->pool_bytes = P;
  b->d_pool = (uint8_t *)dalloc(P ? P : 16);
  if (!b->d_pool) { rs_batch_free(b); set_error("device allocation failed (from_values pool)"); return RS_ENOMEM; }
  RS_LAUNCH(k_fill_from_values, (unsigned)C, 256, 0, C, V, d_v, cstart, b->dev(), b->d_pool);
  dfree(cflag); dfree(cpos); dfree(cstart); dfree(psize); dfree(d_offs); dfree(d_v); dfree(segstart); dfree(d_flag);
  RS_TRY(finalize_batch(b));
  b->h_valid = false;
  b->type_mask = (1u << RS_TAG_ARRAY) | (1u << RS_TAG_BITSET);  // from_values never builds runs
  RS_TRY(fetch_host_meta(b));
  *out = b;
  return RS_OK;
}

// ------------------------------------------------------------ concat / select

namespace {
__global__ void k_shift_u64(uint64_t n, const uint64_t *__restrict__ in, uint64_t add, uint64_t *__restrict__ out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] + add;
}

// new container j of the selection: copy metadata + payload (warp per container)
__global__ void k_select_copy(uint64_t nc_new, uint64_t nb_new, const uint64_t *__restrict__ new_start,
                              const uint64_t *__restrict__ src_start, DevBatch S, const uint64_t *__restrict__ new_off,
                              uint16_t *key, uint8_t *type, uint32_t *card, uint32_t *nn, uint64_t *off,
                              uint8_t *__restrict__ pool) {
  uint64_t j = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (j >= nc_new) return;
  uint64_t lo = 0, hi = nb_new;  // bitmap k with new_start[k] <= j < new_start[k+1]
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (new_start[m] <= j) lo = m; else hi = m;
  }
  uint64_t s = src_start[lo] + (j - new_start[lo]);
  uint32_t bytes = (uint32_t)rs_pad16(rs_payload_bytes(S.type[s], S.n[s]));
  const uint4 *src = (const uint4 *)(S.pool + S.off[s]);
  uint4 *dst = (uint4 *)(pool + new_off[j]);
  for (uint32_t i = lane; i < (bytes >> 4); i += 32) dst[i] = src[i];
  if (lane == 0) {
    key[j] = S.key[s]; type[j] = S.type[s]; card[j] = S.card[s]; nn[j] = S.n[s]; off[j] = new_off[j];
  }
}

__global__ void k_select_sizes(uint64_t nc_new, uint64_t nb_new, const uint64_t *__restrict__ new_start,
                               const uint64_t *__restrict__ src_start, DevBatch S, uint64_t *__restrict__ psize) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j > nc_new) return;
  if (j == nc_new) { psize[j] = 0; return; }
  uint64_t lo = 0, hi = nb_new;
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (new_start[m] <= j) lo = m; else hi = m;
  }
  uint64_t s = src_start[lo] + (j - new_start[lo]);
  psize[j] = rs_pad16(rs_payload_bytes(S.type[s], S.n[s]));
}
}  // namespace

extern "C" int rs_batch_concat(const rs_batch *const *parts, uint64_t nparts, rs_batch **out) {
  RS_TRY(ensure_device());
  uint64_t nb = 0, nc = 0, pool = 0;
  for (uint64_t k = 0; k < nparts; k++) {
    RS_TRY(fetch_host_meta(parts[k]));
    nb += parts[k]->nb; nc += parts[k]->nc; pool += parts[k]->pool_bytes;
  }
  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, nb, nc, pool);
  if (rc) { rs_batch_free(b); return rc; }
  b->h_bm_start.assign(1, 0);
  b->type_mask = 0;
  for (uint64_t k = 0; k < nparts; k++) b->type_mask |= parts[k]->type_mask;
  uint64_t cb = 0, bb = 0, pb = 0;
  for (uint64_t k = 0; k < nparts; k++) {
    const rs_batch *p = parts[k];
    RS_LAUNCH(k_shift_u64, (unsigned)((p->nb + 1 + 255) / 256), 256, 0, p->nb + 1, p->d_bm_start, cb, b->d_bm_start + bb);
    RS_LAUNCH(k_shift_u64, (unsigned)((p->nc + 255) / 256), 256, 0, p->nc, p->d_off, pb, b->d_off + cb);
    if (p->nc) {
      RS_CK(cudaMemcpyAsync(b->d_key + cb, p->d_key, p->nc * 2, cudaMemcpyDeviceToDevice, g_stream));
      RS_CK(cudaMemcpyAsync(b->d_type + cb, p->d_type, p->nc, cudaMemcpyDeviceToDevice, g_stream));
      RS_CK(cudaMemcpyAsync(b->d_card + cb, p->d_card, p->nc * 4, cudaMemcpyDeviceToDevice, g_stream));
      RS_CK(cudaMemcpyAsync(b->d_n + cb, p->d_n, p->nc * 4, cudaMemcpyDeviceToDevice, g_stream));
    }
    if (p->pool_bytes) RS_CK(cudaMemcpyAsync(b->d_pool + pb, p->d_pool, p->pool_bytes, cudaMemcpyDeviceToDevice, g_stream));
    if (p->nb) RS_CK(cudaMemcpyAsync(b->d_bm_card + bb, p->d_bm_card, p->nb * 8, cudaMemcpyDeviceToDevice, g_stream));
    for (uint64_t i = 1; i <= p->nb; i++) b->h_bm_start.push_back(p->h_bm_start[i] + cb);
    cb += p->nc; bb += p->nb; pb += p->pool_bytes;
  }
  b->h_valid = true;
  bool ub = false;
  for (uint64_t k = 0; k < nparts; k++) ub |= parts[k]->ub_pool;
  if (ub) ub_register(b);  // the parts' holes were copied along
  *out = b;
  return RS_OK;
}

extern "C" int rs_batch_select(const rs_batch *S, const uint64_t *idx, uint64_t n, rs_batch **out) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(S));
  std::vector<uint64_t> new_start(n + 1, 0), src_start(n + 1, 0);
  for (uint64_t k = 0; k < n; k++) {
    if (idx[k] >= S->nb) { set_error("bitmap index out of range"); return RS_EARG; }
    src_start[k] = S->h_bm_start[idx[k]];
    new_start[k + 1] = new_start[k] + (S->h_bm_start[idx[k] + 1] - S->h_bm_start[idx[k]]);
  }
  uint64_t nc = new_start[n];
  uint64_t *d_ns = (uint64_t *)dalloc((n + 1) * 8), *d_ss = (uint64_t *)dalloc((n + 1) * 8);
  uint64_t *psize = (uint64_t *)dalloc((nc + 1) * 8), *poff = (uint64_t *)dalloc((nc + 1) * 8);
  if (!d_ns || !d_ss || !psize || !poff) { set_error("device allocation failed (select)"); return RS_ENOMEM; }
  RS_TRY(h2d(d_ns, new_start.data(), (n + 1) * 8));
  RS_TRY(h2d(d_ss, src_start.data(), (n + 1) * 8));
  RS_LAUNCH(k_select_sizes, (unsigned)((nc + 1 + 255) / 256), 256, 0, nc, n, d_ns, d_ss, S->dev(), psize);
  RS_TRY(scan_exclusive<uint64_t>(psize, poff, nc + 1));
  uint64_t P = 0;
  RS_TRY(d2h(&P, poff + nc, 8));
  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, n, nc, P);
  if (rc) { rs_batch_free(b); return rc; }
  RS_CK(cudaMemcpyAsync(b->d_bm_start, d_ns, (n + 1) * 8, cudaMemcpyDeviceToDevice, g_stream));
  RS_LAUNCH(k_select_copy, (unsigned)((nc * 32 + 255) / 256), 256, 0, nc, n, d_ns, d_ss, S->dev(), poff, b->d_key,
            b->d_type, b->d_card, b->d_n, b->d_off, b->d_pool);
  dfree(d_ns); dfree(d_ss); dfree(psize); dfree(poff);
  RS_TRY(finalize_batch(b));
  b->h_bm_start = new_start;
  b->type_mask = S->type_mask;
  b->h_valid = true;
  *out = b;
  return RS_OK;
}

// ------------------------------------------------------ key-range sharding
// Multi-GPU: the 2^16 chunk keys are independent, so a single
// bitmap pair, a wide union or the all-pairs counts shard by contiguous key
// ranges -- each rank restricts its batches to [lo, hi) and the results
// concatenate in key order (counts add up).
namespace {
__global__ void k_key_keep(uint64_t nc, const uint16_t *__restrict__ key, uint32_t lo, uint32_t hi,
                           const uint8_t *__restrict__ type, const uint32_t *__restrict__ n,
                           uint64_t *__restrict__ keep, uint64_t *__restrict__ psize) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c > nc) return;
  const bool k = c < nc && key[c] >= lo && key[c] < hi;
  keep[c] = k;
  psize[c] = k ? rs_pad16(rs_payload_bytes(type[c], n[c])) : 0;
}

// warp per kept container: metadata + payload to the new batch
__global__ void k_key_copy(uint64_t nc, DevBatch S, const uint64_t *__restrict__ keep, const uint64_t *__restrict__ pos,
                           const uint64_t *__restrict__ poff, uint16_t *key, uint8_t *type, uint32_t *card,
                           uint32_t *nn, uint64_t *off, uint8_t *__restrict__ pool) {
  const uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nc || !keep[c]) return;
  const uint64_t j = pos[c];
  const uint32_t nv = (uint32_t)(rs_pad16(rs_payload_bytes(S.type[c], S.n[c])) >> 4);
  const uint4 *src = (const uint4 *)(S.pool + S.off[c]);
  uint4 *dst = (uint4 *)(pool + poff[c]);
  for (uint32_t i = lane; i < nv; i += 32) dst[i] = src[i];
  if (lane == 0) {
    key[j] = S.key[c]; type[j] = S.type[c]; card[j] = S.card[c]; nn[j] = S.n[c]; off[j] = poff[c];
  }
}

__global__ void k_key_bm_start(uint64_t nb, const uint64_t *__restrict__ bm_start, const uint64_t *__restrict__ pos,
                               uint64_t *__restrict__ out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i <= nb) out[i] = pos[bm_start[i]];
}

__global__ void k_key_hist(uint64_t nc, const uint16_t *__restrict__ key, unsigned long long *__restrict__ h) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c < nc) atomicAdd(&h[key[c]], 1ull);
}
}  // namespace

extern "C" int rs_batch_key_range(const rs_batch *S, uint32_t lo, uint32_t hi, rs_batch **out) {
  RS_TRY(ensure_device());
  *out = nullptr;
  if (lo > hi || hi > 65536) { set_error("bad key range"); return RS_EARG; }
  RS_TRY(fetch_host_meta(S));
  RS_TRY(resolve_pending(S));
  const uint64_t nc = S->nc, nb = S->nb;
  uint64_t *keep = (uint64_t *)dalloc((nc + 1) * 8), *pos = (uint64_t *)dalloc((nc + 1) * 8);
  uint64_t *psize = (uint64_t *)dalloc((nc + 1) * 8), *poff = (uint64_t *)dalloc((nc + 1) * 8);
  if (!keep || !pos || !psize || !poff) { set_error("device allocation failed (key range)"); return RS_ENOMEM; }
  RS_LAUNCH(k_key_keep, (unsigned)((nc + 1 + 255) / 256), 256, 0, nc, S->d_key, lo, hi, S->d_type, S->d_n, keep, psize);
  RS_TRY(scan_exclusive<uint64_t>(keep, pos, nc + 1));
  RS_TRY(scan_exclusive<uint64_t>(psize, poff, nc + 1));
  uint64_t tot[2];
  RS_TRY(d2h(&tot[0], pos + nc, 8));
  RS_TRY(d2h(&tot[1], poff + nc, 8));
  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, nb, tot[0], tot[1]);
  if (rc) { rs_batch_free(b); return rc; }
  RS_LAUNCH(k_key_copy, (unsigned)((nc * 32 + 255) / 256), 256, 0, nc, S->dev(), keep, pos, poff, b->d_key, b->d_type,
            b->d_card, b->d_n, b->d_off, b->d_pool);
  RS_LAUNCH(k_key_bm_start, (unsigned)((nb + 1 + 255) / 256), 256, 0, nb, S->d_bm_start, pos, b->d_bm_start);
  dfree(keep); dfree(pos); dfree(psize); dfree(poff);
  RS_TRY(finalize_batch(b));
  b->type_mask = S->type_mask;
  b->h_valid = false;
  RS_TRY(fetch_host_meta(b));
  *out = b;
  return RS_OK;
}

extern "C" int rs_batch_key_histogram(const rs_batch *S, uint64_t *hist) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(S));
  unsigned long long *h = (unsigned long long *)dalloc(65536 * 8);
  if (!h) { set_error("device allocation failed (key histogram)"); return RS_ENOMEM; }
  RS_CK(cudaMemsetAsync(h, 0, 65536 * 8, g_stream));
  RS_LAUNCH(k_key_hist, (unsigned)((S->nc + 255) / 256), 256, 0, S->nc, S->d_key, h);
  RS_TRY(d2h(hist, h, 65536 * 8));
  dfree(h);
  return RS_OK;
}

// ------------------------------------------- wire ingest from device memory
// serde.deserialize (serde.py:87-169) of wire images that are already in HBM
// (e.g. produced on the device, or copied there by the caller): the
// descriptor walk runs on the device too -- a thread per image, twice (count,
// then write), mirroring walk_wire's structural checks in the reference's
// order -- followed by the same payload gather / check kernel as the host
// path.  Any error, structural or payload, sends the images to the host path
// once, which raises the reference's exact first DecodeError: the error path
// is rare, and its message must match byte for byte.
namespace {

__device__ __forceinline__ uint16_t dg16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }
__device__ __forceinline__ uint32_t dg32(const uint8_t *p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Walk image i; emit(k, key, tag, card, n, src_abs) for every container that
// the reference would have accepted before its first structural error.
// Returns true if the image is structurally valid.
template <typename Emit>
__device__ bool dev_walk_image(const uint8_t *buf, uint64_t o0, uint64_t len, Emit emit, uint32_t &nvalid,
                               uint64_t &pool) {
  const uint8_t *d = buf + o0;
  uint64_t off = 0, start = 0;
  nvalid = 0;
  pool = 0;
  auto need = [&](uint64_t nb) -> bool {
    if (len - off < nb) return false;
    start = off;
    off += nb;
    return true;
  };
  if (!need(4)) return false;
  if (d[0] != 'R' || d[1] != 'O' || d[2] != 'A' || d[3] != 'R') return false;
  if (!need(4)) return false;
  const uint32_t count = dg32(d + start);
  int32_t prev_key = -1;
  for (uint32_t k = 0; k < count; k++) {  // descriptor stage: every descriptor before any payload
    if (!need(8)) return false;
    const uint16_t kk = dg16(d + start);
    const uint8_t tag = d[start + 2], pad = d[start + 3];
    if (pad != 0 || tag < 1 || tag > 3 || (int32_t)kk <= prev_key) return false;
    prev_key = kk;
  }
  for (uint32_t k = 0; k < count; k++) {
    const uint8_t *dd = d + 8 + 8ull * k;
    const uint16_t kk = dg16(dd);
    const uint8_t tag = dd[2];
    const uint32_t cc = dg32(dd + 4);
    uint32_t nn;
    if (tag == RS_TAG_ARRAY) {
      if (!(cc >= 1 && cc <= RS_ARRAY_MAX) || !need(2ull * cc)) return false;
      nn = cc;
    } else if (tag == RS_TAG_BITSET) {
      if (!need(8192)) return false;
      nn = RS_WORDS;
    } else {
      if (!need(2)) return false;
      nn = dg16(d + start);
      if (nn == 0 || nn > RS_RUN_MAX_RUNS || !need(4ull * nn)) return false;  // (> 2047 runs: never admissible)
    }
    emit(k, kk, tag, cc, nn, o0 + start);
    nvalid = k + 1;
    pool += rs_pad16(rs_payload_bytes(tag, nn));
  }
  return off == len;
}

__global__ void k_devwire_count(uint64_t n, const uint8_t *__restrict__ buf, const uint64_t *__restrict__ offs,
                                uint64_t *__restrict__ ccount, uint64_t *__restrict__ pbytes, int *__restrict__ bad) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) { ccount[n] = 0; pbytes[n] = 0; return; }
  uint32_t nv;
  uint64_t pool;
  const bool ok = dev_walk_image(buf, offs[i] - offs[0], offs[i + 1] - offs[i],
                                 [](uint32_t, uint16_t, uint8_t, uint32_t, uint32_t, uint64_t) {}, nv, pool);
  ccount[i] = nv;
  pbytes[i] = pool;
  if (!ok) atomicOr(bad, 1);
}

__global__ void k_devwire_write(uint64_t n, const uint8_t *__restrict__ buf, const uint64_t *__restrict__ offs,
                                const uint64_t *__restrict__ cbase, const uint64_t *__restrict__ pbase,
                                uint64_t *__restrict__ bm_start, uint16_t *key, uint8_t *type, uint32_t *card,
                                uint32_t *nn, uint64_t *off, uint64_t *__restrict__ src, unsigned *__restrict__ tmask) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  bm_start[i] = cbase[i];
  if (i == n) return;
  const uint64_t cb = cbase[i];
  uint64_t poff = pbase[i];
  unsigned tm = 0;
  uint32_t nv;
  uint64_t pool;
  dev_walk_image(buf, offs[i] - offs[0], offs[i + 1] - offs[i],
                 [&](uint32_t k, uint16_t kk, uint8_t tag, uint32_t cc, uint32_t n_, uint64_t s) {
                   const uint64_t c = cb + k;
                   key[c] = kk; type[c] = tag; card[c] = cc; nn[c] = n_; off[c] = poff; src[c] = s;
                   poff += rs_pad16(rs_payload_bytes(tag, n_));
                   tm |= 1u << tag;
                 },
                 nv, pool);
  if (tm) atomicOr(tmask, tm);
}

}  // namespace

extern "C" int rs_batch_from_wire_device(const uint8_t *dbuf, const uint64_t *doffs, uint64_t n, rs_batch **out) {
  RS_TRY(ensure_device());
  *out = nullptr;
  uint64_t *ccount = (uint64_t *)dalloc((n + 1) * 8), *pbytes = (uint64_t *)dalloc((n + 1) * 8);
  uint64_t *cbase = (uint64_t *)dalloc((n + 1) * 8), *pbase = (uint64_t *)dalloc((n + 1) * 8);
  int *flags = (int *)dalloc(16);
  if (!ccount || !pbytes || !cbase || !pbase || !flags) { set_error("device allocation failed (device wire)"); return RS_ENOMEM; }
  auto cleanup = [&]() { dfree(ccount); dfree(pbytes); dfree(cbase); dfree(pbase); dfree(flags); };
  // host fallback for malformed images: the exact first error, from the host walk
  auto host_path = [&]() -> int {
    std::vector<uint64_t> h_offs(n + 1);
    int rc = d2h(h_offs.data(), doffs, (n + 1) * 8);
    if (rc) return rc;
    const uint64_t bytes = h_offs[n] - h_offs[0];
    std::vector<uint8_t> h_buf(bytes ? bytes : 1);
    if (bytes) {
      rc = d2h(h_buf.data(), dbuf, bytes);
      if (rc) return rc;
    }
    const uint64_t base = h_offs[0];
    for (auto &o : h_offs) o -= base;
    return rs_batch_from_wire(h_buf.data(), h_offs.data(), n, out);
  };
  RS_CK(cudaMemsetAsync(flags, 0, 16, g_stream));
  const unsigned gn = (unsigned)((n + 1 + 127) / 128);
  RS_LAUNCH(k_devwire_count, gn, 128, 0, n, dbuf, doffs, ccount, pbytes, flags);
  RS_TRY(scan_exclusive<uint64_t>(ccount, cbase, n + 1));
  RS_TRY(scan_exclusive<uint64_t>(pbytes, pbase, n + 1));
  struct { uint64_t C, P; int bad; } h;
  RS_CK(cudaMemcpyAsync(&h.C, cbase + n, 8, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaMemcpyAsync(&h.P, pbase + n, 8, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaMemcpyAsync(&h.bad, flags, 4, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaStreamSynchronize(g_stream));
  if (h.bad) { cleanup(); return host_path(); }
  rs_batch *b = new rs_batch();
  int rc = batch_alloc(b, n, h.C, h.P);
  uint64_t *src = (uint64_t *)dalloc((h.C ? h.C : 1) * 8);
  uint8_t *vcode = (uint8_t *)dalloc(h.C ? h.C : 1);
  uint32_t *vval = (uint32_t *)dalloc((h.C ? h.C : 1) * 4);
  if (rc || !src || !vcode || !vval) {
    rs_batch_free(b); cleanup(); dfree(src); dfree(vcode); dfree(vval);
    set_error("device allocation failed (device wire)");
    return RS_ENOMEM;
  }
  RS_LAUNCH(k_devwire_write, gn, 128, 0, n, dbuf, doffs, cbase, pbase, b->d_bm_start, b->d_key, b->d_type, b->d_card,
            b->d_n, b->d_off, src, (unsigned *)(flags + 2));
  if (h.C)
    RS_LAUNCH(k_wire_gather_validate, (unsigned)((h.C * 32 + 255) / 256), 256, 0, h.C, h.C, dbuf, src, b->dev(),
              b->d_pool, vcode, vval, flags + 1, (uint32_t *)nullptr);
  int hf[2] = {0, 0};
  RS_CK(cudaMemcpyAsync(hf, flags + 1, 8, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaStreamSynchronize(g_stream));
  dfree(src); dfree(vcode); dfree(vval);
  if (hf[0]) { rs_batch_free(b); cleanup(); return host_path(); }
  cleanup();
  b->type_mask = (uint8_t)hf[1];
  b->h_valid = false;
  RS_TRY(finalize_batch(b));
  *out = b;
  return RS_OK;
}
