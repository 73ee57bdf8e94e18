// rs_egress.cu -- results back to the caller: wire images (serde.serialize,
// serde.py:69-84), uint32 arrays (RoaringBitmap.to_array, bitmap.py:136-144)
// and bitmap equality (bitmap.py:87-91).
#include <cub/cub.cuh>
#include <algorithm>
#include "rs_internal.cuh"

using namespace rs;

namespace {

unsigned grid_for(uint64_t n, unsigned block) { return (unsigned)((n + block - 1) / block); }

__device__ __forceinline__ uint64_t bitmap_of(const uint64_t *__restrict__ bm_start, uint64_t nb, uint64_t c) {
  uint64_t lo = 0, hi = nb;
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (bm_start[m] <= c) lo = m; else hi = m;
  }
  return lo;
}

// wire payload bytes (serde.py:76-83): run payloads carry a u16 run count
__global__ void k_wire_psize(uint64_t nc, DevBatch B, uint64_t *__restrict__ psz) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c > nc) return;
  if (c == nc || c >= B.bm_start[B.nb]) { psz[c] = 0; return; }  // (nc may be a capacity)
  uint8_t t = B.type[c];
  uint32_t n = B.n[c];
  psz[c] = t == RS_TAG_ARRAY ? 2ull * n : t == RS_TAG_BITSET ? 8192ull : 2ull + 4ull * n;
}

__global__ void k_wire_imgoff(uint64_t nb, const uint64_t *__restrict__ bm_start, const uint64_t *__restrict__ ps,
                              uint64_t *__restrict__ imgoff) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i <= nb) imgoff[i] = 8 * i + 8 * bm_start[i] + ps[bm_start[i]];
}

__global__ void k_wire_headers(uint64_t nb, const uint64_t *__restrict__ bm_start, const uint64_t *__restrict__ imgoff,
                               uint8_t *__restrict__ out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nb) return;
  uint16_t *h = (uint16_t *)(out + imgoff[i]);
  uint32_t cnt = (uint32_t)(bm_start[i + 1] - bm_start[i]);
  h[0] = 'R' | ('O' << 8);
  h[1] = 'A' | ('R' << 8);
  h[2] = (uint16_t)cnt;
  h[3] = (uint16_t)(cnt >> 16);
}

__device__ void warp_copy_out(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src, uint32_t nbytes, int lane) {
  uintptr_t d = (uintptr_t)dst;
  uint32_t done = 0;
  if ((d & 15) == 0) {
    uint32_t nv = nbytes >> 4;
    for (uint32_t i = lane; i < nv; i += 32) ((uint4 *)dst)[i] = ((const uint4 *)src)[i];
    done = nv << 4;
  } else if ((d & 7) == 0) {
    uint32_t nv = nbytes >> 3;
    for (uint32_t i = lane; i < nv; i += 32) ((uint64_t *)dst)[i] = ((const uint64_t *)src)[i];
    done = nv << 3;
  } else if ((d & 3) == 0) {
    uint32_t nv = nbytes >> 2;
    for (uint32_t i = lane; i < nv; i += 32) ((uint32_t *)dst)[i] = ((const uint32_t *)src)[i];
    done = nv << 2;
  }
  for (uint32_t i = (done >> 1) + lane; i < (nbytes >> 1); i += 32) ((uint16_t *)dst)[i] = ((const uint16_t *)src)[i];
}

__global__ void k_wire_containers(uint64_t nc, uint64_t nb, DevBatch B, const uint64_t *__restrict__ ps,
                                  const uint64_t *__restrict__ imgoff, uint8_t *__restrict__ out) {
  uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  // nc may be a result's entry capacity (no host read-back of its container
  // count): entries past bm_start[nb] are not containers
  if (c >= nc || c >= B.bm_start[nb]) return;
  uint64_t i = bitmap_of(B.bm_start, nb, c);
  uint64_t first = B.bm_start[i], n_i = B.bm_start[i + 1] - first;
  uint8_t t = B.type[c];
  uint32_t n = B.n[c];
  uint8_t *img = out + imgoff[i];
  if (lane == 0) {
    uint16_t *d = (uint16_t *)(img + 8 + 8 * (c - first));
    uint32_t card = B.card[c];
    d[0] = B.key[c];
    d[1] = t;  // tag byte, pad byte 0 (little-endian)
    d[2] = (uint16_t)card;
    d[3] = (uint16_t)(card >> 16);
  }
  uint8_t *pay = img + 8 + 8 * n_i + (ps[c] - ps[first]);
  const uint8_t *src = B.pool + B.off[c];
  if (t == RS_TAG_RUN) {
    if (lane == 0) *(uint16_t *)pay = (uint16_t)n;
    warp_copy_out(pay + 2, src, 4 * n, lane);
  } else {
    warp_copy_out(pay, src, rs_payload_bytes(t, n), lane);
  }
}

// to_array: one CTA per container writes key<<16 | low values in order
constexpr int ET = 256;
__global__ void __launch_bounds__(ET) k_to_u32(uint64_t nc, DevBatch B, const uint64_t *__restrict__ vpos,
                                               uint32_t *__restrict__ out) {
  __shared__ typename cub::BlockScan<uint32_t, ET>::TempStorage scan;
  __shared__ uint32_t run_off[2048];
  uint64_t c = blockIdx.x;
  if (c >= nc) return;
  const int t = threadIdx.x;
  uint8_t type = B.type[c];
  uint32_t n = B.n[c];
  uint32_t hi = (uint32_t)B.key[c] << 16;
  uint32_t *dst = out + vpos[c];
  const uint8_t *src = B.pool + B.off[c];
  if (type == RS_TAG_ARRAY) {
    const uint16_t *v = (const uint16_t *)src;
    for (uint32_t i = t; i < n; i += ET) dst[i] = hi | v[i];
    return;
  }
  if (type == RS_TAG_BITSET) {
    const uint64_t *w = (const uint64_t *)src;
    uint64_t r[4];
    uint32_t pc = 0;
    for (int k = 0; k < 4; k++) { r[k] = w[4 * t + k]; pc += __popcll(r[k]); }
    uint32_t base;
    cub::BlockScan<uint32_t, ET>(scan).ExclusiveSum(pc, base);
    for (int k = 0; k < 4; k++) {
      uint64_t x = r[k];
      while (x) { dst[base++] = hi | ((4 * t + k) * 64 + __ffsll((long long)x) - 1); x &= x - 1; }
    }
    return;
  }
  // runs (_positions_from_runs, containers.py:150-155): prefix of lengths, then
  // one warp per run writes its values
  const uint16_t *rv = (const uint16_t *)src;
  uint32_t ch = (n + ET - 1) / ET, lo = t * ch, hi_r = min(n, lo + ch), s = 0;
  for (uint32_t r = lo; r < hi_r; r++) s += (uint32_t)rv[2 * r + 1] + 1;
  uint32_t base;
  cub::BlockScan<uint32_t, ET>(scan).ExclusiveSum(s, base);
  for (uint32_t r = lo; r < hi_r && r < 2048; r++) { run_off[r] = base; base += (uint32_t)rv[2 * r + 1] + 1; }
  __syncthreads();
  int warp = t >> 5, lane = t & 31;
  for (uint32_t r = warp; r < n && r < 2048; r += ET / 32) {
    uint32_t st = rv[2 * r], len = (uint32_t)rv[2 * r + 1] + 1, o = run_off[r];
    for (uint32_t i = lane; i < len; i += 32) dst[o + i] = hi | (st + i);
  }
}

__global__ void k_card_u64(uint64_t nc, const uint32_t *__restrict__ card, uint64_t *__restrict__ out) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c <= nc) out[c] = c < nc ? card[c] : 0;
}

__global__ void k_bm_gather(uint64_t nb, const uint64_t *__restrict__ bm_start, const uint64_t *__restrict__ pos,
                            uint64_t *__restrict__ out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i <= nb) out[i] = pos[bm_start[i]];
}

// equality: warp per container of pair-aligned container ranges
__global__ void k_equal(uint64_t T, uint64_t npairs, const uint64_t *__restrict__ tbase, DevBatch A, DevBatch B,
                        const uint64_t *__restrict__ a0s, const uint64_t *__restrict__ b0s, uint32_t *__restrict__ eq) {
  uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (t >= T) return;
  uint64_t lo = 0, hi = npairs;
  while (hi - lo > 1) {
    uint64_t m = (lo + hi) >> 1;
    if (tbase[m] <= t) lo = m; else hi = m;
  }
  uint64_t ca = a0s[lo] + (t - tbase[lo]), cb = b0s[lo] + (t - tbase[lo]);
  bool same = A.key[ca] == B.key[cb] && A.type[ca] == B.type[cb] && A.card[ca] == B.card[cb] && A.n[ca] == B.n[cb];
  if (same) {
    uint32_t bytes = rs_payload_bytes(A.type[ca], A.n[ca]);
    const uint16_t *x = (const uint16_t *)(A.pool + A.off[ca]), *y = (const uint16_t *)(B.pool + B.off[cb]);
    bool diff = false;
    for (uint32_t i = lane; i < (bytes >> 1); i += 32) diff |= x[i] != y[i];
    same = !__any_sync(0xffffffffu, diff);
  }
  if (lane == 0 && !same) atomicAnd(&eq[lo], 0u);
}

// SURVEY 8(d) byte accounting of a batch, per container
__global__ void k_stats(uint64_t nc, DevBatch B, unsigned long long *__restrict__ acc) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long pay = 0, cnt[4] = {0, 0, 0, 0};
  if (c < nc) {
    uint8_t t = B.type[c];
    uint32_t n = B.n[c];
    pay = t == RS_TAG_ARRAY ? 2ull * n : t == RS_TAG_BITSET ? 8192ull : 2ull + 4ull * n;
    cnt[t & 3] = 1;
  }
  for (int o = 16; o; o >>= 1) {
    pay += __shfl_xor_sync(0xffffffffu, pay, o);
    for (int k = 1; k < 4; k++) cnt[k] += __shfl_xor_sync(0xffffffffu, cnt[k], o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[0], pay);
    for (int k = 1; k < 4; k++) atomicAdd(&acc[k], cnt[k]);
  }
}

}  // namespace

extern "C" int rs_batch_stats(const rs_batch *b, uint64_t *payload_bytes, uint64_t *descriptor_bytes,
                              uint64_t *type_counts) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(b));
  RS_TRY(resolve_pending(b));
  unsigned long long *acc = (unsigned long long *)dalloc(4 * 8);
  if (!acc) { set_error("device allocation failed (stats)"); return RS_ENOMEM; }
  RS_CK(cudaMemsetAsync(acc, 0, 32, g_stream));
  RS_LAUNCH(k_stats, grid_for(b->nc, 256), 256, 0, b->nc, b->dev(), acc);
  uint64_t h[4];
  RS_TRY(d2h(h, acc, 32));
  dfree(acc);
  if (payload_bytes) *payload_bytes = h[0];
  if (descriptor_bytes) *descriptor_bytes = 8 * b->nc;
  if (type_counts) { type_counts[0] = 0; type_counts[1] = h[1]; type_counts[2] = h[2]; type_counts[3] = h[3]; }
  return RS_OK;
}

static int wire_offsets(const rs_batch *b, uint64_t *&ps, uint64_t *&imgoff) {
  uint64_t *psz = (uint64_t *)dalloc((b->nc + 1) * 8);
  ps = (uint64_t *)dalloc((b->nc + 1) * 8);
  imgoff = (uint64_t *)dalloc((b->nb + 1) * 8);
  if (!psz || !ps || !imgoff) { set_error("device allocation failed (wire)"); return RS_ENOMEM; }
  RS_LAUNCH(k_wire_psize, grid_for(b->nc + 1, 256), 256, 0, b->nc, b->dev(), psz);
  RS_TRY(scan_exclusive<uint64_t>(psz, ps, b->nc + 1));
  RS_LAUNCH(k_wire_imgoff, grid_for(b->nb + 1, 256), 256, 0, b->nb, b->d_bm_start, ps, imgoff);
  dfree(psz);
  return RS_OK;
}

extern "C" int rs_batch_wire_sizes(const rs_batch *b, uint64_t *sizes) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta_nopack(b));
  RS_TRY(resolve_pending(b));
  uint64_t *ps, *imgoff;
  RS_TRY(wire_offsets(b, ps, imgoff));
  std::vector<uint64_t> h(b->nb + 1);
  RS_TRY(d2h(h.data(), imgoff, (b->nb + 1) * 8));
  for (uint64_t i = 0; i < b->nb; i++) sizes[i] = h[i + 1] - h[i];
  dfree(ps);
  dfree(imgoff);
  return RS_OK;
}

extern "C" int rs_batch_to_wire(const rs_batch *b, uint8_t *buf, uint64_t cap, uint64_t *offs) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta_nopack(b));
  RS_TRY(resolve_pending(b));
  uint64_t *ps, *imgoff;
  RS_TRY(wire_offsets(b, ps, imgoff));
  RS_TRY(d2h(offs, imgoff, (b->nb + 1) * 8));
  uint64_t total = offs[b->nb];
  if (total > cap) {
    dfree(ps); dfree(imgoff);
    set_error("wire buffer too small: need " + std::to_string(total));
    return RS_EARG;
  }
  uint8_t *dout = (uint8_t *)dalloc(total ? total : 16);
  if (!dout) { set_error("device allocation failed (wire out)"); return RS_ENOMEM; }
  RS_LAUNCH(k_wire_headers, grid_for(b->nb, 256), 256, 0, b->nb, b->d_bm_start, imgoff, dout);
  RS_LAUNCH(k_wire_containers, grid_for(b->nc * 32, 256), 256, 0, b->nc, b->nb, b->dev(), ps, imgoff, dout);
  RS_TRY(d2h(buf, dout, total));
  dfree(dout); dfree(ps); dfree(imgoff);
  return RS_OK;
}

// Asynchronous export: one host synchronization for the image sizes (the
// layout), then the images are assembled in a stream-ordered device staging
// block and copied to the caller's page-locked buffer on a dedicated export
// stream, so the device->host transfer of one batch overlaps whatever the
// library stream and the ingest copy stream do next (PCIe is full duplex).
namespace {
cudaStream_t g_export = nullptr;
int g_export_dev = -1;
}  // namespace

extern "C" int rs_batch_to_wire_async(const rs_batch *b, uint8_t *buf, uint64_t cap, uint64_t *offs, void **done) {
  RS_TRY(ensure_device());
  if (!b || !offs || !done) { set_error("null batch/offs/done"); return RS_EARG; }
  *done = nullptr;
  // no read-back of the container count: the kernels bound themselves by the
  // device's bm_start, so the image sizes are the call's only synchronization
  RS_TRY(materialize(b));
  if (b->pending) RS_TRY(resolve_pending(b));
  int dev = 0;
  RS_CK(cudaGetDevice(&dev));
  if (!g_export || g_export_dev != dev) {
    RS_CK(cudaStreamCreateWithFlags(&g_export, cudaStreamNonBlocking));
    g_export_dev = dev;
  }
  uint64_t *ps, *imgoff;
  RS_TRY(wire_offsets(b, ps, imgoff));
  RS_TRY(d2h(offs, imgoff, (b->nb + 1) * 8));  // the layout: the one synchronization
  const uint64_t total = offs[b->nb];
  if (total > cap) {
    dfree(ps); dfree(imgoff);
    set_error("wire buffer too small: need " + std::to_string(total));
    return RS_EARG;
  }
  uint8_t *stage = nullptr;
  RS_CK(cudaMallocAsync((void **)&stage, total ? total : 16, g_stream));
  RS_LAUNCH(k_wire_headers, grid_for(b->nb, 256), 256, 0, b->nb, b->d_bm_start, imgoff, stage);
  RS_LAUNCH(k_wire_containers, grid_for(b->nc * 32, 256), 256, 0, b->nc, b->nb, b->dev(), ps, imgoff, stage);
  dfree(ps); dfree(imgoff);
  cudaEvent_t assembled, landed;
  RS_CK(cudaEventCreateWithFlags(&assembled, cudaEventDisableTiming));
  RS_CK(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming));
  RS_CK(cudaEventRecord(assembled, g_stream));
  RS_CK(cudaStreamWaitEvent(g_export, assembled, 0));
  if (total) RS_CK(cudaMemcpyAsync(buf, stage, total, cudaMemcpyDeviceToHost, g_export));
  RS_CK(cudaFreeAsync(stage, g_export));
  RS_CK(cudaEventRecord(landed, g_export));
  RS_CK(cudaEventDestroy(assembled));
  *done = (void *)landed;
  return RS_OK;
}

extern "C" int rs_event_synchronize(void *event) {
  RS_CK(cudaEventSynchronize((cudaEvent_t)event));
  return RS_OK;
}

extern "C" int rs_event_query(void *event) {
  cudaError_t e = cudaEventQuery((cudaEvent_t)event);
  if (e == cudaErrorNotReady) { cudaGetLastError(); return 1; }
  RS_CK(e);
  return RS_OK;
}

extern "C" int rs_batch_to_u32(const rs_batch *b, uint32_t *out, uint64_t cap, uint64_t *offs) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(b));
  RS_TRY(resolve_pending(b));
  uint64_t *cards = (uint64_t *)dalloc((b->nc + 1) * 8), *vpos = (uint64_t *)dalloc((b->nc + 1) * 8),
           *boffs = (uint64_t *)dalloc((b->nb + 1) * 8);
  if (!cards || !vpos || !boffs) { set_error("device allocation failed (to_u32)"); return RS_ENOMEM; }
  RS_LAUNCH(k_card_u64, grid_for(b->nc + 1, 256), 256, 0, b->nc, b->d_card, cards);
  RS_TRY(scan_exclusive<uint64_t>(cards, vpos, b->nc + 1));
  RS_LAUNCH(k_bm_gather, grid_for(b->nb + 1, 256), 256, 0, b->nb, b->d_bm_start, vpos, boffs);
  RS_TRY(d2h(offs, boffs, (b->nb + 1) * 8));
  uint64_t total = offs[b->nb];
  if (total > cap) {
    dfree(cards); dfree(vpos); dfree(boffs);
    set_error("value buffer too small: need " + std::to_string(total));
    return RS_EARG;
  }
  uint32_t *dout = (uint32_t *)dalloc((total ? total : 1) * 4);
  if (!dout) { set_error("device allocation failed (to_u32 out)"); return RS_ENOMEM; }
  RS_LAUNCH(k_to_u32, (unsigned)b->nc, ET, 0, b->nc, b->dev(), vpos, dout);
  RS_TRY(d2h(out, dout, total * 4));
  dfree(dout); dfree(cards); dfree(vpos); dfree(boffs);
  return RS_OK;
}

extern "C" int rs_batch_equal(const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib,
                              uint64_t npairs, uint8_t *eq) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta(A));
  RS_TRY(fetch_host_meta(B));
  RS_TRY(resolve_pending(A));
  RS_TRY(resolve_pending(B));
  std::vector<uint64_t> tbase(npairs + 1, 0), a0s(npairs + 1, 0), b0s(npairs + 1, 0);
  std::vector<uint32_t> init(npairs + 1, 1);
  for (uint64_t p = 0; p < npairs; p++) {
    uint64_t a = ia ? ia[p] : p, b = ib ? ib[p] : p;
    if (a >= A->nb || b >= B->nb) { set_error("pair index out of range"); return RS_EARG; }
    uint64_t na = A->h_bm_start[a + 1] - A->h_bm_start[a], nb = B->h_bm_start[b + 1] - B->h_bm_start[b];
    a0s[p] = A->h_bm_start[a];
    b0s[p] = B->h_bm_start[b];
    if (na != nb) init[p] = 0;
    tbase[p + 1] = tbase[p] + (na == nb ? na : 0);
  }
  uint64_t T = tbase[npairs];
  uint64_t *d_tb = (uint64_t *)dalloc((npairs + 1) * 8), *d_a0 = (uint64_t *)dalloc((npairs + 1) * 8),
           *d_b0 = (uint64_t *)dalloc((npairs + 1) * 8);
  uint32_t *d_eq = (uint32_t *)dalloc((npairs + 1) * 4);
  if (!d_tb || !d_a0 || !d_b0 || !d_eq) { set_error("device allocation failed (equal)"); return RS_ENOMEM; }
  RS_TRY(h2d(d_tb, tbase.data(), (npairs + 1) * 8));
  RS_TRY(h2d(d_a0, a0s.data(), (npairs + 1) * 8));
  RS_TRY(h2d(d_b0, b0s.data(), (npairs + 1) * 8));
  RS_TRY(h2d(d_eq, init.data(), (npairs + 1) * 4));
  RS_LAUNCH(k_equal, grid_for(T * 32, 256), 256, 0, T, npairs, d_tb, A->dev(), B->dev(), d_a0, d_b0, d_eq);
  RS_TRY(d2h(init.data(), d_eq, npairs * 4));
  for (uint64_t p = 0; p < npairs; p++) eq[p] = (uint8_t)(init[p] != 0);
  dfree(d_tb); dfree(d_a0); dfree(d_b0); dfree(d_eq);
  return RS_OK;
}

// ---------------------------------------------------------------- membership
// container_contains (containers.py:258-268) after the key lookup of
// RoaringBitmap.__contains__ (bitmap.py:99-104): binary search of the
// bitmap's key list, then array search / bit test / run search.
namespace {
__global__ void k_contains(uint64_t n, DevBatch B, const uint32_t *__restrict__ ibm,
                           const uint32_t *__restrict__ values, uint8_t *__restrict__ hit) {
  uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t v = values[q], bi = ibm ? ibm[q] : 0;
  const uint16_t key = (uint16_t)(v >> 16), low = (uint16_t)v;
  uint64_t lo = B.bm_start[bi], hi = B.bm_start[bi + 1];
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (B.key[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  uint8_t r = 0;
  if (lo < B.bm_start[bi + 1] && B.key[lo] == key) {
    const uint8_t *src = B.pool + B.off[lo];
    const uint32_t cn = B.n[lo];
    const uint8_t t = B.type[lo];
    if (t == RS_TAG_BITSET) {
      r = (uint8_t)((((const uint64_t *)src)[low >> 6] >> (low & 63)) & 1);
    } else if (t == RS_TAG_ARRAY) {
      const uint16_t *a = (const uint16_t *)src;
      uint32_t l = 0, h = cn;
      while (l < h) {
        uint32_t m = (l + h) >> 1;
        if (a[m] < low) l = m + 1;
        else h = m;
      }
      r = l < cn && a[l] == low;
    } else {  // last run whose start <= low, then low <= start + length
      const uint16_t *rv = (const uint16_t *)src;
      uint32_t l = 0, h = cn;
      while (l < h) {
        uint32_t m = (l + h) >> 1;
        if (rv[2 * m] <= low) l = m + 1;
        else h = m;
      }
      r = l > 0 && (uint32_t)low <= (uint32_t)rv[2 * (l - 1)] + rv[2 * (l - 1) + 1];
    }
  }
  hit[q] = r;
}
}  // namespace

extern "C" int rs_batch_contains(const rs_batch *b, const uint32_t *ibm, const uint32_t *values, uint64_t n,
                                 uint8_t *hit) {
  RS_TRY(ensure_device());
  RS_TRY(resolve_pending(b));
  if (n == 0) return RS_OK;
  if (!values || !hit) { set_error("contains: null values/hit"); return RS_EARG; }
  if (b->nb == 0) { set_error("contains: empty batch"); return RS_EARG; }
  if (ibm)
    for (uint64_t q = 0; q < n; q++)
      if (ibm[q] >= b->nb) { set_error("contains: bitmap index out of range"); return RS_EARG; }
  uint32_t *d_v = (uint32_t *)dalloc(n * 4), *d_i = ibm ? (uint32_t *)dalloc(n * 4) : nullptr;
  uint8_t *d_h = (uint8_t *)dalloc(n);
  if (!d_v || !d_h || (ibm && !d_i)) { set_error("device allocation failed (contains)"); return RS_ENOMEM; }
  RS_TRY(h2d(d_v, values, n * 4));
  if (ibm) RS_TRY(h2d(d_i, ibm, n * 4));
  RS_LAUNCH(k_contains, grid_for(n, 256), 256, 0, n, b->dev(), d_i, d_v, d_h);
  RS_TRY(d2h(hit, d_h, n));
  dfree(d_v); dfree(d_i); dfree(d_h);
  return RS_OK;
}

// ---------------------------------------------------------- content digests
// A 64-bit digest of each bitmap's exact content (keys, types, cardinalities,
// payloads: everything its wire image holds), for parity at full size without
// moving results to the host.  The definition is shared with the oracle
// (oracle/roaring_oracle.c "content digests"):
//   h(c) = mix(key<<48 | tag<<40 | card) + sum of per-unit terms
//   digest(bitmap) = sum_j mix(h(c_j) + (j+1) * K_POS)
namespace {
constexpr uint64_t DG_K_ARRAY = 0x243F6A8885A308D3ull, DG_K_BITSET = 0x13198A2E03707344ull,
                   DG_K_RUN = 0xA4093822299F31D0ull, DG_K_POS = 0x082EFA98EC4E6C89ull;

__device__ __forceinline__ uint64_t dg_mix(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// warp per container: its positional term mix(h(c) + (j+1) K_POS)
__global__ void k_digest_containers(uint64_t nc, uint64_t nb, DevBatch B, uint64_t *__restrict__ term) {
  const uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nc) return;
  const uint8_t t = B.type[c];
  const uint32_t n = B.n[c];
  const uint8_t *p = B.pool + B.off[c];
  uint64_t h = 0;
  if (t == RS_TAG_ARRAY) {
    const uint16_t *v = (const uint16_t *)p;
    for (uint32_t i = lane; i < n; i += 32) h += dg_mix((((uint64_t)i << 16) | v[i]) + DG_K_ARRAY);
  } else if (t == RS_TAG_BITSET) {
    const uint64_t *w = (const uint64_t *)p;
    for (uint32_t i = lane; i < RS_WORDS; i += 32) h += dg_mix(w[i] + (uint64_t)i * DG_K_BITSET);
  } else {
    const uint32_t *r = (const uint32_t *)p;  // (start, length) u16 pairs
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t x = r[i];
      h += dg_mix((((uint64_t)i << 32) | ((uint64_t)(x & 0xFFFF) << 16) | (x >> 16)) + DG_K_RUN);
    }
  }
  for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if (lane == 0) {
    const uint64_t bm = bitmap_of(B.bm_start, nb, c);
    h += dg_mix(((uint64_t)B.key[c] << 48) | ((uint64_t)t << 40) | B.card[c]);
    term[c] = dg_mix(h + (c - B.bm_start[bm] + 1) * DG_K_POS);
  }
}

__global__ void k_digest_bitmaps(uint64_t nb, const uint64_t *__restrict__ bm_start, const uint64_t *__restrict__ term,
                                 uint64_t *__restrict__ out) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nb) return;
  uint64_t s = 0;
  for (uint64_t c = bm_start[w] + lane; c < bm_start[w + 1]; c += 32) s += term[c];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s;
}
}  // namespace

extern "C" int rs_batch_digests(const rs_batch *b, uint64_t *digests, int on_device) {
  RS_TRY(ensure_device());
  RS_TRY(fetch_host_meta_nopack(b));
  if (!on_device) RS_TRY(resolve_pending(b));
  uint64_t *term = (uint64_t *)dalloc((b->nc + 1) * 8);
  uint64_t *dout = on_device ? digests : (uint64_t *)dalloc((b->nb + 1) * 8);
  if (!term || !dout) { set_error("device allocation failed (digests)"); return RS_ENOMEM; }
  RS_LAUNCH(k_digest_containers, grid_for(b->nc * 32, 256), 256, 0, b->nc, b->nb, b->dev(), term);
  RS_LAUNCH(k_digest_bitmaps, grid_for(b->nb * 32, 256), 256, 0, b->nb, b->d_bm_start, term, dout);
  if (!on_device) {
    RS_TRY(d2h(digests, dout, b->nb * 8));
    dfree(dout);
  }
  dfree(term);
  return RS_OK;
}
