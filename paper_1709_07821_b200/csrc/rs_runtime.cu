// rs_runtime.cu -- runtime plumbing: errors, stream, stream-ordered allocation,
// scans/sorts (CUB device primitives), batch lifetime and metadata queries.
#include <cub/cub.cuh>
#include <chrono>
#include <map>
#include <tuple>
#include <mutex>
#include <set>
#include <unordered_map>
#include <cstring>
#include "rs_internal.cuh"

namespace rs {
uint64_t g_dalloc_stats[2] = {0, 0};  // stream switches, cache misses (RS_HOST_TRACE)
cudaStream_t g_stream = nullptr;
uint64_t g_launches = 0;
static thread_local std::string t_err;
static thread_local int64_t t_err_off = -1, t_err_idx = -1;
static int g_device_ok = -1;
static std::mutex g_init_mu;

bool g_prof_on = false;
struct ProfRec { std::string name; cudaEvent_t a, b; uint64_t items; };
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t prof_event() {
  cudaEvent_t e;
  if (!g_event_pool.empty()) { e = g_event_pool.back(); g_event_pool.pop_back(); return e; }
  cudaEventCreate(&e);
  return e;
}
void prof_mark(const char *name, cudaEvent_t a, cudaEvent_t b, uint64_t items) {
  g_prof.push_back({name, a, b, items});
}

// Occupancy of a kernel per (device, kernel, threads, smem), computed once:
// cudaOccupancyMaxActiveBlocksPerMultiprocessor and the attribute queries
// cost microseconds of host time per launch, which small batches (config 1:
// ~10 launches per op) paid on every call.
int occupancy_per_sm(const void *kernel, int threads, size_t smem, int *sms_out) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void *, int, size_t>, int> cache;
  static std::map<int, int> sms;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto si = sms.find(dev);
  if (si == sms.end()) {
    int n = 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    si = sms.emplace(dev, n).first;
  }
  if (sms_out) *sms_out = si->second;
  const auto key = std::make_tuple(dev, kernel, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess || per <= 0) {
    cudaGetLastError();
    per = 1;
  }
  cache.emplace(key, per);
  return per;
}

namespace {
struct HostTrace {
  int on = -1;
  std::chrono::steady_clock::time_point last;
  double ns[32] = {0};
  uint64_t n[32] = {0};
  ~HostTrace() { dump(); }
  void dump() {
    if (on != 1) return;
    fprintf(stderr, "[rs_host] dalloc stream switches %llu, cache misses %llu\n",
            (unsigned long long)g_dalloc_stats[0], (unsigned long long)g_dalloc_stats[1]);
    for (int i = 0; i < 32; i++)
      if (n[i]) fprintf(stderr, "[rs_host] point %2d: %8.2f us avg over %llu\n", i, ns[i] / n[i] * 1e-3,
                        (unsigned long long)n[i]);
  }
} g_ht;
}  // namespace

extern "C" void rs_host_trace_dump(void) { g_ht.dump(); }

void host_mark(int point) {
  if (g_ht.on < 0) {
    const char *v = getenv("RS_HOST_TRACE");
    g_ht.on = v && *v == '1';
  }
  if (!g_ht.on) return;
  auto now = std::chrono::steady_clock::now();
  if (point > 0 && point < 32) {
    g_ht.ns[point] += std::chrono::duration<double, std::nano>(now - g_ht.last).count();
    g_ht.n[point]++;
  }
  g_ht.last = now;
}

void trace(const char *phase) {
  static int on = -1;
  static std::chrono::steady_clock::time_point last;
  if (on < 0) {
    const char *v = getenv("RS_TRACE");
    on = v && *v == '1';
    last = std::chrono::steady_clock::now();
  }
  if (!on) return;
  cudaStreamSynchronize(g_stream);
  auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[rs_trace] %-28s %9.3f ms\n", phase,
          std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

void set_error(const std::string &m, int64_t off, int64_t idx) {
  t_err = m;
  t_err_off = off;
  t_err_idx = idx;
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
           cudaGetErrorString(e), what, file, line);
  set_error(buf);
  return e == cudaErrorMemoryAllocation ? RS_ENOMEM : RS_ECUDA;
}

int ensure_device() {
  std::lock_guard<std::mutex> g(g_init_mu);
  if (g_device_ok == 1) return RS_OK;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device available: roaring_b200 has no CPU fallback");
    return RS_ECUDA;
  }
  cudaMemPool_t pool;
  int dev = 0;
  RS_CK(cudaGetDevice(&dev));
  RS_CK(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = UINT64_MAX;  // keep freed blocks cached in the pool
  RS_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  g_device_ok = 1;
  return RS_OK;
}

// Caching allocator: freed blocks go to size-class free lists and are reused
// in stream order on the single library stream (an op's scratch and result
// pools are the same sizes step after step), so steady-state ops never call
// into the driver.  Small blocks round to powers of two, large ones to 2 MB;
// a cached block is reused when it is at most 1/8 larger than the request.
static std::mutex g_alloc_mu;
static std::multimap<size_t, void *> g_free_blocks;
static std::unordered_map<void *, size_t> g_block_size;
static cudaStream_t g_alloc_stream = nullptr;

static size_t round_block(size_t b) {
  if (b <= (1u << 20)) {
    size_t r = 256;
    while (r < b) r <<= 1;
    return r;
  }
  return (b + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
}

static void release_cached_locked() {
  for (auto &kv : g_free_blocks) {
    cudaFreeAsync(kv.second, g_stream);
    g_block_size.erase(kv.second);
  }
  g_free_blocks.clear();
}

void *dalloc(size_t bytes) {
  std::lock_guard<std::mutex> g(g_alloc_mu);
  if (g_alloc_stream != g_stream) {  // cached blocks are ordered on the old stream
    g_dalloc_stats[0]++;
    cudaStreamSynchronize(g_alloc_stream);
    g_alloc_stream = g_stream;
  }
  const size_t r = round_block(bytes ? bytes : 16);
  auto it = g_free_blocks.lower_bound(r);
  if (it != g_free_blocks.end() && it->first <= r + r / 8) {
    void *p = it->second;
    g_free_blocks.erase(it);
    return p;
  }
  void *p = nullptr;
  g_dalloc_stats[1]++;
  if (cudaMallocAsync(&p, r, g_stream) != cudaSuccess) {
    cudaGetLastError();
    release_cached_locked();
    cudaStreamSynchronize(g_stream);
    if (cudaMallocAsync(&p, r, g_stream) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  g_block_size[p] = r;
  return p;
}

void dfree(void *p) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_alloc_mu);
  auto it = g_block_size.find(p);
  if (it == g_block_size.end()) {
    cudaFreeAsync(p, g_stream);
    return;
  }
  g_free_blocks.emplace(it->second, p);
}

int d2h(void *h, const void *d, size_t bytes) {
  if (bytes) RS_CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, g_stream));
  RS_CK(cudaStreamSynchronize(g_stream));
  return RS_OK;
}

int h2d(void *d, const void *h, size_t bytes) {
  if (bytes) RS_CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, g_stream));
  return RS_OK;
}

// Fork/join of independent launches (the per-type-pair class kernels of one
// op): side streams wait on an event recorded on the library stream, the
// library stream waits on an event recorded on every side stream used.
namespace {
std::vector<cudaStream_t> g_side;
std::vector<cudaEvent_t> g_side_ev;
cudaEvent_t g_fork_ev = nullptr;
int g_side_dev = -1;
}  // namespace

int Fork::begin(int nside) {
  int dev = 0;
  RS_CK(cudaGetDevice(&dev));
  if (g_side_dev != dev) {  // streams and events belong to a device
    g_side.clear();
    g_side_ev.clear();
    RS_CK(cudaEventCreateWithFlags(&g_fork_ev, cudaEventDisableTiming));
    g_side_dev = dev;
  }
  while ((int)g_side.size() < nside) {
    cudaStream_t st;
    cudaEvent_t ev;
    RS_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    RS_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    g_side.push_back(st);
    g_side_ev.push_back(ev);
  }
  saved = g_stream;
  n = nside;
  used = 0;
  RS_CK(cudaEventRecord(g_fork_ev, saved));
  for (int i = 0; i < n; i++) RS_CK(cudaStreamWaitEvent(g_side[i], g_fork_ev, 0));
  return RS_OK;
}

void Fork::next() {
  if (n && used < n) g_stream = g_side[used++];
}

int Fork::end() {
  if (!n) return RS_OK;
  g_stream = saved;
  for (int i = 0; i < used; i++) {
    RS_CK(cudaEventRecord(g_side_ev[i], g_side[i]));
    RS_CK(cudaStreamWaitEvent(saved, g_side_ev[i], 0));
  }
  n = 0;
  return RS_OK;
}

// An op's small host->device upload (a few KB): a plain cudaMemcpyAsync from
// pageable memory, which the driver stages through the command stream itself.
// Measured on the pipelined e2e path (bulk ingest saturating PCIe on the copy
// stream): pageable 80 ms/step, pinned DMA 91 ms (queues on the copy engine
// behind the bulk transfer), a kernel pulling from mapped host memory 94 ms.
int h2d_small(void *d, const void *h, size_t bytes) {
  if (bytes) RS_CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, g_stream));
  return RS_OK;
}

// Short scans (the per-op entry/keep/ub arrays of small batches) run in one
// CTA: one launch instead of CUB's two plus its temp allocation.  The CTA is
// 1024 threads wide with 16 (u32) / 8 (u64) values per thread, so up to
// 16 K / 8 K values take one pass: each pass is a load latency plus a block
// scan (~2.5 us), and a 256 x 8 CTA spent ~20 us on 15 K values in 8 passes
// (two such scans per op).
constexpr int SCAN_T = 1024;
constexpr uint64_t SCAN_SMALL_MAX = 16384;
template <typename T>
constexpr int scan_v() { return sizeof(T) == 4 ? 16 : 8; }

template <typename T, bool INCL>
__global__ void __launch_bounds__(SCAN_T) k_scan_small(const T *in, T *out, uint32_t n) {
  constexpr int SCAN_V = scan_v<T>();
  __shared__ T wsum[SCAN_T / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T carry = 0;
  for (uint32_t base = 0; base < n; base += SCAN_T * SCAN_V) {
    // thread-serial sums around one block scan of the per-thread totals
    T v[SCAN_V], sum = 0;
    const uint32_t i0 = base + threadIdx.x * SCAN_V;
#pragma unroll
    for (int k = 0; k < SCAN_V; k++) {
      v[k] = i0 + k < n ? in[i0 + k] : T(0);
      sum += v[k];
    }
    // block exclusive scan of `sum`: warp shuffles, then the 32 warp totals
    T x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    T wt = lane < SCAN_T / 32 ? wsum[lane] : T(0), wx = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, wx, o);
      if (lane >= o) wx += y;
    }
    const T wbase = __shfl_sync(0xffffffffu, wx - wt, w);  // warps before w
    const T tot = __shfl_sync(0xffffffffu, wx, 31);
    const T excl = wbase + x - sum;
    T run = excl + carry;
#pragma unroll
    for (int k = 0; k < SCAN_V; k++) {
      if (INCL) run += v[k];
      if (i0 + k < n) out[i0 + k] = run;
      if (!INCL) run += v[k];
    }
    carry += tot;
    __syncthreads();
  }
}

template <typename T, bool INCL>
static int scan_impl(const T *in, T *out, uint64_t n) {
  if (n == 0) return RS_OK;
  if (n <= SCAN_SMALL_MAX) {
    k_scan_small<T, INCL><<<1, SCAN_T, 0, g_stream>>>(in, out, (uint32_t)n);
    RS_CK(cudaGetLastError());
    g_launches += 1;
    return RS_OK;
  }
  size_t tmp = 0;
  if (INCL) RS_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, (int64_t)n, g_stream));
  else RS_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)n, g_stream));
  void *t = dalloc(tmp);
  if (!t) { set_error("device allocation failed (scan)"); return RS_ENOMEM; }
  if (INCL) RS_CK(cub::DeviceScan::InclusiveSum(t, tmp, in, out, (int64_t)n, g_stream));
  else RS_CK(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int64_t)n, g_stream));
  g_launches += 2;
  dfree(t);
  return RS_OK;
}

template <typename T>
int scan_exclusive(const T *in, T *out, uint64_t n) { return scan_impl<T, false>(in, out, n); }
template <typename T>
int scan_inclusive(const T *in, T *out, uint64_t n) { return scan_impl<T, true>(in, out, n); }

template int scan_exclusive<uint32_t>(const uint32_t *, uint32_t *, uint64_t);
template int scan_exclusive<uint64_t>(const uint64_t *, uint64_t *, uint64_t);
template int scan_inclusive<uint32_t>(const uint32_t *, uint32_t *, uint64_t);
template int scan_inclusive<uint64_t>(const uint64_t *, uint64_t *, uint64_t);

int sort_u64(uint64_t *keys, uint64_t n, int end_bit, int begin_bit) {
  if (n <= 1) return RS_OK;
  uint64_t *alt = (uint64_t *)dalloc(n * 8);
  if (!alt) { set_error("device allocation failed (sort)"); return RS_ENOMEM; }
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  size_t tmp = 0;
  RS_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, (int64_t)n, begin_bit, end_bit, g_stream));
  void *t = dalloc(tmp);
  if (!t) { dfree(alt); set_error("device allocation failed (sort)"); return RS_ENOMEM; }
  RS_CK(cub::DeviceRadixSort::SortKeys(t, tmp, db, (int64_t)n, begin_bit, end_bit, g_stream));
  g_launches += (end_bit - begin_bit + 7) / 8 + 2;
  if (db.Current() != keys)
    RS_CK(cudaMemcpyAsync(keys, db.Current(), n * 8, cudaMemcpyDeviceToDevice, g_stream));
  dfree(t);
  dfree(alt);
  return RS_OK;
}

int batch_alloc(rs_batch *b, uint64_t nb, uint64_t nc, uint64_t pool_bytes) {
  b->nb = nb;
  b->nc = nc;
  b->cap_c = nc;
  b->pool_bytes = pool_bytes;
  b->d_bm_start = (uint64_t *)dalloc((nb + 1) * 8);
  b->d_bm_card = (uint64_t *)dalloc((nb + 1) * 8);
  uint64_t c = nc ? nc : 1;
  b->d_key = (uint16_t *)dalloc(c * 2);
  b->d_type = (uint8_t *)dalloc(c);
  b->d_card = (uint32_t *)dalloc(c * 4);
  b->d_n = (uint32_t *)dalloc(c * 4);
  b->d_off = (uint64_t *)dalloc(c * 8);
  b->d_pool = (uint8_t *)dalloc(pool_bytes ? pool_bytes : 16);
  if (!b->d_bm_start || !b->d_bm_card || !b->d_key || !b->d_type || !b->d_card || !b->d_n ||
      !b->d_off || !b->d_pool) {
    set_error("device allocation failed (batch)");
    return RS_ENOMEM;
  }
  return RS_OK;
}

void batch_release(rs_batch *b) {
  if (b->ub_pool) ub_unregister(b);
  if (b->pending) {
    drop_staged(b);
    dfree(b->pending->d_any); dfree(b->pending->d_vcode); dfree(b->pending->d_vval);
    delete b->pending;
    b->pending = nullptr;
  }
  dfree(b->d_bm_start); dfree(b->d_bm_card); dfree(b->d_key); dfree(b->d_type);
  dfree(b->d_card); dfree(b->d_n); dfree(b->d_off); dfree(b->d_pool);
  b->d_bm_start = nullptr; b->d_bm_card = nullptr; b->d_key = nullptr; b->d_type = nullptr;
  b->d_card = nullptr; b->d_n = nullptr; b->d_off = nullptr; b->d_pool = nullptr;
}

int fetch_host_meta_nopack(const rs_batch *cb) {
  RS_TRY(materialize(cb));
  rs_batch *b = const_cast<rs_batch *>(cb);
  if (!b->h_valid) {
    b->h_bm_start.resize(b->nb + 1);
    RS_TRY(d2h(b->h_bm_start.data(), b->d_bm_start, (b->nb + 1) * 8));
    b->nc = b->h_bm_start[b->nb];
    b->h_valid = true;
  }
  return RS_OK;
}

int fetch_host_meta(const rs_batch *cb) {
  RS_TRY(fetch_host_meta_nopack(cb));
  // the stream is synchronized (or was, when h_valid was set): pack an
  // upper-bound pool now, so a batch the host keeps using holds at most
  // ~1.25x its containers' bytes (bitmap.py:318-328 shrink_to_fit semantics).
  // Exports (wire images, digests) read the pool in place and skip this.
  rs_batch *b = const_cast<rs_batch *>(cb);
  if (b->ub_pool) RS_TRY(repack_pool(b));
  return RS_OK;
}

// ------------------------------------------------------- pool repacking
namespace {
std::mutex g_ub_mu;
std::set<rs_batch *> g_ub_live;   // results whose pool still holds its upper-bound slots
uint64_t g_ub_bytes = 0;

__global__ void k_pool_sizes(uint64_t nc, const uint8_t *__restrict__ type, const uint32_t *__restrict__ n,
                             uint64_t *__restrict__ psize) {
  uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c < nc) psize[c] = rs_pad16(rs_payload_bytes(type[c], n[c]));
  else if (c == nc) psize[c] = 0;
}

// warp per container: payload to its packed offset (16-byte units)
__global__ void k_repack(uint64_t nc, DevBatch S, const uint64_t *__restrict__ new_off, uint8_t *__restrict__ pool) {
  uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nc) return;
  const uint32_t nv = (uint32_t)(rs_pad16(rs_payload_bytes(S.type[c], S.n[c])) >> 4);
  const uint4 *src = (const uint4 *)(S.pool + S.off[c]);
  uint4 *dst = (uint4 *)(pool + new_off[c]);
  for (uint32_t i = lane; i < nv; i += 32) __stcs(dst + i, __ldcs(src + i));
}

uint64_t ub_high_water() {
  static uint64_t mark = 0;
  if (!mark) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    mark = std::max<uint64_t>(tot / 8, 1ull << 30);
  }
  return mark;
}
}  // namespace

void ub_register(rs_batch *b) {
  std::lock_guard<std::mutex> g(g_ub_mu);
  b->ub_pool = true;
  if (g_ub_live.insert(b).second) g_ub_bytes += b->pool_bytes;
}

void ub_unregister(rs_batch *b) {
  std::lock_guard<std::mutex> g(g_ub_mu);
  if (g_ub_live.erase(b)) g_ub_bytes -= b->pool_bytes;
  b->ub_pool = false;
}

int repack_pool(rs_batch *b) {
  ub_unregister(b);
  const uint64_t nc = b->nc;
  uint64_t *psize = (uint64_t *)dalloc((nc + 1) * 8), *poff = (uint64_t *)dalloc((nc + 1) * 8);
  if (!psize || !poff) { dfree(psize); dfree(poff); set_error("device allocation failed (repack)"); return RS_ENOMEM; }
  RS_LAUNCH(k_pool_sizes, (unsigned)((nc + 1 + 255) / 256), 256, 0, nc, b->d_type, b->d_n, psize);
  RS_TRY(scan_exclusive<uint64_t>(psize, poff, nc + 1));
  uint64_t used = 0;
  RS_TRY(d2h(&used, poff + nc, 8));
  // keep the pool when it is already within 1.25x of its containers' bytes
  if (4 * b->pool_bytes <= 5 * used + 4096) {
    dfree(psize); dfree(poff);
    return RS_OK;
  }
  uint8_t *np = (uint8_t *)dalloc(used ? used : 16);
  if (!np) { dfree(psize); dfree(poff); set_error("device allocation failed (repack pool)"); return RS_ENOMEM; }
  if (nc) RS_LAUNCH(k_repack, (unsigned)((nc * 32 + 255) / 256), 256, 0, nc, b->dev(), poff, np);
  RS_CK(cudaMemcpyAsync(b->d_off, poff, nc * 8, cudaMemcpyDeviceToDevice, g_stream));
  dfree(b->d_pool);
  b->d_pool = np;
  b->pool_bytes = used;
  dfree(psize); dfree(poff);
  return RS_OK;
}

int ub_reserve(uint64_t bytes) {
  std::vector<rs_batch *> victims;
  {
    std::lock_guard<std::mutex> g(g_ub_mu);
    if (g_ub_bytes + bytes <= ub_high_water()) return RS_OK;
    victims.assign(g_ub_live.begin(), g_ub_live.end());
  }
  for (rs_batch *v : victims) RS_TRY(fetch_host_meta(v));  // packs it
  return RS_OK;
}

// RoaringBitmap.__len__ (bitmap.py:77-82): one warp per bitmap sums its cards
// (one thread per bitmap when bitmaps hold few containers, e.g. config 3's
// single-container bitmaps, where a warp would leave 31 lanes idle).
__global__ void k_bm_card(uint64_t nb, const uint64_t *__restrict__ bm_start,
                          const uint32_t *__restrict__ card, uint64_t *__restrict__ out) {
  uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= nb) return;
  uint64_t s = 0;
  for (uint64_t c = bm_start[w] + lane; c < bm_start[w + 1]; c += 32) s += card[c];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s;
}

__global__ void k_bm_card_thread(uint64_t nb, const uint64_t *__restrict__ bm_start,
                                 const uint32_t *__restrict__ card, uint64_t *__restrict__ out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nb) return;
  uint64_t s = 0;
  for (uint64_t c = bm_start[i]; c < bm_start[i + 1]; c++) s += card[c];
  out[i] = s;
}

// few bitmaps holding many containers (a wide union's result): a CTA per
// bitmap instead of a lone warp walking tens of thousands of cards
// few bitmaps holding many containers (a wide union's result): CTAs of 256
// threads split each bitmap's cards (blockIdx.y) and add their block sums
// into out, which is zeroed first
__global__ void __launch_bounds__(256) k_bm_card_split(uint64_t nb, const uint64_t *__restrict__ bm_start,
                                                       const uint32_t *__restrict__ card,
                                                       unsigned long long *__restrict__ out) {
  __shared__ uint64_t red[8];
  const uint64_t b = blockIdx.x;
  const uint64_t c0 = bm_start[b], c1 = bm_start[b + 1];
  uint64_t s = 0;
  for (uint64_t c = c0 + blockIdx.y * 256ull + threadIdx.x; c < c1; c += 256ull * gridDim.y) s += card[c];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t tot = 0;
    for (int w = 0; w < 8; w++) tot += red[w];
    if (tot) atomicAdd(&out[b], (unsigned long long)tot);
  }
}

int finalize_batch(rs_batch *b) {
  if (b->nb && b->nb <= 1024 && b->nc >= 256 * b->nb) {
    const unsigned split = (unsigned)std::min<uint64_t>(std::max<uint64_t>(b->nc / b->nb / 2048, 1), 64);
    RS_CK(cudaMemsetAsync(b->d_bm_card, 0, b->nb * 8, g_stream));
    dim3 grid((unsigned)b->nb, split);
    k_bm_card_split<<<grid, 256, 0, g_stream>>>(b->nb, b->d_bm_start, b->d_card,
                                                (unsigned long long *)b->d_bm_card);
    ++g_launches;
    RS_CK(cudaGetLastError());
    return RS_OK;
  }
  if (b->nb && b->nc <= 4 * b->nb) {
    RS_LAUNCH(k_bm_card_thread, (unsigned)((b->nb + 255) / 256), 256, 0, b->nb, b->d_bm_start, b->d_card,
              b->d_bm_card);
    return RS_OK;
  }
  uint64_t threads = b->nb * 32;
  RS_LAUNCH(k_bm_card, (unsigned)((threads + 255) / 256), 256, 0, b->nb, b->d_bm_start, b->d_card,
            b->d_bm_card);
  return RS_OK;
}
}  // namespace rs

using namespace rs;

extern "C" {

const char *rs_last_error(void) { return rs::t_err.c_str(); }
int64_t rs_last_error_offset(void) { return rs::t_err_off; }
int64_t rs_last_error_index(void) { return rs::t_err_idx; }
const char *rs_version(void) { return "roaring_b200 0.1.0 (sm_100a)"; }
uint64_t rs_kernel_launches(void) { return rs::g_launches; }

int rs_set_device(int device) {
  RS_CK(cudaSetDevice(device));
  {
    std::lock_guard<std::mutex> g(rs::g_init_mu);
    rs::g_device_ok = -1;  // re-run the pool setup for this device
  }
  return ensure_device();
}

int rs_set_stream(void *stream) {
  RS_TRY(ensure_device());
  g_stream = (cudaStream_t)stream;
  return RS_OK;
}
void *rs_get_stream(void) { return (void *)g_stream; }

int rs_synchronize(void) {
  RS_TRY(ensure_device());
  RS_CK(cudaStreamSynchronize(g_stream));
  return RS_OK;
}

int rs_host_alloc(void **ptr, uint64_t bytes) {
  RS_TRY(ensure_device());
  RS_CK(cudaMallocHost(ptr, bytes ? bytes : 16));
  return RS_OK;
}
int rs_host_free(void *ptr) {
  RS_CK(cudaFreeHost(ptr));
  return RS_OK;
}

int rs_event_record(void **event) {
  RS_TRY(ensure_device());
  cudaEvent_t e;
  RS_CK(cudaEventCreate(&e));
  RS_CK(cudaEventRecord(e, g_stream));
  *event = (void *)e;
  return RS_OK;
}
int rs_event_elapsed(void *start, void *stop, float *ms) {
  RS_CK(cudaEventSynchronize((cudaEvent_t)stop));
  RS_CK(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
  return RS_OK;
}
int rs_event_destroy(void *event) {
  RS_CK(cudaEventDestroy((cudaEvent_t)event));
  return RS_OK;
}

int rs_profile_enable(int on) {
  RS_TRY(ensure_device());
  rs::g_prof_on = on != 0;
  return RS_OK;
}

int rs_profile_reset(void) {
  RS_CK(cudaStreamSynchronize(g_stream));
  for (auto &r : rs::g_prof) { rs::g_event_pool.push_back(r.a); rs::g_event_pool.push_back(r.b); }
  rs::g_prof.clear();
  return RS_OK;
}

int rs_profile_query(const char *name, double *total_ms, uint64_t *launches, uint64_t *items) {
  RS_CK(cudaStreamSynchronize(g_stream));
  double t = 0;
  uint64_t n = 0, it = 0;
  for (auto &r : rs::g_prof) {
    if (r.name != name) continue;
    float ms = 0;
    RS_CK(cudaEventElapsedTime(&ms, r.a, r.b));
    t += ms;
    n++;
    it += r.items;
  }
  *total_ms = t;
  *launches = n;
  if (items) *items = it;
  return RS_OK;
}

int rs_batch_free(rs_batch *b) {
  if (!b) return RS_OK;
  host_mark(0);
  batch_release(b);
  delete b;
  host_mark(20);
  return RS_OK;
}

uint64_t rs_batch_len(const rs_batch *b) { return b ? b->nb : 0; }

int rs_batch_info(const rs_batch *b, uint64_t *n_bitmaps, uint64_t *n_containers,
                  uint64_t *pool_bytes) {
  if (!b) { set_error("null batch"); return RS_EARG; }
  RS_TRY(fetch_host_meta(b));
  if (n_bitmaps) *n_bitmaps = b->nb;
  if (n_containers) *n_containers = b->nc;
  if (pool_bytes) *pool_bytes = b->pool_bytes;
  return RS_OK;
}

int rs_batch_cardinalities(const rs_batch *b, uint64_t *out) {
  if (!b) { set_error("null batch"); return RS_EARG; }
  RS_TRY(resolve_pending(b));
  return d2h(out, b->d_bm_card, b->nb * 8);
}

int rs_batch_cardinalities_device(const rs_batch *b, uint64_t *dout) {
  if (!b || !dout) { set_error("null batch/out"); return RS_EARG; }
  RS_TRY(materialize(b));
  if (b->nb) RS_CK(cudaMemcpyAsync(dout, b->d_bm_card, b->nb * 8, cudaMemcpyDeviceToDevice, g_stream));
  return RS_OK;
}

int rs_batch_container_counts(const rs_batch *b, uint64_t *out) {
  RS_TRY(fetch_host_meta(b));
  for (uint64_t i = 0; i < b->nb; i++) out[i] = b->h_bm_start[i + 1] - b->h_bm_start[i];
  return RS_OK;
}

}  // extern "C"
