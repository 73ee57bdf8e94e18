// rs_internal.cuh -- shared host/device definitions of the B200 Roaring library.
//
// Data layout in HBM: a batch of N bitmaps is a CSR over a flat
// container table (structure of arrays) plus one payload pool:
//   bm_start u64[N+1]   containers of bitmap i are [bm_start[i], bm_start[i+1])
//   key  u16[C]          chunk key (high 16 bits), strictly increasing per bitmap
//   type u8[C]           1 array / 2 bitset / 3 run (containers.py:31-33)
//   card u32[C]          cardinality (1..65536)
//   n    u32[C]          array: #values, run: #runs, bitset: 1024 (words)
//   off  u64[C]          byte offset of the payload in pool, 16-byte aligned
//   pool u8[P]           array: u16[n]; bitset: u64[1024]; run: u16 (start,len)[n]
// Payloads are 16-byte aligned so bitsets are read with 128-bit loads; pools
// produced by ops may hold holes (each result gets its upper-bound slot).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "../../include/roaring_b200.h"

#define RS_TAG_ARRAY 1
#define RS_TAG_BITSET 2
#define RS_TAG_RUN 3
#define RS_ARRAY_MAX 4096
#define RS_RUN_MAX_RUNS 2047
#define RS_WORDS 1024
#define RS_NONE 0xFFFFFFFFu

struct DevBatch {
  uint64_t nb, nc;
  const uint64_t *bm_start;
  const uint16_t *key;
  const uint8_t *type;
  const uint32_t *card;
  const uint32_t *n;
  const uint64_t *off;
  const uint8_t *pool;
  const uint64_t *bm_card;
};

// Deferred payload validation of an asynchronously ingested batch
// (rs_batch_from_wire_async): the device flags plus what the host needs to
// format the reference's DecodeError once they are read back.
struct rs_pending {
  int *d_any = nullptr;
  uint8_t *d_vcode = nullptr;
  uint32_t *d_vval = nullptr;
  std::vector<uint32_t> card;
  std::vector<uint64_t> src, offs;  // payload start in the staged bytes; image offsets
  void *slot = nullptr;              // staging slot until first use (materialize)
  uint64_t meta_bytes = 0;           // metadata section at the head of the slot
  bool failed = false;
  std::string msg;
  int64_t offset = -1, index = -1;
};

struct rs_batch {
  uint64_t nb = 0, nc = 0, cap_c = 0, pool_bytes = 0;
  uint64_t *d_bm_start = nullptr;
  uint16_t *d_key = nullptr;
  uint8_t *d_type = nullptr;
  uint32_t *d_card = nullptr;
  uint32_t *d_n = nullptr;
  uint64_t *d_off = nullptr;
  uint8_t *d_pool = nullptr;
  uint64_t *d_bm_card = nullptr;
  // host mirror of bm_start (fetched lazily for op results)
  std::vector<uint64_t> h_bm_start;
  bool h_valid = false;
  // container types that may be present (bit t = type t); lets the op
  // pipeline skip type-pair classes that cannot occur
  uint8_t type_mask = 0xFF;
  int single = -1;  // 1 = every bitmap holds exactly one container (cached)
  // pool laid out by per-result upper bounds (op / union results): it may
  // hold holes until repack_pool() packs it (at the first host query, or when
  // the live upper-bound reservations pass the high-water mark)
  bool ub_pool = false;
  rs_pending *pending = nullptr;  // payload checks not yet read back
  DevBatch dev() const {
    DevBatch d;
    d.nb = nb; d.nc = nc; d.bm_start = d_bm_start; d.key = d_key; d.type = d_type;
    d.card = d_card; d.n = d_n; d.off = d_off; d.pool = d_pool; d.bm_card = d_bm_card;
    return d;
  }
};

// ------------------------------------------------------------ host runtime
namespace rs {
extern cudaStream_t g_stream;
extern uint64_t g_launches;
void set_error(const std::string &m, int64_t off = -1, int64_t idx = -1);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);
void *dalloc(size_t bytes);   // stream-ordered (cudaMallocAsync); nullptr on failure
void dfree(void *p);
int ensure_device();
int batch_alloc(rs_batch *b, uint64_t nb, uint64_t nc, uint64_t pool_bytes);
void batch_release(rs_batch *b);
int fetch_host_meta(const rs_batch *b);   // fills h_bm_start (synchronizes); packs an upper-bound pool
int fetch_host_meta_nopack(const rs_batch *b);  // same, leaving the pool as it is (egress paths)
int finalize_batch(rs_batch *b);          // computes d_bm_card from containers
// Upper-bound result pools: register a fresh result (its reservation counts
// toward the high-water mark), pack one pool to its containers' bytes
// (synchronizes), and pack every registered pool when the reservations
// exceed the mark -- called before an op reserves a new result pool.
void ub_register(rs_batch *b);
void ub_unregister(rs_batch *b);
int repack_pool(rs_batch *b);
int ub_reserve(uint64_t bytes);
int resolve_pending(const rs_batch *b);    // reads deferred checks; RS_EDECODE on failure
int materialize(const rs_batch *b);        // queue a deferred batch's unpack/gather (first use)
void drop_staged(rs_batch *b);             // release an unused deferred batch's staging slot
template <typename T> int scan_exclusive(const T *in, T *out, uint64_t n);
template <typename T> int scan_inclusive(const T *in, T *out, uint64_t n);
// LSD radix sort of bits [begin_bit, end_bit) (stable: equal keys keep their order)
int sort_u64(uint64_t *keys, uint64_t n, int end_bit, int begin_bit = 0);
int d2h(void *h, const void *d, size_t bytes);   // synchronous on g_stream
// RS_TRACE=1: synchronize and print host wall time per phase (diagnostics only)
// cached cudaOccupancyMaxActiveBlocksPerMultiprocessor (+ the device's SM count)
int occupancy_per_sm(const void *kernel, int threads, size_t smem, int *sms_out);
// RS_HOST_TRACE=1: accumulated host nanoseconds between numbered points of
// the per-op host path, printed at exit (diagnostics only; no synchronization)
void host_mark(int point);
void trace(const char *phase);
// live per-kernel timing (bench roofline): events around tagged launches
extern bool g_prof_on;
void prof_mark(const char *name, cudaEvent_t a, cudaEvent_t b, uint64_t items);
cudaEvent_t prof_event();
int h2d(void *d, const void *h, size_t bytes);   // async on g_stream
int h2d_small(void *d, const void *h, size_t bytes);  // small upload (see rs_runtime.cu)
// Fork/join of independent launches onto side streams: begin(n) forks n
// streams off the library stream, next() points g_stream at the next one (no
// allocation may happen until end()), end() joins them back and restores it.
struct Fork {
  cudaStream_t saved = nullptr;
  int n = 0, used = 0;
  int begin(int nside);
  void next();
  int end();
  ~Fork() { end(); }  // an early error return still joins and restores the stream
};
}  // namespace rs

#define RS_CK(x)                                                                   \
  do {                                                                             \
    cudaError_t _e = (x);                                                          \
    if (_e != cudaSuccess) return rs::cuda_fail(_e, #x, __FILE__, __LINE__);       \
  } while (0)

#define RS_LAUNCH(kernel, grid, block, smem, ...)                                  \
  do {                                                                             \
    if ((grid) > 0) {                                                              \
      kernel<<<(grid), (block), (smem), rs::g_stream>>>(__VA_ARGS__);              \
      ++rs::g_launches;                                                            \
      RS_CK(cudaGetLastError());                                                   \
    }                                                                              \
  } while (0)

// Time one launch with events on the launch stream when profiling is on.
#define RS_LAUNCH_PROF(name, items, kernel, grid, block, smem, ...)                 \
  do {                                                                             \
    if ((grid) > 0) {                                                              \
      cudaEvent_t _pa = nullptr, _pb = nullptr;                                    \
      if (rs::g_prof_on) { _pa = rs::prof_event(); cudaEventRecord(_pa, rs::g_stream); } \
      kernel<<<(grid), (block), (smem), rs::g_stream>>>(__VA_ARGS__);              \
      ++rs::g_launches;                                                            \
      RS_CK(cudaGetLastError());                                                   \
      if (rs::g_prof_on) {                                                         \
        _pb = rs::prof_event();                                                    \
        cudaEventRecord(_pb, rs::g_stream);                                        \
        rs::prof_mark(name, _pa, _pb, (uint64_t)(items));                          \
      }                                                                            \
    }                                                                              \
  } while (0)

#define RS_TRY(x)                                                                  \
  do {                                                                             \
    int _rc = (x);                                                                 \
    if (_rc != RS_OK) return _rc;                                                  \
  } while (0)

// ------------------------------------------------------------ device helpers
__host__ __device__ inline uint64_t rs_pad16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// payload bytes of a container in the pool layout (not the wire layout)
__host__ __device__ inline uint32_t rs_payload_bytes(uint8_t type, uint32_t n) {
  return type == RS_TAG_ARRAY ? 2u * n : (type == RS_TAG_BITSET ? 8192u : 4u * n);
}

// _run_admissible, containers.py:202-205
__host__ __device__ inline bool rs_run_admissible(uint32_t card, uint32_t nruns) {
  return card > RS_ARRAY_MAX ? nruns <= RS_RUN_MAX_RUNS : 2u * nruns < card;
}

// _word_op, kernels/scalar.py:27-36
__device__ __forceinline__ uint64_t rs_word_op(int op, uint64_t x, uint64_t y) {
  return op == RS_OP_AND ? (x & y) : op == RS_OP_OR ? (x | y) : op == RS_OP_XOR ? (x ^ y) : (x & ~y);
}

// Does the result of container_pairwise(op, a, b) go through
// container_normalize(run ...) (run result possible)?  SURVEY App. A /
// containers.py:487-503: run x run (all ops), run x array (or, andnot, xor),
// array x run (or, xor).  Everything else picks array/bitset by cardinality.
__host__ __device__ inline bool rs_consider_run(uint8_t ta, uint8_t tb, int op) {
  if (ta == RS_TAG_RUN && tb == RS_TAG_RUN) return true;
  if (ta == RS_TAG_RUN && tb == RS_TAG_ARRAY) return op != RS_OP_AND;
  if (ta == RS_TAG_ARRAY && tb == RS_TAG_RUN) return op == RS_OP_OR || op == RS_OP_XOR;
  return false;
}

// Upper bound on the pool bytes of container_pairwise(op, a, b)'s result.
__host__ __device__ inline uint32_t rs_result_ub(uint8_t ta, uint32_t ca, uint8_t tb, uint32_t cb,
                                                  int op) {
  uint32_t ub = 8192;
  if (ta == RS_TAG_ARRAY && tb == RS_TAG_ARRAY) {
    if (op == RS_OP_AND) ub = 2u * (ca < cb ? ca : cb);
    else if (op == RS_OP_ANDNOT) ub = 2u * ca;
    else ub = 2u * (ca + cb) < 8192u ? 2u * (ca + cb) : 8192u;
  } else if (ta == RS_TAG_ARRAY && (op == RS_OP_AND || op == RS_OP_ANDNOT)) {
    ub = 2u * ca;  // array x {bitset,run}: and/andnot keep a subset of a
  } else if (tb == RS_TAG_ARRAY && op == RS_OP_AND) {
    ub = 2u * cb;  // {bitset,run} x array: and keeps a subset of b
  }
  return ub;
}
