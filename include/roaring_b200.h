/*
 * roaring_b200.h -- C ABI of the B200-native Roaring set-operation library.
 *
 * The drop-in boundary for the reference's bitmap API
 * (/root/reference/pkg/src/roaringset).  Everything here is plain C: opaque
 * handles, pointers and sizes, no torch types.  A batch (rs_batch) is a
 * device-resident collection of Roaring bitmaps in a flattened layout
 * (DESIGN.md "Data layout in HBM"); every operation is batched over many
 * bitmap pairs and runs hand-written sm_100a kernels.  There is no CPU
 * fallback: on a machine without a usable CUDA device every compute entry
 * point fails with RS_ECUDA.
 *
 * Conventions (mirroring the reference):
 *   - ops are 0=and 1=or 2=andnot 3=xor, the order of kernels/_shared.py:8;
 *     anything else -> RS_EOP (the reference's ValueError "unknown op").
 *   - inputs are never mutated (bitmap.py:8-9,170) except by
 *     rs_batch_run_optimize, which mutates by contract (bitmap.py:308-316).
 *   - results are fresh batches owned by the caller (rs_batch_free).
 *   - return value: RS_OK (0) or an error code; rs_last_error() (thread-local)
 *     carries the message, rs_last_error_offset()/rs_last_error_index() the
 *     DecodeError byte offset and the failing image.
 *   - all work is queued on the library stream (rs_set_stream); entry points
 *     that return host data synchronize that stream.
 */
#ifndef ROARING_B200_H
#define ROARING_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rs_batch rs_batch;

enum {
  RS_OK = 0,
  RS_EOP = 1,      /* unknown op: ValueError (bitmap.py:171-172, containers.py:456-457) */
  RS_EDECODE = 2,  /* malformed wire image: DecodeError(offset) (serde.py:55-60) */
  RS_EVALUE = 3,   /* value outside 32 bits: ValueError (bitmap.py:49-50) */
  RS_EARG = 4,     /* bad argument (index out of range, size mismatch, ...) */
  RS_ECUDA = 5,    /* CUDA error or no device: the product never falls back to the CPU */
  RS_ENOMEM = 6,   /* device allocation failed */
  RS_ESHAPE = 7    /* container-level call on images that are not one container each */
};

enum { RS_OP_AND = 0, RS_OP_OR = 1, RS_OP_ANDNOT = 2, RS_OP_XOR = 3 };

/* ---- errors / runtime -------------------------------------------------- */
const char *rs_last_error(void);
int64_t rs_last_error_offset(void);
int64_t rs_last_error_index(void);
const char *rs_version(void);
/* Select the CUDA device (one process per GPU; call before any other entry point). */
int rs_set_device(int device);
/* Set the CUDA stream (cudaStream_t as void*) all calls of this process use; NULL = library default. */
int rs_set_stream(void *stream);
void *rs_get_stream(void);
int rs_synchronize(void);
/* Pinned host memory for zero-staging H2D/D2H (used by the e2e path). */
int rs_host_alloc(void **ptr, uint64_t bytes);
int rs_host_free(void *ptr);
/* Device timing helpers on the library stream (milliseconds). */
int rs_event_record(void **event);
int rs_event_elapsed(void *start, void *stop, float *ms);
int rs_event_destroy(void *event);
/* Number of this library's kernels launched since load (bench gpu_launches). */
uint64_t rs_kernel_launches(void);
/* Live per-kernel timing: with profiling on, the hot kernels are bracketed by
 * CUDA events on the launch stream; query sums them per kernel name
 * ("bitset_pair", "array_pair", "generic_pair", "copy", "bitset_count",
 * "array_count", "generic_count", "union_fold", "allpairs"). */
int rs_profile_enable(int on);
int rs_profile_reset(void);
int rs_profile_query(const char *name, double *total_ms, uint64_t *launches, uint64_t *items);

/* ---- ingest ------------------------------------------------------------- */
/* serde.deserialize (serde.py:87-169) for n wire images concatenated in
 * buf with offsets offs[0..n].  buf is a host pointer.  Structural checks run
 * on the host walk; payload checks (sortedness, popcount, run rules) run in a
 * device kernel.  The first failing image raises RS_EDECODE with the
 * reference's offset and message. */
int rs_batch_from_wire(const uint8_t *buf, const uint64_t *offs, uint64_t n, rs_batch **out);
/* Same result, asynchronous: the host walk runs now (structural errors are
 * raised here, through the synchronous path), the payload bytes are copied on
 * the library's copy stream and checked by a kernel queued on the library
 * stream, and the call returns without waiting.  buf must stay untouched
 * until rs_batch_wait (pinned memory makes the copy truly asynchronous).
 * Payload errors are reported by rs_batch_wait -- or by the first call that
 * returns values to the host -- with the same offset and message as the
 * synchronous path; results computed from a batch that then fails are
 * meaningless (but stay in bounds). */
int rs_batch_from_wire_async(const uint8_t *buf, const uint64_t *offs, uint64_t n, rs_batch **out);
/* Same result from images already in DEVICE memory (dbuf, doffs[0..n] both
 * device pointers, offsets relative to dbuf[0] at doffs[0]): the descriptor
 * walk runs on the device as well (a thread per image), so no host round
 * trip of the bytes; a malformed image is reported exactly as by
 * rs_batch_from_wire (the error path copies the images to the host). */
int rs_batch_from_wire_device(const uint8_t *dbuf, const uint64_t *doffs, uint64_t n, rs_batch **out);
/* Read back the deferred payload checks: RS_OK or RS_EDECODE (repeatable). */
int rs_batch_wait(const rs_batch *b);

/* RoaringBitmap.from_values (bitmap.py:40-62) for n bitmaps whose uint32
 * values are concatenated in vals with offsets offs[0..n] (any order,
 * duplicates allowed; sorted input takes the fast path).  `on_device` != 0
 * means vals/offs are device pointers. */
int rs_batch_from_u32(const uint32_t *vals, const uint64_t *offs, uint64_t n, int on_device,
                      rs_batch **out);

int rs_batch_free(rs_batch *b);
/* Algorithmic size of a batch: payload bytes in the SURVEY 8(d) accounting
 * (array 2*card, bitset 8192, run 2+4*runs), 8-byte descriptors, and the
 * container count per type (u64[4], index = tag). */
int rs_batch_stats(const rs_batch *b, uint64_t *payload_bytes, uint64_t *descriptor_bytes,
                   uint64_t *type_counts);
/* Number of bitmaps (host-side, never synchronizes). */
uint64_t rs_batch_len(const rs_batch *b);
/* Number of bitmaps, total containers, payload-pool bytes.  An op result's
 * pool, laid out by per-container upper bounds, is packed here first, so
 * pool_bytes is at most ~1.25x the containers' bytes. */
int rs_batch_info(const rs_batch *b, uint64_t *n_bitmaps, uint64_t *n_containers,
                  uint64_t *pool_bytes);
/* Per-bitmap cardinality (RoaringBitmap.__len__, bitmap.py:77-82) -> host u64[n]. */
int rs_batch_cardinalities(const rs_batch *b, uint64_t *out);
/* Same into DEVICE memory dout (u64[n]), stream-ordered, no synchronization. */
int rs_batch_cardinalities_device(const rs_batch *b, uint64_t *dout);
/* Per-bitmap container counts -> host u64[n]. */
int rs_batch_container_counts(const rs_batch *b, uint64_t *out);
/* Concatenate batches (bitmaps in order) into a new batch. */
int rs_batch_concat(const rs_batch *const *parts, uint64_t nparts, rs_batch **out);
/* Copy of bitmaps idx[0..n) (host indices) into a new batch (RoaringBitmap.copy). */
int rs_batch_select(const rs_batch *b, const uint64_t *idx, uint64_t n, rs_batch **out);

/* Multi-GPU key-range sharding: a copy of every bitmap
 * restricted to the chunk keys in [lo, hi) (0 <= lo <= hi <= 65536); and the
 * number of containers per chunk key over the whole batch (host u64[65536]),
 * to balance the ranges. */
int rs_batch_key_range(const rs_batch *b, uint32_t lo, uint32_t hi, rs_batch **out);
int rs_batch_key_histogram(const rs_batch *b, uint64_t *hist);

/* ---- egress ------------------------------------------------------------- */
/* serde.serialize (serde.py:69-84): wire size of every image -> host u64[n]. */
int rs_batch_wire_sizes(const rs_batch *b, uint64_t *sizes);
/* All images concatenated into host buf (capacity cap) with offs[0..n] out. */
int rs_batch_to_wire(const rs_batch *b, uint8_t *buf, uint64_t cap, uint64_t *offs);
/* Same images, asynchronously: the image sizes are read back (one
 * synchronization of the library stream: offs[0..n] are valid on return),
 * the images are assembled on the device and copied into buf on the
 * library's export stream, and the call returns; *done is a CUDA event
 * (rs_event_synchronize / rs_event_query / rs_event_destroy) that completes
 * when the bytes have landed.  buf should be page-locked (rs_host_alloc) for
 * the copy to overlap; the batch may be freed as soon as the call returns. */
int rs_batch_to_wire_async(const rs_batch *b, uint8_t *buf, uint64_t cap, uint64_t *offs, void **done);
int rs_event_synchronize(void *event);
/* RS_OK when the event has completed, 1 while it is pending. */
int rs_event_query(void *event);
/* RoaringBitmap.to_array (bitmap.py:136-144): all bitmaps' values into host
 * out (capacity cap values) with offs[0..n] out. */
int rs_batch_to_u32(const rs_batch *b, uint32_t *out, uint64_t cap, uint64_t *offs);
/* Content digest of every bitmap: a 64-bit hash of exactly what its wire
 * image holds (keys, container types, cardinalities, payloads), computed on
 * the device -- equal bitmaps (bitmap.py:87-91) have equal digests.  For
 * checking results at full size against another implementation without
 * moving them (the definition is in DESIGN.md section 5).  digests: host
 * u64[n] (synchronizes) or, with on_device != 0, device u64[n]. */
int rs_batch_digests(const rs_batch *b, uint64_t *digests, int on_device);
/* Bitmap-level equality (bitmap.py:87-91): eq[p] = A[ia[p]] == B[ib[p]], host u8 out. */
int rs_batch_equal(const rs_batch *A, const rs_batch *B, const uint32_t *ia, const uint32_t *ib,
                   uint64_t npairs, uint8_t *eq);
/* Membership (RoaringBitmap.__contains__, bitmap.py:99-104 ->
 * container_contains, containers.py:258-268), batched: hit[q] = values[q] in
 * bitmap ibm[q] (ibm NULL = bitmap 0 for every query).  Host arrays in/out;
 * one thread per query on the device. */
int rs_batch_contains(const rs_batch *b, const uint32_t *ibm, const uint32_t *values, uint64_t n,
                      uint8_t *hit);

/* ---- the hot path ------------------------------------------------------- */
/* RoaringBitmap.op (bitmap.py:169-210) for npairs pairs: out bitmap p =
 * A[ia[p]] op B[ib[p]].  ia/ib are host arrays of bitmap indices, or NULL for
 * the identity pairing (p, p).  Result container types follow
 * container_pairwise (containers.py:450-529) exactly; empty results are
 * dropped; unmatched containers are copied (OR/XOR both sides, ANDNOT A). */
int rs_pairwise(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia,
                const uint32_t *ib, uint64_t npairs, rs_batch **out);

/* RoaringBitmap.op_cardinality (bitmap.py:212-241): counts[p] =
 * |A[ia[p]] op B[ib[p]]|.  `counts` is a host u64[npairs] (synchronizes) or,
 * with counts_on_device != 0, a device u64[npairs] written asynchronously. */
int rs_pairwise_cardinality(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia,
                            const uint32_t *ib, uint64_t npairs, uint64_t *counts,
                            int counts_on_device);

/* container_pairwise (containers.py:450-529) over container pairs: both
 * batches hold one-container bitmaps; pair p combines the single containers
 * of A[ia[p]] and B[ib[p]] (keys ignored; the result takes A's key).  An
 * empty result becomes an empty bitmap.  RS_ESHAPE if an image has != 1
 * container. */
int rs_container_pairwise(int op, const rs_batch *A, const rs_batch *B, const uint32_t *ia,
                          const uint32_t *ib, uint64_t npairs, rs_batch **out);
/* container_pairwise_cardinality (containers.py:554-570), same pairing. */
int rs_container_pairwise_cardinality(int op, const rs_batch *A, const rs_batch *B,
                                      const uint32_t *ia, const uint32_t *ib, uint64_t npairs,
                                      uint64_t *counts, int counts_on_device);

/* RoaringBitmap.union_many (bitmap.py:257-304) over bitmaps idx[0..n) of `in`
 * in that order (idx NULL = all, in order) -> a batch holding one bitmap.
 * Container types replay the reference's sequential fold. */
int rs_union_many(const rs_batch *in, const uint64_t *idx, uint64_t n, rs_batch **out);

/* All unordered pairs i<j of `in` (row-major): inter[k] = |B_i ∩ B_j| and
 * uni[k] = |B_i ∪ B_j| (op_cardinality and/or, bitmap.py:212-241).  Host
 * u64[n(n-1)/2] each (uni may be NULL). */
int rs_all_pairs_cardinality(const rs_batch *in, uint64_t *inter, uint64_t *uni);

/* RoaringBitmap.run_optimize (bitmap.py:308-316) on every bitmap, in place;
 * changed[i] (host u8[n], may be NULL) = 1 if any container changed type. */
int rs_batch_run_optimize(rs_batch *b, uint8_t *changed);

#ifdef __cplusplus
}
#endif
#endif /* ROARING_B200_H */
