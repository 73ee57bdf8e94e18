// rs_umma.cuh -- all-pairs |A AND B| of one chunk key's containers on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Config 5 asks for op_cardinality("and") over every bitmap pair
// (bitmap.py:212-241 -> container_pairwise_cardinality, containers.py:532-570).
// Grouped by chunk key, the containers of one key form m bit-rows of 65,536
// bits (densified to 8 KB), and all their pairwise intersection counts are the
// Gram matrix G = X X^T over {0,1}: a GEMM.  On CUDA cores this is bound by
// the POPC issue rate (16/clk/SM); the tensor cores multiply 0/1 bytes.  Each
// CTA owns one tile: A = 128 rows starting at r0, B = NB <= 256 rows starting
// at c0, both of one key.  When r0 == c0 the A rows are the first 128 rows of
// the B operand -- one expansion feeds both descriptors -- so a key with
// m <= 256 containers is one tile (pairs u < v with u < 128) plus, past 128,
// a small corner left to the CUDA-core tiles.
//   * warps 0-7 (producers) stream 256-bit K chunks of the rows from HBM (4
//     chunks prefetched in registers), expand bits to bytes {0,1} in shared
//     memory in the canonical K-major SWIZZLE_128B layout, and arrive on the
//     stage's `full` mbarrier;
//   * warp 8 lane 0 issues 8 x tcgen05.mma (M=128, N=NB, K=32) per chunk into
//     an s32 accumulator in TMEM and frees the stage with tcgen05.commit ->
//     `empty`;
//   * after the last chunk every warp reads a quarter of the accumulator rows
//     (TMEM lanes 32(w%4)..) and half of the columns back with tcgen05.ld and
//     adds the upper-triangle counts into the N x N matrix.
// Counts are exact: at most 65,536 per pair, accumulated in s32.
#pragma once
#include "rs_internal.cuh"

namespace rsu {

constexpr int UM = 128;                 // tile rows (A operand, TMEM lanes)
constexpr int UNMAX = 256;              // tile columns (B operand rows), at most
constexpr int UKC = 256;                // K bits per smem chunk
constexpr int UACH = UM * UKC;          // expanded separate-A bytes per chunk (32 KB)
constexpr int URING = 192 * 1024;       // stage ring: as many stages as fit (<= UMAXST)
constexpr int UMAXST = 6;
constexpr int UPF = 4;                  // raw chunks prefetched in registers
constexpr int UPROD = 256;              // producer threads
constexpr int UTHREADS = UPROD + 32;    // + the MMA-issuer warp
constexpr size_t USMEM = (size_t)URING + 256;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B (8-row x 128-byte
// atoms, 1024 B apart along M/N), Blackwell descriptor version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;                 // descriptor version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: D s32, A and B unsigned 8-bit, K-major.
__host__ __device__ constexpr uint32_t idesc_u8(int m, int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// Byte offset of (row, k) in one operand chunk of `rows` rows:
// [k/128 atom][row/8][row%8][128 B], the 16-byte units of each 128-byte row
// XOR-swizzled by row%8.
__device__ __forceinline__ uint32_t sw_off(int row, int k, int rows) {
  return (k >> 7) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 127) >> 4) ^ (row & 7)) << 4);
}

// 4 bits -> 4 bytes {0,1} (the four shifted copies never overlap)
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return ((n & 0xF) * 0x00204081u) & 0x01010101u; }

__device__ __forceinline__ void ubar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void ubar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nUW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra UW_%=;\n}\n" ::"r"(su32(bar)), "r"(phase)
      : "memory");
}
__device__ __forceinline__ void ubar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

// Expand NW consecutive words (bits k0 ..) of one row into `dst`.
template <int NW>
__device__ __forceinline__ void expand_words(uint8_t *dst, int row, int rows, int k0, const uint64_t *x) {
#pragma unroll
  for (int w = 0; w < NW; w++) {
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const uint32_t s = (uint32_t)(x[w] >> (16 * h));
      *(uint4 *)(dst + sw_off(row, k0 + w * 64 + h * 16, rows)) =
          make_uint4(spread4(s), spread4(s >> 4), spread4(s >> 8), spread4(s >> 12));
    }
  }
}

}  // namespace rsu
