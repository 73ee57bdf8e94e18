// rs_umma.cuh -- all-pairs |A AND B| of one chunk key's containers on the
// 5th-generation tensor cores (tcgen05.mma kind::mxf4, accumulators in TMEM).
//
// Config 5 asks for op_cardinality("and") over every bitmap pair
// (bitmap.py:212-241 -> container_pairwise_cardinality, containers.py:532-570).
// Grouped by chunk key, the containers of one key form m bit-rows of 65,536
// bits (densified to 8 KB), and all their pairwise intersection counts are the
// Gram matrix G = X X^T over {0,1}: a GEMM.  On CUDA cores this is bound by
// the POPC issue rate (16/clk/SM); the tensor cores multiply 0/1 values
// packed as 4-bit E2M1 (bit -> nibble 0x2 = 1.0) with unit E8M0 block scales,
// K = 64 per instruction -- twice the K of kind::i8 at the same issue rate
// (N/2 cycles per 128 x N MMA, tools/umma_rate_probe.cu), and half the
// expanded shared-memory bytes.  Products and sums of 0/1 are exact in the f32
// accumulator (counts <= 65,536 < 2^24).  Each
// CTA owns one tile: A = 128 rows starting at r0, B = NB <= 256 rows starting
// at c0, both of one key.  When r0 == c0 the A rows are the first 128 rows of
// the B operand -- one expansion feeds both descriptors -- so a key with
// m <= 256 containers is one tile (pairs u < v with u < 128) plus, past 128,
// a small corner left to the CUDA-core tiles.
//   * warp 9 lane 0 streams the raw rows with 2D tensor TMA (box: 128 rows x
//     128 bytes = four 256-bit K chunks, SWIZZLE_128B) into a raw ring;
//   * warps 0-7 (producers) each expand whole chunks (warp c % 8 takes chunk
//     c, so eight chunks are in flight): per row, the 32 raw bytes (two
//     conflict-free 128-bit loads) become one 128-byte K-major SWIZZLE_128B
//     atom row of nibbles (nib32: 7 integer ops per 32 bits), then the warp
//     arrives on the stage's `full` mbarrier;
//   * warp 8 lane 0 issues 4 x tcgen05.mma (M=128, N=NB, K=64) per chunk into
//     an f32 accumulator in TMEM and frees the stage with tcgen05.commit ->
//     `empty`; the block scales are 0x7F bytes filled once into TMEM columns
//     256..287 (every scale-factor layout then reads 1.0);
//   * after the last chunk every warp reads a quarter of the accumulator rows
//     (TMEM lanes 32(w%4)..) and half of the columns back with tcgen05.ld and
//     adds the upper-triangle counts into the N x N matrix.
// Counts are exact: at most 65,536 per pair.  Within each 32-bit word the K
// order is permuted (see nib32), identically for every row, which a dot
// product does not see.
#pragma once
#include "rs_internal.cuh"

namespace rsu {

constexpr int UM = 128;                 // tile rows (A operand, TMEM lanes)
constexpr int UNMAX = 256;              // tile columns (B operand rows), at most
constexpr int UKC = 256;                // K bits per smem chunk
constexpr int UROWB = UKC / 2;          // expanded bytes per row and chunk (one 128-byte atom row)
constexpr int UTMEM = 512;              // TMEM columns: accumulator (<= 256), A stages, block scales
constexpr int UACOL = 256;              // A operand stages: 32 columns (one 256-bit K chunk of 128 rows) each
constexpr int USCOL = 480;              // unit block scales (SFA at 480, SFB at 496)
constexpr int URING = 192 * 1024;       // expanded stages, then as many raw stages as fit
constexpr int UNST = 4;                 // expanded stages = producer groups = TMEM A stages (256..383)
constexpr int URAWMAX = 8;              // raw TMA stages in flight (barrier slots)
constexpr int UBOXR = 32;               // raw TMA box: rows
constexpr int UBOXB = 128;              // raw TMA box: bytes of K (4 chunks)
constexpr int UBOX = UBOXR * UBOXB;     // 4 KB
constexpr int UPROD = 512;              // producer threads: UNST groups of four warps
constexpr int UTHREADS = UPROD + 64;    // + the MMA-issuer warp + the TMA warp
constexpr size_t USMEM = (size_t)URING + 2048;  // + alignment slack and the barriers

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

// Instruction descriptor, kind::mxf4 block-scaled: A and B E2M1 (MXF4 format
// 1), E8M0 scales, K-major, dense K = 64, scale-factor ids 0; D is f32.
__host__ __device__ constexpr uint32_t idesc_mxf4(int m, int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((uint32_t)(m >> 4) << 24);
}

// Byte offset of (row, k) in one operand chunk of `rows` rows:
// [k/128 atom][row/8][row%8][128 B], the 16-byte units of each 128-byte row
// XOR-swizzled by row%8.
__device__ __forceinline__ uint32_t sw_off(int row, int k, int rows) {
  return (k >> 7) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 127) >> 4) ^ (row & 7)) << 4);
}

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

// 32 bits -> 32 nibbles {0, 0x2 = E2M1 1.0} in one 16-byte unit: nibble j of
// word i holds bit 4j + i (a fixed K permutation within the word).
__device__ __forceinline__ uint4 nib32(uint32_t x) {
  constexpr uint32_t M2 = 0x22222222u;
  return make_uint4((x << 1) & M2, x & M2, (x >> 1) & M2, (x >> 2) & M2);
}

// one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(p));
  return p != 0;
}

// D[tmem] (+)= A[ta] x B[db] (kind::mxf4, unit block scales at sfa / sfb)
__device__ __forceinline__ void umma_mxf4(uint32_t tmem, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t sfa,
                                          uint32_t sfb, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem),
      "r"(ta), "l"(db), "r"(idesc), "r"((uint32_t)acc), "r"(sfa), "r"(sfb)
      : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes (lane = thread) <- e
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&e)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(e[0]), "r"(e[1]), "r"(e[2]), "r"(e[3]), "r"(e[4]), "r"(e[5]), "r"(e[6]), "r"(e[7]), "r"(e[8]), "r"(e[9]),
      "r"(e[10]), "r"(e[11]), "r"(e[12]), "r"(e[13]), "r"(e[14]), "r"(e[15]), "r"(e[16]), "r"(e[17]), "r"(e[18]),
      "r"(e[19]), "r"(e[20]), "r"(e[21]), "r"(e[22]), "r"(e[23]), "r"(e[24]), "r"(e[25]), "r"(e[26]), "r"(e[27]),
      "r"(e[28]), "r"(e[29]), "r"(e[30]), "r"(e[31])
      : "memory");
}

// Expand one row's 256-bit chunk (two 16-byte raw units) into its 128-byte
// atom row of an operand chunk of `rows` rows.
__device__ __forceinline__ void expand_row(uint8_t *dst, int row, int rows, uint4 lo, uint4 hi) {
  const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int u = 0; u < 8; u++) *(uint4 *)(dst + sw_off(row, 16 * u, rows)) = nib32(w[u]);
}

}  // namespace rsu
