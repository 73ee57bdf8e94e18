// Probe: all-pairs |row_i AND row_j| of 128 bit-rows via tcgen05.mma kind::i8.
// Bits are expanded to u8 {0,1} in shared memory (canonical K-major, no
// swizzle: 8-row x 16-byte core matrices), the accumulator is s32 in TMEM,
// read back with tcgen05.ld.  Checks against a CPU popcount and times the
// full 65536-bit K.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#ifndef FP8
#define FP8 0
#endif
#ifndef MXF4
#define MXF4 0   // packed E2M1 (1.0 = 0x2 per nibble), kind::mxf4 with unit E8M0 block scales
#endif
constexpr int M = 128;          // rows (A) = cols (B): Gram tile
#ifndef KCH
#define KCH 256
#endif
#ifndef NST
#define NST 2
#endif
constexpr int KC = KCH;         // K elements (bits) per smem chunk
constexpr int NS = NST;         // smem stages
constexpr int CHUNK_BYTES = MXF4 ? M * KC / 2 : M * KC;   // u8 expanded: 32 KB (4-bit: 16 KB)
constexpr int NT = 256;         // threads: thread t expands half of row t & 127
constexpr int PF = 4;           // chunks of raw words prefetched in registers

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifndef SW128
#define SW128 1
#endif
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  if (SW128) d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// byte offset of (row, k) inside a chunk: SW128 K-major = [k/128 atom][row/8][row%8][128 B, 16-B units ^ row%8];
// no swizzle = [row/8][k/16][row%8][16 B]
__device__ __forceinline__ uint32_t koff(int row, int k) {
  if (SW128) return (k >> 7) * (M * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 127) >> 4) ^ (row & 7)) << 4);
  return (row >> 3) * (KC / 16) * 128 + (k >> 4) * 128 + (row & 7) * 16;
}

// kind::i8 instruction descriptor: D s32, A/B unsigned 8-bit, K-major, N, M
// (FP8: kind::f8f6f4, D f32, A/B E4M3)
__host__ __device__ constexpr uint32_t idesc_mxf4(int m, int n) {
  return (1u << 7) | (1u << 10)          // a/b format: MXF4 E2M1
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | (1u << 23)                    // scale format E8M0
         | ((uint32_t)(m >> 4) << 24);   // M >> 4 (sf ids 0, K64)
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return ((FP8 ? 1u : 2u) << 4)         // c_format S32 (F32 for FP8)
         | (0u << 7) | (0u << 10)       // a/b format: unsigned 8-bit
         | (0u << 15) | (0u << 16)      // K-major A and B
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(m >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nS_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra S_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ void mbar_sleep(uint64_t *bar, uint32_t phase) {
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    if (ok) break;
    __nanosleep(64);
  }
}

// expand 4 bits n -> 4 bytes {0,1} (FP8: {0, 0x38 = E4M3 1.0})
__device__ __forceinline__ uint32_t spread4(uint32_t n) {
  const uint32_t b = ((n & 0xF) * 0x00204081u) & 0x01010101u;
  return FP8 ? b * 0x38u : b;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialized: warps 0-7 expand (producers), warp 8 lane 0 issues MMAs.
// full[s]: 8 producer-warp arrivals; empty[s]: tcgen05.commit of the MMAs.
__global__ void __launch_bounds__(NT + 32, 1) k_gram(const uint64_t *__restrict__ rows, int kwords, uint32_t *out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *full = (uint64_t *)(sm + NS * CHUNK_BYTES);
  uint64_t *empty = full + NS;
  uint64_t *done = empty + NS;
  uint32_t *tslot = (uint32_t *)(done + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int i = 0; i < NS; i++) { mbar_init(&full[i], NT / 32); mbar_init(&empty[i], 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(MXF4 ? 512 : 128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
#if MXF4
  if (warp < 4) {  // unit E8M0 scales (0x7F = 2^0) in columns 256..287 of every lane
    const uint32_t one = 0x7F7F7F7Fu;
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((uint32_t)(32 * warp) << 16) + 256 + c), "r"(one)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#endif
  const int nchunks = kwords * 64 / KC;
  if (warp == NT / 32) {  // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = MXF4 ? idesc_mxf4(M, M) : idesc_i8(M, M);
      for (int c = 0; c < nchunks; c++) {
        const int b = c % NS;
        if (mode & 16) mbar_spin(&full[b], (c / NS) & 1);
        else if (!(mode & 32)) mbar_wait(&full[b], (c / NS) & 1);
        if (!(mode & 64)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = smem_u32(sm + b * CHUNK_BYTES);
#pragma unroll
        for (int s = 0; s < ((mode & 2) ? 1 : (MXF4 ? KC / 64 : KC / 32)); s++) {
          const uint64_t da = SW128 ? sdesc(base + (s >> 2) * (M * 128) + (s & 3) * 32, 16, 1024)
                                    : sdesc(base + s * 256, 128, (KC / 16) * 128);
          const uint32_t acc = (c | s) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
#if MXF4
              "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
              ::"r"(tmem), "l"(da), "l"(da), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 272)
              : "memory");
#else
#if FP8
              "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
#else
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
#endif
              "l"(da), "l"(da), "r"(idesc), "r"(acc)
              : "memory");
#endif
        }
        if (!(mode & 32))
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[b]))
                       : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(done))
                   : "memory");
    }
  } else {  // ---------------- expansion producers
    const int row = t & (M - 1), half = t >> 7;
    const uint64_t *src = rows + (size_t)row * kwords + half * (KC / 128);
    uint64_t x[PF][KC / 128];
#pragma unroll
    for (int p = 0; p < PF; p++)
#pragma unroll
      for (int w = 0; w < KC / 128; w++) x[p][w] = p < nchunks ? src[p * (KC / 64) + w] : 0;
    for (int c0 = 0; c0 < nchunks; c0 += PF) {
#pragma unroll
      for (int p = 0; p < PF; p++) {
        const int c = c0 + p;
        if (c >= nchunks) break;
        const int b = c % NS;
        uint8_t *bufb = sm + b * CHUNK_BYTES;
        if (c >= NS) {
          if (mode & 32) {}
          else if (mode & 128) mbar_sleep(&empty[b], ((c - NS) / NS) & 1);
          else if (mode & 16) mbar_spin(&empty[b], ((c - NS) / NS) & 1);
          else if (mode & 4) { if (lane == 0) mbar_wait(&empty[b], ((c - NS) / NS) & 1); __syncwarp(); }
          else mbar_wait(&empty[b], ((c - NS) / NS) & 1);
        }
        if (!(mode & 1)) {
          const int k0 = half * (KC / 2);
#pragma unroll
          for (int w = 0; w < KC / 128; w++) {
            const uint64_t xv = x[p][w];
#if MXF4
            // 32 bits -> 32 nibbles (16 bytes); K order within the 8 bits is
            // permuted (0,4,1,5,..), identically for every row
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const uint32_t s = (uint32_t)(xv >> (32 * h));
              uint4 v;
              v.x = (spread4(s) << 1) | (spread4(s >> 4) << 5);
              v.y = (spread4(s >> 8) << 1) | (spread4(s >> 12) << 5);
              v.z = (spread4(s >> 16) << 1) | (spread4(s >> 20) << 5);
              v.w = (spread4(s >> 24) << 1) | (spread4(s >> 28) << 5);
              *(uint4 *)(bufb + koff(row, (k0 + w * 64 + h * 32) / 2)) = v;  // koff takes a byte index
            }
#else
#pragma unroll
            for (int h = 0; h < 4; h++) {
              const uint32_t s = (uint32_t)(xv >> (16 * h));
              uint4 v = make_uint4(spread4(s), spread4(s >> 4), spread4(s >> 8), spread4(s >> 12));
              *(uint4 *)(bufb + koff(row, k0 + w * 64 + h * 16)) = v;
            }
#endif
            x[p][w] = c + PF < nchunks ? src[(c + PF) * (KC / 64) + w] : 0;
          }
        }
        if (!(mode & 8)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[b]);
      }
    }
  }
  if (mode & 128) mbar_sleep(done, 0);
  else mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4)
    for (int c0 = 0; c0 < M; c0 += 32) {
      uint32_t v[32];
      const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; j++) out[t * M + c0 + j] = (FP8 || MXF4) ? (uint32_t)__uint_as_float(v[j]) : v[j];
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(MXF4 ? 512 : 128) : "memory");
}

int main(int argc, char **argv) {
  const int kwords = argc > 1 ? atoi(argv[1]) : 16;  // 64-bit words per row
  std::vector<uint64_t> h((size_t)M * kwords);
  uint64_t s = 12345;
  for (auto &x : h) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t a = s;
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    x = a ^ (s >> 17) ^ (a & s);  // density ~ 1/2 .. mixed
  }
  uint64_t *d;
  uint32_t *dout;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&dout, M * M * 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = NS * CHUNK_BYTES + 256;
  cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_gram<<<1, NT + 32, smem>>>(d, kwords, dout, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  std::vector<uint32_t> o(M * M);
  cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M; i++)
    for (int j = 0; j < M; j++) {
      uint32_t ref = 0;
      for (int w = 0; w < kwords; w++) ref += __builtin_popcountll(h[(size_t)i * kwords + w] & h[(size_t)j * kwords + w]);
      if (ref != o[i * M + j]) {
        if (bad < 5) printf("mismatch (%d,%d): got %u want %u\n", i, j, o[i * M + j], ref);
        bad++;
      }
    }
  printf("correctness: %s (%d mismatches of %d)\n", bad ? "FAIL" : "ok", bad, M * M);
  // timing: 148 CTAs x full 65536-bit rows
  if (kwords >= 64) {
    const int modes[] = {0, 128, 3, 3 | 128, 1, 1 | 128, 3 | 32 | 128, 1 | 32 | 128};
    for (int mode : modes) {
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      k_gram<<<148, NT + 32, smem>>>(d, kwords, dout, mode);
      cudaEventRecord(a);
      for (int r = 0; r < 10; r++) k_gram<<<148, NT + 32, smem>>>(d, kwords, dout, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double macs = 148.0 * M * M * 64.0 * kwords;
      printf("mode %2d (1 noexp 2 one-mma 16 spin 32 nosync) 148 CTAs x 128x128x65536: %.3f ms/launch, %.1f T MAC/s, %.0f clk/chunk\n", mode, ms / 10,
             macs / (ms / 10 * 1e-3) / 1e12, ms / 10 * 1e-3 * 1.965e9 / (kwords * 64 / KC));
    }
  }
  return bad != 0;
}
