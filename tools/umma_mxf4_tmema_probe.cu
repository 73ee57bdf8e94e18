// Probe: tcgen05.mma kind::mxf4 with the A operand in TMEM (written by
// tcgen05.st from registers) and B in shared memory (K-major SWIZZLE_128B):
// 128 x 128 Gram tile of 128 random 256-bit rows (one K chunk, 4 MMAs),
// checked against a CPU popcount.  Establishes the TMEM column order of A:
// column j holds the same 32-bit word as bytes 4j..4j+3 of the B atom row.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t sw_off(int row, int k, int rows) {
  return (k >> 7) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((((k & 127) >> 4) ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint4 nib32(uint32_t x) {
  constexpr uint32_t M2 = 0x22222222u;
  return make_uint4((x << 1) & M2, x & M2, (x >> 1) & M2, (x >> 2) & M2);
}

__global__ void __launch_bounds__(128, 1) k(const uint32_t *rows, float *out, int mode) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // expand row t: 8 raw words -> 32 expanded words
  uint32_t e[32];
  for (int u = 0; u < 8; u++) {
    const uint4 v = nib32(rows[t * 8 + u]);
    e[4 * u] = v.x; e[4 * u + 1] = v.y; e[4 * u + 2] = v.z; e[4 * u + 3] = v.w;
    *(uint4 *)(sm + sw_off(t, 16 * u, 128)) = v;
  }
  // A: columns 288..319 of lane t
  const uint32_t acol = 288;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + ((uint32_t)(32 * warp) << 16) + acol),
      "r"(e[0]), "r"(e[1]), "r"(e[2]), "r"(e[3]), "r"(e[4]), "r"(e[5]), "r"(e[6]), "r"(e[7]), "r"(e[8]), "r"(e[9]),
      "r"(e[10]), "r"(e[11]), "r"(e[12]), "r"(e[13]), "r"(e[14]), "r"(e[15]), "r"(e[16]), "r"(e[17]), "r"(e[18]),
      "r"(e[19]), "r"(e[20]), "r"(e[21]), "r"(e[22]), "r"(e[23]), "r"(e[24]), "r"(e[25]), "r"(e[26]), "r"(e[27]),
      "r"(e[28]), "r"(e[29]), "r"(e[30]), "r"(e[31])
      : "memory");
  {  // unit scales at 256..287
    const uint32_t one = 0x7F7F7F7Fu;
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((uint32_t)(32 * warp) << 16) + 256 + c), "r"(one) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | (1u << 23) | (8u << 24);
    for (int kk = 0; kk < 4; kk++) {
      const uint64_t db = sw128_desc(su32(sm) + 32 * kk);
      const uint32_t acc = kk ? 1u : 0u;
      if (mode == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n}\n"
                     ::"r"(tmem), "r"(tmem + acol + 8 * kk), "l"(db), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 272)
                     : "memory");
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                     ::"r"(tmem), "l"(db), "l"(db), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 272)
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < 128; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; j++) out[t * 128 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
  std::vector<uint32_t> h(128 * 8);
  uint64_t s = 99;
  for (auto &x : h) { s = s * 6364136223846793005ull + 1442695040888963407ull; x = (uint32_t)(s >> 29); }
  uint32_t *d; float *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 128 * 128 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  for (int mode = 0; mode < 2; mode++) {
    k<<<1, 128, 32 * 1024>>>(d, o, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> r(128 * 128);
    cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128; i++)
      for (int j = 0; j < 128; j++) {
        int ref = 0;
        for (int u = 0; u < 8; u++) ref += __builtin_popcount(h[i * 8 + u] & h[j * 8 + u]);
        if ((int)r[i * 128 + j] != ref) { if (bad < 3) printf("  (%d,%d) got %g want %d\n", i, j, r[i * 128 + j], ref); bad++; }
      }
    printf("mode %d (%s): %s, %d mismatches\n", mode, mode ? "A smem" : "A tmem", cudaGetErrorString(e), bad);
  }
  return 0;
}
