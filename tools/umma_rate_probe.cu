// Probe: raw tcgen05.mma issue rate by kind and N (no operand traffic): one
// CTA per SM, one thread issues R MMAs on a fixed zeroed shared-memory tile,
// then commits and waits.  Prints SM cycles per MMA and MACs/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  if constexpr (KIND == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
  else if constexpr (KIND == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
  else if constexpr (KIND == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 272) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_rate(int n, int reps, unsigned long long *cyc, int commit_every, uint32_t fill) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 64 * 1024 / 16; i += 128) ((uint4 *)sm)[i] = make_uint4(fill, fill * 3u, fill ^ (i * 0x9E3779B9u), fill);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  {
    const uint32_t one = 0x7F7F7F7Fu;
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                       tmem + ((uint32_t)(32 * warp) << 16) + 256 + c), "r"(one) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    uint32_t idesc;
    if (KIND == 0) idesc = (2u << 4) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    else if (KIND == 1) idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    else if (KIND == 2) idesc = (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | (8u << 24);
    else idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);  // bf16 -> f32
    const uint64_t da = sdesc(smem_u32(sm)), db = sdesc(smem_u32(sm + 32768));
    const unsigned long long c0 = clock64();
    for (int r = 0; r < reps; r++) {
#pragma unroll
      for (int s = 0; s < 4; s++) mma<KIND>(tmem, da + 2 * s, db + 2 * s, idesc, (r | s) ? 1u : 0u);
      if (commit_every && (r % commit_every) == commit_every - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
    const unsigned long long c1 = clock64();
    if (blockIdx.x == 0) *cyc = c1 - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int KIND>
void run(const char *name, int kper, int ce = 0, uint32_t fill = 0) {
  unsigned long long *d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_rate<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int n : {128, 256}) {
    const int reps = 2000;
    k_rate<KIND><<<148, 128, 64 * 1024>>>(n, reps, d, ce, fill);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / (reps * 4.0);
    printf("%-8s fill=%08x commit/%d N=%3d: %s  %.1f clk/MMA  %.0f MAC/clk/SM (M=128, K=%d)\n", name, fill, ce, n, cudaGetErrorString(e), per,
           128.0 * n * kper / per, kper);
  }
  cudaFree(d);
}

int main() {
  run<2>("mxf4", 64, 0);
  run<2>("mxf4", 64, 1);
  run<2>("mxf4", 64, 4);
  run<2>("mxf4", 64, 64);
  run<2>("mxf4", 64, 1999);
  return 0;
}
