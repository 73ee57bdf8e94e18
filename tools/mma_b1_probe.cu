// Probe: is mma.sync.m16n8k256 .b1 .and.popc correct and fast on sm_100a?
// Correctness: one warp computes a 16x8 tile over K=256*KT bits and compares
// with __popc.  Throughput: many warps issue back-to-back MMAs.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_b1(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// A: 16 rows x K bits (row-major, u32 words); B: 8 cols x K bits (col-major = 8 rows of K bits)
__global__ void k_tile(const uint32_t *A, const uint32_t *B, int KW, int *C) {
  int lane = threadIdx.x, g = lane >> 2, t4 = lane & 3;
  int d[4] = {0, 0, 0, 0};
  for (int kb = 0; kb < KW; kb += 8) {  // 8 u32 words = 256 bits per MMA
    uint32_t a[4] = {A[g * KW + kb + t4], A[(g + 8) * KW + kb + t4], A[g * KW + kb + 4 + t4],
                     A[(g + 8) * KW + kb + 4 + t4]};
    uint32_t b[2] = {B[g * KW + kb + t4], B[g * KW + kb + 4 + t4]};
    mma_b1(d, a, b);
  }
  C[g * 8 + 2 * t4] = d[0];
  C[g * 8 + 2 * t4 + 1] = d[1];
  C[(g + 8) * 8 + 2 * t4] = d[2];
  C[(g + 8) * 8 + 2 * t4 + 1] = d[3];
}

__global__ void k_rate(int iters, int *out) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
  int d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0}, d2[4] = {0, 0, 0, 0}, d3[4] = {0, 0, 0, 0};
  for (int i = 0; i < iters; i++) {
    mma_b1(d0, a, b);
    mma_b1(d1, a, b);
    mma_b1(d2, a, b);
    mma_b1(d3, a, b);
    a[0] ^= d0[0];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = d0[0] + d1[1] + d2[2] + d3[3];
}

int main() {
  const int KW = 64;  // 2048 bits
  uint32_t hA[16 * KW], hB[8 * KW];
  srand(7);
  for (auto &x : hA) x = (uint32_t)rand() * 2654435761u ^ rand();
  for (auto &x : hB) x = (uint32_t)rand() * 2246822519u ^ rand();
  uint32_t *dA, *dB;
  int *dC, hC[128];
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dC, sizeof hC);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  k_tile<<<1, 32>>>(dA, dB, KW, dC);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 16; i++)
    for (int j = 0; j < 8; j++) {
      int ref = 0;
      for (int k = 0; k < KW; k++) ref += __builtin_popcount(hA[i * KW + k] & hB[j * KW + k]);
      if (ref != hC[i * 8 + j]) bad++;
    }
  printf("correctness: %s (%d/128 mismatches) err=%s\n", bad ? "FAIL" : "ok", bad, cudaGetErrorString(e));
  int *dout;
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  cudaMalloc(&dout, blocks * threads * sizeof(int));
  k_rate<<<blocks, threads>>>(16, dout);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_rate<<<blocks, threads>>>(iters, dout);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double mmas = (double)blocks * (threads / 32) * iters * 4;
  double bitops = mmas * 16 * 8 * 256;  // AND+POPC-accumulate per bit
  printf("rate: %.3f ms, %.1f T mma/s, %.1f T bit-ops/s (= %.2f T 64-bit word-pairs/s)\n", ms, mmas / ms / 1e9,
         bitops / ms / 1e9, bitops / 64 / ms / 1e9);
  return 0;
}
