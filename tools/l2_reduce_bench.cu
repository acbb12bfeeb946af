// Microbenchmark: L2 fp32 reduction bandwidth on B200, the resource a
// single-pass attention backward with a dQ reduce-add would lean on.
// Each CTA repeatedly adds a 32 KB tile into a 4 MB (L2-resident) fp32
// accumulator, either with red.global.add.v4.f32 from registers or with a
// 1-D TMA bulk reduce (cp.reduce.async.bulk ... add.f32) from shared memory.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void red_v4(float* acc, int tiles, int iters) {
  const int tid = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const int tile = (blockIdx.x * 7 + it * 13) % tiles;
    float* base = acc + (size_t)tile * 8192;   // 32 KB tile
    for (int i = tid * 4; i < 8192; i += blockDim.x * 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(base + i), "f"(1.f),
                   "f"(1.f), "f"(1.f), "f"(1.f)
                   : "memory");
  }
}

__global__ void bulk_reduce(float* acc, int tiles, int iters) {
  extern __shared__ __align__(128) float sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    for (int it = 0; it < iters; ++it) {
      const int tile = (blockIdx.x * 7 + it * 13) % tiles;
      float* base = acc + (size_t)tile * 8192;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::
                       "l"(base), "r"(s), "r"(32768)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int tiles = 128;             // 4 MB accumulator
  float* acc;
  cudaMalloc(&acc, (size_t)tiles * 8192 * 4);
  cudaMemset(acc, 0, (size_t)tiles * 8192 * 4);
  cudaFuncSetAttribute(bulk_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148, 296, 592}) {
    const int iters = 200;
    for (int mode = 0; mode < 2; ++mode) {
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(a);
        if (mode == 0) red_v4<<<grid, 256>>>(acc, tiles, iters);
        else bulk_reduce<<<grid, 128, 32768>>>(acc, tiles, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)grid * iters * 32768;
      printf("{\"mode\": \"%s\", \"grid\": %d, \"ms\": %.3f, \"TBps\": %.2f}\n",
             mode ? "bulk_reduce" : "red_v4", grid, ms, bytes / ms / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
