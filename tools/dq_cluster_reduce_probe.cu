// Probe: can a KV-parallel single-pass backward afford its dQ reduction if
// a thread-block cluster pre-reduces the dQ partials in distributed shared
// memory (DSMEM) before one TMA bulk reduce-add per cluster goes to L2?
// (VERDICT r01 "next" 3; DESIGN.md §4 "The single-pass backward, measured".)
//
// Model of one fused dK/dV/dQ step per CTA: a 128 x 128 fp32 dQ partial
// (64 KB, here already in shared memory - the real kernel would first drain it
// from TMEM) must be summed over the C CTAs of the cluster, which own
// consecutive 128-row KV tiles of the same head group and walk the query
// steps in the same order.  Per step:
//   1. cluster barrier (every partial of this step is in place)
//   2. CTA r sums slice r (64 KB / C) of all C partials over DSMEM
//      (ld.shared::cluster.v4.f32) into a local staging slice
//   3. one cp.reduce.async.bulk .add.f32 of the slice into the global dQ
//      tile of this step (L2), 1/C of the 64 KB per CTA
//   4. cluster barrier (partials may be overwritten by the next step)
// The global dQ working set is 16 query steps x 8 head groups x 64 KB (8 MB,
// L2-resident), clusters of one head group hit the same tile in the same
// step as the real kernel would (stagger 0) or spread over the steps.
//
// Output (JSON lines): clocks per step per CTA, DSMEM bytes per clock per SM,
// and the L2 reduce bytes per step, for C = 1 (no DSMEM: every CTA reduces
// its whole 64 KB into L2) and C = 2, 4, 8, 16.  A fused step has ~2560 clk
// of tensor work (five 128x128x128 MMAs at 8192 FLOP/clk/SM); the reduction
// must fit beside it on otherwise idle warps.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace cg = cooperative_groups;

constexpr int kTileFloats = 128 * 128;       // 64 KB
constexpr int kThreads = 256;
constexpr int kQSteps = 16;
constexpr int kGroups = 8;

__device__ __forceinline__ float4 ld_dsmem_v4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

template <int C>
__global__ void __launch_bounds__(kThreads, 1)
probe(float* __restrict__ dq, int steps, int stagger, long long* __restrict__ clk_out) {
  extern __shared__ __align__(1024) float sm[];
  float* part = sm;                    // this CTA's 64 KB partial
  float* stage = sm + kTileFloats;     // reduced slice (64 KB / C)
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t rank = C > 1 ? cluster.block_rank() : 0;
  const int cl = blockIdx.x / C;
  const int group = cl % kGroups;
  for (int i = threadIdx.x; i < kTileFloats; i += kThreads) part[i] = 1.f + (i & 7);
  constexpr int kSlice = kTileFloats / C;        // floats per CTA slice
  const uint32_t part_u = (uint32_t)__cvta_generic_to_shared(part);
  const uint32_t stage_u = (uint32_t)__cvta_generic_to_shared(stage);
  __syncthreads();
  if (C > 1) cluster.sync();
  const long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int qs = (s + stagger * cl) % kQSteps;
    float* gdst = dq + ((size_t)group * kQSteps + qs) * kTileFloats + (size_t)rank * kSlice;
    if (C == 1) {
      // no cluster: the whole partial goes to L2
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                gdst),
            "r"(part_u), "r"(kTileFloats * 4)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();
      continue;
    }
    // 2. sum slice `rank` of every CTA's partial (DSMEM), rotating the source
    //    order so the C CTAs do not all read the same peer at once
    for (int i = threadIdx.x * 4; i < kSlice; i += kThreads * 4) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const uint32_t src = (rank + j) % C;
        const float4 v = ld_dsmem_v4(mapa(part_u + (rank * kSlice + i) * 4, src));
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      *reinterpret_cast<float4*>(stage + i) = acc;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // 3. one bulk reduce-add of the slice into L2
    if (threadIdx.x == 0) {
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
          "r"(stage_u), "r"(kSlice * 4)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    // 4. nobody overwrites a partial or the staging slice before all reads
    cluster.sync();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk_out[blockIdx.x] = t1 - t0;
}

template <int C>
void run(float* dq, long long* clk, int sms, int stagger) {
  const int ctas = (sms / C) * C;
  const size_t smem = (size_t)kTileFloats * 4 + (size_t)kTileFloats * 4 / C;
  cudaFuncSetAttribute(probe<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(probe<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int steps = 400;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe<C>, dq, steps, stagger, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("{\"cluster\": %d, \"error\": \"%s\"}\n", C, cudaGetErrorString(e));
      return;
    }
    cudaEventElapsedTime(&ms, a, b);
  }
  static long long h[1024];
  cudaMemcpy(h, clk, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double mean = 0, mx = 0;
  for (int i = 0; i < ctas; ++i) {
    mean += (double)h[i];
    mx = h[i] > mx ? (double)h[i] : mx;
  }
  mean /= ctas;
  const double clk_step = mean / steps;
  const double dsmem_bytes = C > 1 ? (double)kTileFloats * 4 * (C - 1) / C : 0.0;  // remote reads
  const double l2_bytes = (double)kTileFloats * 4 / C;
  printf("{\"cluster\": %d, \"ctas\": %d, \"stagger\": %d, \"clk_per_step\": %.0f, "
         "\"clk_per_step_max\": %.0f, \"ms\": %.3f, \"dsmem_remote_B_per_clk_per_sm\": %.1f, "
         "\"l2_reduce_bytes_per_step_per_cta\": %.0f, \"l2_reduce_TBps\": %.2f}\n",
         C, ctas, stagger, clk_step, mx / steps, ms, dsmem_bytes / clk_step, l2_bytes,
         l2_bytes * ctas * steps / (ms * 1e-3) / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* dq;
  long long* clk;
  cudaMalloc(&dq, (size_t)kGroups * kQSteps * kTileFloats * 4);
  cudaMemset(dq, 0, (size_t)kGroups * kQSteps * kTileFloats * 4);
  cudaMalloc(&clk, sizeof(long long) * 1024);
  for (int stagger : {0, 1}) {
    run<1>(dq, clk, sms, stagger);
    run<2>(dq, clk, sms, stagger);
    run<4>(dq, clk, sms, stagger);
    run<8>(dq, clk, sms, stagger);
    run<16>(dq, clk, sms, stagger);
  }
  printf("{\"status\": \"%s\", \"sms\": %d}\n", cudaGetErrorString(cudaGetLastError()), sms);
  return 0;
}
