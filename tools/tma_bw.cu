// L2 -> SMEM TMA throughput probe (NOT part of the product library).
//
// Every CTA (one per SM, 148 x waves) streams 128-row x 128-col bf16 tiles
// (two SW128 panels = 32 KB, the K / V / Q / dO tiles of the attention
// kernels) through a STAGES-deep ring: wait full -> release, no compute.
// All CTAs of a group read the same tile sequence (like the dQ kernel's K/V
// stream, shared by the 64 query-tile CTAs of a kv head), so the data sits in
// L2.  mode 0: each CTA loads both tiles of a step itself (unicast); mode 1:
// cluster of 2, each CTA loads ONE tile and multicasts it to both CTAs.
// Reports bytes landed per SM per SM clock (clock64 of CTA 0) and TB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC \
//        -o build/tma_bw.so tools/tma_bw.cu -cudart static
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2502_02406_b200/csrc/lvx_sm100.cuh"

using namespace lvx::sm100;

namespace {

constexpr int kTile = 128 * 128 * 2;   // 32 KB
constexpr int kStages = 3;             // ring of (tile A | tile B) = 64 KB per stage

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(128, 1)
tma_bw_kernel(const __grid_constant__ CUtensorMap tm, int steps, int ntiles,
              long long* clk_out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * 2 * kTile);
  uint64_t* empty = full + kStages;
  const uint32_t rank = MODE == 1 ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MODE == 1 ? 2 : 1);   // both CTAs of the pair released it
    }
    fence_barrier_init();
  }
  if (MODE == 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
  } else {
    __syncthreads();
  }
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int grp = (blockIdx.x >> 1) % 8;   // 8 groups of CTAs share a tile sequence
    for (int i = 0; i < steps; ++i) {
      const int s = i % kStages, u = i / kStages;
      if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
      mbar_arrive_expect_tx(&full[s], 2 * kTile);
      const int tile = (grp * 1009 + i) % ntiles;
      uint8_t* dst = sm + s * 2 * kTile;
      if (MODE == 0) {
        for (int t = 0; t < 2; ++t)
          for (int pn = 0; pn < 2; ++pn)
            tma_load_3d(dst + t * kTile + pn * 128 * 128, &tm, &full[s], pn * 64,
                        (2 * tile + t) * 128, 0);
      } else {   // this CTA's tile, multicast to both CTAs (same smem offset, same barrier)
        for (int pn = 0; pn < 2; ++pn)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
              ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(
                  smem_u32(dst + rank * kTile + pn * 128 * 128)),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&full[s])), "r"(pn * 64),
              "r"((int)((2 * tile + rank) * 128)), "r"(0), "h"((uint16_t)0x3)
              : "memory");
      }
      mbar_wait(&full[s], u & 1);   // landed: release it (to both CTAs in mode 1)
      if (MODE == 0) {
        mbar_arrive(&empty[s]);
      } else {
        mbar_arrive(&empty[s]);
        uint32_t peer;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer)
                     : "r"(smem_u32(&empty[s])), "r"(rank ^ 1u));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(peer)
                     : "memory");
      }
    }
  }
  __syncthreads();
  if (MODE == 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk_out = clock64() - t0;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

}  // namespace

// buf: [rows][128] bf16 (rows = 256 * ntiles); grid CTAs; returns 0 / -3.
extern "C" int tma_bw_run(const void* buf, int ntiles, int ctas, int steps, int mode,
                          long long* clk_dev, void* stream) {
  CUtensorMap m;
  cuuint64_t dims[3] = {128, (cuuint64_t)ntiles * 256, 1};
  cuuint64_t strides[2] = {256, (cuuint64_t)ntiles * 256 * 256};
  cuuint32_t box[3] = {64, 128, 1}, estr[3] = {1, 1, 1};
  if (encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(buf), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return -3;
  const int smem = 1024 + kStages * 2 * kTile + 2 * kStages * 8;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mode == 0) {
    cudaFuncSetAttribute(tma_bw_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma_bw_kernel<0><<<ctas, 128, smem, st>>>(m, steps, ntiles, clk_dev);
  } else {
    cudaFuncSetAttribute(tma_bw_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tma_bw_kernel<1>, m, steps, ntiles, clk_dev);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
