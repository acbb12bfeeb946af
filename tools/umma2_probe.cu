// 2-CTA (cta_group::2) tcgen05 probe — groundwork for a 2-CTA dK/dV kernel
// (DESIGN.md §8).  NOT part of the product library.
//
// D[256 x 128] (fp32) = A[256 x 64] . B[128 x 64]^T (bf16, K-major), one cluster
// of two CTAs: CTA r loads A rows [128 r, 128 r + 128) and B rows [64 r, 64 r + 64)
// (A split by M, B split by N — cute's SM100_MMA_F16BF16_2x1SM_SS layouts); the
// leader (rank 0) issues ONE M=256 MMA chain, whose commit is multicast to both
// CTAs' barriers; each CTA drains its own 128 TMEM lanes.  The peer's TMA bytes
// complete on the leader's barrier (shared::cluster address with bit 24 clear).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC \
//        -o build/umma2_probe.so tools/umma2_probe.cu -cudart static
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2502_02406_b200/csrc/lvx_sm100.cuh"

using namespace lvx::sm100;

namespace {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
             float* D) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];   // 128 rows x 64 bf16 (one SW128 panel)
  __shared__ __align__(1024) uint8_t sB[64 * 128];    // 64 rows x 64 bf16
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {   // same warp in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;

  if (threadIdx.x == 0) {
    // both CTAs load their halves; the bytes complete on the LEADER's barrier
    const uint32_t lead_full = smem_u32(&full) & 0xFEFFFFFFu;
    if (rank == 0) mbar_arrive_expect_tx(&full, 2 * (128 * 128 + 64 * 128));
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sA)),
        "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(lead_full), "r"(0), "r"((int)(128 * rank)),
        "r"(0)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sB)),
        "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(lead_full), "r"(0), "r"((int)(64 * rank)),
        "r"(0)
        : "memory");
  }
  if (rank == 0 && warp == 0) {
    mbar_wait(&full, 0);
    tc_fence_after();
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) |
                               ((256u >> 4) << 24);   // bf16 x bf16 -> f32, K-major, N=128, M=256
    if (elect_one()) {
      const uint64_t da = umma_desc_sw128(smem_u32(sA), 0, 1024);
      const uint64_t db = umma_desc_sw128(smem_u32(sB), 0, 1024);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = kk > 0;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(da + (uint64_t)((kk * 32) >> 4)), "l"(db + (uint64_t)((kk * 32) >> 4)),
            "r"(idesc), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
          " [%0], %1;" ::"r"(smem_u32(&done)), "h"((uint16_t)0x3));
    }
    __syncwarp();
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  float* row = D + (size_t)(128 * rank + warp * 32 + lane) * 128;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(tl + c * 32, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) row[c * 32 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

bool map2d(CUtensorMap* m, const void* base, int rows, int box_rows) {
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {128, (cuuint64_t)rows * 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1}, estr[3] = {1, 1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// A: [256, 64] bf16, B: [128, 64] bf16 (row-major, K contiguous); D: [256, 128] fp32.
extern "C" int umma2_probe(const void* A, const void* B, float* D, void* stream) {
  CUtensorMap ma, mb;
  if (!map2d(&ma, A, 256, 128) || !map2d(&mb, B, 128, 64)) return -3;
  probe_kernel<<<2, 128, 0, static_cast<cudaStream_t>(stream)>>>(ma, mb, D);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
