// GEMMs of the cross-attention layer's projections on B200: the K/V
// recompute from the shared visual tokens (mllm.py:296-300, :358-360), the
// Q / O projections and their backward (kernels.py:227-254).
//
//   C[M, N] (+)= op(A)[M, K] op(B)[K, N]   row-major storage, bf16 in,
//                                          fp32 accumulate, bf16 out
//
// tcgen05 kernel (bf16): persistent, one CTA per SM, 128 x 256 output tiles,
// 64-deep K blocks in a 4-stage TMA ring (48 KB per stage, 128-byte swizzle),
// fp32 accumulators double-buffered in TMEM (2 x 256 columns) so the
// epilogue of tile t overlaps the main loop of tile t+1.  Warp roles:
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMA-fed MMA issuer, M = 128, N = 256, K = 16 per instruction
//   warps 2-5   epilogue: tcgen05.ld of their 32-lane quadrant, bf16 pack,
//               16-byte stores (or fp32 reduce-adds for split-K partials)
// Operand majors come from the transposes, so no operand is ever copied:
//   A not transposed: stored [M, K] -> K-major tile (one 128 x 64 box)
//   A transposed:     stored [K, M] -> MN-major tile (two 64 x 64 boxes)
//   B not transposed: stored [K, N] -> MN-major tile (four 64 x 64 boxes)
//   B transposed:     stored [N, K] -> K-major tile (one 256 x 64 box)
// Tall-K products with few output tiles (weight gradients x^T dOut over the
// rank's visual rows) split K so every SM gets work; the partials are
// stored as fp32 slices (one per split, stream-ordered scratch); the last
// split to finish a tile's rows (an atomic count per epilogue warp) sums the
// slices in split order and writes C, so the result is the same bits on every
// run and no CTA ever waits for another.
//
// Exact SIMT kernel for f32 / f64 (and bf16 views TMA cannot describe): one
// output element per thread, accumulated in fp32 (bf16, f32) or f64.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>

#include "lvx_common.cuh"
#include "lvx_sm100.cuh"

namespace lvx {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;          // 16 KB
constexpr int B_BYTES = BN * BK * 2;          // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int GEMM_THREADS = 192;
constexpr int GEMM_SMEM = STAGES * STAGE_BYTES + 1024 /* align */ + 256 /* barriers */;

struct GemmParams {
  int M, N, K;
  int m_tiles, n_tiles, kb_total, kb_per_split, splits, units;
  __nv_bfloat16* C;
  int64_t ldc;
  float* Cf;          // fp32 output: split-K scratch or the caller's fp32 C, else null
  int64_t ldcf;       // its leading dimension
  int* counters;      // split-K: per (tile, CTA of the pair, epilogue warp) count of the
                      // splits whose slice is written (null: one split)
  int64_t split_stride;   // split-K: elements between the fp32 slices in Cf
  float* Cout;        // split-K with an fp32 C: the caller's C (else the bf16 C above)
  int64_t ldcout;
  int f32_store;      // into Cf: 1 store (one split, overwrite), 0 reduce-add
  int accumulate;     // bf16 C += A B
};

// Split-K: after a split has stored its fp32 slice of a warp's 32 rows, one
// atomic per warp counts it (release: fence first); the warp that completes
// the count (acquire: fence after) sums the slices in split order 0, 1, ...
// for its rows and writes C (bf16 or fp32, + C when accumulating).  Nothing
// waits, so concurrent GEMMs on other streams cannot deadlock it.
__device__ __forceinline__ bool splitk_last(int* counter, int splits, int lane) {
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(counter, 1) == splits - 1;
    if (last) __threadfence();
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  return last != 0;
}

// Split-K slices are private scratch, laid out per epilogue warp as
// [32-column chunk c][float4 g][lane] (8192 floats = the warp's 32 rows x 256
// columns), so every slice store and every reduction load of a warp is one
// contiguous 512-byte run.  The completing warp sums its block over the
// splits in order and writes its rows of C.
constexpr int kSliceBlock = 32 * 256;

__device__ __forceinline__ void splitk_reduce_block(const GemmParams& p, const float* blk0,
                                                    int row0, int n0, int lane) {
  const int row = row0 + lane;
  const float4* b4 = reinterpret_cast<const float4*>(blk0);
  const int64_t ss = p.split_stride / 4;   // float4s between splits
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
#pragma unroll
    for (int gp = 0; gp < 4; ++gp) {
      float v[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int idx = (c * 8 + 2 * gp + h) * 32 + lane;
        float4 t = b4[idx];
        for (int sp = 1; sp < p.splits; ++sp) {
          const float4 o = b4[sp * ss + idx];
          t.x += o.x; t.y += o.y; t.z += o.z; t.w += o.w;
        }
        v[4 * h] = t.x; v[4 * h + 1] = t.y; v[4 * h + 2] = t.z; v[4 * h + 3] = t.w;
      }
      const int col = n0 + c * 32 + gp * 8;
      if (row >= p.M || col >= p.N) continue;
      if (p.Cout) {
        float4* d = reinterpret_cast<float4*>(p.Cout + (int64_t)row * p.ldcout + col);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4 t = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
          if (p.accumulate) {
            const float4 o = d[h];
            t.x += o.x; t.y += o.y; t.z += o.z; t.w += o.w;
          }
          d[h] = t;
        }
      } else {
        uint4* d4 = reinterpret_cast<uint4*>(p.C + (int64_t)row * p.ldc + col);
        if (p.accumulate) {
          const uint4 old = *d4;
          const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 o2 = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
            v[2 * e] += __bfloat162float(o2.x);
            v[2 * e + 1] += __bfloat162float(o2.y);
          }
        }
        *d4 = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                         pack_bf16(v[6], v[7]));
      }
    }
  }
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto decode = [&](int u, int& m0, int& n0, int& kb0, int& kb1) {
    // split slowest (the splits running side by side share their K range of
    // A and B in L2; split fastest measured 0.64x at the Flamingo weight
    // gradient), then N: one A row band meets every B tile
    const int tiles = p.m_tiles * p.n_tiles;
    const int split = u / tiles, t = u % tiles;
    m0 = (t / p.n_tiles) * BM;
    n0 = (t % p.n_tiles) * BN;
    kb0 = split * p.kb_per_split;
    kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      int it = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        int m0, n0, kb0, kb1;
        decode(u, m0, n0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          uint8_t* sa = sm + s * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_3d(sa, &tmA, &full[s], k0, m0, 0);
          } else {
            tma_load_3d(sa, &tmA, &full[s], m0, k0, 0);
            tma_load_3d(sa + 8192, &tmA, &full[s], m0 + 64, k0, 0);
          }
          if (!B_MN) {
            tma_load_3d(sb, &tmB, &full[s], k0, n0, 0);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) tma_load_3d(sb + j * 8192, &tmB, &full[s], n0 + 64 * j, k0, 0);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
    const uint32_t base = smem_u32(sm);
    int it = 0, lt = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++lt) {
      int m0, n0, kb0, kb1;
      decode(u, m0, n0, kb0, kb1);
      const int buf = lt & 1;
      if (lt >= 2) mbar_wait(&acc_empty[buf], ((lt >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t acc = tmem + buf * BN;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = base + s * STAGE_BYTES, sb = sa + A_BYTES;
          const uint64_t da = A_MN ? umma_desc_sw128(sa, 8192, 1024) : umma_desc_sw128(sa, 0, 1024);
          const uint64_t db = B_MN ? umma_desc_sw128(sb, 8192, 1024) : umma_desc_sw128(sb, 0, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: 16 elements = 32 bytes along the swizzled row;
            // MN-major: 16 K rows of 128 bytes
            const uint64_t oa = A_MN ? (uint64_t)((kk * 16 * 128) >> 4) : (uint64_t)((kk * 32) >> 4);
            const uint64_t ob = B_MN ? (uint64_t)((kk * 16 * 128) >> 4) : (uint64_t)((kk * 32) >> 4);
            mma_bf16_ss(acc, da + oa, db + ob, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          if (kb + 1 == kb1) mma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                  // TMEM lane quadrant of this warp
    int lt = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++lt) {
      int m0, n0, kb0, kb1;
      decode(u, m0, n0, kb0, kb1);
      const int buf = lt & 1;
      mbar_wait(&acc_full[buf], (lt >> 1) & 1);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const uint32_t tbase = tmem + buf * BN + ((uint32_t)(q * 32) << 16);
      const bool sk = p.counters != nullptr;
      const int64_t wblk = ((int64_t)(u % (p.m_tiles * p.n_tiles)) * 4 + q) * kSliceBlock;
      float* cf = sk ? p.Cf + (int64_t)(kb0 / p.kb_per_split) * p.split_stride + wblk : p.Cf;
      const bool store = p.f32_store == 1;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        tmem_wait_ld();
        if (sk) {   // this split's slice, [c][g][lane] (coalesced)
          float4* w4 = reinterpret_cast<float4*>(cf) + c * 8 * 32 + lane;
#pragma unroll
          for (int g = 0; g < 8; ++g)
            w4[g * 32] = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                     __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3]));
          continue;
        }
        const int col0 = n0 + c * 32;
        if (row >= p.M || col0 >= p.N) continue;
        if (p.Cf) {
          float* dst = cf + (int64_t)row * p.ldcf + col0;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (col0 + 4 * g >= p.N) break;
            const float4 v4 = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                          __uint_as_float(r[4 * g + 2]),
                                          __uint_as_float(r[4 * g + 3]));
            if (store) {
              *reinterpret_cast<float4*>(dst + 4 * g) = v4;
            } else
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * g),
                           "f"(v4.x), "f"(v4.y), "f"(v4.z), "f"(v4.w)
                           : "memory");
          }
        } else {
          __nv_bfloat16* dst = p.C + (int64_t)row * p.ldc + col0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (col0 + 8 * g >= p.N) break;
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * g + e]);
            uint4* d4 = reinterpret_cast<uint4*>(dst + 8 * g);
            if (p.accumulate) {
              const uint4 old = *d4;
              const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const __nv_bfloat162 o2 = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
                v[2 * e] += __bfloat162float(o2.x);
                v[2 * e + 1] += __bfloat162float(o2.y);
              }
            }
            *d4 = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                             pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (sk && splitk_last(p.counters + (size_t)(u % (p.m_tiles * p.n_tiles)) * 4 + q,
                            p.splits, lane))
        splitk_reduce_block(p, p.Cf + wblk, m0 + q * 32, n0, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- CTA pairs
// The same GEMM on cta_group::2: a pair of CTAs (one cluster) owns a
// 256 x 256 output tile; the leader issues M = 256, N = 256 MMAs for both.
// Operands split as the pair MMA reads them: A by M (each CTA its 128 rows),
// B by N (each CTA 128 of the 256 columns), so each CTA stages 32 KB per
// 64-deep K block instead of 48 KB and its tensor core reads 2/3 of the
// operand bytes per FLOP of the 1-CTA kernel.  Each CTA's TMEM holds its 128
// rows x 256 fp32 columns, double-buffered.  Barriers: `full` (the leader's,
// expecting both CTAs' TMA bytes), `empty` / `acc_full` (multicast commits
// into both CTAs), `acc_empty` (the leader's, 256 epilogue arrivals).
constexpr int P_STAGES = 6;
constexpr int P_A_BYTES = 128 * BK * 2;       // this CTA's M half of A: 16 KB
constexpr int P_B_BYTES = 128 * BK * 2;       // this CTA's N half of B: 16 KB
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int PAIR_SMEM = P_STAGES * P_STAGE_BYTES + 1024 + 256;

template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
gemm_bf16_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* acc_full = empty + P_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto decode = [&](int u, int& m0, int& n0, int& kb0, int& kb1) {
    const int tiles = p.m_tiles * p.n_tiles;
    const int split = u / tiles, t = u % tiles;   // split slowest (see gemm_bf16_kernel)
    m0 = (t / p.n_tiles) * 256;
    n0 = (t % p.n_tiles) * 256;
    kb0 = split * p.kb_per_split;
    kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (elect_one()) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      int it = 0;
      for (int u = pair; u < p.units; u += npairs) {
        int m0, n0, kb0, kb1;
        decode(u, m0, n0, kb0, kb1);
        const int ma = m0 + 128 * (int)rank, nb = n0 + 128 * (int)rank;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % P_STAGES;
          if (it >= P_STAGES) mbar_wait(&empty[s], ((it / P_STAGES) - 1) & 1);
          uint8_t* sa = sm + s * P_STAGE_BYTES;
          uint8_t* sb = sa + P_A_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * P_STAGE_BYTES);
          const uint32_t lf = leader_addr(&full[s]);
          const int k0 = kb * BK;
          const uint64_t pol = l2_evict_last();
          if (!A_MN) {
            tma2_load_3d(sa, &tmA, lf, k0, ma, 0, pol);
          } else {
            tma2_load_3d(sa, &tmA, lf, ma, k0, 0, pol);
            tma2_load_3d(sa + 8192, &tmA, lf, ma + 64, k0, 0, pol);
          }
          if (!B_MN) {
            tma2_load_3d(sb, &tmB, lf, k0, nb, 0, pol);
          } else {
            tma2_load_3d(sb, &tmB, lf, nb, k0, 0, pol);
            tma2_load_3d(sb + 8192, &tmB, lf, nb + 64, k0, 0, pol);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(256, 256, A_MN, B_MN);
      const uint32_t base = smem_u32(sm);
      int it = 0, lt = 0;
      for (int u = pair; u < p.units; u += npairs, ++lt) {
        int m0, n0, kb0, kb1;
        decode(u, m0, n0, kb0, kb1);
        const int buf = lt & 1;
        if (lt >= 2) mbar_wait_cluster(&acc_empty[buf], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * 256;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % P_STAGES;
          mbar_wait_cluster(&full[s], (it / P_STAGES) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = base + s * P_STAGE_BYTES, sb = sa + P_A_BYTES;
            const uint64_t da = A_MN ? umma_desc_sw128(sa, 8192, 1024) : umma_desc_sw128(sa, 0, 1024);
            const uint64_t db = B_MN ? umma_desc_sw128(sb, 8192, 1024) : umma_desc_sw128(sb, 0, 1024);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t oa = A_MN ? (uint64_t)((kk * 16 * 128) >> 4) : (uint64_t)((kk * 32) >> 4);
              const uint64_t ob = B_MN ? (uint64_t)((kk * 16 * 128) >> 4) : (uint64_t)((kk * 32) >> 4);
              mma2_bf16_ss(acc, da + oa, db + ob, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            }
            mma2_commit_mc(&empty[s]);
            if (kb + 1 == kb1) mma2_commit_mc(&acc_full[buf]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    int lt = 0;
    for (int u = pair; u < p.units; u += npairs, ++lt) {
      int m0, n0, kb0, kb1;
      decode(u, m0, n0, kb0, kb1);
      const int buf = lt & 1;
      mbar_wait(&acc_full[buf], (lt >> 1) & 1);
      tc_fence_after();
      const int row = m0 + 128 * (int)rank + q * 32 + lane;
      const uint32_t tbase = tmem + buf * 256 + ((uint32_t)(q * 32) << 16);
      const bool sk = p.counters != nullptr;
      const int64_t wblk =
          (((int64_t)(u % (p.m_tiles * p.n_tiles)) * 2 + rank) * 4 + q) * kSliceBlock;
      float* cf = sk ? p.Cf + (int64_t)(kb0 / p.kb_per_split) * p.split_stride + wblk : p.Cf;
      const bool store = p.f32_store == 1;
#pragma unroll 1
      for (int c = 0; c < 256 / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        tmem_wait_ld();
        if (sk) {   // this split's slice, [c][g][lane] (coalesced)
          float4* w4 = reinterpret_cast<float4*>(cf) + c * 8 * 32 + lane;
#pragma unroll
          for (int g = 0; g < 8; ++g)
            w4[g * 32] = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                     __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3]));
          continue;
        }
        const int col0 = n0 + c * 32;
        if (row >= p.M || col0 >= p.N) continue;
        if (p.Cf) {
          float* dst = cf + (int64_t)row * p.ldcf + col0;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (col0 + 4 * g >= p.N) break;
            const float4 v4 = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                          __uint_as_float(r[4 * g + 2]),
                                          __uint_as_float(r[4 * g + 3]));
            if (store) {
              *reinterpret_cast<float4*>(dst + 4 * g) = v4;
            } else
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * g),
                           "f"(v4.x), "f"(v4.y), "f"(v4.z), "f"(v4.w)
                           : "memory");
          }
        } else {
          __nv_bfloat16* dst = p.C + (int64_t)row * p.ldc + col0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (col0 + 8 * g >= p.N) break;
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * g + e]);
            uint4* d4 = reinterpret_cast<uint4*>(dst + 8 * g);
            if (p.accumulate) {
              const uint4 old = *d4;
              const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const __nv_bfloat162 o2 = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
                v[2 * e] += __bfloat162float(o2.x);
                v[2 * e + 1] += __bfloat162float(o2.y);
              }
            }
            *d4 = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                             pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
          }
        }
      }
      tc_fence_before();
      if (rank == 0) mbar_arrive(&acc_empty[buf]);
      else mbar_arrive_cluster(leader_addr(&acc_empty[buf]));
      if (sk && splitk_last(p.counters +
                                ((size_t)(u % (p.m_tiles * p.n_tiles)) * 2 + rank) * 4 + q,
                            p.splits, lane))
        splitk_reduce_block(p, p.Cf + wblk, m0 + 128 * (int)rank + q * 32, n0, lane);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

// ---------------------------------------------------------------- SIMT
// One output element per thread; op(A)[m, k] = A[m * lda + k] or A[k * lda + m].
template <typename T, typename Acc, typename TO = T>
__global__ void gemm_simt_kernel(const T* __restrict__ A, int64_t lda, bool ta,
                                 const T* __restrict__ B, int64_t ldb, bool tb, TO* __restrict__ C,
                                 int64_t ldc, int64_t M, int64_t N, int64_t K, bool accumulate) {
  constexpr int TS = 16;
  __shared__ Acc sa[TS][TS + 1], sb[TS][TS + 1];
  const int64_t m = (int64_t)blockIdx.y * TS + threadIdx.y;
  const int64_t n = (int64_t)blockIdx.x * TS + threadIdx.x;
  Acc acc = 0;
  for (int64_t k0 = 0; k0 < K; k0 += TS) {
    const int64_t ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
    const int64_t mA = (int64_t)blockIdx.y * TS + threadIdx.y;
    sa[threadIdx.y][threadIdx.x] =
        (mA < M && ka < K) ? to_acc<Acc>(ta ? A[ka * lda + mA] : A[mA * lda + ka]) : Acc(0);
    sb[threadIdx.y][threadIdx.x] =
        (n < N && kb < K) ? to_acc<Acc>(tb ? B[n * ldb + kb] : B[kb * ldb + n]) : Acc(0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TS; ++k) acc += sa[threadIdx.y][k] * sb[k][threadIdx.x];
    __syncthreads();
  }
  if (m < M && n < N) {
    TO* c = C + m * ldc + n;
    *c = from_acc<TO>(accumulate ? acc + to_acc<Acc>(*c) : acc);
  }
}

template <typename T, typename Acc, typename TO = T>
int launch_simt(const GemmCall& g, cudaStream_t st) {
  dim3 block(16, 16), grid((unsigned)((g.N + 15) / 16), (unsigned)((g.M + 15) / 16));
  if (grid.y > 65535) return LVX_EUNSUPPORTED;
  gemm_simt_kernel<T, Acc, TO><<<grid, block, 0, st>>>(
      static_cast<const T*>(g.a), g.lda, g.ta, static_cast<const T*>(g.b), g.ldb, g.tb,
      static_cast<TO*>(g.c), g.ldc, g.M, g.N, g.K, g.accumulate);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

// 2-D bf16 map of a row-major [rows, cols] matrix (leading dimension ld),
// box (64 columns, box_rows rows), 128-byte swizzle
bool map2d(CUtensorMap* m, const void* p, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto fn = tensor_map_encoder();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2 * (cuuint64_t)rows};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(p), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tc_ok(const GemmCall& g) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const int64_t ldc_align = g.c_dtype == LVX_F32 ? 4 : 8;   // 16-byte rows
  return g.dtype == LVX_BF16 && is_sm100() && g.M > 0 && g.N > 0 && g.K > 0 && al16(g.a) &&
         al16(g.b) && al16(g.c) && g.lda % 8 == 0 && g.ldb % 8 == 0 && g.ldc % ldc_align == 0 &&
         g.N % 8 == 0 && g.M < (1ll << 31) && g.N < (1ll << 31) && g.K < (1ll << 31);
}

// The split-K scratch comes from the device's default stream-ordered pool.
// By default the pool returns freed memory to the driver at every
// synchronisation, so the next cudaMallocAsync maps it again (~0.1-0.2 ms,
// measured: a 0.18 ms weight-gradient GEMM took 0.35 ms per call); keep it.
bool keep_pool_memory() {
  static std::atomic<unsigned> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const unsigned bit = dev < 32 ? 1u << dev : 0u;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return false;
  uint64_t keep = ~0ull;
  if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess)
    return false;
  done.fetch_or(bit, std::memory_order_release);
  return true;
}

// Split K so the work units fill whole waves of `slots` (SMs, or CTA pairs):
// maximise units / (waves x slots) over splits with >= 8 K blocks each; more
// splits only when they raise that efficiency by > 2 % (each split adds an
// M x N fp32 reduce-add pass).
int plan_splits(int tiles, int kb_total, int slots) {
  int best = 1;
  double best_eff = (double)tiles / (double)(((tiles + slots - 1) / slots) * slots);
  for (int s = 2; s <= 16 && kb_total / s >= 8; ++s) {
    const int units = tiles * s;
    const double eff = (double)units / (double)(((units + slots - 1) / slots) * slots);
    if (eff > best_eff + 0.02) {
      best = s;
      best_eff = eff;
    }
  }
  return best;
}

template <bool A_MN, bool B_MN>
int launch_tc(const GemmCall& g, cudaStream_t st) {
  const int sms = device_sms();
  // CTA pairs for every product with at least two 256-row bands; the 1-CTA
  // kernel for thin ones (fewer rows than a pair tile wastes half of it)
  const bool pairs = g.M >= 256;
  const int tm = pairs ? 256 : BM, tn = pairs ? 256 : BN;
  const int box_m = pairs ? 128 : BM, box_n = pairs ? 128 : BN;
  CUtensorMap ta, tb;
  // A: [M, K] K-major box of box_m rows; [K, M] MN-major boxes of 64 K rows
  const bool okA = A_MN ? map2d(&ta, g.a, g.K, g.M, g.lda, 64) : map2d(&ta, g.a, g.M, g.K, g.lda, box_m);
  const bool okB = B_MN ? map2d(&tb, g.b, g.K, g.N, g.ldb, 64) : map2d(&tb, g.b, g.N, g.K, g.ldb, box_n);
  if (!okA || !okB) return LVX_ECUDA;
  GemmParams p{};
  p.M = (int)g.M;
  p.N = (int)g.N;
  p.K = (int)g.K;
  p.m_tiles = (int)((g.M + tm - 1) / tm);
  p.n_tiles = (int)((g.N + tn - 1) / tn);
  p.kb_total = (int)((g.K + BK - 1) / BK);
  const int slots = pairs ? sms / 2 : sms;
  const int tiles = p.m_tiles * p.n_tiles;
  const int splits = plan_splits(tiles, p.kb_total, slots);
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.units = tiles * p.splits;
  p.C = static_cast<__nv_bfloat16*>(g.c);
  p.ldc = g.ldc;
  p.accumulate = g.accumulate ? 1 : 0;
  float* scratch = nullptr;
  if (p.splits > 1) {
    // split K: per-split fp32 slices + per-warp counters in one stream-ordered
    // allocation; the last split of each tile's rows reduces them in order
    // and writes C (see splitk_last), so there is no finish kernel
    if (!keep_pool_memory()) return LVX_ECUDA;
    const size_t ncnt = (size_t)p.m_tiles * p.n_tiles * (pairs ? 2 : 1) * 4;   // warps
    const size_t slice = ncnt * kSliceBlock;   // floats per split (padded tiles)
    const size_t cnt_off = ((size_t)p.splits * slice * 4 + 255) / 256 * 256;
    if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), cnt_off + ncnt * sizeof(int), st) !=
        cudaSuccess)
      return LVX_ECUDA;
    p.counters = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) + cnt_off);
    if (cudaMemsetAsync(p.counters, 0, ncnt * sizeof(int), st) != cudaSuccess)
      return LVX_ECUDA;
    p.Cf = scratch;
    p.ldcf = 0;   // slices are [warp block][c][g][lane], not row-major
    p.split_stride = (int64_t)slice;
    if (g.c_dtype == LVX_F32) {
      p.Cout = static_cast<float*>(g.c);
      p.ldcout = g.ldc;
    }
  } else if (g.c_dtype == LVX_F32) {
    // fp32 C, one split: stored directly, or reduce-added when accumulating
    // (one add per element, so deterministic): fire-and-forget in L2, where a
    // load-add-store made the epilogue wait on every load (measured 0.38 ->
    // 0.75 ms per dY GEMM of the C4 layer)
    p.C = nullptr;
    p.Cf = static_cast<float*>(g.c);
    p.ldcf = g.ldc;
    p.f32_store = g.accumulate ? 0 : 1;
  }
  if (pairs) {
    auto kern = gemm_bf16_pair_kernel<A_MN, B_MN>;
    static std::atomic<unsigned> attr_done{0};
    if (!ensure_smem_attr(kern, PAIR_SMEM, attr_done)) return LVX_ECUDA;
    kern<<<2 * std::min(p.units, slots), GEMM_THREADS, PAIR_SMEM, st>>>(ta, tb, p);
  } else {
    auto kern = gemm_bf16_kernel<A_MN, B_MN>;
    static std::atomic<unsigned> attr_done{0};
    if (!ensure_smem_attr(kern, GEMM_SMEM, attr_done)) return LVX_ECUDA;
    kern<<<std::min(p.units, slots), GEMM_THREADS, GEMM_SMEM, st>>>(ta, tb, p);
  }
  note_launch();
  if (scratch) cudaFreeAsync(scratch, st);
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

}  // namespace

int gemm(const GemmCall& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return LVX_OK;
  if (g.K <= 0) {   // empty contraction: C = 0, or unchanged when accumulating
    if (g.accumulate) return LVX_OK;
    const size_t es = g.c_dtype == LVX_F64 ? 8 : (g.c_dtype == LVX_F32 ? 4 : 2);
    return cudaMemset2DAsync(g.c, g.ldc * es, 0, g.N * es, g.M, st) == cudaSuccess ? LVX_OK
                                                                                    : LVX_ECUDA;
  }
  if (g.c_dtype == LVX_F32 && g.dtype == LVX_BF16 && !tc_ok(g))
    return launch_simt<__nv_bfloat16, float, float>(g, st);
  if (tc_ok(g)) {
    if (!g.ta && !g.tb) return launch_tc<false, true>(g, st);
    if (!g.ta && g.tb) return launch_tc<false, false>(g, st);
    if (g.ta && !g.tb) return launch_tc<true, true>(g, st);
    return launch_tc<true, false>(g, st);
  }
  switch (g.dtype) {
    case LVX_BF16: return launch_simt<__nv_bfloat16, float>(g, st);
    case LVX_F32: return launch_simt<float, float>(g, st);
    case LVX_F64: return launch_simt<double, double>(g, st);
    default: return LVX_EDTYPE;
  }
}

}  // namespace lvx
