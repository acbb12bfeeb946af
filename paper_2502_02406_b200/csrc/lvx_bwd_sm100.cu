// tcgen05/TMEM/TMA blockwise attention backward for B200 (sm_100a).
//
// Replaces kernels.py:192-224 blockwise_attention_backward for bf16 inputs
// with d in {64, 128}:  P = exp(S - L), dV = P^T dO, dP = dO V^T,
// dS = P (dP - D), dQ = scale dS K, dK = scale dS^T Q.
//
// Two deterministic kernels instead of one kernel with dQ atomics (a dQ
// atomic stream of 64 KB per (KV tile, Q tile) pair would need ~7 TB/s of L2
// reductions at full tensor rate):
//   bwd_dkv_kernel  KV-parallel.  One CTA owns a 128-row KV tile; dK, dV
//                   accumulate in TMEM over every 128-row query step of the
//                   GQA group (kernels.py:258-262 accumulate over rounds on
//                   top of this in fp32 HBM accumulators).
//                   MMAs: S^T = K Q^T, dP^T = V dO^T (SS); dV += P^T dO,
//                   dK += dS^T Q (TS: P^T / dS^T live in TMEM as bf16, written
//                   over the S^T / dP^T columns they came from).
//   bwd_dq_kernel   Q-parallel, one 128-row query tile per CTA (Q, dO copied
//                   into TMEM), 128-row K/V steps, split over the KV block.
//                   S = Q K^T, dP = dO V^T, dQ += dS K (all TS).
// Softmax statistics enter pre-scaled and negated, nL = -L log2(e) (-inf on
// padding rows, so P = 0 there) and nD = -D, packed by bwd_prep_kernel into
// 16-byte aligned rows, so the element math is FFMA2 / FADD2 / FMUL2 pairs.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "lvx_common.cuh"
#include "lvx_sm100.cuh"

namespace lvx {
namespace {

using namespace sm100;

constexpr int kStep = 64;      // q rows per step (dkv kernel) / kv rows per step (dq kernel)
constexpr float kLog2e = 1.4426950408889634f;
// Polynomial exp2 shares, tuned in the power-capped bench step
// (tools/ab_bench.sh): dQ 1/8 (3/8 was best isolated at ~1.8 GHz; at the
// bench's ~1.4 GHz cap 1/8 measured +0.2-0.7 %), dK/dV 2/8 (1/8: -0.4 %, 0/8:
// -1.7 %); the forward keeps 3/8 (2/8 even, 1/8 -0.4 %)
#ifndef LVX_DQ_POLY
#define LVX_DQ_POLY 1
#endif
#ifndef LVX_DKV_POLY
#define LVX_DKV_POLY 2
#endif
// At d = 64 the MMAs take half as long per step while the exponentials do
// not, so the softmax side is rebalanced toward the FMA pipe (same-box A/B,
// tools/ab_poly.sh: c4gath dQ +3-5 %, dK/dV +1 %; d = 128 unchanged).
#ifndef LVX_DQ_POLY64
#define LVX_DQ_POLY64 2
#endif
#ifndef LVX_DKV_POLY64
#define LVX_DKV_POLY64 3
#endif
template <int D>
constexpr int kPolyPairsD = D == 64 ? LVX_DQ_POLY64 : LVX_DQ_POLY;   // of every 8 column pairs, exp2 by polynomial (FMA pipe)
template <int D>
constexpr int kPolyPairsDkvD = D == 64 ? LVX_DKV_POLY64 : LVX_DKV_POLY;   // the dK/dV kernel's phase A
#ifndef LVX_DKV_CHUNKS
#define LVX_DKV_CHUNKS 2
#endif
constexpr int kDkvChunks = LVX_DKV_CHUNKS;   // P^T publication chunks per step (dK/dV kernel)
#ifndef LVX_DKV_ARRIVALS
#define LVX_DKV_ARRIVALS 256
#endif
constexpr int kDkvArrivals = LVX_DKV_ARRIVALS;   // per hand-off barrier: 256 threads or 8 warps

// Profiling switches (p.debug) compile to nothing in the product build
#ifdef LVX_BWD_DEBUG_MODES
#define BWD_DBG(cond) (cond)
#else
#define BWD_DBG(cond) false
#endif

// LVX_DQ_TRACE=<query tile> (profiling builds only, tools/dq_trace.py): the same
// for one dQ CTA (split 0, head group 0), [role][kv step][event]
#ifdef LVX_DQ_TRACE
__device__ long long g_dq_trace[4][128][8];
#define DQ_STAMP(role, step, ev)                                                       \
  do {                                                                                 \
    if (blockIdx.x == LVX_DQ_TRACE && blockIdx.y == 0 && blockIdx.z == 0 &&            \
        (step) < 128 && lane == 0)                                                     \
      g_dq_trace[role][step][ev] = clock64();                                          \
  } while (0)
#else
#define DQ_STAMP(role, step, ev) \
  do {                           \
  } while (0)
#endif

// LVX_DKV_TRACE=<cta x> (profiling builds only, tools/dkv_trace.py): clock64
// stamps of one dK/dV CTA's hand-offs, [role][step][event]
#ifdef LVX_DKV_TRACE
__device__ long long g_dkv_trace[4][64][8];
#define DKV_STAMP(role, step, ev)                                                  \
  do {                                                                             \
    if (blockIdx.x == LVX_DKV_TRACE && blockIdx.y == 0 && (step) < 64 && lane == 0) \
      g_dkv_trace[role][step][ev] = clock64();                                     \
  } while (0)
#else
#define DKV_STAMP(role, step, ev) \
  do {                            \
  } while (0)
#endif

// ------------------------------------------------------------------- prep
__global__ void bwd_prep_kernel(View3<const float> L, View3<const float> Dv, int hq, int rows,
                                int rows_pad, float* __restrict__ Lp, float* __restrict__ Dp) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)hq * rows_pad) return;
  const int h = (int)(idx / rows_pad), r = (int)(idx % rows_pad);
  if (r < rows) {
    Lp[idx] = -*L.at(h, r) * kLog2e;
    Dp[idx] = -*Dv.at(h, r);
  } else {
    Lp[idx] = -INFINITY;
    Dp[idx] = 0.f;
  }
}

struct BwdParams {
  int hq, hkv, G, rows_q, rows_kv, rows_pad;
  int tq64;           // 64-row query steps per head (dkv kernel)
  int tpq;            // 128-row query tiles per head (dq kernel)
  int n_tiles;        // 128-row kv tiles
  int tiles_per_split, splits;
  float scale_log2, scale;
  const float* Lp;    // [hq][rows_pad]
  const float* Dp;
  int accumulate;     // dK / dV: TMA reduce-add into the fp32 accumulators (else store)
  void* dk_ptr; void* dv_ptr;     // outputs [hkv][rows_kv][D] (strided): fp32, or bf16
  int out_bf16;                   //   when overwriting in the input dtype
  int64_t dk_hs, dk_rs, dv_hs, dv_rs;
  float* ws_dq;       // [splits][hq][rows_q][D]
  int debug;          // LVX_BWD_DEBUG, honoured only by -DLVX_BWD_DEBUG_MODES builds
                      // (tools/build_variant.sh; profiling): 1 = skip exp / dS math,
                      // 2 = also skip Q/dO reloads (dkv), 3 = skip reloads only,
                      // 4 = skip the dK/dV drain, 5 = no nL/nD shared loads (dkv)
};

// ============================================================ dK / dV kernel
// 128-row query steps so every SS MMA has N = 128 (A 4 KB + B 4 KB per 64
// clk = the 128 B/clk SMEM read rate; 64-row steps re-read the 128-row A
// operand twice as often and capped the kernel at ~80 % of peak).  TMEM:
//   R1 [0,128)    S^T(i), then P^T(i) packed bf16 (columns [0,32) + [64,96))
//   R2 [128,256)  dP^T(i), then dS^T(i) packed bf16 (the same columns of R2)
//   dV [256, 256+D), dK [256+D, 256+2D)
// Two-phase softmax per step: phase A turns S^T into P^T (the exponentials)
// and releases dV(i) in kDkvChunks chunks, then S^T(i+1); phase B turns dP^T into
// dS^T while the tensor pipe runs dV(i) / S^T(i+1), then releases dK(i) and
// dP^T(i+1).  P stays in fp32 registers between the phases (R1 is
// overwritten by S^T(i+1) as soon as dV(i) has read it).  Two softmax
// warpgroups split the 128 query columns, each packing into its own columns.
template <int D>
struct DkvCfg {
  static constexpr int PANELS = D / 64;
  static constexpr int KV_BYTES = 128 * D * 2;             // resident K (or V) tile
  static constexpr int QT_BYTES = 128 * D * 2;             // one Q (or dO) 128-row step tile
  // separate rings: Q (+ the step's nL / nD rows) is released after dK, dO
  // after dV, so each load gets more than one step of lead time (the L2 ->
  // SMEM stream of all CTAs runs at ~75 % of the chip's TMA throughput)
  static constexpr int QSTAGES = D == 128 ? 3 : 4, GSTAGES = D == 128 ? 2 : 4;
  // nD (read in phase B, until dK) rides with Q, nL (read in phase A, before
  // dV) with dO
  static constexpr int OFF_G = QSTAGES * QT_BYTES;                // dO tiles
  static constexpr int OFF_LD = OFF_G + GSTAGES * QT_BYTES;      // nD rows [QSTAGES][512]
  static constexpr int OFF_LL = OFF_LD + QSTAGES * 512;          // nL rows [GSTAGES][512]
  static constexpr int NBAR = 1 + 2 * QSTAGES + 2 * GSTAGES + 4 + kDkvChunks;
  static constexpr int RING = OFF_LL + GSTAGES * 512;
  // no alignment pad at d = 128 (it would not fit 227 KB): the kernel traps
  // unless the dynamic shared memory base is 1024-byte aligned
  static constexpr int PAD = D == 128 ? 0 : 1024;
  static constexpr int SMEM = PAD + 2 * KV_BYTES + RING + NBAR * 8 + 16;
  static constexpr int R1 = 0, R2 = 128, DV_COL = 256, DK_COL = 256 + D;
  static_assert(8 * 32 * D * 4 <= OFF_LD, "epilogue staging must fit the Q/dO rings");
  static_assert(SMEM <= 232448, "227 KB of shared memory per CTA");
};

// dK / dV softmax, shared by the 1-CTA and CTA-pair kernels.  Thread = one kv
// row (TMEM lane); warpgroup wg owns query columns [64 wg, 64 wg + 64) of S^T
// / dP^T and packs its bf16 P^T / dS^T into the first 32 of those columns, so
// the two warpgroups never touch each other's columns.  P^T is published in
// kDkvChunks chunks (query columns 64/kDkvChunks c .. of each wg) so the dV
// MMAs of the first chunks run while later ones are still exponentiated.
// The TS MMA k-step kk (query rows 16 kk ..) reads A at column dkv_a_col(kk).
__device__ __forceinline__ uint32_t dkv_a_col(int kk) { return (kk >> 2) * 64 + (kk & 3) * 8; }
// k-step j (0 .. 8/kDkvChunks - 1) of chunk c, both warpgroups' columns
__device__ __forceinline__ int dkv_chunk_kk(int c, int j) {
  constexpr int kpw = 4 / kDkvChunks;
  return (j / kpw) * 4 + c * kpw + j % kpw;
}

// phase A: P^T = exp2(S^T c + nL[q]) over this thread's 64 columns at tS; the
// fp32 P^T stays in pf for phase B; arrive(c) after each packed chunk is stored
template <int D, class Arrive>
__device__ __forceinline__ void dkv_phase_a(uint32_t tS, uint32_t lds, float2 sc2, int debug,
                                            float2 (&pf)[32], Arrive&& arrive) {
  constexpr int kPolyPairsDkv = kPolyPairsDkvD<D>;
  constexpr int CW = 64 / kDkvChunks;   // query columns per chunk
  uint32_t sv[2][32];
  tmem_ld32(tS, sv[0]);
  tmem_ld32(tS + 32, sv[1]);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < kDkvChunks; ++c) {
    uint32_t pp[CW / 2];
    if (BWD_DBG(debug == 1 || debug == 2)) {   // profiling: no exp math
#pragma unroll
      for (int c2 = 0; c2 < CW; c2 += 2) {
        const int col = c * CW + c2;
        pp[c2 / 2] = sv[col / 32][col % 32];
        pf[col / 2] = u2f2(sv[col / 32][col % 32], sv[col / 32][col % 32 + 1]);
      }
    } else {
#pragma unroll
      for (int c4 = 0; c4 < CW; c4 += 4) {
        const int col = c * CW + c4, hh = col / 32, k = col % 32, pi = col / 2;
        const float4 l4 = BWD_DBG(debug == 5) ? make_float4(-1.f, -1.f, -1.f, -1.f)
                                              : ld_shared_f4(lds + col * 4);   // -L log2 e per q
        const float2 x0 = ffma2(u2f2(sv[hh][k], sv[hh][k + 1]), sc2, make_float2(l4.x, l4.y));
        const float2 x1 =
            ffma2(u2f2(sv[hh][k + 2], sv[hh][k + 3]), sc2, make_float2(l4.z, l4.w));
        // phase A is MUFU-bound: some pairs on the FMA pipe
        const float2 p0 =
            (pi % 8) < kPolyPairsDkv ? ex2_poly2(x0) : make_float2(ex2(x0.x), ex2(x0.y));
        const float2 p1 =
            ((pi + 1) % 8) < kPolyPairsDkv ? ex2_poly2(x1) : make_float2(ex2(x1.x), ex2(x1.y));
        pp[c4 / 2] = pack_bf16(p0.x, p0.y);
        pp[c4 / 2 + 1] = pack_bf16(p1.x, p1.y);
        pf[pi] = p0;
        pf[pi + 1] = p1;
      }
    }
    tmem_st_n(tS + c * (CW / 2), pp);   // over columns this thread has already read
    tmem_wait_st();
    tc_fence_before();
    arrive(c);
  }
}

// phase B: dS^T = P^T (dP^T + nD[q]) over this thread's 64 columns at tP,
// packed into the first 32 of them; arrive() once stored
template <class Arrive>
__device__ __forceinline__ void dkv_phase_b(uint32_t tP, uint32_t ldd, int debug,
                                            const float2 (&pf)[32], Arrive&& arrive) {
  uint32_t gv[2][32], dd[32];
  tmem_ld32(tP, gv[0]);
  tmem_ld32(tP + 32, gv[1]);
  tmem_wait_ld();
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    if (BWD_DBG(debug == 1 || debug == 2)) {
#pragma unroll
      for (int e = 0; e < 16; ++e) dd[hh * 16 + e] = gv[hh][2 * e];
    } else {
#pragma unroll
      for (int c4 = 0; c4 < 32; c4 += 4) {
        const float4 d4 = BWD_DBG(debug == 5) ? make_float4(0.f, 0.f, 0.f, 0.f)
                                              : ld_shared_f4(ldd + (hh * 32 + c4) * 4);   // -D per q
        const int pi = (hh * 32 + c4) / 2;
        const float2 t0 = fadd2(u2f2(gv[hh][c4], gv[hh][c4 + 1]), make_float2(d4.x, d4.y));
        const float2 t1 = fadd2(u2f2(gv[hh][c4 + 2], gv[hh][c4 + 3]), make_float2(d4.z, d4.w));
        const float2 r0 = fmul2(pf[pi], t0);
        const float2 r1 = fmul2(pf[pi + 1], t1);
        dd[pi] = pack_bf16(r0.x, r0.y);
        dd[pi + 1] = pack_bf16(r1.x, r1.y);
      }
    }
  }
  tmem_st32(tP, dd);
  tmem_wait_st();
  tc_fence_before();
  arrive();
}

template <int D>
__global__ void __launch_bounds__(384, 1)
bwd_dkv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG,
               const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV,
               const BwdParams p) {
  using C = DkvCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint8_t* sK = sm;
  uint8_t* sV = sK + C::KV_BYTES;
  uint8_t* sSlot = sV + C::KV_BYTES;          // Q tiles | dO tiles | nL/nD rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSlot + C::RING);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;                // Q(i), nD(i)
  uint64_t* q_empty = q_full + C::QSTAGES;    // after dK(i)
  uint64_t* g_full = q_empty + C::QSTAGES;    // dO(i), nL(i)
  uint64_t* g_empty = g_full + C::GSTAGES;    // after dV(i)
  uint64_t* s_full = g_empty + C::GSTAGES;    // S^T(i) in R1
  uint64_t* p_ready = s_full + 1;             // [kDkvChunks]: P^T(i) chunks in R1 (256 each)
  uint64_t* dp_full = p_ready + kDkvChunks;   // dP^T(i) in R2
  uint64_t* ds_ready = dp_full + 1;           // dS^T(i) packed in R2 (256 arrivals)
  uint64_t* dkv_done = ds_ready + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128, g = blockIdx.y;
  const int nsteps = p.G * p.tpq;

  if (C::PAD == 0 && (raw_u & 1023u)) __trap();   // SW128 tiles need 1024-byte alignment
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::QSTAGES; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < C::GSTAGES; ++s) {
      mbar_init(&g_full[s], 1);
      mbar_init(&g_empty[s], 1);
    }
    mbar_init(s_full, 1);
    for (int c = 0; c < kDkvChunks; ++c) mbar_init(&p_ready[c], kDkvArrivals);
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, kDkvArrivals);
    mbar_init(dkv_done, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // 12 warps: softmax warpgroups 0-1 hold P in fp32 between the phases (setmaxnreg
  // 224), warpgroup 2 = producer, MMA issuer and two idle warps (56).
  if (warp == 8) {
    // ------------------------------------------------------------ producer
    reg_dealloc<56>();
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmG);
      // L2 policy: this CTA's K/V tile is read once (evict first); the GQA
      // group's Q / dO / L / D are swept by every CTA of the group (evict last)
      const uint64_t once = l2_evict_first(), shared = l2_evict_last();
      mbar_arrive_expect_tx(kv_full, 2 * C::KV_BYTES);
      for (int pn = 0; pn < C::PANELS; ++pn) {
        tma_load_3d_hint(sK + pn * 128 * 128, &tmK, kv_full, pn * 64, n0, g, once);
        tma_load_3d_hint(sV + pn * 128 * 128, &tmV, kv_full, pn * 64, n0, g, once);
      }
      // in pipe order a Q slot frees (dK(i - QSTAGES)) before a dO slot (dV(i - GSTAGES))
      for (int i = 0; i < nsteps; ++i) {
        const int sq = i % C::QSTAGES, uq = i / C::QSTAGES;
        const int sg = i % C::GSTAGES, ug = i / C::GSTAGES;
        const int h = g * p.G + i / p.tpq, r0 = (i % p.tpq) * 128;
        const bool reload = !BWD_DBG((p.debug == 2 || p.debug == 3) && i >= C::QSTAGES);
        if (uq > 0) mbar_wait(&q_empty[sq], (uq - 1) & 1);
        DKV_STAMP(3, i, 0);
        if (!reload) {   // profiling: no reloads (stale data)
          mbar_arrive(&q_full[sq]);
        } else {
          uint8_t* qt = sSlot + sq * C::QT_BYTES;
          mbar_arrive_expect_tx(&q_full[sq], C::QT_BYTES + 512);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_3d_hint(qt + pn * 128 * 128, &tmQ, &q_full[sq], pn * 64, r0, h, shared);
          bulk_load_hint(sSlot + C::OFF_LD + sq * 512, p.Dp + (size_t)h * p.rows_pad + r0, 512,
                         &q_full[sq], shared);
        }
        if (ug > 0) mbar_wait(&g_empty[sg], (ug - 1) & 1);
        DKV_STAMP(3, i, 1);
        if (!reload || BWD_DBG((p.debug == 2 || p.debug == 3) && i >= C::GSTAGES)) {
          mbar_arrive(&g_full[sg]);
        } else {
          uint8_t* gt = sSlot + C::OFF_G + sg * C::QT_BYTES;
          mbar_arrive_expect_tx(&g_full[sg], C::QT_BYTES + 512);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_3d_hint(gt + pn * 128 * 128, &tmG, &g_full[sg], pn * 64, r0, h, shared);
          bulk_load_hint(sSlot + C::OFF_LL + sg * 512, p.Lp + (size_t)h * p.rows_pad + r0, 512,
                         &g_full[sg], shared);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------- MMA issuer (converged warp)
    reg_dealloc<56>();
    constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idKV = idesc_bf16(128, D, false, true);
    const uint64_t dk0 = umma_desc_sw128(smem_u32(sK), 0, 1024);
    const uint64_t dv0 = umma_desc_sw128(smem_u32(sV), 0, 1024);
    const uint64_t ds0 = umma_desc_sw128(smem_u32(sSlot), 0, 1024);        // K-major Q / dO
    const uint64_t dm0 = umma_desc_sw128(smem_u32(sSlot), 128 * 128, 1024);  // MN-major Q / dO
    auto qoff = [&](int i) { return (uint64_t)(((i % C::QSTAGES) * C::QT_BYTES) >> 4); };
    auto goff = [&](int i) {
      return (uint64_t)((C::OFF_G + (i % C::GSTAGES) * C::QT_BYTES) >> 4);
    };
    auto issue_st = [&](uint64_t a0, uint32_t col, uint64_t boff, uint64_t* bar) {
      // col R1: S^T = K Q^T ; col R2: dP^T = V dO^T   (M=128 kv, N=128 q, K=D)
      if (elect_one()) {
        const uint64_t b = ds0 + boff;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t o = ((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4;
          mma_bf16_ss(tmem + col, a0 + o, b + o, idS, kk > 0);
        }
        mma_commit(bar);
      }
      __syncwarp();
    };
    auto issue_acc = [&](int i, uint32_t acc_col, uint32_t a_col, uint64_t boff, int c) {
      // dV += P^T dO (a_col R1, dO) ; dK += dS^T Q (a_col R2, Q); chunk c
      if (elect_one()) {
        const uint64_t b = dm0 + boff;
#pragma unroll
        for (int j = 0; j < 8 / kDkvChunks; ++j) {
          const int kk = dkv_chunk_kk(c, j);
          mma_bf16_ts(tmem + acc_col, tmem + a_col + dkv_a_col(kk), b + ((kk * 16 * 128) >> 4),
                      idKV, (i > 0 || c > 0 || j > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
    mbar_wait(kv_full, 0);
    tc_fence_after();
    mbar_wait(&q_full[0], 0);
    tc_fence_after();
    issue_st(dk0, C::R1, qoff(0), s_full);
    mbar_wait(&g_full[0], 0);
    tc_fence_after();
    issue_st(dv0, C::R2, goff(0), dp_full);
    for (int i = 0; i < nsteps; ++i) {
      const uint32_t ph = i & 1;
#pragma unroll
      for (int c = 0; c < kDkvChunks; ++c) {                  // dV(i), as P^T chunks land
        mbar_wait(&p_ready[c], ph);
        DKV_STAMP(2, i, c);
        tc_fence_after();
        issue_acc(i, C::DV_COL, C::R1, goff(i), c);
      }
      commit(&g_empty[i % C::GSTAGES]);                       // dO(i) slot after dV(i)
      if (i + 1 < nsteps) {
        mbar_wait(&q_full[(i + 1) % C::QSTAGES], ((i + 1) / C::QSTAGES) & 1);
        DKV_STAMP(2, i, 4);
        tc_fence_after();
        issue_st(dk0, C::R1, qoff(i + 1), s_full);            // S^T(i+1) after dV(i) read R1
      }
      mbar_wait(ds_ready, ph);
      DKV_STAMP(2, i, 5);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < kDkvChunks; ++c) issue_acc(i, C::DK_COL, C::R2, qoff(i), c);   // dK(i)
      commit(&q_empty[i % C::QSTAGES]);                       // Q(i), nL / nD(i) after dK(i)
      if (i + 1 < nsteps) {
        mbar_wait(&g_full[(i + 1) % C::GSTAGES], ((i + 1) / C::GSTAGES) & 1);
        DKV_STAMP(2, i, 6);
        tc_fence_after();
        issue_st(dv0, C::R2, goff(i + 1), dp_full);           // dP^T(i+1)
      }
    }
    if (elect_one()) mma_commit(dkv_done);
    __syncwarp();
  } else if (warp >= 10) {
    reg_dealloc<56>();
  } else {
    // -------------- softmax: kv row per thread, 64 of the 128 query columns per wg
    reg_alloc<224>();
    const int wg = warp >> 2, q4 = warp & 3;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    for (int i = 0; i < nsteps; ++i) {
      const uint32_t ph = i & 1;
      const uint32_t ldl = smem_u32(sSlot + C::OFF_LL + (i % C::GSTAGES) * 512) + wg * 256;
      const uint32_t ldd = smem_u32(sSlot + C::OFF_LD + (i % C::QSTAGES) * 512) + wg * 256;
      mbar_wait(&g_full[i % C::GSTAGES], (i / C::GSTAGES) & 1);   // nL(i)
      mbar_wait(s_full, ph);
      if (q4 == 0) DKV_STAMP(wg, i, 0);
      tc_fence_after();
      float2 pf[32];     // P^T in fp32 for phase B
      auto arrive = [&](uint64_t* bar) {
        if constexpr (kDkvArrivals == 8) {   // one lane per warp after the warp converges
          __syncwarp();
          if (lane == 0) mbar_arrive(bar);
        } else {
          mbar_arrive(bar);
        }
      };
      dkv_phase_a<D>(tl + C::R1 + wg * 64, ldl, sc2, p.debug, pf, [&](int c) {
        arrive(&p_ready[c]);
        if (q4 == 0) DKV_STAMP(wg, i, 1 + c);
      });
      mbar_wait(dp_full, ph);
      if (q4 == 0) DKV_STAMP(wg, i, 5);
      tc_fence_after();
      dkv_phase_b(tl + C::R2 + wg * 64, ldd, p.debug, pf, [&]() { arrive(ds_ready); });
      if (q4 == 0) DKV_STAMP(wg, i, 6);
    }
    // epilogue: warpgroup 0 drains dV, warpgroup 1 drains scale * dK.  Each warp
    // stages its 32 rows in the (now idle) Q/dO ring with the 128B swizzle, then
    // either stores them row-contiguously (whole 128-byte lines per 8 lanes) or,
    // when accumulating, hands them to TMA as 32x32 fp32 reduce-add boxes (the
    // add happens in L2, no read-modify-write through the SM).
    mbar_wait(dkv_done, 0);
    tc_fence_after();
    const uint32_t col = wg ? C::DK_COL : C::DV_COL;
    const float mul = wg ? p.scale : 1.f;
    uint8_t* stage = sSlot + warp * (32 * D * 4);
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tl + col + c * 32, v);
      tmem_wait_ld();
      const uint32_t rowbase = smem_u32(stage + c * 4096) + lane * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        st_shared_v4(rowbase + ((q ^ (lane & 7)) << 4),
                     __float_as_uint(__uint_as_float(v[4 * q]) * mul),
                     __float_as_uint(__uint_as_float(v[4 * q + 1]) * mul),
                     __float_as_uint(__uint_as_float(v[4 * q + 2]) * mul),
                     __float_as_uint(__uint_as_float(v[4 * q + 3]) * mul));
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (!p.accumulate && p.out_bf16 && !BWD_DBG(p.debug == 4)) {
      // overwrite in bf16: each 8-lane group packs 64 columns of one row (two
      // staged 32-column chunks) into one full 128-byte line
      __nv_bfloat16* base = static_cast<__nv_bfloat16*>(wg ? p.dk_ptr : p.dv_ptr);
      const int64_t hs = wg ? p.dk_hs : p.dv_hs, rs = wg ? p.dk_rs : p.dv_rs;
#pragma unroll 1
      for (int cp = 0; cp < D / 64; ++cp) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + (lane >> 3), q8 = lane & 7;
          const int c = cp * 2 + (q8 >> 2), qq = (q8 & 3) * 2;
          const uint32_t rb = smem_u32(stage + c * 4096) + rr * 128;
          const float4 a = ld_shared_f4(rb + ((qq ^ (rr & 7)) << 4));
          const float4 b = ld_shared_f4(rb + (((qq + 1) ^ (rr & 7)) << 4));
          const int grow = n0 + q4 * 32 + rr;
          if (grow < p.rows_kv)
            *reinterpret_cast<uint4*>(base + g * hs + (int64_t)grow * rs + cp * 64 + q8 * 8) =
                make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y),
                           pack_bf16(b.z, b.w));
        }
      }
    } else if (!p.accumulate && !BWD_DBG(p.debug == 4)) {   // 4: profiling, no drain
      // overwrite: each 8-lane group stores one full 128-byte row segment
      // (STG.128, whole lines); measured ~5 % faster than TMA tensor stores here
      float* base = static_cast<float*>(wg ? p.dk_ptr : p.dv_ptr);
      const int64_t hs = wg ? p.dk_hs : p.dv_hs, rs = wg ? p.dk_rs : p.dv_rs;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + (lane >> 3), q = lane & 7;
          const int grow = n0 + q4 * 32 + rr;
          const float4 val = ld_shared_f4(smem_u32(stage + c * 4096) + rr * 128 +
                                          ((q ^ (rr & 7)) << 4));
          if (grow < p.rows_kv)
            *reinterpret_cast<float4*>(base + g * hs + (int64_t)grow * rs + c * 32 + q * 4) = val;
        }
      }
    } else if (p.accumulate && lane == 0 && !BWD_DBG(p.debug == 4)) {   // reduce-add in L2
      const CUtensorMap* m = wg ? &tmDK : &tmDV;
      const uint64_t pol = l2_evict_first();   // written once, not re-read here
      for (int c = 0; c < D / 32; ++c)
        tma_reduce_add_3d(m, stage + c * 4096, c * 32, n0 + q4 * 32, g, pol);
      bulk_commit();
      bulk_wait_read0();
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#ifdef LVX_DKV2_PROBE   // CTA-pair variant: measured 19 % slower, not in the product build
// ================================================================ dK / dV on CTA pairs
// The same algorithm as bwd_dkv_kernel on cta_group::2 (M = 256 KV rows per
// pair, 128 per CTA): the leader issues S^T = K Q^T, dP^T = V dO^T (SS) and
// dV += P^T dO, dK += dS^T Q (TS) for the pair.  B splits by N (cute's 2x1SM
// layouts), so each CTA stages the query HALF of Q / dO (64 rows, B of S^T /
// dP^T) and the d HALF (128 rows x 64 cols, B of dV / dK): per-CTA operand
// reads drop from 192 to 128 KB per 128-row step, the SMEM ceiling of the
// 1-CTA kernel.  Softmax, epilogue and TMEM layout are the 1-CTA kernel's;
// each CTA's softmax warps arrive on the LEADER's p_ready / ds_ready (16).
// Registers: warpgroup 2 -> 72 (the issuer keeps more descriptors than the
// 1-CTA one), softmax -> 216: (168 - 72) x 128 >= (216 - 168) x 256, else
// setmaxnreg.inc waits forever for registers nobody frees.
template <int D>
struct Dkv2Cfg {
  static constexpr int PANELS = D / 64;
  static constexpr int KV_BYTES = 128 * D * 2;             // own K (or V) rows
  static constexpr int QH_BYTES = 64 * D * 2;              // query half: 64 rows x D
  static constexpr int DH_BYTES = 128 * 64 * 2;            // d half: 128 rows x 64 cols
  static constexpr int OFF_QQ = 0, OFF_GQ = QH_BYTES, OFF_QD = 2 * QH_BYTES,
                       OFF_GD = 2 * QH_BYTES + DH_BYTES, OFF_LD = 2 * QH_BYTES + 2 * DH_BYTES;
  static constexpr int SLOT = ((OFF_LD + 1024 + 1023) / 1024) * 1024;
  static constexpr int STAGES = 2;
  static constexpr int QT_BYTES = QH_BYTES;   // (epilogue staging uses the slots only)
  static constexpr int NBAR = 1 + 3 * STAGES + 4 + kDkvChunks;
  static constexpr int SMEM = 1024 + 2 * KV_BYTES + STAGES * SLOT + NBAR * 8 + 16;
  static constexpr int R1 = 0, R2 = 128, DV_COL = 256, DK_COL = 256 + D;
  static_assert(D == 128, "the d halves are one 128-byte panel each");
  static_assert(8 * 32 * D * 4 <= STAGES * SLOT, "epilogue staging must fit the Q/dO ring");
};

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
bwd_dkv2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG,
                const __grid_constant__ CUtensorMap tmQh, const __grid_constant__ CUtensorMap tmGh,
                const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV,
                const BwdParams p) {
  using C = Dkv2Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint8_t* sK = sm;
  uint8_t* sV = sK + C::KV_BYTES;
  uint8_t* sSlot = sV + C::KV_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSlot + C::STAGES * C::SLOT);
  uint64_t* kv_full = bars;                   // leader: K / V of both CTAs
  uint64_t* qd_full = bars + 1;               // leader: Q / dO halves of both CTAs
  uint64_t* ld_full = qd_full + C::STAGES;    // local: this CTA's nL / nD rows
  uint64_t* qd_empty = ld_full + C::STAGES;   // both (multicast commit)
  uint64_t* s_full = qd_empty + C::STAGES;    // both
  uint64_t* p_ready = s_full + 1;             // leader [kDkvChunks]: 512 arrivals each
  uint64_t* dp_full = p_ready + kDkvChunks;   // both
  uint64_t* ds_ready = dp_full + 1;           // leader: 512
  uint64_t* dkv_done = ds_ready + 1;          // both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int n0 = (blockIdx.x >> 1) * 256 + (int)rank * 128, g = blockIdx.y;
  const int nsteps = p.G * p.tpq;
  // one arrival per softmax thread of both CTAs on the leader's copy of bar (512)
  auto arrive_pair = [&](uint64_t* bar) {
    if (rank == 0) mbar_arrive(bar);
    else mbar_arrive_cluster(leader_addr(bar));
  };

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&qd_full[s], 1);
      mbar_init(&ld_full[s], 1);
      mbar_init(&qd_empty[s], 1);
    }
    mbar_init(s_full, 1);
    for (int c = 0; c < kDkvChunks; ++c) mbar_init(&p_ready[c], 512);
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, 512);
    mbar_init(dkv_done, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ producer (both CTAs)
    reg_dealloc<72>();
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmQh);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmG);
      tma_prefetch(&tmGh);
      const uint64_t once = l2_evict_first(), shared = l2_evict_last();
      if (rank == 0) mbar_arrive_expect_tx(kv_full, 2 * 2 * C::KV_BYTES);
      const uint32_t lkv = leader_addr(kv_full);
      for (int pn = 0; pn < C::PANELS; ++pn) {
        tma2_load_3d(sK + pn * 128 * 128, &tmK, lkv, pn * 64, n0, g, once);
        tma2_load_3d(sV + pn * 128 * 128, &tmV, lkv, pn * 64, n0, g, once);
      }
      for (int i = 0; i < nsteps; ++i) {
        const int s = i % C::STAGES, u = i / C::STAGES;
        if (u > 0) mbar_wait(&qd_empty[s], (u - 1) & 1);
        const int h = g * p.G + i / p.tpq, r0 = (i % p.tpq) * 128;
        uint8_t* slot = sSlot + s * C::SLOT;
        if (rank == 0)
          mbar_arrive_expect_tx(&qd_full[s], 2 * (2 * C::QH_BYTES + 2 * C::DH_BYTES));
        const uint32_t lq = leader_addr(&qd_full[s]);
        for (int pn = 0; pn < C::PANELS; ++pn) {   // query half: rows r0 + 64 rank
          tma2_load_3d(slot + C::OFF_QQ + pn * 64 * 128, &tmQh, lq, pn * 64,
                       r0 + 64 * (int)rank, h, shared);
          tma2_load_3d(slot + C::OFF_GQ + pn * 64 * 128, &tmGh, lq, pn * 64,
                       r0 + 64 * (int)rank, h, shared);
        }
        // d half: all 128 query rows, columns [64 rank, 64 rank + 64)
        tma2_load_3d(slot + C::OFF_QD, &tmQ, lq, 64 * (int)rank, r0, h, shared);
        tma2_load_3d(slot + C::OFF_GD, &tmG, lq, 64 * (int)rank, r0, h, shared);
        const size_t off = (size_t)h * p.rows_pad + r0;
        mbar_arrive_expect_tx(&ld_full[s], 1024);
        bulk_load_hint(slot + C::OFF_LD, p.Lp + off, 512, &ld_full[s], shared);
        bulk_load_hint(slot + C::OFF_LD + 512, p.Dp + off, 512, &ld_full[s], shared);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------- MMA issuer (leader, converged warp)
    reg_dealloc<72>();
    if (rank == 0) {
      constexpr uint32_t idS = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idKV = idesc_bf16(256, D, false, true);
      const uint64_t dk0 = umma_desc_sw128(smem_u32(sK), 0, 1024);
      const uint64_t dv0 = umma_desc_sw128(smem_u32(sV), 0, 1024);
      const uint64_t dh0 = umma_desc_sw128(smem_u32(sSlot), 0, 1024);   // query halves, K-major
      const uint64_t dm0 = umma_desc_sw128(smem_u32(sSlot), 0, 1024);   // d halves, MN-major
      auto qslot = [&](int i) { return (uint64_t)(((i % C::STAGES) * C::SLOT) >> 4); };
      auto issue_st = [&](int i, uint64_t a0, uint32_t col, uint32_t boff, uint64_t* bar) {
        // col R1: S^T = K Q^T ; col R2: dP^T = V dO^T   (M=256 kv, N=128 q, K=D)
        if (elect_one()) {
          const uint64_t b = dh0 + qslot(i) + (boff >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oa = ((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4;
            const uint32_t ob = ((kk >> 2) * (64 * 128) + (kk & 3) * 32) >> 4;
            mma2_bf16_ss(tmem + col, a0 + oa, b + ob, idS, kk > 0);
          }
          mma2_commit_mc(bar);
        }
        __syncwarp();
      };
      auto issue_acc = [&](int i, uint32_t acc_col, uint32_t a_col, uint32_t boff, int c) {
        // dV += P^T dO (a_col R1, d half of dO) ; dK += dS^T Q (a_col R2, d half of Q)
        if (elect_one()) {
          const uint64_t b = dm0 + qslot(i) + (boff >> 4);
#pragma unroll
          for (int j = 0; j < 8 / kDkvChunks; ++j) {
            const int kk = dkv_chunk_kk(c, j);
            mma2_bf16_ts(tmem + acc_col, tmem + a_col + dkv_a_col(kk),
                         b + ((kk * 16 * 128) >> 4), idKV, (i > 0 || c > 0 || j > 0) ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      mbar_wait_cluster(kv_full, 0);
      tc_fence_after();
      mbar_wait_cluster(&qd_full[0], 0);
      tc_fence_after();
      issue_st(0, dk0, C::R1, C::OFF_QQ, s_full);
      issue_st(0, dv0, C::R2, C::OFF_GQ, dp_full);
      for (int i = 0; i < nsteps; ++i) {
        const uint32_t ph = i & 1;
#pragma unroll
        for (int c = 0; c < kDkvChunks; ++c) {                 // dV(i), as P^T chunks land
          mbar_wait_cluster(&p_ready[c], ph);
          tc_fence_after();
          issue_acc(i, C::DV_COL, C::R1, C::OFF_GD, c);
        }
        if (i + 1 < nsteps) {
          mbar_wait_cluster(&qd_full[(i + 1) % C::STAGES], ((i + 1) / C::STAGES) & 1);
          tc_fence_after();
          issue_st(i + 1, dk0, C::R1, C::OFF_QQ, s_full);      // S^T(i+1)
        }
        mbar_wait_cluster(ds_ready, ph);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kDkvChunks; ++c) issue_acc(i, C::DK_COL, C::R2, C::OFF_QD, c);   // dK(i)
        if (elect_one()) mma2_commit_mc(&qd_empty[i % C::STAGES]);
        __syncwarp();
        if (i + 1 < nsteps) issue_st(i + 1, dv0, C::R2, C::OFF_GQ, dp_full);   // dP^T(i+1)
      }
      if (elect_one()) mma2_commit_mc(dkv_done);
      __syncwarp();
    }
  } else if (warp >= 10) {
    reg_dealloc<72>();
  } else {
    // -------------- softmax: kv row per thread, 64 of the 128 query columns per wg
    reg_alloc<216>();
    const int wg = warp >> 2, q4 = warp & 3;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    for (int i = 0; i < nsteps; ++i) {
      const int s = i % C::STAGES;
      const uint32_t ph = i & 1;
      const uint32_t lds = smem_u32(sSlot + s * C::SLOT + C::OFF_LD) + wg * 256;
      // phase A: P^T = exp2(S^T * c + nL[q]), 32 columns at a time
      mbar_wait(&ld_full[s], (i / C::STAGES) & 1);   // this CTA's nL / nD rows
      mbar_wait(s_full, ph);
      tc_fence_after();
      float2 pf[32];     // P^T in fp32 for phase B
      dkv_phase_a<D>(tl + C::R1 + wg * 64, lds, sc2, p.debug, pf,
                  [&](int hh) { arrive_pair(&p_ready[hh]); });
      mbar_wait(dp_full, ph);
      tc_fence_after();
      dkv_phase_b(tl + C::R2 + wg * 64, lds + 512, p.debug, pf, [&]() { arrive_pair(ds_ready); });
    }
    // epilogue (as bwd_dkv_kernel): this CTA's 128 rows, staged in its Q/dO ring
    mbar_wait(dkv_done, 0);
    tc_fence_after();
    const uint32_t col = wg ? C::DK_COL : C::DV_COL;
    const float mul = wg ? p.scale : 1.f;
    uint8_t* stage = sSlot + warp * (32 * D * 4);
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tl + col + c * 32, v);
      tmem_wait_ld();
      const uint32_t rowbase = smem_u32(stage + c * 4096) + lane * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        st_shared_v4(rowbase + ((q ^ (lane & 7)) << 4),
                     __float_as_uint(__uint_as_float(v[4 * q]) * mul),
                     __float_as_uint(__uint_as_float(v[4 * q + 1]) * mul),
                     __float_as_uint(__uint_as_float(v[4 * q + 2]) * mul),
                     __float_as_uint(__uint_as_float(v[4 * q + 3]) * mul));
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (!p.accumulate && p.out_bf16 && !BWD_DBG(p.debug == 4)) {
      // overwrite in bf16: each 8-lane group packs 64 columns of one row (two
      // staged 32-column chunks) into one full 128-byte line
      __nv_bfloat16* base = static_cast<__nv_bfloat16*>(wg ? p.dk_ptr : p.dv_ptr);
      const int64_t hs = wg ? p.dk_hs : p.dv_hs, rs = wg ? p.dk_rs : p.dv_rs;
#pragma unroll 1
      for (int cp = 0; cp < D / 64; ++cp) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + (lane >> 3), q8 = lane & 7;
          const int c = cp * 2 + (q8 >> 2), qq = (q8 & 3) * 2;
          const uint32_t rb = smem_u32(stage + c * 4096) + rr * 128;
          const float4 a = ld_shared_f4(rb + ((qq ^ (rr & 7)) << 4));
          const float4 b = ld_shared_f4(rb + (((qq + 1) ^ (rr & 7)) << 4));
          const int grow = n0 + q4 * 32 + rr;
          if (grow < p.rows_kv)
            *reinterpret_cast<uint4*>(base + g * hs + (int64_t)grow * rs + cp * 64 + q8 * 8) =
                make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y),
                           pack_bf16(b.z, b.w));
        }
      }
    } else if (!p.accumulate && !BWD_DBG(p.debug == 4)) {   // 4: profiling, no drain
      // overwrite: each 8-lane group stores one full 128-byte row segment
      // (STG.128, whole lines); measured ~5 % faster than TMA tensor stores here
      float* base = static_cast<float*>(wg ? p.dk_ptr : p.dv_ptr);
      const int64_t hs = wg ? p.dk_hs : p.dv_hs, rs = wg ? p.dk_rs : p.dv_rs;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + (lane >> 3), q = lane & 7;
          const int grow = n0 + q4 * 32 + rr;
          const float4 val = ld_shared_f4(smem_u32(stage + c * 4096) + rr * 128 +
                                          ((q ^ (rr & 7)) << 4));
          if (grow < p.rows_kv)
            *reinterpret_cast<float4*>(base + g * hs + (int64_t)grow * rs + c * 32 + q * 4) = val;
        }
      }
    } else if (p.accumulate && lane == 0 && !BWD_DBG(p.debug == 4)) {   // reduce-add in L2
      const CUtensorMap* m = wg ? &tmDK : &tmDV;
      const uint64_t pol = l2_evict_first();   // written once, not re-read here
      for (int c = 0; c < D / 32; ++c)
        tma_reduce_add_3d(m, stage + c * 4096, c * 32, n0 + q4 * 32, g, pol);
      bulk_commit();
      bulk_wait_read0();
    }
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

#endif  // LVX_DKV2_PROBE

// ================================================================ dQ kernel
// Q-parallel, one 128-row query tile per CTA, split over the KV block in
// 128-row steps.  Q and dO are copied once into TMEM so that all three MMAs
// read A from TMEM (TS) and SMEM holds only a 3-stage K/V ring.  TMEM:
//   [0,128) S(j)   [128,256) dP(j), then dS(j) packed bf16   [256,256+D) dQ
//   [384,448) Q    [448,512) dO          (bf16 pairs; D = 128)
// Two softmax warpgroups split the 128 kv columns of a step.  Phase A turns
// S into P (kept packed in registers) and releases S(j+1); phase B turns dP
// into dS over dP and releases dQ(j) -> dP(j+1) (tensor-pipe order).
template <int D>
struct DqCfg {
  static constexpr int PANELS = D / 64;
  static constexpr int Q_BYTES = 128 * D * 2;
  static constexpr int KVT_BYTES = 128 * D * 2;
  static constexpr int SLOT = 2 * KVT_BYTES;             // K | V, also Q | dO staging
  static constexpr int STAGES = D == 128 ? 3 : 6;
  static constexpr int NBAR = 2 + 2 * STAGES + 6;
  static constexpr int SMEM = 1024 + STAGES * SLOT + NBAR * 8 + 16;
  static constexpr int S_COL = 0, DP_COL = 128, DQ_COL = 256, Q_COL = 384,
                       G_COL = 384 + D / 2;
  static constexpr int QSLOT = STAGES - 1;                  // where Q / dO are staged
};

template <int D>
__global__ void __launch_bounds__(320, 1)
bwd_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmG,
              const BwdParams p) {
  using C = DqCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint8_t* sKV = sm;                          // STAGES x (K | V)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::STAGES * C::SLOT);
  uint64_t* qd_full = bars;                   // Q / dO staged in slot QSLOT
  uint64_t* q_ready = bars + 1;               // Q / dO copied into TMEM (256)
  uint64_t* kv_full = bars + 2;
  uint64_t* kv_empty = kv_full + C::STAGES;
  uint64_t* s_full = kv_empty + C::STAGES;    // S(j) in TMEM
  uint64_t* s_read = s_full + 1;              // softmax has read S(j) (256)
  uint64_t* dp_full = s_read + 1;             // dP(j) in TMEM
  uint64_t* ds_full = dp_full + 1;            // dS(j) packed over dP (256)
  uint64_t* dq_done = ds_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tt = blockIdx.x, split = blockIdx.y, g = blockIdx.z;
  const int kv_t0 = split * p.tiles_per_split;
  const int nt = min(p.n_tiles, kv_t0 + p.tiles_per_split) - kv_t0;
  const int qh = g * p.G + tt / p.tpq, row0 = (tt % p.tpq) * 128;

  if (threadIdx.x == 0) {
    mbar_init(qd_full, 1);
    mbar_init(q_ready, 256);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_read, 256);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmG);
      uint8_t* qs = sKV + C::QSLOT * C::SLOT;
      mbar_arrive_expect_tx(qd_full, 2 * C::Q_BYTES);
      for (int pn = 0; pn < C::PANELS; ++pn) {
        tma_load_3d(qs + pn * 128 * 128, &tmQ, qd_full, pn * 64, row0, qh);
        tma_load_3d(qs + C::Q_BYTES + pn * 128 * 128, &tmG, qd_full, pn * 64, row0, qh);
      }
      for (int j = 0; j < nt; ++j) {
        const int s = j % C::STAGES, u = j / C::STAGES;
        if (u > 0) mbar_wait(&kv_empty[s], (u - 1) & 1);
        else if (s == C::QSLOT) mbar_wait(q_ready, 0);   // Q / dO have left this slot
        DQ_STAMP(3, j, 0);
        uint8_t* slot = sKV + s * C::SLOT;
        mbar_arrive_expect_tx(&kv_full[s], C::SLOT);
        const int kr = (kv_t0 + j) * 128;
        for (int pn = 0; pn < C::PANELS; ++pn) {
          tma_load_3d(slot + pn * 128 * 128, &tmK, &kv_full[s], pn * 64, kr, g);
          tma_load_3d(slot + C::KVT_BYTES + pn * 128 * 128, &tmV, &kv_full[s], pn * 64, kr, g);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------- MMA issuer (converged warp)
    constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idQ = idesc_bf16(128, D, false, true);
    const uint64_t dkv0 = umma_desc_sw128(smem_u32(sKV), 0, 1024);          // K-major K / V
    const uint64_t dkm0 = umma_desc_sw128(smem_u32(sKV), 128 * 128, 1024);  // MN-major K
    auto kslot = [&](int j) { return (uint64_t)(((j % C::STAGES) * C::SLOT) >> 4); };
    auto issue_sdp = [&](int j, uint32_t a_col, uint32_t col, uint32_t boff, uint64_t* bar) {
      if (elect_one()) {   // S = Q K^T / dP = dO V^T, A (Q / dO) from TMEM
        const uint64_t b = dkv0 + kslot(j) + (boff >> 4);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t o = ((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4;
          mma_bf16_ts(tmem + col, tmem + a_col + kk * 8, b + o, idS, kk > 0);
        }
        mma_commit(bar);
      }
      __syncwarp();
    };
    auto wait_kv = [&](int j) {
      mbar_wait(&kv_full[j % C::STAGES], (j / C::STAGES) & 1);
      tc_fence_after();
    };
    mbar_wait(q_ready, 0);
    tc_fence_after();
    wait_kv(0);
    issue_sdp(0, C::Q_COL, C::S_COL, 0, s_full);
    issue_sdp(0, C::G_COL, C::DP_COL, C::KVT_BYTES, dp_full);
    for (int j = 0; j < nt; ++j) {
      const uint32_t ph = j & 1;
      if (j + 1 < nt) {
        wait_kv(j + 1);
        DQ_STAMP(2, j, 0);
        mbar_wait(s_read, ph);
        DQ_STAMP(2, j, 1);
        tc_fence_after();
        issue_sdp(j + 1, C::Q_COL, C::S_COL, 0, s_full);            // S(j+1)
      }
      mbar_wait(ds_full, ph);
      DQ_STAMP(2, j, 2);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t b = dkm0 + kslot(j);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)   // dQ += dS K (A = dS packed over dP)
          mma_bf16_ts(tmem + C::DQ_COL, tmem + C::DP_COL + dkv_a_col(kk),
                      b + ((kk * 16 * 128) >> 4), idQ, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&kv_empty[j % C::STAGES]);
      }
      __syncwarp();
      if (j + 1 < nt) issue_sdp(j + 1, C::G_COL, C::DP_COL, C::KVT_BYTES, dp_full);   // dP(j+1)
    }
    if (elect_one()) mma_commit(dq_done);
    __syncwarp();
  } else {
    // ------------- softmax: query row per thread, 64 of the 128 kv columns per wg
    const int wg = warp >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    {   // stage Q (wg 0) / dO (wg 1) rows into TMEM as bf16 pairs (A operands)
      mbar_wait(qd_full, 0);
      const uint32_t base = smem_u32(sKV + C::QSLOT * C::SLOT + wg * C::Q_BYTES) + r * 128;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {      // one 64-column (128 B) panel per chunk
        uint32_t v[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {          // 16-byte chunks, 128B swizzle
          uint32_t a, b2, c2, d2;
          const uint32_t addr = base + c * 128 * 128 + ((q ^ (r & 7)) << 4);
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(a), "=r"(b2), "=r"(c2), "=r"(d2) : "r"(addr));
          v[q * 4] = a; v[q * 4 + 1] = b2; v[q * 4 + 2] = c2; v[q * 4 + 3] = d2;
        }
        tmem_st32(tl + (wg ? C::G_COL : C::Q_COL) + c * 32, v);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(q_ready);
    }
    const int row = row0 + r;
    const size_t prow = (size_t)qh * p.rows_pad + row;
    const float2 nl2 = make_float2(p.Lp[prow], p.Lp[prow]);   // -L log2 e
    const float2 nd2 = make_float2(p.Dp[prow], p.Dp[prow]);   // -D
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    for (int j = 0; j < nt; ++j) {
      const uint32_t ph = j & 1;
      const int nvalid = min(128, p.rows_kv - (kv_t0 + j) * 128) - wg * 64;
      // phase A: P = exp2(S*c + nL) in registers.  S(j) is released as soon as
      // it is loaded (P never goes back to TMEM here), so S(j+1) overlaps the
      // exponentials instead of waiting for them.
      mbar_wait(s_full, ph);
      if (q4 == 0) DQ_STAMP(wg, j, 0);
      tc_fence_after();
      uint32_t sv[2][32];
      tmem_ld32(tl + C::S_COL + wg * 64, sv[0]);
      tmem_ld32(tl + C::S_COL + wg * 64 + 32, sv[1]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_read);
      float2 pf[32];   // P in fp32 until phase B (only dS feeds an MMA here)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (BWD_DBG(p.debug == 1)) {
#pragma unroll
          for (int e = 0; e < 16; ++e) pf[hh * 16 + e] = u2f2(sv[hh][2 * e], sv[hh][2 * e + 1]);
          continue;
        }
        // full and ragged KV steps are separate instantiations (otherwise the
        // column mask is if-converted into selects on every element)
        auto pa = [&](auto masked) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int c = hh * 32 + e;
            float2 x = ffma2(u2f2(sv[hh][e], sv[hh][e + 1]), sc2, nl2);
            if constexpr (decltype(masked)::value) {
              x.x = c < nvalid ? x.x : -INFINITY;
              x.y = c + 1 < nvalid ? x.y : -INFINITY;
            }
            const float2 pq = (((c / 2) * 3) % 8) < kPolyPairsD<D> && !decltype(masked)::value
                                  ? ex2_poly2(x)
                                  : make_float2(ex2(x.x), ex2(x.y));
            pf[c / 2] = pq;
          }
        };
        if (nvalid < 64)
          pa(std::true_type{});
        else
          pa(std::false_type{});
      }
      if (q4 == 0) DQ_STAMP(wg, j, 1);
      // phase B: dS = P (dP + nD), packed into the first half of this
      // warpgroup's own dP columns (the two warpgroups never share columns)
      mbar_wait(dp_full, ph);
      if (q4 == 0) DQ_STAMP(wg, j, 2);
      tc_fence_after();
      uint32_t gv[2][32], dd[32];
      tmem_ld32(tl + C::DP_COL + wg * 64, gv[0]);
      tmem_ld32(tl + C::DP_COL + wg * 64 + 32, gv[1]);
      tmem_wait_ld();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (BWD_DBG(p.debug == 1)) {
#pragma unroll
          for (int e = 0; e < 16; ++e) dd[hh * 16 + e] = gv[hh][2 * e];
          continue;
        }
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int pi = (hh * 32 + e) / 2;
          const float2 r2 = fmul2(pf[pi], fadd2(u2f2(gv[hh][e], gv[hh][e + 1]), nd2));
          dd[pi] = pack_bf16(r2.x, r2.y);
        }
      }
      tmem_st32(tl + C::DP_COL + wg * 64, dd);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (q4 == 0) DQ_STAMP(wg, j, 3);
    }
    // epilogue: warpgroup w drains dQ columns [w*D/2, (w+1)*D/2) of its rows
    mbar_wait(dq_done, 0);
    tc_fence_after();
    const bool valid = row < p.rows_q;
    float* dst = p.ws_dq + (((size_t)split * p.hq + qh) * p.rows_q + row) * D;
#pragma unroll 1
    for (int c = wg * (D / 64); c < (wg + 1) * (D / 64); ++c) {
      uint32_t v[32];
      tmem_ld32(tl + C::DQ_COL + c * 32, v);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + e) =
              make_float4(__uint_as_float(v[e]) * p.scale, __uint_as_float(v[e + 1]) * p.scale,
                          __uint_as_float(v[e + 2]) * p.scale, __uint_as_float(v[e + 3]) * p.scale);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#ifdef LVX_DQ2_PROBE   // CTA-pair variant: measured 20-29 % slower, not in the product build
// ================================================================ dQ on CTA pairs
// bwd_dq_kernel on cta_group::2: a pair = two query tiles of the same GQA
// group and KV split (M = 256 query rows, 128 per CTA); the leader issues
// S = Q K^T, dP = dO V^T and dQ += dS K for both.  B splits by N, so each CTA
// stages only its half of every B operand per 128-row KV step: K and V rows
// [64 rank, 64 rank + 64) (B of S / dP, both 64-column panels) and the d-panel
// `rank` of K over all 128 rows (B of dQ) — 48 KB instead of 64 KB, which
// takes the per-SM L2 -> SMEM stream (the 1-CTA kernel's bound) below the
// tensor rate.  The overlap of the two K halves is loaded twice: the leader's
// descriptors address both CTAs' SMEM at the same offsets.  Softmax, TMEM
// layout and epilogue are the 1-CTA kernel's; each CTA's softmax threads
// arrive on the LEADER's q_ready / s_read / ds_full (512).
struct Dq2Cfg {
  static constexpr int D = 128;
  static constexpr int Q_BYTES = 128 * D * 2;
  static constexpr int HALF = 64 * 128;                        // 64 rows x one 128-byte panel
  static constexpr int OFF_SB = 0, OFF_QB = 2 * HALF, OFF_VB = 4 * HALF;
  static constexpr int SLOT = 6 * HALF;                        // 48 KB
  static constexpr int STAGES = 4;
  static constexpr int QSLOT = 2;                              // Q | dO staged over slots 2-3
  static constexpr int NBAR = 3 + 2 * STAGES + 5;
  static constexpr int SMEM = 1024 + STAGES * SLOT + NBAR * 8 + 16;
  static constexpr int S_COL = 0, DP_COL = 128, DQ_COL = 256, Q_COL = 384, G_COL = 448;
  static_assert((STAGES - QSLOT) * SLOT >= 2 * Q_BYTES, "Q / dO staging must fit");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
bwd_dq2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmKh, const __grid_constant__ CUtensorMap tmVh,
               const __grid_constant__ CUtensorMap tmG, const BwdParams p) {
  using C = Dq2Cfg;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint8_t* sKV = sm;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::STAGES * C::SLOT);
  uint64_t* qd_full = bars;                   // local: Q / dO staged
  uint64_t* q_local = bars + 1;               // local: this CTA's Q / dO in TMEM (256)
  uint64_t* q_ready = bars + 2;               // leader: both CTAs' Q / dO in TMEM (512)
  uint64_t* kv_full = bars + 3;               // leader: both CTAs' K / V halves
  uint64_t* kv_empty = kv_full + C::STAGES;   // both (multicast commit)
  uint64_t* s_full = kv_empty + C::STAGES;    // both
  uint64_t* s_read = s_full + 1;              // leader (512)
  uint64_t* dp_full = s_read + 1;             // both
  uint64_t* ds_full = dp_full + 1;            // leader (512)
  uint64_t* dq_done = ds_full + 1;            // both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int tt = blockIdx.x, split = blockIdx.y, g = blockIdx.z;
  const int kv_t0 = split * p.tiles_per_split;
  const int nt = min(p.n_tiles, kv_t0 + p.tiles_per_split) - kv_t0;
  const int qh = g * p.G + tt / p.tpq, row0 = (tt % p.tpq) * 128;
  auto arrive_pair = [&](uint64_t* bar) {
    if (rank == 0) mbar_arrive(bar);
    else mbar_arrive_cluster(leader_addr(bar));
  };

  if (threadIdx.x == 0) {
    mbar_init(qd_full, 1);
    mbar_init(q_local, 256);
    mbar_init(q_ready, 512);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_read, 512);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 512);
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmKh);
      tma_prefetch(&tmVh);
      tma_prefetch(&tmG);
      uint8_t* qs = sKV + C::QSLOT * C::SLOT;
      mbar_arrive_expect_tx(qd_full, 2 * C::Q_BYTES);
      for (int pn = 0; pn < 2; ++pn) {
        tma_load_3d(qs + pn * 128 * 128, &tmQ, qd_full, pn * 64, row0, qh);
        tma_load_3d(qs + C::Q_BYTES + pn * 128 * 128, &tmG, qd_full, pn * 64, row0, qh);
      }
      const uint64_t pol = l2_evict_last();   // the pair's K / V step is read by 64 CTAs
      for (int j = 0; j < nt; ++j) {
        const int s = j % C::STAGES, u = j / C::STAGES;
        if (u > 0) mbar_wait(&kv_empty[s], (u - 1) & 1);
        else if (s >= C::QSLOT) mbar_wait(q_local, 0);   // Q / dO have left these slots
        uint8_t* slot = sKV + s * C::SLOT;
        if (rank == 0) mbar_arrive_expect_tx(&kv_full[s], 2 * C::SLOT);
        const uint32_t lb = leader_addr(&kv_full[s]);
        const int kr = (kv_t0 + j) * 128, mine = kr + 64 * (int)rank;
        for (int pn = 0; pn < 2; ++pn) {
          tma2_load_3d(slot + C::OFF_SB + pn * C::HALF, &tmKh, lb, pn * 64, mine, g, pol);
          tma2_load_3d(slot + C::OFF_VB + pn * C::HALF, &tmVh, lb, pn * 64, mine, g, pol);
        }
        tma2_load_3d(slot + C::OFF_QB, &tmK, lb, 64 * (int)rank, kr, g, pol);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------- MMA issuer (leader, converged warp)
    if (rank == 0) {
      constexpr uint32_t idS = idesc_bf16(256, 128, false, false);
      constexpr uint32_t idQ = idesc_bf16(256, D, false, true);
      const uint64_t dh0 = umma_desc_sw128(smem_u32(sKV), 0, 1024);   // 64-row halves, K-major
      const uint64_t dm0 = umma_desc_sw128(smem_u32(sKV + C::OFF_QB), 0, 1024);   // MN-major K
      auto kslot = [&](int j) { return (uint64_t)(((j % C::STAGES) * C::SLOT) >> 4); };
      auto issue_sdp = [&](int j, uint32_t a_col, uint32_t col, uint32_t boff, uint64_t* bar) {
        if (elect_one()) {   // S = Q K^T / dP = dO V^T, A (Q / dO) from TMEM
          const uint64_t b = dh0 + kslot(j) + (boff >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t o = ((kk >> 2) * C::HALF + (kk & 3) * 32) >> 4;
            mma2_bf16_ts(tmem + col, tmem + a_col + kk * 8, b + o, idS, kk > 0);
          }
          mma2_commit_mc(bar);
        }
        __syncwarp();
      };
      auto wait_kv = [&](int j) {
        mbar_wait_cluster(&kv_full[j % C::STAGES], (j / C::STAGES) & 1);
        tc_fence_after();
      };
      mbar_wait_cluster(q_ready, 0);
      tc_fence_after();
      wait_kv(0);
      issue_sdp(0, C::Q_COL, C::S_COL, C::OFF_SB, s_full);
      issue_sdp(0, C::G_COL, C::DP_COL, C::OFF_VB, dp_full);
      for (int j = 0; j < nt; ++j) {
        const uint32_t ph = j & 1;
        if (j + 1 < nt) {
          wait_kv(j + 1);
          mbar_wait_cluster(s_read, ph);
          tc_fence_after();
          issue_sdp(j + 1, C::Q_COL, C::S_COL, C::OFF_SB, s_full);            // S(j+1)
        }
        mbar_wait_cluster(ds_full, ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t b = dm0 + kslot(j);
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)   // dQ += dS K (A = dS packed over dP)
            mma2_bf16_ts(tmem + C::DQ_COL, tmem + C::DP_COL + dkv_a_col(kk),
                         b + ((kk * 16 * 128) >> 4), idQ, (j > 0 || kk > 0) ? 1u : 0u);
          mma2_commit_mc(&kv_empty[j % C::STAGES]);
        }
        __syncwarp();
        if (j + 1 < nt) issue_sdp(j + 1, C::G_COL, C::DP_COL, C::OFF_VB, dp_full);   // dP(j+1)
      }
      if (elect_one()) mma2_commit_mc(dq_done);
      __syncwarp();
    }
  } else {
    // ------------- softmax: query row per thread, 64 of the 128 kv columns per wg
    const int wg = warp >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    {   // stage Q (wg 0) / dO (wg 1) rows into TMEM as bf16 pairs (A operands)
      mbar_wait(qd_full, 0);
      const uint32_t base = smem_u32(sKV + C::QSLOT * C::SLOT + wg * C::Q_BYTES) + r * 128;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t v[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint32_t a, b2, c2, d2;
          const uint32_t addr = base + c * 128 * 128 + ((q ^ (r & 7)) << 4);
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(a), "=r"(b2), "=r"(c2), "=r"(d2) : "r"(addr));
          v[q * 4] = a; v[q * 4 + 1] = b2; v[q * 4 + 2] = c2; v[q * 4 + 3] = d2;
        }
        tmem_st32(tl + (wg ? C::G_COL : C::Q_COL) + c * 32, v);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(q_local);
      arrive_pair(q_ready);
    }
    const int row = row0 + r;
    const size_t prow = (size_t)qh * p.rows_pad + row;
    const float2 nl2 = make_float2(p.Lp[prow], p.Lp[prow]);   // -L log2 e
    const float2 nd2 = make_float2(p.Dp[prow], p.Dp[prow]);   // -D
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    for (int j = 0; j < nt; ++j) {
      const uint32_t ph = j & 1;
      const int nvalid = min(128, p.rows_kv - (kv_t0 + j) * 128) - wg * 64;
      mbar_wait(s_full, ph);
      tc_fence_after();
      uint32_t sv[2][32];
      tmem_ld32(tl + C::S_COL + wg * 64, sv[0]);
      tmem_ld32(tl + C::S_COL + wg * 64 + 32, sv[1]);
      tmem_wait_ld();
      tc_fence_before();
      arrive_pair(s_read);
      float2 pf[32];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        auto pa = [&](auto masked) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int c = hh * 32 + e;
            float2 x = ffma2(u2f2(sv[hh][e], sv[hh][e + 1]), sc2, nl2);
            if constexpr (decltype(masked)::value) {
              x.x = c < nvalid ? x.x : -INFINITY;
              x.y = c + 1 < nvalid ? x.y : -INFINITY;
            }
            const float2 pq = (((c / 2) * 3) % 8) < kPolyPairsD<D> && !decltype(masked)::value
                                  ? ex2_poly2(x)
                                  : make_float2(ex2(x.x), ex2(x.y));
            pf[c / 2] = pq;
          }
        };
        if (nvalid < 64)
          pa(std::true_type{});
        else
          pa(std::false_type{});
      }
      mbar_wait(dp_full, ph);
      tc_fence_after();
      uint32_t gv[2][32], dd[32];
      tmem_ld32(tl + C::DP_COL + wg * 64, gv[0]);
      tmem_ld32(tl + C::DP_COL + wg * 64 + 32, gv[1]);
      tmem_wait_ld();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int pi = (hh * 32 + e) / 2;
          const float2 r2 = fmul2(pf[pi], fadd2(u2f2(gv[hh][e], gv[hh][e + 1]), nd2));
          dd[pi] = pack_bf16(r2.x, r2.y);
        }
      }
      tmem_st32(tl + C::DP_COL + wg * 64, dd);
      tmem_wait_st();
      tc_fence_before();
      arrive_pair(ds_full);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    const bool valid = row < p.rows_q;
    float* dst = p.ws_dq + (((size_t)split * p.hq + qh) * p.rows_q + row) * D;
#pragma unroll 1
    for (int c = wg * (D / 64); c < (wg + 1) * (D / 64); ++c) {
      uint32_t v[32];
      tmem_ld32(tl + C::DQ_COL + c * 32, v);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + e) =
              make_float4(__uint_as_float(v[e]) * p.scale, __uint_as_float(v[e + 1]) * p.scale,
                          __uint_as_float(v[e + 2]) * p.scale, __uint_as_float(v[e + 3]) * p.scale);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}
#endif  // LVX_DQ2_PROBE

// dq (+)= sum_s ws_dq[s]  (fixed order, deterministic)
template <int D>
__global__ void dq_combine_kernel(const float* __restrict__ ws, int splits, int hq, int rows,
                                  View3<float> dQ, int accumulate) {
  constexpr int PER = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (int64_t)hq * rows) return;
  const int h = (int)(gw / rows), i = (int)(gw % rows);
  const size_t stride = (size_t)hq * rows * D;
  float acc[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) acc[e] = 0.f;
  // batches of B splits with every load in flight; summation order unchanged
  constexpr int B = D == 64 ? 16 : 8;
  for (int s0 = 0; s0 < splits; s0 += B) {
    float v[B][PER];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float* src = ws + (size_t)(s0 + b) * stride + (size_t)gw * D + lane * PER;
      const bool live = s0 + b < splits;
      if constexpr (PER == 4) {
        const float4 t = live ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0, 0, 0, 0);
        v[b][0] = t.x; v[b][1] = t.y; v[b][2] = t.z; v[b][3] = t.w;
      } else {
        const float2 t = live ? __ldg(reinterpret_cast<const float2*>(src)) : make_float2(0, 0);
        v[b][0] = t.x; v[b][1] = t.y;
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (s0 + b >= splits) break;
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] += v[b][e];
    }
  }
  float* o = dQ.at(h, i) + lane * PER;
#pragma unroll
  for (int e = 0; e < PER; ++e) o[e] = accumulate ? o[e] + acc[e] : acc[e];
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

__global__ void zero_kernel(View3<float> A) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= A.heads * A.rows * A.d) return;
  const int64_t c = idx % A.d, r = (idx / A.d) % A.rows, h = idx / (A.d * A.rows);
  A.at(h, r)[c] = 0.f;
}

int fill_zero_f32(const lvx_view* v, cudaStream_t st) {
  const int64_t total = v->heads * v->rows * v->d;
  if (!total) return LVX_OK;
  zero_kernel<<<ceil_div(total, 256), 256, 0, st>>>(make_view<float>(v));
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

struct BwdPlan {
  int tq64, tpq, pairs, rows_pad, n_tiles, tiles_per_split, splits;
};

BwdPlan plan_bwd(const lvx_view* q, const lvx_view* k) {
  BwdPlan pl{};
  const int G = (int)(q->heads / k->heads);
  pl.tq64 = (int)ceil_div(q->rows, kStep);
  pl.tpq = (int)ceil_div(q->rows, 128);
  pl.rows_pad = pl.tpq * 128;
  pl.pairs = G * pl.tpq;                       // one 128-row query tile per dQ CTA
  pl.n_tiles = (int)ceil_div(k->rows, 128);
  const int64_t units0 = (int64_t)pl.pairs * k->heads;
  const int sms = device_sms();
  int best = 1;
  double best_score = -1.0;
  const int max_s = (int)std::max<int64_t>(1, std::min<int64_t>(64, pl.n_tiles / 2));
  for (int s = 1; s <= max_s; ++s) {
    const int tps = (int)ceil_div(pl.n_tiles, s);
    const int real_s = (int)ceil_div(pl.n_tiles, tps);
    const int64_t units = units0 * real_s;
    const int64_t waves = ceil_div(units, sms);
    const double eff = (double)units / (double)(waves * sms);
    // partial dQ traffic relative to the split's work (fp32 write + read)
    const double score = eff / (1.0 + 1.6 * real_s / pl.n_tiles);
    if (score > best_score + 1e-9) {
      best_score = score;
      best = s;
    }
  }
  pl.tiles_per_split = (int)ceil_div(pl.n_tiles, best);
  pl.splits = (int)ceil_div(pl.n_tiles, pl.tiles_per_split);
  return pl;
}

bool f32_rows_ok(const lvx_view* v) {
  return v->dtype == LVX_F32 && (reinterpret_cast<uintptr_t>(v->data) & 15) == 0 &&
         v->row_stride % 4 == 0 && (v->heads <= 1 || v->head_stride % 4 == 0);
}

// bf16 outputs (dK / dV overwritten in the input dtype): 16-byte aligned rows
bool bf16_rows_ok(const lvx_view* v) {
  return v->dtype == LVX_BF16 && (reinterpret_cast<uintptr_t>(v->data) & 15) == 0 &&
         v->row_stride % 8 == 0 && (v->heads <= 1 || v->head_stride % 8 == 0);
}

void fill_params(BwdParams& p, const BwdPlan& pl, const lvx_view* q, const lvx_view* k,
                 double scale, void* ws) {
  p.hq = (int)q->heads;
  p.hkv = (int)k->heads;
  p.G = p.hq / p.hkv;
  p.rows_q = (int)q->rows;
  p.rows_kv = (int)k->rows;
  p.rows_pad = pl.rows_pad;
  p.tq64 = pl.tq64;
  p.tpq = pl.tpq;
  p.n_tiles = pl.n_tiles;
  p.tiles_per_split = pl.tiles_per_split;
  p.splits = pl.splits;
  p.scale = (float)scale;
  p.scale_log2 = (float)(scale * 1.4426950408889634);
#ifdef LVX_BWD_DEBUG_MODES
  const char* dbg = getenv("LVX_BWD_DEBUG");
  p.debug = dbg ? atoi(dbg) : 0;
#endif
  char* w = static_cast<char*>(ws);
  const size_t lp_bytes = align256((size_t)p.hq * p.rows_pad * 4);
  p.Lp = reinterpret_cast<float*>(w);
  p.Dp = reinterpret_cast<float*>(w + lp_bytes);
  p.ws_dq = reinterpret_cast<float*>(w + 2 * lp_bytes);
}

int launch_prep(const BwdParams& p, const lvx_view* L, const lvx_view* Dv, cudaStream_t st) {
  const int64_t total = (int64_t)p.hq * p.rows_pad;
  bwd_prep_kernel<<<ceil_div(total, 256), 256, 0, st>>>(
      View3<const float>{static_cast<const float*>(L->data), L->heads, L->rows, 1, L->head_stride,
                         L->row_stride},
      View3<const float>{static_cast<const float*>(Dv->data), Dv->heads, Dv->rows, 1,
                         Dv->head_stride, Dv->row_stride},
      p.hq, p.rows_q, p.rows_pad, const_cast<float*>(p.Lp), const_cast<float*>(p.Dp));
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

template <int D>
int launch_dkv(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* dO,
               BwdParams p, const lvx_view* dk, const lvx_view* dvv, int accumulate,
               cudaStream_t st) {
  CUtensorMap mq128, mg128, mk128, mv128, mdk{}, mdv{};
  if (!make_tma_3d(&mq128, q, 128) || !make_tma_3d(&mg128, dO, 128) ||
      !make_tma_3d(&mk128, k, 128) || !make_tma_3d(&mv128, v, 128))
    return LVX_ECUDA;
  if (accumulate && (!make_tma_f32_3d(&mdk, dk, 32) || !make_tma_f32_3d(&mdv, dvv, 32)))
    return LVX_ECUDA;
  static std::atomic<unsigned> attr_done{0};
  if (!ensure_smem_attr(bwd_dkv_kernel<D>, DkvCfg<D>::SMEM, attr_done)) return LVX_ECUDA;
  p.accumulate = accumulate;
  p.dk_ptr = dk->data;
  p.dv_ptr = dvv->data;
  p.out_bf16 = dk->dtype == LVX_BF16;
  p.dk_hs = dk->head_stride;
  p.dk_rs = dk->row_stride;
  p.dv_hs = dvv->head_stride;
  p.dv_rs = dvv->row_stride;
  bwd_dkv_kernel<D><<<dim3((unsigned)ceil_div(k->rows, 128), (unsigned)k->heads), 384,
                      DkvCfg<D>::SMEM, st>>>(mq128, mk128, mv128, mg128, mdk, mdv, p);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

#ifdef LVX_DKV2_PROBE
int launch_dkv2(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* dO,
                BwdParams p, const lvx_view* dk, const lvx_view* dvv, int accumulate,
                cudaStream_t st) {
  CUtensorMap mq128, mg128, mq64, mg64, mk128, mv128, mdk{}, mdv{};
  if (!make_tma_3d(&mq128, q, 128) || !make_tma_3d(&mg128, dO, 128) ||
      !make_tma_3d(&mq64, q, 64) || !make_tma_3d(&mg64, dO, 64) ||
      !make_tma_3d(&mk128, k, 128) || !make_tma_3d(&mv128, v, 128))
    return LVX_ECUDA;
  if (accumulate && (!make_tma_f32_3d(&mdk, dk, 32) || !make_tma_f32_3d(&mdv, dvv, 32)))
    return LVX_ECUDA;
  static std::atomic<unsigned> attr_done{0};
  if (!ensure_smem_attr(bwd_dkv2_kernel<128>, Dkv2Cfg<128>::SMEM, attr_done)) return LVX_ECUDA;
  p.accumulate = accumulate;
  p.dk_ptr = dk->data;
  p.dv_ptr = dvv->data;
  p.out_bf16 = dk->dtype == LVX_BF16;
  p.dk_hs = dk->head_stride;
  p.dk_rs = dk->row_stride;
  p.dv_hs = dvv->head_stride;
  p.dv_rs = dvv->row_stride;
  const unsigned pairs = (unsigned)ceil_div(k->rows, 256);
  bwd_dkv2_kernel<128><<<dim3(2 * pairs, (unsigned)k->heads), 384, Dkv2Cfg<128>::SMEM, st>>>(
      mq128, mk128, mv128, mg128, mq64, mg64, mdk, mdv, p);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

#endif  // LVX_DKV2_PROBE

template <int D>
int launch_dq(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* dO,
              const BwdParams& p, const BwdPlan& pl, cudaStream_t st) {
  CUtensorMap mq128, mg128, mk128, mv128;
  if (!make_tma_3d(&mq128, q, 128) || !make_tma_3d(&mg128, dO, 128) ||
      !make_tma_3d(&mk128, k, 128) || !make_tma_3d(&mv128, v, 128))
    return LVX_ECUDA;
  static std::atomic<unsigned> attr_done{0};
  if (!ensure_smem_attr(bwd_dq_kernel<D>, DqCfg<D>::SMEM, attr_done)) return LVX_ECUDA;
  bwd_dq_kernel<D><<<dim3(pl.pairs, pl.splits, (unsigned)k->heads), 320, DqCfg<D>::SMEM, st>>>(
      mq128, mk128, mv128, mg128, p);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

#ifdef LVX_DQ2_PROBE
int launch_dq2(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* dO,
               const BwdParams& p, const BwdPlan& pl, cudaStream_t st) {
  CUtensorMap mq128, mg128, mk128, mk64, mv64;
  if (!make_tma_3d(&mq128, q, 128) || !make_tma_3d(&mg128, dO, 128) ||
      !make_tma_3d(&mk128, k, 128) || !make_tma_3d(&mk64, k, 64) || !make_tma_3d(&mv64, v, 64))
    return LVX_ECUDA;
  static std::atomic<unsigned> attr_done{0};
  if (!ensure_smem_attr(bwd_dq2_kernel, Dq2Cfg::SMEM, attr_done)) return LVX_ECUDA;
  bwd_dq2_kernel<<<dim3(pl.pairs, pl.splits, (unsigned)k->heads), 320, Dq2Cfg::SMEM, st>>>(
      mq128, mk128, mk64, mv64, mg128, p);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}
#endif  // LVX_DQ2_PROBE

}  // namespace

bool tc_bwd_eligible(const lvx_view* q, const lvx_view* k, const lvx_view* v) {
  if (q->dtype != LVX_BF16 || (q->d != 64 && q->d != 128)) return false;
  if (!tma_view_ok(q) || !tma_view_ok(k) || !tma_view_ok(v)) return false;
  if (k->heads == 0 || q->heads % k->heads) return false;
  return is_sm100();
}

bool tc_bwd_outputs_ok(const lvx_view* dO, const lvx_view* a, const lvx_view* b) {
  auto ok = [](const lvx_view* x) { return !x || f32_rows_ok(x) || bf16_rows_ok(x); };
  return tma_view_ok(dO) && ok(a) && ok(b);
}

size_t tc_bwd_workspace(const lvx_view* q, const lvx_view* k) {
  if (q->rows == 0 || k->rows == 0) return 256;
  const BwdPlan pl = plan_bwd(q, k);
  const size_t lp = align256((size_t)q->heads * pl.rows_pad * 4);
  return 2 * lp + align256((size_t)pl.splits * q->heads * q->rows * q->d * 4);
}

int tc_bwd_dq_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                      const lvx_view* L, const lvx_view* D, const lvx_view* dO, double scale,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
  if (q->rows == 0 || k->rows == 0) return LVX_OK;
  if (ws_bytes < tc_bwd_workspace(q, k)) return LVX_EWORKSPACE;
  const BwdPlan pl = plan_bwd(q, k);
  BwdParams p{};
  fill_params(p, pl, q, k, scale, ws);
  int s = launch_prep(p, L, D, st);
  if (s) return s;
#ifdef LVX_DQ2_PROBE
  if (q->d == 128 && pl.pairs % 2 == 0) return launch_dq2(q, k, v, dO, p, pl, st);
#endif
  return q->d == 128 ? launch_dq<128>(q, k, v, dO, p, pl, st) : launch_dq<64>(q, k, v, dO, p, pl, st);
}

int tc_bwd_dq_finish(const lvx_view* q, const lvx_view* k, const lvx_view* dq, int accumulate,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  if (q->rows == 0) return LVX_OK;
  if (ws_bytes < tc_bwd_workspace(q, k)) return LVX_EWORKSPACE;
  const BwdPlan pl = plan_bwd(q, k);
  BwdParams p{};
  fill_params(p, pl, q, k, 1.0, ws);
  const int64_t rows_total = (int64_t)p.hq * p.rows_q;
  if (k->rows == 0) {   // no contribution: dq (+)= 0
    if (accumulate) return LVX_OK;
    return fill_zero_f32(dq, st);
  }
  if (q->d == 128)
    dq_combine_kernel<128><<<ceil_div(rows_total * 32, 256), 256, 0, st>>>(
        p.ws_dq, p.splits, p.hq, p.rows_q, make_view<float>(dq), accumulate);
  else
    dq_combine_kernel<64><<<ceil_div(rows_total * 32, 256), 256, 0, st>>>(
        p.ws_dq, p.splits, p.hq, p.rows_q, make_view<float>(dq), accumulate);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

int tc_bwd_dkv(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
               const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dk,
               const lvx_view* dv, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (k->rows == 0) return LVX_OK;
  if (q->rows == 0) {
    if (accumulate) return LVX_OK;
    int s = fill_empty_zero(dk, st);
    return s ? s : fill_empty_zero(dv, st);
  }
  if (ws_bytes < tc_bwd_workspace(q, k)) return LVX_EWORKSPACE;
  const BwdPlan pl = plan_bwd(q, k);
  BwdParams p{};
  fill_params(p, pl, q, k, scale, ws);
  int s = launch_prep(p, L, D, st);
  if (s) return s;
#ifdef LVX_DKV2_PROBE
  // CTA-pair kernel (d = 128), probe builds only: bit-identical to the 1-CTA
  // kernel and equal with the softmax stubbed (1423 vs 1457 TFLOP/s at
  // c2gath), but 19 % slower with real math (1008-1013 vs 1242-1251 at
  // c2full): the pair's two tensor cores wait for the slower CTA's softmax at
  // both hand-offs of every step.
  const char* two = getenv("LVX_DKV_2CTA");
  if (q->d == 128 && two && atoi(two) == 1)
    return launch_dkv2(q, k, v, dO, p, dk, dv, accumulate, st);
#endif
  return q->d == 128 ? launch_dkv<128>(q, k, v, dO, p, dk, dv, accumulate, st)
                     : launch_dkv<64>(q, k, v, dO, p, dk, dv, accumulate, st);
}

}  // namespace lvx

#ifdef LVX_DKV_TRACE
extern "C" int lvx_dbg_dkv_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, lvx::g_dkv_trace, sizeof(lvx::g_dkv_trace)) == cudaSuccess ? 0
                                                                                             : -3;
}
#endif

#ifdef LVX_DQ_TRACE
extern "C" int lvx_dbg_dq_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, lvx::g_dq_trace, sizeof(lvx::g_dq_trace)) == cudaSuccess ? 0 : -3;
}
#endif
