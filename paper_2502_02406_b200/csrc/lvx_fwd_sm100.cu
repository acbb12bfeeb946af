// tcgen05/TMEM/TMA blockwise attention forward for B200 (sm_100a).
//
// Replaces kernels.py:105-141 blockwise_attention for bf16 inputs with
// d in {64, 128}; the split combine + prior merge kernel replaces the
// merge_states call that follows it in lvx_forward (strategies.py:207-213)
// and ring_forward (strategies.py:299-301).
//
// One CTA = one kv head g, two 128-row query tiles of that head's GQA group
// (so each K/V tile fetched into shared memory feeds 256 query rows), and one
// split of the resident KV block.  With a single query tile per kv head (MHA,
// <= 128 rows; KVP instantiation) the two tiles are the same Q against the
// even / odd KV tiles of the split, each writing its own split partial.  Warp roles (384
// threads, kThreads; warps 10-11 only donate registers via setmaxnreg):
//   warps 0-3  softmax for query tile 0 (TMEM lanes 0-127, one row per thread)
//   warps 4-7  softmax for query tile 1
//   warp  8    TMA producer: Q tiles once, then K_j / V_j into a 5-slot
//              128B-swizzled ring (10 slots at d=64)
//   warp  9    TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 columns): S_t = Q_t K_j^T at cols [128t, 128t+128), O_t at
// [256 + t*D, 256 + (t+1)*D).  The softmax warps write P_t =
// exp2(S_t*scale*log2e - m) as bf16 pairs back OVER S_t, in two published
// halves (single pass against the running reference max m, a per-half
// row-sum vote; the exact two-pass path when a vote fails), and PV_t is a TS
// MMA reading P_t from TMEM, issued per half.  tcgen05.mma runs in issue
// order, so the stream PV_t(j) -> QK_t(j+1) needs no extra barrier and the
// commit after QK_t(j) also proves PV_t(j-1) done.  The running max is
// updated lazily: O in TMEM is rescaled only when the row max grows by more
// than 2^8 (or a vote failed), which is exact (P, l and O always share one
// reference max).
// Each split writes a normalised partial (O, L) in fp32 to the workspace;
// fwd_combine_kernel merges the splits (and the prior ring state) in a fixed
// order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "lvx_common.cuh"
#include "lvx_sm100.cuh"

namespace lvx {
namespace {

using namespace sm100;

constexpr int kBM = 128;   // query rows per tile (TMEM lanes)
constexpr int kBN = 128;   // kv rows per tile
constexpr int kThreads = 384;   // softmax WGs 0-1, WG 2 = producer, MMA, 2 idle warps
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr float kFastBound = 4096.f;       // single-pass acceptance bound on a P row sum
// Both halves' scores come out of TMEM in one round trip before the first
// half is exponentiated (one load latency per tile instead of two): same-box
// A/B +0.5-0.8 % forward (tools/ab_fwd_prefetch.sh, profiles/r02_ab_fwd_prefetch.txt)
#ifndef LVX_FWD_PREFETCH
#define LVX_FWD_PREFETCH 1
#endif
#ifndef LVX_FWD_POLY
#define LVX_FWD_POLY 3
#endif
#ifndef LVX_FWD_POLY64
#define LVX_FWD_POLY64 LVX_FWD_POLY
#endif
template <int D>
constexpr int kPolyPairsD = D == 64 ? LVX_FWD_POLY64 : LVX_FWD_POLY;   // of every 8 column pairs, exp2 by polynomial

// LVX_FWD_TRACE=<split> (profiling builds only, tools/fwd_trace.py): clock64
// stamps of CTA (pair 0, split, head 0), [role][kv tile][event]
#ifdef LVX_FWD_TRACE
__device__ long long g_fwd_trace[4][128][6];
#define FWD_STAMP(role, j, ev)                                                              \
  do {                                                                                      \
    if (blockIdx.x == 0 && blockIdx.y == LVX_FWD_TRACE && blockIdx.z == 0 && (j) < 128 &&   \
        lane == 0)                                                                          \
      g_fwd_trace[role][j][ev] = clock64();                                                 \
  } while (0)
#else
#define FWD_STAMP(role, j, ev) \
  do {                         \
  } while (0)
#endif

template <int D>
struct FwdCfg {
  static constexpr int PANELS = D / 64;      // 128-byte (64 x bf16) column panels
  static constexpr int Q_BYTES = kBM * D * 2;
  static constexpr int KV_BYTES = kBN * D * 2;
  static constexpr int STAGES = D == 128 ? 5 : 10;
  static constexpr int NBAR = 1 + 2 * STAGES + 10;
  static constexpr int SMEM = 1024 + 2 * Q_BYTES + STAGES * KV_BYTES + NBAR * 8 + 16;
  static constexpr int S_COL0 = 0;
  static constexpr int O_COL0 = 256;
};

struct FwdParams {
  int hq, hkv, G, rows_q, rows_kv;
  int tpq;              // 128-row tiles per query head
  int n_tiles;          // 128-row kv tiles in the block
  int tiles_per_split;
  int splits;           // workspace partials (2 per CTA split in kv_pair mode)
  int kv_pair;          // one query tile per kv head: the CTA's two tiles take the
                        // even / odd KV tiles of its split with the same Q
  float scale_log2;     // scale * log2(e)
  float* ws_o;          // [splits][hq][rows_q][D]
  float* ws_l;          // [splits][hq][rows_q]
};

template <int D, bool KVP>
__global__ void __launch_bounds__(kThreads, 1)
fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, const FwdParams p) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw_u + 1023u) & ~1023u) - raw_u);
  uint8_t* sQ = sm;
  uint8_t* sKV = sQ + 2 * C::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::STAGES * C::KV_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::STAGES;
  uint64_t* s_full = kv_empty + C::STAGES;   // [2]
  uint64_t* p_full = s_full + 2;             // [2 t + h]: half h of P_t (128 each)
  uint64_t* o_done = p_full + 4;             // [2]
  uint64_t* pv0_done = o_done + 2;           // [2]: PV_t(j) over the first half
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = blockIdx.x, split = blockIdx.y, g = blockIdx.z;
  const int kv_t0 = split * p.tiles_per_split;
  const int nt = min(p.n_tiles, kv_t0 + p.tiles_per_split) - kv_t0;
  bool active[2];
  int qh[2], row0[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int tt = 2 * pair + t;
    active[t] = tt < p.G * p.tpq;
    qh[t] = g * p.G + tt / p.tpq;
    row0[t] = (tt % p.tpq) * kBM;
  }
  // kv_pair: tile t runs over KV tiles kv_t0 + 2 j + t (nt is even), one Q
  constexpr bool kvp = KVP;   // == p.kv_pair (a separate instantiation: no cost to the normal path)
  if (kvp) {
    active[1] = active[0];
    qh[1] = qh[0];
    row0[1] = row0[0];
  }
  const int ns = kvp ? nt / 2 : nt;   // KV steps per query tile
  // load index L of the K / V tile QK_t(j) / PV_t(j) reads: (K_j, V_j)
  // pairs, or (K_2j, K_2j+1, V_2j, V_2j+1) quads in kv_pair mode
  auto k_load = [&](int t, int j) { return kvp ? 4 * j + t : 2 * j; };
  auto v_load = [&](int t, int j) { return kvp ? 4 * j + 2 + t : 2 * j + 1; };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[2 * t], 128);
      mbar_init(&p_full[2 * t + 1], 128);
      mbar_init(&o_done[t], 1);
      mbar_init(&pv0_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Registers move from warpgroup 2 (TMA + MMA issue) to the softmax
  // warpgroups, which hold a packed P tile plus two S chunks in flight.  Each
  // role resizes inside its own branch so ptxas sizes each region separately.
  if (warp == 8) {
    // ------------------------------------------------------------ producer
    reg_dealloc<56>();
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      const uint32_t qbytes = (kvp ? active[0] : active[0] + active[1]) * C::Q_BYTES;
      mbar_arrive_expect_tx(q_full, qbytes);
      for (int t = 0; t < (kvp ? 1 : 2); ++t)
        if (active[t])
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_3d(sQ + t * C::Q_BYTES + pn * kBM * 128, &tmQ, q_full, pn * 64, row0[t],
                        qh[t]);
      for (int L = 0; L < 2 * nt; ++L) {
        const int s = L % C::STAGES, u = L / C::STAGES;
        if (u > 0) mbar_wait(&kv_empty[s], (u - 1) & 1);
        const bool is_v = kvp ? (L & 3) >= 2 : (L & 1);
        const int kvt = kvp ? 2 * (L >> 2) + (L & 1) : L >> 1;
        const CUtensorMap* m = is_v ? &tmV : &tmK;
        mbar_arrive_expect_tx(&kv_full[s], C::KV_BYTES);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_3d(sKV + s * C::KV_BYTES + pn * kBN * 128, m, &kv_full[s], pn * 64,
                      (kv_t0 + kvt) * kBN, g);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    reg_dealloc<56>();
    // Tensor-pipe order per KV tile j and query tile t:
    //   ... PV_t(j-1) -> QK_t(j) -> [softmax_t(j) writes P over S_t] -> PV_t(j) -> QK_t(j+1)
    // tcgen05.mma executes in issue order, so QK_t(j+1) overwrites S_t/P_t only
    // after PV_t(j) has consumed P_t, and the s_full commit after QK_t(j)
    // also certifies that PV_t(j-1) is complete (O_t stable for a rescale).
    // The whole warp runs the schedule (waits are warp-wide); one elected lane
    // issues.  Descriptors are built once per tile and advanced by adding the
    // byte offset >> 4 to the low word.
    {
      constexpr uint32_t idQK = idesc_bf16(kBM, kBN, false, false);
      constexpr uint32_t idPV = idesc_bf16(kBM, D, false, true);
      const uint64_t dq0 = umma_desc_sw128(smem_u32(sQ), 0, 1024);
      const uint64_t dkv0 = umma_desc_sw128(smem_u32(sKV), 0, 1024);
      const uint64_t dv0 = umma_desc_sw128(smem_u32(sKV), kBN * 128, 1024);
      auto slot_of = [&](int L) { return L % C::STAGES; };
      auto wait_load = [&](int L) {
        mbar_wait(&kv_full[slot_of(L)], (L / C::STAGES) & 1);
        tc_fence_after();
      };
      auto issue_qk = [&](int t, int j) {
        if (elect_one()) {
          const uint64_t a = dq0 + (((kvp ? 0 : t) * C::Q_BYTES) >> 4);
          const uint64_t b = dkv0 + ((slot_of(k_load(t, j)) * C::KV_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t ao = ((kk >> 2) * (kBM * 128) + (kk & 3) * 32) >> 4;
            const uint32_t bo = ((kk >> 2) * (kBN * 128) + (kk & 3) * 32) >> 4;
            mma_bf16_ss(tmem + C::S_COL0 + t * kBN, a + ao, b + bo, idQK, kk > 0);
          }
          mma_commit(&s_full[t]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j, int kk0, int kk1, uint64_t* bar) {
        if (elect_one()) {
          const uint64_t b = dv0 + ((slot_of(v_load(t, j)) * C::KV_BYTES) >> 4);
#pragma unroll
          for (int kk = kk0; kk < kk1; ++kk)   // A = P_t in TMEM (bf16, 8 cols per K=16)
            mma_bf16_ts(tmem + C::O_COL0 + t * D, tmem + C::S_COL0 + t * kBN + kk * 8,
                        b + ((kk * 16 * 128) >> 4), idPV, (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit(bar);
        }
        __syncwarp();
      };
      auto release = [&](int L) {
        if (elect_one()) mma_commit(&kv_empty[slot_of(L)]);
        __syncwarp();
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      const int nk = kvp ? 2 : 1;   // K (and V) loads per step and tile pair
      for (int t = 0; t < nk; ++t) wait_load(k_load(t, 0));
      for (int t = 0; t < 2; ++t)
        if (active[t]) issue_qk(t, 0);
      for (int t = 0; t < nk; ++t) release(k_load(t, 0));   // K_0 consumed
      for (int j = 0; j < ns; ++j) {
        for (int t = 0; t < nk; ++t) wait_load(v_load(t, j));     // V_j
        FWD_STAMP(2, j, 0);
        if (j + 1 < ns)
          for (int t = 0; t < nk; ++t) wait_load(k_load(t, j + 1));   // K_{j+1}
        FWD_STAMP(2, j, 1);
        for (int t = 0; t < 2; ++t) {
          if (!active[t]) continue;
          mbar_wait(&p_full[2 * t], j & 1);   // PV over kv rows [0, 64) as soon as they land
          tc_fence_after();
          issue_pv(t, j, 0, kBN / 32, &pv0_done[t]);
          mbar_wait(&p_full[2 * t + 1], j & 1);
          FWD_STAMP(2, j, 2 + t);
          tc_fence_after();
          issue_pv(t, j, kBN / 32, kBN / 16, &o_done[t]);
          if (j + 1 < ns) issue_qk(t, j + 1);
        }
        for (int t = 0; t < nk; ++t) release(v_load(t, j));       // V_j consumed
        if (j + 1 < ns)
          for (int t = 0; t < nk; ++t) release(k_load(t, j + 1));   // K_{j+1} consumed
      }
    }
  } else if (warp >= 10) {
    reg_dealloc<56>();   // idle warps of warpgroup 2
  } else {
    // ------------------------------------------------------------ softmax
    reg_alloc<224>();
    const int t = warp >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    if (active[t]) {
      const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < ns; ++j) {
        mbar_wait(&s_full[t], j & 1);   // QK_t(j) done, hence PV_t(j-1) done
        if (q4 == 0) FWD_STAMP(t, j, 0);
        tc_fence_after();
        const int nvalid = min(kBN, p.rows_kv - (kv_t0 + (kvp ? 2 * j + t : j)) * kBN);
        const uint32_t sa = tl + C::S_COL0 + t * kBN;
        // Single pass (j > 0): exponentiate against the current reference max
        // m_used without looking for the row max first.  The row sum bounds
        // every element, so if no row's sum exceeds 2^kFastLog2 no P element
        // does either and P is final.  P stays packed in registers until the
        // warp knows that, so S is still intact in TMEM for the two-pass path
        // below when a row's scores grew (rare after the first tiles; that
        // path then moves m_used to the exact row max).  Packed FFMA2/FADD2
        // halve the FMA-pipe issue per element.
        // Single pass in two halves of 64 columns (j > 0): a half is final when
        // no row's partial sum exceeds the bound (every P element of it is then
        // <= the bound), so it is packed over its own, already read, scores and
        // published at once — PV_t(j) runs on kv rows [0, 64) while [64, 128)
        // is exponentiated.  If the first half fails, S is intact and the tile
        // takes the exact two-pass path.  If only the second fails, the first
        // half is already in PV: wait for it (pv0_done), rescale O and l to the
        // new row max and redo the second half from its intact scores.
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        int fail_half = j > 0 ? 2 : 0;   // 2: both halves single-pass
        if (j > 0) {
          const float2 nm2 = make_float2(-m_used, -m_used);
#if LVX_FWD_PREFETCH
          // both halves' scores in one TMEM round trip (one load latency per tile)
          uint32_t sall[4][32];
          tmem_ld32(sa, sall[0]);
          tmem_ld32(sa + 32, sall[1]);
          tmem_ld32(sa + 64, sall[2]);
          tmem_ld32(sa + 96, sall[3]);
          tmem_wait_ld();
#endif
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t pk[2][16];
            float2 acc = make_float2(0.f, 0.f);
            auto half = [&](auto masked, auto poly) {
#if LVX_FWD_PREFETCH
              const uint32_t (&s0)[32] = sall[2 * h];
              const uint32_t (&s1)[32] = sall[2 * h + 1];
#else
              uint32_t s0[32], s1[32];
              tmem_ld32(sa + h * 64, s0);
              tmem_ld32(sa + h * 64 + 32, s1);
              tmem_wait_ld();
#endif
              auto chunk = [&](const uint32_t (&sv)[32], int c) {
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                  float2 x = ffma2(u2f2(sv[e], sv[e + 1]), sc2, nm2);
                  if constexpr (decltype(masked)::value) {
                    const int col = c * 32 + e;
                    x.x = col < nvalid ? x.x : -INFINITY;
                    x.y = col + 1 < nvalid ? x.y : -INFINITY;
                  }
                  const float2 pp = ((((c * 16 + e / 2) * 3) % 8) < decltype(poly)::value)
                                        ? ex2_poly2(x)
                                        : make_float2(ex2(x.x), ex2(x.y));
                  acc = fadd2(acc, pp);
                  pk[c & 1][e / 2] = pack_bf16(pp.x, pp.y);
                }
              };
              chunk(s0, 2 * h);
              chunk(s1, 2 * h + 1);
            };
            using I = std::integral_constant<int, 0>;
            if (nvalid < kBN) half(std::true_type{}, I{});
            else half(std::false_type{}, std::integral_constant<int, kPolyPairsD<D>>{});
            const float rs = acc.x + acc.y;
            if (__any_sync(0xffffffffu, !(rs <= kFastBound))) {   // also inf / NaN
              fail_half = h;
              break;
            }
            tmem_st16(sa + (2 * h) * 16, pk[0]);
            tmem_st16(sa + (2 * h + 1) * 16, pk[1]);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[2 * t + h]);
            l += rs;
          }
        }
        if (fail_half < 2) {
          // exact path over halves h0 .. 1 (h0 = 1: the first half is in PV)
          const int h0 = fail_half;
          float mx = -INFINITY;
          for (int c = 2 * h0; c < 4; ++c) {
            uint32_t sv[32];
            tmem_ld32(sa + c * 32, sv);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e < nvalid) mx = fmaxf(mx, __uint_as_float(sv[e]));
          }
          mx *= p.scale_log2;
          // a failed single pass moves to the exact max; the first tile too
          const bool need = mx > m_used + (j > 0 ? 0.f : kRescaleThreshold);
          const float alpha = need ? ex2(m_used - mx) : 1.f;
          if (__any_sync(0xffffffffu, need && j > 0)) {   // lazy rescale of O_t in TMEM
            if (h0 == 1) {   // O must include PV_t(j) over the first half
              mbar_wait(&pv0_done[t], j & 1);
              tc_fence_after();
            }
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t ov[32];
              const uint32_t oa = tl + C::O_COL0 + t * D + c * 32;
              tmem_ld32(oa, ov);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
              tmem_st32(oa, ov);
            }
          }
          if (need) {
            l *= alpha;
            m_used = mx;
          }
          for (int h = h0; h < 2; ++h) {
            float rs = 0.f;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              const int c = 2 * h + cc;
              uint32_t sv[32], pk[16];
              tmem_ld32(sa + c * 32, sv);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const int col = c * 32 + e;
                float p0 = ex2(fmaf(__uint_as_float(sv[e]), p.scale_log2, -m_used));
                float p1 = ex2(fmaf(__uint_as_float(sv[e + 1]), p.scale_log2, -m_used));
                p0 = col < nvalid ? p0 : 0.f;
                p1 = col + 1 < nvalid ? p1 : 0.f;
                rs += p0 + p1;
                pk[e / 2] = pack_bf16(p0, p1);
              }
              tmem_st16(sa + c * 16, pk);   // packed columns [16c, 16c + 16): scores read
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[2 * t + h]);
            l += rs;
          }
        }
        if (q4 == 0) FWD_STAMP(t, j, 1);
        if (q4 == 0) FWD_STAMP(t, j, 2 + (int)(fail_half == 2));   // 3: single pass accepted
        if (q4 == 0 && fail_half == 1) FWD_STAMP(t, j, 4);         // 4: second-half fallback
      }
      // epilogue: O / l and L = (m + log2 l) ln 2 into this split's partial
      mbar_wait(&o_done[t], (ns - 1) & 1);
      tc_fence_after();
      const int row = row0[t] + r;
      const bool valid = row < p.rows_q;
      const float inv = 1.f / l;
      const int ws_split = kvp ? 2 * split + t : split;   // this tile's partial
      const size_t slot = ((size_t)ws_split * p.hq + qh[t]) * p.rows_q + row;
      float* dst = p.ws_o + slot * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32(tl + C::O_COL0 + t * D + c * 32, ov);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            float4 v4 = make_float4(__uint_as_float(ov[e]) * inv, __uint_as_float(ov[e + 1]) * inv,
                                    __uint_as_float(ov[e + 2]) * inv,
                                    __uint_as_float(ov[e + 3]) * inv);
            *reinterpret_cast<float4*>(dst + c * 32 + e) = v4;
          }
        }
      }
      if (valid) p.ws_l[slot] = (m_used + log2f(l)) * 0.69314718055994530942f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Split combine + merge with the prior state (fixed order, deterministic):
//   L = log sum_s exp(L_s);  O = sum_s exp(L_s - L) O_s
//   then (O, L) = merge_states(prior, (O, L))   (kernels.py:144-161)
template <int D>
__global__ void fwd_combine_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_l,
                                   int splits, int hq, int rows, View3<const float> PO,
                                   View3<const float> PL, bool has_prior, View3<float> O,
                                   View3<float> L) {
  constexpr int PER = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= (int64_t)hq * rows) return;
  const int h = (int)(gw / rows), i = (int)(gw % rows);
  const size_t stride = (size_t)hq * rows;
  // The split LSEs are read lane-parallel (split s0 + lane), their max is a
  // warp reduction (order-free) and each weight w_s = exp(L_s - max) is
  // broadcast from its lane; the O rows of the splits are read in batches of
  // B with every load in flight (with one query tile per head there are few
  // rows and up to 128 splits, so a load-use chain per split would leave the
  // kernel latency-bound).  O and the weight total are summed in the order
  // s = 0, 1, ... exactly as a sequential loop would (deterministic).
  constexpr int B = D == 64 ? 16 : 8;
  float mx = -INFINITY;
  for (int s = lane; s < splits; s += 32) mx = fmaxf(mx, __ldg(ws_l + (size_t)s * stride + gw));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float acc[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) acc[e] = 0.f;
  float tot = 0.f;
  for (int c0 = 0; c0 < splits; c0 += 32) {
    const int sl = c0 + lane;
    const float wl = sl < splits ? __expf(__ldg(ws_l + (size_t)sl * stride + gw) - mx) : 0.f;
    const int nc = min(32, splits - c0);
    for (int b0 = 0; b0 < nc; b0 += B) {
      float v[B][PER];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const bool live = b0 + b < nc;
        const float* src = ws_o + ((size_t)(c0 + b0 + b) * stride + gw) * D + lane * PER;
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
        const float w = __shfl_sync(0xffffffffu, wl, (b0 + b) & 31);
        if (b0 + b >= nc) break;
        tot += w;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] += w * v[b][e];
      }
    }
  }
  float lse = mx + __logf(tot);
  const float inv = 1.f / tot;
#pragma unroll
  for (int e = 0; e < PER; ++e) acc[e] *= inv;
  if (has_prior) {
    const float lp = *PL.at(h, i);
    const float hi = fmaxf(lp, lse);
    const float lm = (hi == -INFINITY) ? -INFINITY : hi + log1pf(__expf(fminf(lp, lse) - hi));
    const float safe = (lm == -INFINITY) ? 0.f : lm;
    const float wp = __expf(lp - safe), wd = __expf(lse - safe);
    const float* po = PO.at(h, i) + lane * PER;
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = wp * po[e] + wd * acc[e];
    lse = lm;
  }
  float* o = O.at(h, i) + lane * PER;
#pragma unroll
  for (int e = 0; e < PER; ++e) o[e] = acc[e];
  if (lane == 0) *L.at(h, i) = lse;
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return encode_fn(); }

// bf16 [heads, rows, d] view -> 3-D TMA map with a (64, 128, 1) box, 128B swizzle.
bool make_tma_3d(CUtensorMap* m, const lvx_view* v, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t rs = (uint64_t)v->row_stride * 2;
  uint64_t hs = (uint64_t)v->head_stride * 2;
  if (v->heads <= 1) hs = rs * (uint64_t)(v->rows > 0 ? v->rows : 1);
  cuuint64_t dims[3] = {(cuuint64_t)v->d, (cuuint64_t)v->rows, (cuuint64_t)v->heads};
  cuuint64_t strides[2] = {rs, hs};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, v->data, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tma_f32_3d(CUtensorMap* m, const lvx_view* v, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t rs = (uint64_t)v->row_stride * 4;
  uint64_t hs = (uint64_t)v->head_stride * 4;
  if (v->heads <= 1) hs = rs * (uint64_t)(v->rows > 0 ? v->rows : 1);
  cuuint64_t dims[3] = {(cuuint64_t)v->d, (cuuint64_t)v->rows, (cuuint64_t)v->heads};
  cuuint64_t strides[2] = {rs, hs};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, v->data, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// SM count of the current device.  The grid plans depend only on this and the
// shapes, so a workspace query, _partial and _finish always agree (the ring
// hops run on copy engines and take no SM, so the plans use all of them).
int device_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms <= 0) {
    cudaGetLastError();
    sms = 148;
  }
  return sms;
}

bool is_sm100() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached = (major == 10 && minor == 0) ? 1 : 0;
  }
  return cached == 1;
}

bool tma_view_ok(const lvx_view* v) {
  return v->dtype == LVX_BF16 && (reinterpret_cast<uintptr_t>(v->data) & 15) == 0 &&
         (v->row_stride * 2) % 16 == 0 && (v->heads <= 1 || (v->head_stride * 2) % 16 == 0) &&
         v->row_stride >= v->d && v->rows < (1ll << 31);
}

namespace {

struct FwdPlan {
  int tpq, pairs, n_tiles, tiles_per_split;
  int grid_splits;   // CTA splits of the KV block
  int splits;        // workspace partials: grid_splits, x2 in kv_pair mode
  bool kv_pair;
};

FwdPlan plan_fwd(const lvx_view* q, const lvx_view* k) {
  FwdPlan pl{};
  const int G = (int)(q->heads / k->heads);
  pl.tpq = (int)ceil_div(q->rows, kBM);
  pl.pairs = (int)ceil_div((int64_t)G * pl.tpq, 2);
  pl.n_tiles = (int)ceil_div(k->rows, kBN);
  // one query tile per kv head (MHA rounds with <= 128 query rows): pair the
  // KV tiles of each split instead, so both softmax warpgroups ping-pong
  pl.kv_pair = G * pl.tpq == 1 && pl.n_tiles >= 2 && pl.n_tiles % 2 == 0;
  const int64_t units0 = (int64_t)pl.pairs * k->heads;
  const int sms = device_sms();
  // maximise modelled throughput: wave efficiency / (1 + partial-state traffic)
  int best_tps = pl.n_tiles;
  double best_score = -1.0;
  const int max_s = (int)std::max<int64_t>(1, std::min<int64_t>(64, pl.n_tiles / 2));
  for (int s = 1; s <= max_s; ++s) {
    int tps = (int)ceil_div(pl.n_tiles, s);
    if (pl.kv_pair) tps += tps & 1;   // even tile counts in every split
    const int real_s = (int)ceil_div(pl.n_tiles, tps);
    const int64_t units = units0 * real_s;
    const int64_t waves = ceil_div(units, sms);
    const double eff = (double)units / (double)(waves * sms);
    const double score = eff / (1.0 + 2.4 * real_s / pl.n_tiles);
    if (score > best_score + 1e-9) {
      best_score = score;
      best_tps = tps;
    }
  }
  pl.tiles_per_split = best_tps;
  pl.grid_splits = (int)ceil_div(pl.n_tiles, pl.tiles_per_split);
  pl.splits = pl.grid_splits * (pl.kv_pair ? 2 : 1);
  return pl;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

template <int D>
int launch_fwd(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale, void* ws,
               cudaStream_t st) {
  const FwdPlan pl = plan_fwd(q, k);
  CUtensorMap mq, mk, mv;
  if (!make_tma_3d(&mq, q, kBM) || !make_tma_3d(&mk, k, kBN) || !make_tma_3d(&mv, v, kBN))
    return LVX_ECUDA;
  FwdParams p{};
  p.hq = (int)q->heads;
  p.hkv = (int)k->heads;
  p.G = p.hq / p.hkv;
  p.rows_q = (int)q->rows;
  p.rows_kv = (int)k->rows;
  p.tpq = pl.tpq;
  p.n_tiles = pl.n_tiles;
  p.tiles_per_split = pl.tiles_per_split;
  p.splits = pl.splits;
  p.kv_pair = pl.kv_pair ? 1 : 0;
  p.scale_log2 = (float)(scale * 1.4426950408889634);
  const size_t n = (size_t)q->heads * q->rows;
  p.ws_o = static_cast<float*>(ws);
  p.ws_l = reinterpret_cast<float*>(static_cast<char*>(ws) + align256(pl.splits * n * D * 4));
  dim3 grid(pl.pairs, pl.grid_splits, (unsigned)k->heads);
  constexpr int smem = FwdCfg<D>::SMEM;
  if (pl.kv_pair) {
    static std::atomic<unsigned> attr_done{0};
    if (!ensure_smem_attr(fwd_kernel<D, true>, smem, attr_done)) return LVX_ECUDA;
    fwd_kernel<D, true><<<grid, kThreads, smem, st>>>(mq, mk, mv, p);
  } else {
    static std::atomic<unsigned> attr_done{0};
    if (!ensure_smem_attr(fwd_kernel<D, false>, smem, attr_done)) return LVX_ECUDA;
    fwd_kernel<D, false><<<grid, kThreads, smem, st>>>(mq, mk, mv, p);
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

}  // namespace

bool tc_fwd_eligible(const lvx_view* q, const lvx_view* k, const lvx_view* v) {
  if (q->dtype != LVX_BF16 || (q->d != 64 && q->d != 128)) return false;
  if (!tma_view_ok(q) || !tma_view_ok(k) || !tma_view_ok(v)) return false;
  if (k->heads == 0 || q->heads % k->heads) return false;
  return is_sm100();
}

size_t tc_fwd_workspace(const lvx_view* q, const lvx_view* k) {
  if (k->rows == 0 || q->rows == 0) return 256;
  const FwdPlan pl = plan_fwd(q, k);
  const size_t n = (size_t)q->heads * q->rows;
  return align256(pl.splits * n * q->d * 4) + align256(pl.splits * n * 4);
}

int tc_fwd_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
                   void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < tc_fwd_workspace(q, k)) return LVX_EWORKSPACE;
  return q->d == 128 ? launch_fwd<128>(q, k, v, scale, ws, st)
                     : launch_fwd<64>(q, k, v, scale, ws, st);
}

int tc_fwd_finish(const lvx_view* q, const lvx_view* k, const lvx_view* po, const lvx_view* pl_,
                  const lvx_view* o, const lvx_view* l, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  if (ws_bytes < tc_fwd_workspace(q, k)) return LVX_EWORKSPACE;
  const FwdPlan pl = plan_fwd(q, k);
  const size_t n = (size_t)q->heads * q->rows;
  const float* wo = static_cast<const float*>(ws);
  const float* wl =
      reinterpret_cast<const float*>(static_cast<const char*>(ws) + align256(pl.splits * n * q->d * 4));
  const bool prior = po && pl_;
  View3<const float> POv{}, PLv{};
  if (prior) {
    POv = View3<const float>{static_cast<const float*>(po->data), po->heads, po->rows, po->d,
                             po->head_stride, po->row_stride};
    PLv = View3<const float>{static_cast<const float*>(pl_->data), pl_->heads, pl_->rows, 1,
                             pl_->head_stride, pl_->row_stride};
  }
  const int threads = 256;
  const int64_t blocks = ceil_div((int64_t)n * 32, threads);
  if (q->d == 128)
    fwd_combine_kernel<128><<<blocks, threads, 0, st>>>(wo, wl, pl.splits, (int)q->heads,
                                                        (int)q->rows, POv, PLv, prior,
                                                        make_view<float>(o), make_view<float>(l));
  else
    fwd_combine_kernel<64><<<blocks, threads, 0, st>>>(wo, wl, pl.splits, (int)q->heads,
                                                       (int)q->rows, POv, PLv, prior,
                                                       make_view<float>(o), make_view<float>(l));
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

}  // namespace lvx

#ifdef LVX_FWD_TRACE
extern "C" int lvx_dbg_fwd_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, lvx::g_fwd_trace, sizeof(lvx::g_fwd_trace)) == cudaSuccess ? 0
                                                                                             : -3;
}
#endif
