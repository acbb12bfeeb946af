// Exact-parity SIMT kernels (CUDA cores) for the LV-XAttn path.
//
// These serve F32/F64 inputs (the reference package's dtypes) and any head
// dim up to 256.  F32 and F64 inputs are computed in float64 internally,
// exactly as the reference does (kernels.py:3-8), so F32 results are the
// rounding of the f64 computation; BF16 inputs that the tensor-core path
// cannot take are computed in float32.  Reductions run in a fixed order, so
// repeated runs are bit-identical (tests/test_strategies.py:239-249).
//
//   simt_fwd_kernel      kernels.py:105-141 blockwise_attention (+ fused
//                        merge with a prior state, kernels.py:144-161)
//   simt_bwd_dq_kernel   kernels.py:192-224, the dQ half
//   simt_bwd_dkv_kernel  kernels.py:192-224, the dK/dV half (GQA summed)
//   merge_kernel         kernels.py:144-161 merge_states
//   row_stats_kernel     kernels.py:164-169 attention_row_stats
#include <type_traits>

#include "lvx_common.cuh"

namespace lvx {
namespace {

constexpr int kWarps = 4;     // warps per block; one (head,row) per warp
constexpr int kMaxD = 256;

template <typename Acc>
struct SimtCfg {};

// ---------------------------------------------------------------------------
// forward: one warp per (q head, q row); KV walked in tiles of 32 rows with
// lane j owning score j of the tile; running (m, l) rescale once per tile.
// ---------------------------------------------------------------------------
template <typename Tin, typename Ts, typename Acc, int DPL>
__global__ void __launch_bounds__(kWarps * 32)
simt_fwd_kernel(View3<const Tin> Q, View3<const Tin> K, View3<const Tin> V, Acc scale,
                View3<const Ts> PO, View3<const Ts> PL, bool has_prior, View3<Ts> O,
                View3<Ts> L) {
  __shared__ Acc qs[kWarps][32 * DPL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + w;
  const int64_t rows = Q.rows, d = Q.d;
  if (gw >= Q.heads * rows) return;
  const int64_t h = gw / rows, i = gw % rows;
  const int64_t hk = h / (Q.heads / K.heads);
  const Tin* qrow = Q.at(h, i);
  for (int c = lane; c < d; c += 32) qs[w][c] = to_acc<Acc>(qrow[c]);
  __syncwarp();

  Acc o[DPL];
#pragma unroll
  for (int c = 0; c < DPL; ++c) o[c] = 0;
  Acc m = neg_inf<Acc>(), l = 0;
  const int64_t nkv = K.rows;
  for (int64_t j0 = 0; j0 < nkv; j0 += 32) {
    const int64_t j = j0 + lane;
    Acc s = neg_inf<Acc>();
    if (j < nkv) {
      const Tin* krow = K.at(hk, j);
      Acc acc = 0;
      for (int64_t c = 0; c < d; ++c) acc += qs[w][c] * to_acc<Acc>(krow[c]);
      s = scale * acc;
    }
    const Acc m_new = fmax(m, warp_max(s));
    const Acc p = (j < nkv) ? exp_acc(s - m_new) : Acc(0);
    const Acc alpha = exp_acc(m - m_new);  // first tile: exp(-inf) = 0
    l = alpha * l + warp_sum(p);
#pragma unroll
    for (int c = 0; c < DPL; ++c) o[c] *= alpha;
    const int cnt = (int)(nkv - j0 < 32 ? nkv - j0 : 32);
    for (int jj = 0; jj < cnt; ++jj) {
      const Acc pj = __shfl_sync(0xffffffffu, p, jj);
      const Tin* vrow = V.at(hk, j0 + jj);
#pragma unroll
      for (int c = 0; c < DPL; ++c) {
        const int64_t col = lane + 32 * c;
        if (col < d) o[c] += pj * to_acc<Acc>(vrow[col]);
      }
    }
    m = m_new;
  }
  Acc lse;
  if (nkv == 0) {
    lse = neg_inf<Acc>();
#pragma unroll
    for (int c = 0; c < DPL; ++c) o[c] = 0;
  } else {
    const Acc inv = Acc(1) / l;
#pragma unroll
    for (int c = 0; c < DPL; ++c) o[c] *= inv;
    lse = m + log_acc(l);
  }
  if (has_prior) {  // merge_states(prior, delta), kernels.py:144-161
    // the reference merges the delta after rounding it to the state dtype
    const Acc lp = to_acc<Acc>(*PL.at(h, i));
    const Acc ld = to_acc<Acc>(from_acc<Ts, Acc>(lse));
    const Acc lm = logaddexp(lp, ld);
    const Acc safe = isinf(lm) && lm < 0 ? Acc(0) : lm;
    const Acc wp = exp_acc(lp - safe), wd = exp_acc(ld - safe);
    const Ts* po = PO.at(h, i);
#pragma unroll
    for (int c = 0; c < DPL; ++c) {
      const int64_t col = lane + 32 * c;
      if (col < d) {
        const Acc dlt = to_acc<Acc>(from_acc<Ts, Acc>(o[c]));
        o[c] = wp * to_acc<Acc>(po[col]) + wd * dlt;
      }
    }
    lse = lm;
  }
  Ts* orow = O.at(h, i);
#pragma unroll
  for (int c = 0; c < DPL; ++c) {
    const int64_t col = lane + 32 * c;
    if (col < d) orow[col] = from_acc<Ts, Acc>(o[c]);
  }
  if (lane == 0) *L.at(h, i) = from_acc<Ts, Acc>(lse);
}

// ---------------------------------------------------------------------------
// backward dQ: one warp per (q head, q row)
// ---------------------------------------------------------------------------
template <typename Tin, typename Ts, typename Acc, int DPL>
__global__ void __launch_bounds__(kWarps * 32)
simt_bwd_dq_kernel(View3<const Tin> Q, View3<const Tin> K, View3<const Tin> V,
                   View3<const Ts> Lv, View3<const Ts> Dv, View3<const Tin> dO, Acc scale,
                   View3<Ts> dQ, bool accumulate) {
  __shared__ Acc qs[kWarps][32 * DPL];
  __shared__ Acc gs[kWarps][32 * DPL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + w;
  const int64_t rows = Q.rows, d = Q.d;
  if (gw >= Q.heads * rows) return;
  const int64_t h = gw / rows, i = gw % rows;
  const int64_t hk = h / (Q.heads / K.heads);
  for (int c = lane; c < d; c += 32) {
    qs[w][c] = to_acc<Acc>(Q.at(h, i)[c]);
    gs[w][c] = to_acc<Acc>(dO.at(h, i)[c]);
  }
  __syncwarp();
  const Acc Li = to_acc<Acc>(*Lv.at(h, i)), Di = to_acc<Acc>(*Dv.at(h, i));
  Acc dq[DPL];
#pragma unroll
  for (int c = 0; c < DPL; ++c) dq[c] = 0;
  const int64_t nkv = K.rows;
  for (int64_t j0 = 0; j0 < nkv; j0 += 32) {
    const int64_t j = j0 + lane;
    Acc ds = 0;
    if (j < nkv) {
      const Tin* krow = K.at(hk, j);
      const Tin* vrow = V.at(hk, j);
      Acc s = 0, dp = 0;
      for (int64_t c = 0; c < d; ++c) {
        s += qs[w][c] * to_acc<Acc>(krow[c]);
        dp += gs[w][c] * to_acc<Acc>(vrow[c]);
      }
      const Acc p = exp_acc(scale * s - Li);
      ds = p * (dp - Di);
    }
    const int cnt = (int)(nkv - j0 < 32 ? nkv - j0 : 32);
    for (int jj = 0; jj < cnt; ++jj) {
      const Acc dsj = __shfl_sync(0xffffffffu, ds, jj);
      const Tin* krow = K.at(hk, j0 + jj);
#pragma unroll
      for (int c = 0; c < DPL; ++c) {
        const int64_t col = lane + 32 * c;
        if (col < d) dq[c] += dsj * to_acc<Acc>(krow[col]);
      }
    }
  }
  Ts* out = dQ.at(h, i);
#pragma unroll
  for (int c = 0; c < DPL; ++c) {
    const int64_t col = lane + 32 * c;
    if (col < d) {
      Acc val = scale * dq[c];
      if (accumulate) val += to_acc<Acc>(out[col]);
      out[col] = from_acc<Ts, Acc>(val);
    }
  }
}

// ---------------------------------------------------------------------------
// backward dK/dV: one warp per (kv head, kv row); walks all query rows of
// every q head in the GQA group (ascending head, then row: fixed order)
// ---------------------------------------------------------------------------
template <typename Tin, typename Ts, typename Acc, int DPL>
__global__ void __launch_bounds__(kWarps * 32)
simt_bwd_dkv_kernel(View3<const Tin> Q, View3<const Tin> K, View3<const Tin> V,
                    View3<const Ts> Lv, View3<const Ts> Dv, View3<const Tin> dO, Acc scale,
                    View3<Ts> dK, View3<Ts> dV, bool accumulate) {
  __shared__ Acc ks[kWarps][32 * DPL];
  __shared__ Acc vs[kWarps][32 * DPL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + w;
  const int64_t nkv = K.rows, d = K.d;
  if (gw >= K.heads * nkv) return;
  const int64_t hk = gw / nkv, j = gw % nkv;
  for (int c = lane; c < d; c += 32) {
    ks[w][c] = to_acc<Acc>(K.at(hk, j)[c]);
    vs[w][c] = to_acc<Acc>(V.at(hk, j)[c]);
  }
  __syncwarp();
  Acc dk[DPL], dv[DPL];
#pragma unroll
  for (int c = 0; c < DPL; ++c) dk[c] = dv[c] = 0;
  const int64_t G = Q.heads / K.heads, rows = Q.rows;
  for (int64_t g = 0; g < G; ++g) {
    const int64_t h = hk * G + g;
    for (int64_t i0 = 0; i0 < rows; i0 += 32) {
      const int64_t i = i0 + lane;
      Acc p = 0, ds = 0;
      if (i < rows) {
        const Tin* qrow = Q.at(h, i);
        const Tin* grow = dO.at(h, i);
        Acc s = 0, dp = 0;
        for (int64_t c = 0; c < d; ++c) {
          s += to_acc<Acc>(qrow[c]) * ks[w][c];
          dp += to_acc<Acc>(grow[c]) * vs[w][c];
        }
        p = exp_acc(scale * s - to_acc<Acc>(*Lv.at(h, i)));
        ds = p * (dp - to_acc<Acc>(*Dv.at(h, i)));
      }
      const int cnt = (int)(rows - i0 < 32 ? rows - i0 : 32);
      for (int ii = 0; ii < cnt; ++ii) {
        const Acc pi = __shfl_sync(0xffffffffu, p, ii);
        const Acc dsi = __shfl_sync(0xffffffffu, ds, ii);
        const Tin* qrow = Q.at(h, i0 + ii);
        const Tin* grow = dO.at(h, i0 + ii);
#pragma unroll
        for (int c = 0; c < DPL; ++c) {
          const int64_t col = lane + 32 * c;
          if (col < d) {
            dv[c] += pi * to_acc<Acc>(grow[col]);
            dk[c] += dsi * to_acc<Acc>(qrow[col]);
          }
        }
      }
    }
  }
  Ts* ok = dK.at(hk, j);
  Ts* ov = dV.at(hk, j);
#pragma unroll
  for (int c = 0; c < DPL; ++c) {
    const int64_t col = lane + 32 * c;
    if (col < d) {
      Acc a = scale * dk[c], b = dv[c];
      if (accumulate) {
        a += to_acc<Acc>(ok[col]);
        b += to_acc<Acc>(ov[col]);
      }
      ok[col] = from_acc<Ts, Acc>(a);
      ov[col] = from_acc<Ts, Acc>(b);
    }
  }
}

// ---------------------------------------------------------------------------
// merge_states: one warp per (head, row), lanes over d
// ---------------------------------------------------------------------------
template <typename Ts>
__global__ void merge_kernel(View3<const Ts> OA, View3<const Ts> LA, View3<const Ts> OB,
                             View3<const Ts> LB, View3<Ts> O, View3<Ts> L) {
  using Acc = double;  // the reference merges in f64 (kernels.py:152-160)
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= O.heads * O.rows) return;
  const int64_t h = gw / O.rows, i = gw % O.rows;
  const Acc la = to_acc<Acc>(*LA.at(h, i)), lb = to_acc<Acc>(*LB.at(h, i));
  const Acc lm = logaddexp(la, lb);
  const Acc safe = (isinf(lm) && lm < 0) ? 0.0 : lm;
  const Acc wa = exp(la - safe), wb = exp(lb - safe);
  const Ts* a = OA.at(h, i);
  const Ts* b = OB.at(h, i);
  Ts* o = O.at(h, i);
  for (int64_t c = lane; c < O.d; c += 32)
    o[c] = from_acc<Ts, Acc>(wa * to_acc<Acc>(a[c]) + wb * to_acc<Acc>(b[c]));
  __syncwarp();
  if (lane == 0) *L.at(h, i) = from_acc<Ts, Acc>(lm);
}

// f32 states: compute in f32 when used by the bf16 perf path is unnecessary —
// the merge is HBM-bound either way, so one f64-internal kernel serves all.

template <typename Ts, typename Tg>
__global__ void row_stats_kernel(View3<const Ts> O, View3<const Tg> dO, View3<Ts> D) {
  using Acc = double;  // kernels.py:168 sums in f64
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= O.heads * O.rows) return;
  const int64_t h = gw / O.rows, i = gw % O.rows;
  const Ts* o = O.at(h, i);
  const Tg* g = dO.at(h, i);
  Acc acc = 0;
  for (int64_t c = lane; c < O.d; c += 32) acc += to_acc<Acc>(o[c]) * to_acc<Acc>(g[c]);
  acc = warp_sum(acc);
  if (lane == 0) *D.at(h, i) = from_acc<Ts, Acc>(acc);
}

// f32 states (the bf16 tensor-core path's O / L / D): HBM-bound, so one
// 16-byte vector per thread, LPR = d/4 lanes per row (a power of two <= 32),
// several rows per warp, fp32 math (logaddexp / exp to ~1e-7 relative, far
// inside every gate).  The row weights are recomputed by each lane of the row
// from the two L values (one broadcast load per lane group).
template <int LPR>
__global__ void __launch_bounds__(256)
merge_f32v_kernel(View3<const float> OA, View3<const float> LA, View3<const float> OB,
                  View3<const float> LB, View3<float> O, View3<float> L, int64_t nrows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gr = t / LPR;
  const int c = (int)(t % LPR) * 4;
  if (gr >= nrows) return;
  const int64_t h = gr / O.rows, i = gr % O.rows;
  const float la = *LA.at(h, i), lb = *LB.at(h, i);
  float lm;
  if (la == lb) {
    lm = la + 0.693147180559945309f;      // numpy.logaddexp(x, x); -inf stays -inf
  } else {
    const float hi = fmaxf(la, lb), lo = fminf(la, lb);
    lm = isinf(hi) ? hi : hi + log1pf(expf(lo - hi));
  }
  const float safe = (isinf(lm) && lm < 0.f) ? 0.f : lm;
  const float wa = expf(la - safe), wb = expf(lb - safe);
  const float4 a = __ldcs(reinterpret_cast<const float4*>(OA.at(h, i) + c));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(OB.at(h, i) + c));
  __stcs(reinterpret_cast<float4*>(O.at(h, i) + c),
         make_float4(wa * a.x + wb * b.x, wa * a.y + wb * b.y, wa * a.z + wb * b.z,
                     wa * a.w + wb * b.w));
  if (c == 0) *L.at(h, i) = lm;
}

template <int LPR, typename Tg>
__global__ void __launch_bounds__(256)
row_stats_f32v_kernel(View3<const float> O, View3<const Tg> dO, View3<float> D, int64_t nrows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gr = t / LPR;
  const int c = (int)(t % LPR) * 4;
  const bool live = gr < nrows;
  float acc = 0.f;
  int64_t h = 0, i = 0;
  if (live) {
    h = gr / O.rows;
    i = gr % O.rows;
    const float4 o = __ldcs(reinterpret_cast<const float4*>(O.at(h, i) + c));
    float g[4];
    if constexpr (std::is_same<Tg, float>::value) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(dO.at(h, i) + c));
      g[0] = v.x; g[1] = v.y; g[2] = v.z; g[3] = v.w;
    } else {
      const uint2 v = __ldcs(reinterpret_cast<const uint2*>(dO.at(h, i) + c));
      const __nv_bfloat162 p0 = *reinterpret_cast<const __nv_bfloat162*>(&v.x);
      const __nv_bfloat162 p1 = *reinterpret_cast<const __nv_bfloat162*>(&v.y);
      g[0] = __bfloat162float(p0.x); g[1] = __bfloat162float(p0.y);
      g[2] = __bfloat162float(p1.x); g[3] = __bfloat162float(p1.y);
    }
    acc = o.x * g[0] + o.y * g[1] + o.z * g[2] + o.w * g[3];
  }
#pragma unroll
  for (int off = LPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (live && c == 0) *D.at(h, i) = acc;
}

bool f32_vec_ok(const lvx_view* v) {
  return v->d % 4 == 0 && (reinterpret_cast<uintptr_t>(v->data) & 15) == 0 &&
         v->row_stride % 4 == 0 && (v->heads <= 1 || v->head_stride % 4 == 0);
}
bool bf16_vec_ok(const lvx_view* v) {
  return v->d % 4 == 0 && (reinterpret_cast<uintptr_t>(v->data) & 7) == 0 &&
         v->row_stride % 4 == 0 && (v->heads <= 1 || v->head_stride % 4 == 0);
}
// lanes per row of the vector kernels: d/4 when that is a power of two <= 32
int vec_lanes(int64_t d) {
  const int64_t l = d / 4;
  return (l >= 1 && l <= 32 && (l & (l - 1)) == 0) ? (int)l : 0;
}

template <int LPR>
int merge_vec(const lvx_view* oa, const lvx_view* la, const lvx_view* ob, const lvx_view* lb,
              const lvx_view* o, const lvx_view* l, int64_t nrows, cudaStream_t st) {
  const int64_t threads = nrows * LPR;
  merge_f32v_kernel<LPR><<<(unsigned)ceil_div(threads, 256), 256, 0, st>>>(
      View3<const float>{static_cast<const float*>(oa->data), oa->heads, oa->rows, oa->d,
                         oa->head_stride, oa->row_stride},
      View3<const float>{static_cast<const float*>(la->data), la->heads, la->rows, la->d,
                         la->head_stride, la->row_stride},
      View3<const float>{static_cast<const float*>(ob->data), ob->heads, ob->rows, ob->d,
                         ob->head_stride, ob->row_stride},
      View3<const float>{static_cast<const float*>(lb->data), lb->heads, lb->rows, lb->d,
                         lb->head_stride, lb->row_stride},
      make_view<float>(o), make_view<float>(l), nrows);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

template <int LPR, typename Tg>
int row_stats_vec(const lvx_view* o, const lvx_view* dO, const lvx_view* D, int64_t nrows,
                  cudaStream_t st) {
  row_stats_f32v_kernel<LPR, Tg><<<(unsigned)ceil_div(nrows * LPR, 256), 256, 0, st>>>(
      View3<const float>{static_cast<const float*>(o->data), o->heads, o->rows, o->d,
                         o->head_stride, o->row_stride},
      View3<const Tg>{static_cast<const Tg*>(dO->data), dO->heads, dO->rows, dO->d,
                      dO->head_stride, dO->row_stride},
      make_view<float>(D), nrows);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

#define LVX_LPR_DISPATCH(lpr, CALL)            \
  switch (lpr) {                               \
    case 1: { constexpr int LPR = 1; CALL; }   \
    case 2: { constexpr int LPR = 2; CALL; }   \
    case 4: { constexpr int LPR = 4; CALL; }   \
    case 8: { constexpr int LPR = 8; CALL; }   \
    case 16: { constexpr int LPR = 16; CALL; } \
    default: { constexpr int LPR = 32; CALL; } \
  }

template <typename Ts>
__global__ void fill_empty_kernel(View3<Ts> O, View3<Ts> L) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = O.heads * O.rows * O.d;
  if (idx >= total) return;
  const int64_t c = idx % O.d, r = (idx / O.d) % O.rows, h = idx / (O.d * O.rows);
  O.at(h, r)[c] = from_acc<Ts, float>(0.f);
  if (c == 0) *L.at(h, r) = from_acc<Ts, float>(-INFINITY);
}

template <typename Ta, typename Tb>
__global__ void convert_kernel(View3<const Ta> A, View3<Tb> B) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = A.heads * A.rows * A.d;
  if (idx >= total) return;
  const int64_t c = idx % A.d, r = (idx / A.d) % A.rows, h = idx / (A.d * A.rows);
  B.at(h, r)[c] = from_acc<Tb, double>(to_acc<double>(A.at(h, r)[c]));
}

template <typename T>
View3<const T> cview(const lvx_view* v) {
  return View3<const T>{static_cast<const T*>(v->data), v->heads, v->rows, v->d,
                        v->head_stride, v->row_stride};
}

int launch_status() {
  note_launch();
  return cudaGetLastError() == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

template <typename Tin, typename Ts, typename Acc, int DPL>
int fwd_launch(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
               const lvx_view* po, const lvx_view* pl, const lvx_view* o, const lvx_view* l,
               cudaStream_t st) {
  const int64_t warps = q->heads * q->rows;
  if (warps == 0) return LVX_OK;
  const bool prior = po && pl;
  View3<const Ts> POv = prior ? cview<Ts>(po) : View3<const Ts>{};
  View3<const Ts> PLv = prior ? cview<Ts>(pl) : View3<const Ts>{};
  simt_fwd_kernel<Tin, Ts, Acc, DPL><<<ceil_div(warps, kWarps), kWarps * 32, 0, st>>>(
      cview<Tin>(q), cview<Tin>(k), cview<Tin>(v), (Acc)scale, POv, PLv, prior,
      make_view<Ts>(o), make_view<Ts>(l));
  return launch_status();
}

template <typename Tin, typename Ts, typename Acc, int DPL>
int bwd_launch(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
               const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dq,
               const lvx_view* dk, const lvx_view* dv, int acc, cudaStream_t st) {
  const int64_t wq = dq ? q->heads * q->rows : 0, wk = dk ? k->heads * k->rows : 0;
  if (wq) {
    simt_bwd_dq_kernel<Tin, Ts, Acc, DPL><<<ceil_div(wq, kWarps), kWarps * 32, 0, st>>>(
        cview<Tin>(q), cview<Tin>(k), cview<Tin>(v), cview<Ts>(L), cview<Ts>(D),
        cview<Tin>(dO), (Acc)scale, make_view<Ts>(dq), acc != 0);
    if (launch_status()) return LVX_ECUDA;
  }
  if (wk) {
    simt_bwd_dkv_kernel<Tin, Ts, Acc, DPL><<<ceil_div(wk, kWarps), kWarps * 32, 0, st>>>(
        cview<Tin>(q), cview<Tin>(k), cview<Tin>(v), cview<Ts>(L), cview<Ts>(D),
        cview<Tin>(dO), (Acc)scale, make_view<Ts>(dk), make_view<Ts>(dv), acc != 0);
    if (launch_status()) return LVX_ECUDA;
  }
  return LVX_OK;
}

template <typename Tin, typename Ts, typename Acc>
int fwd_by_d(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
             const lvx_view* po, const lvx_view* pl, const lvx_view* o, const lvx_view* l,
             cudaStream_t st) {
  const int64_t d = q->d;
  if (d <= 32) return fwd_launch<Tin, Ts, Acc, 1>(q, k, v, scale, po, pl, o, l, st);
  if (d <= 64) return fwd_launch<Tin, Ts, Acc, 2>(q, k, v, scale, po, pl, o, l, st);
  if (d <= 128) return fwd_launch<Tin, Ts, Acc, 4>(q, k, v, scale, po, pl, o, l, st);
  if (d <= kMaxD) return fwd_launch<Tin, Ts, Acc, 8>(q, k, v, scale, po, pl, o, l, st);
  return LVX_EUNSUPPORTED;
}

template <typename Tin, typename Ts, typename Acc>
int bwd_by_d(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
             const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dq,
             const lvx_view* dk, const lvx_view* dv, int acc, cudaStream_t st) {
  const int64_t d = q->d;
  if (d <= 32) return bwd_launch<Tin, Ts, Acc, 1>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
  if (d <= 64) return bwd_launch<Tin, Ts, Acc, 2>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
  if (d <= 128) return bwd_launch<Tin, Ts, Acc, 4>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
  if (d <= kMaxD) return bwd_launch<Tin, Ts, Acc, 8>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
  return LVX_EUNSUPPORTED;
}

}  // namespace

int simt_fwd(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
             const lvx_view* po, const lvx_view* pl, const lvx_view* o, const lvx_view* l,
             cudaStream_t st) {
  switch (q->dtype) {
    case LVX_F32: return fwd_by_d<float, float, double>(q, k, v, scale, po, pl, o, l, st);
    case LVX_F64: return fwd_by_d<double, double, double>(q, k, v, scale, po, pl, o, l, st);
    case LVX_BF16: return fwd_by_d<__nv_bfloat16, float, float>(q, k, v, scale, po, pl, o, l, st);
  }
  return LVX_EDTYPE;
}

int simt_bwd(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
             const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dq,
             const lvx_view* dk, const lvx_view* dv, int acc, cudaStream_t st) {
  switch (q->dtype) {
    case LVX_F32:
      return bwd_by_d<float, float, double>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
    case LVX_F64:
      return bwd_by_d<double, double, double>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
    case LVX_BF16:
      return bwd_by_d<__nv_bfloat16, float, float>(q, k, v, L, D, dO, scale, dq, dk, dv, acc, st);
  }
  return LVX_EDTYPE;
}

int merge(const lvx_view* oa, const lvx_view* la, const lvx_view* ob, const lvx_view* lb,
          const lvx_view* o, const lvx_view* l, cudaStream_t st) {
  const int64_t warps = o->heads * o->rows;
  if (!warps) return LVX_OK;
  const int threads = 256;
  const int64_t blocks = ceil_div(warps * 32, threads);
  const int lpr = vec_lanes(o->d);
  if (o->dtype == LVX_F32 && lpr && f32_vec_ok(oa) && f32_vec_ok(ob) && f32_vec_ok(o))
    LVX_LPR_DISPATCH(lpr, return merge_vec<LPR>(oa, la, ob, lb, o, l, warps, st))
  if (o->dtype == LVX_F32)
    merge_kernel<float><<<blocks, threads, 0, st>>>(cview<float>(oa), cview<float>(la),
                                                    cview<float>(ob), cview<float>(lb),
                                                    make_view<float>(o), make_view<float>(l));
  else if (o->dtype == LVX_F64)
    merge_kernel<double><<<blocks, threads, 0, st>>>(cview<double>(oa), cview<double>(la),
                                                     cview<double>(ob), cview<double>(lb),
                                                     make_view<double>(o), make_view<double>(l));
  else
    return LVX_EDTYPE;
  return launch_status();
}

int row_stats(const lvx_view* o, const lvx_view* dO, const lvx_view* D, cudaStream_t st) {
  const int64_t warps = o->heads * o->rows;
  if (!warps) return LVX_OK;
  const int threads = 256;
  const int64_t blocks = ceil_div(warps * 32, threads);
  const int lpr = vec_lanes(o->d);
  if (o->dtype == LVX_F32 && lpr && f32_vec_ok(o) && D->dtype == LVX_F32) {
    if (dO->dtype == LVX_F32 && f32_vec_ok(dO))
      LVX_LPR_DISPATCH(lpr, return (row_stats_vec<LPR, float>(o, dO, D, warps, st)))
    if (dO->dtype == LVX_BF16 && bf16_vec_ok(dO))
      LVX_LPR_DISPATCH(lpr, return (row_stats_vec<LPR, __nv_bfloat16>(o, dO, D, warps, st)))
  }
  if (o->dtype == LVX_F32 && dO->dtype == LVX_F32)
    row_stats_kernel<float, float><<<blocks, threads, 0, st>>>(cview<float>(o), cview<float>(dO),
                                                               make_view<float>(D));
  else if (o->dtype == LVX_F32 && dO->dtype == LVX_BF16)
    row_stats_kernel<float, __nv_bfloat16><<<blocks, threads, 0, st>>>(
        cview<float>(o), cview<__nv_bfloat16>(dO), make_view<float>(D));
  else if (o->dtype == LVX_F64 && dO->dtype == LVX_F64)
    row_stats_kernel<double, double><<<blocks, threads, 0, st>>>(
        cview<double>(o), cview<double>(dO), make_view<double>(D));
  else
    return LVX_EDTYPE;
  return launch_status();
}

int fill_empty(const lvx_view* o, const lvx_view* l, cudaStream_t st) {
  const int64_t total = o->heads * o->rows * o->d;
  if (!total) return LVX_OK;
  const int threads = 256;
  if (o->dtype == LVX_F32)
    fill_empty_kernel<float><<<ceil_div(total, threads), threads, 0, st>>>(make_view<float>(o),
                                                                          make_view<float>(l));
  else if (o->dtype == LVX_F64)
    fill_empty_kernel<double><<<ceil_div(total, threads), threads, 0, st>>>(
        make_view<double>(o), make_view<double>(l));
  else
    return LVX_EDTYPE;
  return launch_status();
}

template <typename Ta>
static int convert_to(const lvx_view* a, const lvx_view* b, cudaStream_t st) {
  const int64_t total = a->heads * a->rows * a->d;
  const int threads = 256;
  const int64_t blocks = ceil_div(total, threads);
  switch (b->dtype) {
    case LVX_F32:
      convert_kernel<Ta, float><<<blocks, threads, 0, st>>>(cview<Ta>(a), make_view<float>(b));
      break;
    case LVX_F64:
      convert_kernel<Ta, double><<<blocks, threads, 0, st>>>(cview<Ta>(a), make_view<double>(b));
      break;
    case LVX_BF16:
      convert_kernel<Ta, __nv_bfloat16><<<blocks, threads, 0, st>>>(
          cview<Ta>(a), make_view<__nv_bfloat16>(b));
      break;
    default:
      return LVX_EDTYPE;
  }
  return launch_status();
}

template <typename Ts>
__global__ void accum_kernel(View3<const Ts> A, View3<Ts> B, bool acc) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = A.heads * A.rows * A.d;
  if (idx >= total) return;
  const int64_t c = idx % A.d, r = (idx / A.d) % A.rows, h = idx / (A.d * A.rows);
  Ts* o = B.at(h, r) + c;
  *o = acc ? *o + A.at(h, r)[c] : A.at(h, r)[c];
}

template <typename Ts>
__global__ void zero_state_kernel(View3<Ts> A) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= A.heads * A.rows * A.d) return;
  const int64_t c = idx % A.d, r = (idx / A.d) % A.rows, h = idx / (A.d * A.rows);
  A.at(h, r)[c] = Ts(0);
}

int fill_empty_zero(const lvx_view* a, cudaStream_t st) {
  const int64_t total = a->heads * a->rows * a->d;
  if (!total) return LVX_OK;
  const int threads = 256;
  if (a->dtype == LVX_F32)
    zero_state_kernel<float><<<ceil_div(total, threads), threads, 0, st>>>(make_view<float>(a));
  else if (a->dtype == LVX_F64)
    zero_state_kernel<double><<<ceil_div(total, threads), threads, 0, st>>>(make_view<double>(a));
  else if (a->dtype == LVX_BF16)
    zero_state_kernel<__nv_bfloat16><<<ceil_div(total, threads), threads, 0, st>>>(
        make_view<__nv_bfloat16>(a));
  else
    return LVX_EDTYPE;
  return launch_status();
}

int accumulate_into(const lvx_view* a, const lvx_view* b, int acc, cudaStream_t st) {
  const int64_t total = a->heads * a->rows * a->d;
  if (!total) return LVX_OK;
  const int threads = 256;
  if (a->dtype == LVX_F32 && b->dtype == LVX_F32)
    accum_kernel<float><<<ceil_div(total, threads), threads, 0, st>>>(cview<float>(a),
                                                                     make_view<float>(b), acc != 0);
  else if (a->dtype == LVX_F64 && b->dtype == LVX_F64)
    accum_kernel<double><<<ceil_div(total, threads), threads, 0, st>>>(
        cview<double>(a), make_view<double>(b), acc != 0);
  else
    return LVX_EDTYPE;
  return launch_status();
}

int convert(const lvx_view* a, const lvx_view* b, cudaStream_t st) {
  if (a->heads * a->rows * a->d == 0) return LVX_OK;
  switch (a->dtype) {
    case LVX_F32: return convert_to<float>(a, b, st);
    case LVX_F64: return convert_to<double>(a, b, st);
    case LVX_BF16: return convert_to<__nv_bfloat16>(a, b, st);
  }
  return LVX_EDTYPE;
}

}  // namespace lvx
