// Projections of the cross-attention layer: project / project_backward
// (reference kernels.py:227-254) and the MLLM K/V recompute from the shared
// visual tokens (mllm.py:296-300 forward, :358-360 backward).
//
// The GEMMs run on the hand-written tcgen05 kernel of lvx_gemm_sm100.cu (bf16
// in, fp32 accumulate) or its exact SIMT sibling (f32 / f64).  The head
// layout is folded into the GEMM's leading dimensions, so [heads, S, d]
// outputs that are column blocks of one [S, heads*d] matrix (head_stride == d:
// the layout the recompute layer keeps) take ONE GEMM with N = heads*d; any
// other head stride one GEMM per head.  No copies.
#include <cuda_runtime.h>

#include "lvx_common.cuh"

namespace lvx {
namespace {

size_t esize(int32_t dt) { return dt == LVX_F64 ? 8 : (dt == LVX_F32 ? 4 : 2); }

// Row-major C[M,N] (ldc) = op(A)[M,K] op(B)[K,N] (+ C), batched over `batch`
// operand / output element strides sA / sB / sC (one launch per batch entry:
// only views whose heads are not column blocks of one matrix get here).
int gemm_rm(cudaStream_t st, int32_t dt, bool ta, bool tb, int64_t M, int64_t N, int64_t K,
            const void* A, int64_t lda, int64_t sA, const void* B, int64_t ldb, int64_t sB,
            void* C, int64_t ldc, int64_t sC, int batch, bool accumulate) {
  if (dt != LVX_BF16 && dt != LVX_F32 && dt != LVX_F64) return LVX_EDTYPE;
  const int64_t es = (int64_t)esize(dt);
  for (int b = 0; b < batch; ++b) {
    GemmCall g{dt, M, N, K,
               static_cast<const char*>(A) + b * sA * es, lda, ta,
               static_cast<const char*>(B) + b * sB * es, ldb, tb,
               static_cast<char*>(C) + b * sC * es, ldc, accumulate, dt};
    const int s = gemm(g, st);
    if (s) return s;
  }
  return LVX_OK;
}

bool mat_ok(const lvx_matrix* m) {
  return m && m->rows >= 0 && m->cols >= 0 && m->row_stride >= m->cols &&
         (m->data || m->rows == 0 || m->cols == 0);
}

const char* at(const void* p, int64_t elems, int32_t dt) {
  return static_cast<const char*>(p) + elems * (int64_t)esize(dt);
}

int project_impl(cudaStream_t h, const lvx_matrix* x, const lvx_matrix* w, const lvx_view* out) {
  const int64_t heads = out->heads, S = x->rows, e = x->cols, d = out->d;
  if (w->rows != e || w->cols != heads * d || out->rows != S) return LVX_EINVAL;
  if (out->head_stride == d || heads == 1)   // [S, heads*d] column blocks: one GEMM
    return gemm_rm(h, x->dtype, false, false, S, heads * d, e, x->data, x->row_stride, 0,
                   w->data, w->row_stride, 0, out->data, out->row_stride, 0, 1, false);
  return gemm_rm(h, x->dtype, false, false, S, d, e, x->data, x->row_stride, 0, w->data,
                 w->row_stride, d, out->data, out->row_stride, out->head_stride, (int)heads,
                 false);
}

}  // namespace
}  // namespace lvx

using namespace lvx;

extern "C" {

int lvx_project(const lvx_matrix* x, const lvx_matrix* w, const lvx_view* out, void* stream) {
  if (!mat_ok(x) || !mat_ok(w) || !out || out->heads < 1 || out->d < 1) return LVX_EINVAL;
  if (x->dtype != w->dtype || x->dtype != out->dtype) return LVX_EDTYPE;
  cudaStream_t h = static_cast<cudaStream_t>(stream);
  return project_impl(h, x, w, out);
}

int lvx_kv_recompute(const lvx_matrix* y, const lvx_matrix* w_k, const lvx_matrix* w_v,
                     const lvx_view* k_out, const lvx_view* v_out, void* stream) {
  if (!mat_ok(y) || !mat_ok(w_k) || !mat_ok(w_v) || !k_out || !v_out) return LVX_EINVAL;
  if (y->dtype != w_k->dtype || y->dtype != w_v->dtype || y->dtype != k_out->dtype ||
      y->dtype != v_out->dtype)
    return LVX_EDTYPE;
  if (k_out->heads != v_out->heads || k_out->d != v_out->d || k_out->rows != v_out->rows)
    return LVX_EINVAL;
  cudaStream_t h = static_cast<cudaStream_t>(stream);
  const int64_t hd = k_out->heads * k_out->d;
  const int32_t dt = y->dtype;
  // [W_K | W_V] adjacent in one weight and K | V adjacent in one [S, 2 hkv d]
  // output: the whole recompute is ONE GEMM y @ [W_K | W_V]
  const bool fused = w_v->data == at(w_k->data, hd, dt) && w_v->row_stride == w_k->row_stride &&
                     v_out->data == at(k_out->data, hd, dt) && k_out->head_stride == k_out->d &&
                     v_out->head_stride == v_out->d && k_out->row_stride == v_out->row_stride &&
                     w_k->cols == hd && w_v->cols == hd;
  if (fused) {
    lvx_matrix w{w_k->data, w_k->rows, 2 * hd, w_k->row_stride, dt, 0};
    lvx_view out{k_out->data, 2 * k_out->heads, k_out->rows, k_out->d, k_out->d,
                 k_out->row_stride, dt, 0};
    return project_impl(h, y, &w, &out);
  }
  int s = project_impl(h, y, w_k, k_out);
  return s ? s : project_impl(h, y, w_v, v_out);
}

int lvx_project_bwd(const lvx_matrix* x, const lvx_matrix* w, const lvx_view* dout,
                    const lvx_matrix* dx, const lvx_matrix* dw, void* stream) {
  if (!mat_ok(x) || !mat_ok(w) || !dout || !mat_ok(dx) || !mat_ok(dw)) return LVX_EINVAL;
  const int32_t dt = x->dtype;
  if (w->dtype != dt || dout->dtype != dt || dx->dtype != dt || dw->dtype != dt)
    return LVX_EDTYPE;
  const int64_t heads = dout->heads, S = x->rows, e = x->cols, d = dout->d;
  if (dout->rows != S || w->rows != e || w->cols != heads * d || dx->rows != S ||
      dx->cols != e || dw->rows != e || dw->cols != heads * d)
    return LVX_EINVAL;
  cudaStream_t h = static_cast<cudaStream_t>(stream);
  const bool flat = dout->head_stride == d || heads == 1;
  int s;
  // dX = dOut_flat W^T (kernels.py:250)
  if (flat) {
    s = gemm_rm(h, dt, false, true, S, e, heads * d, dout->data, dout->row_stride, 0, w->data,
                w->row_stride, 0, dx->data, dx->row_stride, 0, 1, false);
  } else {
    s = LVX_OK;
    for (int64_t hh = 0; hh < heads && !s; ++hh)
      s = gemm_rm(h, dt, false, true, S, e, d, at(dout->data, hh * dout->head_stride, dt),
                  dout->row_stride, 0, at(w->data, hh * d, dt), w->row_stride, 0, dx->data,
                  dx->row_stride, 0, 1, hh > 0);
  }
  if (s) return s;
  // dW = x^T dOut_flat (kernels.py:251)
  if (flat)
    return gemm_rm(h, dt, true, false, e, heads * d, S, x->data, x->row_stride, 0, dout->data,
                   dout->row_stride, 0, dw->data, dw->row_stride, 0, 1, false);
  return gemm_rm(h, dt, true, false, e, d, S, x->data, x->row_stride, 0, dout->data,
                 dout->row_stride, dout->head_stride, dw->data, dw->row_stride, d, (int)heads,
                 false);
}

}  // extern "C"

extern "C" int lvx_gemm(const lvx_matrix* a, int ta, const lvx_matrix* b, int tb,
                        const lvx_matrix* c, int accumulate, void* stream) {
  if (!mat_ok(a) || !mat_ok(b) || !mat_ok(c)) return LVX_EINVAL;
  if (a->dtype != b->dtype) return LVX_EDTYPE;
  // c in the operands' dtype, or fp32 for bf16 operands (an fp32 accumulator)
  if (c->dtype != a->dtype && !(a->dtype == LVX_BF16 && c->dtype == LVX_F32)) return LVX_EDTYPE;
  const int64_t M = ta ? a->cols : a->rows, K = ta ? a->rows : a->cols;
  const int64_t Kb = tb ? b->cols : b->rows, N = tb ? b->rows : b->cols;
  if (K != Kb || c->rows != M || c->cols != N) return LVX_EINVAL;
  GemmCall g{a->dtype, M, N, K, a->data, a->row_stride, ta != 0, b->data, b->row_stride,
             tb != 0, c->data, c->row_stride, accumulate != 0, c->dtype};
  return gemm(g, static_cast<cudaStream_t>(stream));
}
