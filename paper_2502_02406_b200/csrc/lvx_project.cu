// Projections of the cross-attention layer: project / project_backward
// (reference kernels.py:227-254) and the MLLM K/V recompute from the shared
// visual tokens (mllm.py:296-300 forward, :358-360 backward).
//
// These are plain GEMMs and run on cuBLAS (bf16 in, fp32 accumulate; f32 and
// f64 without TF32).  The head layout is folded into the GEMM's leading
// dimensions and batch strides, so [heads, S, d] outputs that are column
// blocks of one [S, heads*d] matrix (head_stride == d: the layout the
// recompute layer keeps) take ONE GEMM with N = heads*d, and any other
// head stride takes one strided-batched GEMM over heads.  No copies.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <mutex>

#include "lvx_common.cuh"

namespace lvx {
namespace {

constexpr int kMaxDevices = 64;

// One cuBLAS handle per device, created on first use; calls are serialised
// because a handle's stream binding is shared state.
std::mutex g_mu;
cublasHandle_t g_handle[kMaxDevices] = {};

cublasHandle_t handle_for_current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  if (!g_handle[dev]) {
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    g_handle[dev] = h;
  }
  return g_handle[dev];
}

bool gemm_types(int32_t dt, cudaDataType_t* t, cublasComputeType_t* c) {
  switch (dt) {
    case LVX_BF16: *t = CUDA_R_16BF; *c = CUBLAS_COMPUTE_32F; return true;
    case LVX_F32: *t = CUDA_R_32F; *c = CUBLAS_COMPUTE_32F_PEDANTIC; return true;
    case LVX_F64: *t = CUDA_R_64F; *c = CUBLAS_COMPUTE_64F; return true;
    default: return false;
  }
}

size_t esize(int32_t dt) { return dt == LVX_F64 ? 8 : (dt == LVX_F32 ? 4 : 2); }

// Row-major C[M,N] (ldc) = op(A)[M,K] op(B)[K,N] + beta C, batched with element
// strides sA / sB / sC (batch 1 = plain GEMM).  Column-major cuBLAS sees the
// transposes: C^T = op(B)^T op(A)^T.
int gemm_rm(cublasHandle_t h, int32_t dt, bool ta, bool tb, int64_t M, int64_t N, int64_t K,
            const void* A, int64_t lda, int64_t sA, const void* B, int64_t ldb, int64_t sB,
            void* C, int64_t ldc, int64_t sC, int batch, bool accumulate) {
  cudaDataType_t t;
  cublasComputeType_t ct;
  if (!gemm_types(dt, &t, &ct)) return LVX_EDTYPE;
  if (M <= 0 || N <= 0 || batch <= 0) return LVX_OK;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || lda > INT32_MAX || ldb > INT32_MAX ||
      ldc > INT32_MAX)
    return LVX_EUNSUPPORTED;
  const float a32 = 1.f, b32 = accumulate ? 1.f : 0.f;
  const double a64 = 1.0, b64 = accumulate ? 1.0 : 0.0;
  const void* alpha = dt == LVX_F64 ? static_cast<const void*>(&a64) : &a32;
  const void* beta = dt == LVX_F64 ? static_cast<const void*>(&b64) : &b32;
  const cublasOperation_t opB = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t opA = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
  if (K == 0) {   // empty contraction: C = 0 (or unchanged when accumulating)
    if (accumulate) return LVX_OK;
    cudaStream_t st = nullptr;
    cublasGetStream(h, &st);
    for (int b = 0; b < batch; ++b)
      if (cudaMemset2DAsync(static_cast<char*>(C) + (int64_t)b * sC * (int64_t)esize(dt),
                            ldc * esize(dt), 0, N * esize(dt), M, st) != cudaSuccess)
        return LVX_ECUDA;
    return LVX_OK;
  }
  cublasStatus_t s;
  if (batch == 1)
    s = cublasGemmEx(h, opB, opA, (int)N, (int)M, (int)K, alpha, B, t, (int)ldb, A, t, (int)lda,
                     beta, C, t, (int)ldc, ct, CUBLAS_GEMM_DEFAULT);
  else
    s = cublasGemmStridedBatchedEx(h, opB, opA, (int)N, (int)M, (int)K, alpha, B, t, (int)ldb,
                                   sB, A, t, (int)lda, sA, beta, C, t, (int)ldc, sC, batch, ct,
                                   CUBLAS_GEMM_DEFAULT);
  return s == CUBLAS_STATUS_SUCCESS ? LVX_OK : LVX_ECUDA;
}

bool mat_ok(const lvx_matrix* m) {
  return m && m->rows >= 0 && m->cols >= 0 && m->row_stride >= m->cols &&
         (m->data || m->rows == 0 || m->cols == 0);
}

const char* at(const void* p, int64_t elems, int32_t dt) {
  return static_cast<const char*>(p) + elems * (int64_t)esize(dt);
}

int project_impl(cublasHandle_t h, const lvx_matrix* x, const lvx_matrix* w, const lvx_view* out) {
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
  std::lock_guard<std::mutex> lk(g_mu);
  cublasHandle_t h = handle_for_current_device();
  if (!h || cublasSetStream(h, static_cast<cudaStream_t>(stream)) != CUBLAS_STATUS_SUCCESS)
    return LVX_ECUDA;
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
  std::lock_guard<std::mutex> lk(g_mu);
  cublasHandle_t h = handle_for_current_device();
  if (!h || cublasSetStream(h, static_cast<cudaStream_t>(stream)) != CUBLAS_STATUS_SUCCESS)
    return LVX_ECUDA;
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
  std::lock_guard<std::mutex> lk(g_mu);
  cublasHandle_t h = handle_for_current_device();
  if (!h || cublasSetStream(h, static_cast<cudaStream_t>(stream)) != CUBLAS_STATUS_SUCCESS)
    return LVX_ECUDA;
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
