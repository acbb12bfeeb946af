// Shared helpers for the LV-XAttn B200 kernels: view descriptors, dtype
// conversion and warp reductions.  sm_100a only.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>

#include "../../include/lvx_b200.h"

namespace lvx {

// Device-side copy of an lvx_view with the pointer typed.
template <typename T>
struct View3 {
  T* p;
  int64_t heads, rows, d, hs, rs;
  __host__ __device__ T* at(int64_t h, int64_t r) const { return p + h * hs + r * rs; }
};

template <typename T>
inline View3<T> make_view(const lvx_view* v) {
  return View3<T>{static_cast<T*>(v->data), v->heads, v->rows, v->d, v->head_stride,
                  v->row_stride};
}

template <typename Acc, typename T>
__device__ __forceinline__ Acc to_acc(T x) { return static_cast<Acc>(x); }
template <>
__device__ __forceinline__ float to_acc<float, __nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <>
__device__ __forceinline__ double to_acc<double, __nv_bfloat16>(__nv_bfloat16 x) {
  return static_cast<double>(__bfloat162float(x));
}

template <typename T, typename Acc>
__device__ __forceinline__ T from_acc(Acc x) { return static_cast<T>(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16, float>(float x) {
  return __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16, double>(double x) {
  return __float2bfloat16_rn(static_cast<float>(x));
}

template <typename Acc>
__device__ __forceinline__ Acc warp_sum(Acc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename Acc>
__device__ __forceinline__ Acc warp_max(Acc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float exp_acc(float x) { return expf(x); }
__device__ __forceinline__ double exp_acc(double x) { return exp(x); }
__device__ __forceinline__ float log_acc(float x) { return logf(x); }
__device__ __forceinline__ double log_acc(double x) { return log(x); }
__device__ __forceinline__ float log1p_acc(float x) { return log1pf(x); }
__device__ __forceinline__ double log1p_acc(double x) { return log1p(x); }

template <typename Acc>
__device__ __forceinline__ Acc neg_inf() { return -INFINITY; }

// numpy.logaddexp semantics: equal arguments give x + log 2, -inf/-inf stays -inf
template <typename Acc>
__device__ __forceinline__ Acc logaddexp(Acc a, Acc b) {
  if (a == b) return a + static_cast<Acc>(0.693147180559945309417232121458);
  Acc hi = fmax(a, b), lo = fmin(a, b);
  if (isinf(hi)) return hi;  // +-inf dominates (both -inf handled above)
  return hi + log1p_acc(exp_acc(lo - hi));
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lvx

// Internal entry points implemented per translation unit (not part of the ABI).
namespace lvx {
// diagnostic count of kernel launches issued by this library (lvx_kernel_launches)
void note_launch(int n = 1);
int simt_fwd(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
             const lvx_view* prior_o, const lvx_view* prior_l, const lvx_view* o,
             const lvx_view* l, cudaStream_t st);
// dq / dk+dv halves are selected by non-null outputs
int simt_bwd(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
             const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dq,
             const lvx_view* dk, const lvx_view* dv, int accumulate, cudaStream_t st);
// zero an F32/F64 view
int fill_empty_zero(const lvx_view* a, cudaStream_t st);
// dst (+)= src, state dtypes, same shapes
int accumulate_into(const lvx_view* src, const lvx_view* dst, int accumulate, cudaStream_t st);
int merge(const lvx_view* oa, const lvx_view* la, const lvx_view* ob, const lvx_view* lb,
          const lvx_view* o, const lvx_view* l, cudaStream_t st);
int row_stats(const lvx_view* o, const lvx_view* dO, const lvx_view* D, cudaStream_t st);
int fill_empty(const lvx_view* o, const lvx_view* l, cudaStream_t st);
int convert(const lvx_view* src, const lvx_view* dst, cudaStream_t st);

// tcgen05 (sm_100a) kernels, lvx_fwd_sm100.cu / lvx_bwd_sm100.cu
bool tc_fwd_eligible(const lvx_view* q, const lvx_view* k, const lvx_view* v);
size_t tc_fwd_workspace(const lvx_view* q, const lvx_view* k);
int tc_fwd_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
                   void* ws, size_t ws_bytes, cudaStream_t st);
int tc_fwd_finish(const lvx_view* q, const lvx_view* k, const lvx_view* prior_o,
                  const lvx_view* prior_l, const lvx_view* o, const lvx_view* l, void* ws,
                  size_t ws_bytes, cudaStream_t st);
bool tc_bwd_eligible(const lvx_view* q, const lvx_view* k, const lvx_view* v);
bool tc_bwd_outputs_ok(const lvx_view* dO, const lvx_view* a, const lvx_view* b);
size_t tc_bwd_workspace(const lvx_view* q, const lvx_view* k);
int tc_bwd_dq_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                      const lvx_view* L, const lvx_view* D, const lvx_view* dO, double scale,
                      void* ws, size_t ws_bytes, cudaStream_t st);
int tc_bwd_dq_finish(const lvx_view* q, const lvx_view* k, const lvx_view* dq, int accumulate,
                     void* ws, size_t ws_bytes, cudaStream_t st);
int tc_bwd_dkv(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
               const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dk,
               const lvx_view* dv, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st);

// GEMMs (lvx_gemm_sm100.cu): C[M, N] (+)= op(A) op(B), row-major storage;
// op(A) = A^T when ta (A stored [K, M]), op(B) = B^T when tb (B stored [N, K]).
struct GemmCall {
  int32_t dtype;
  int64_t M, N, K;
  const void* a;
  int64_t lda;
  bool ta;
  const void* b;
  int64_t ldb;
  bool tb;
  void* c;
  int64_t ldc;
  bool accumulate;
  int32_t c_dtype;   // = dtype, or LVX_F32 for bf16 operands into an fp32 C
};
int gemm(const GemmCall& g, cudaStream_t st);
// cuTensorMapEncodeTiled through the runtime's driver entry point (null if absent)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

// Raise a kernel's dynamic shared memory limit once per device: function
// attributes belong to the device's context, so a process driving several
// GPUs needs the call on each (bit d of `done` = device d).
template <typename F>
inline bool ensure_smem_attr(F* fn, int bytes, std::atomic<unsigned>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const unsigned bit = dev < 32 ? 1u << dev : 0u;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return false;
  done.fetch_or(bit, std::memory_order_release);
  return true;
}

}  // namespace lvx
