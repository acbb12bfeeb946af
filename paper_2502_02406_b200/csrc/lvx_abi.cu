// C-ABI entry points (include/lvx_b200.h): argument validation and routing
// to the tcgen05 kernels (BF16, d in {64,128}) or the exact SIMT kernels.
#include <atomic>

#include "lvx_common.cuh"

using namespace lvx;

namespace lvx {
static std::atomic<unsigned long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
}  // namespace lvx

namespace {

bool valid_view(const lvx_view* v) {
  return v && v->heads >= 0 && v->rows >= 0 && v->d >= 1 && v->head_stride >= 0 &&
         v->row_stride >= 0 && (v->data || v->heads * v->rows * v->d == 0);
}

bool dtype_ok(int dt) { return dt == LVX_F32 || dt == LVX_F64 || dt == LVX_BF16; }

int state_dtype(int in) { return in == LVX_F64 ? LVX_F64 : LVX_F32; }

bool same_hr(const lvx_view* a, const lvx_view* b) {
  return a->heads == b->heads && a->rows == b->rows;
}

// kernels.py:62-73 validate_qkv, extended to GQA (hq a multiple of hkv)
int check_qkv(const lvx_view* q, const lvx_view* k, const lvx_view* v) {
  if (!valid_view(q) || !valid_view(k) || !valid_view(v)) return LVX_EINVAL;
  if (!dtype_ok(q->dtype) || k->dtype != q->dtype || v->dtype != q->dtype) return LVX_EDTYPE;
  if (k->heads != v->heads || k->heads == 0 || q->heads % k->heads) return LVX_EINVAL;
  if (k->rows != v->rows || q->d != k->d || v->d != q->d) return LVX_EINVAL;
  return LVX_OK;
}

int check_state(const lvx_view* o, const lvx_view* l, const lvx_view* q) {
  if (!valid_view(o) || !valid_view(l)) return LVX_EINVAL;
  if (o->dtype != state_dtype(q->dtype) || l->dtype != o->dtype) return LVX_EDTYPE;
  if (!same_hr(o, q) || o->d != q->d || !same_hr(l, q)) return LVX_EINVAL;
  return LVX_OK;
}

}  // namespace

extern "C" {

int lvx_abi_version(void) { return LVX_ABI_VERSION; }

unsigned long long lvx_kernel_launches(void) {
  return g_launches.load(std::memory_order_relaxed);
}

const char* lvx_strerror(int s) {
  switch (s) {
    case LVX_OK: return "ok";
    case LVX_EINVAL: return "invalid shape, stride or argument";
    case LVX_EDTYPE: return "unsupported or mismatched dtype";
    case LVX_ECUDA: return "CUDA error";
    case LVX_EUNSUPPORTED: return "no kernel for this configuration";
    case LVX_EWORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

int lvx_tc_eligible(const lvx_view* q, const lvx_view* k) {
  if (!q || !k) return 0;
  return tc_fwd_eligible(q, k, k) ? 1 : 0;
}

// SIMT path scratch: one delta state [hq, rows_q, d] + [hq, rows_q] in the
// state dtype.  tcgen05 path: per-split partial states.
static size_t simt_fwd_ws(const lvx_view* q) {
  const size_t e = q->dtype == LVX_F64 ? 8 : 4;
  const size_t n = (size_t)q->heads * (size_t)q->rows;
  return ((n * (size_t)q->d * e + 255) / 256) * 256 + ((n * e + 255) / 256) * 256;
}

static void simt_ws_views(const lvx_view* q, void* ws, lvx_view* o, lvx_view* l) {
  const size_t e = q->dtype == LVX_F64 ? 8 : 4;
  const size_t n = (size_t)q->heads * (size_t)q->rows;
  const int dt = state_dtype(q->dtype);
  *o = lvx_view{ws, q->heads, q->rows, q->d, q->rows * q->d, q->d, dt, 0};
  char* lp = static_cast<char*>(ws) + ((n * (size_t)q->d * e + 255) / 256) * 256;
  *l = lvx_view{lp, q->heads, q->rows, 1, q->rows, 1, dt, 0};
}

size_t lvx_blockwise_fwd_workspace(const lvx_view* q, const lvx_view* k) {
  if (!q || !k) return 0;
  return tc_fwd_eligible(q, k, k) ? tc_fwd_workspace(q, k) : simt_fwd_ws(q);
}

int lvx_fwd_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
                    void* ws, size_t ws_bytes, void* stream) {
  int s = check_qkv(q, k, v);
  if (s) return s;
  if (ws_bytes < lvx_blockwise_fwd_workspace(q, k)) return LVX_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q->heads * q->rows == 0 || k->rows == 0) return LVX_OK;
  if (tc_fwd_eligible(q, k, v)) return tc_fwd_partial(q, k, v, scale, ws, ws_bytes, st);
  lvx_view o, l;
  simt_ws_views(q, ws, &o, &l);
  return simt_fwd(q, k, v, scale, nullptr, nullptr, &o, &l, st);
}

int lvx_fwd_finish(const lvx_view* q, const lvx_view* k, const lvx_view* prior_o,
                   const lvx_view* prior_l, const lvx_view* o, const lvx_view* l, void* ws,
                   size_t ws_bytes, void* stream) {
  if (!valid_view(q) || !valid_view(k) || !dtype_ok(q->dtype)) return LVX_EINVAL;
  int s = check_state(o, l, q);
  if (s) return s;
  const bool prior = prior_o && prior_l;
  if ((prior_o != nullptr) != (prior_l != nullptr)) return LVX_EINVAL;
  if (prior && (s = check_state(prior_o, prior_l, q))) return s;
  if (ws_bytes < lvx_blockwise_fwd_workspace(q, k)) return LVX_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q->heads * q->rows == 0) return LVX_OK;
  if (k->rows == 0) {  // empty KV block -> empty state (kernels.py:119-120)
    if (prior) {
      if (prior_o->data == o->data && prior_l->data == l->data) return LVX_OK;
      if ((s = convert(prior_o, o, st))) return s;
      return convert(prior_l, l, st);
    }
    return fill_empty(o, l, st);
  }
  if (tc_fwd_eligible(q, k, k))
    return tc_fwd_finish(q, k, prior ? prior_o : nullptr, prior ? prior_l : nullptr, o, l, ws,
                         ws_bytes, st);
  lvx_view wo, wl;
  simt_ws_views(q, ws, &wo, &wl);
  if (prior) return merge(prior_o, prior_l, &wo, &wl, o, l, st);
  if ((s = convert(&wo, o, st))) return s;
  return convert(&wl, l, st);
}

int lvx_blockwise_fwd(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
                      const lvx_view* prior_o, const lvx_view* prior_l, const lvx_view* o,
                      const lvx_view* l, void* ws, size_t ws_bytes, void* stream) {
  int s = lvx_fwd_partial(q, k, v, scale, ws, ws_bytes, stream);
  if (s) return s;
  return lvx_fwd_finish(q, k, prior_o, prior_l, o, l, ws, ws_bytes, stream);
}

int lvx_merge_states(const lvx_view* oa, const lvx_view* la, const lvx_view* ob,
                     const lvx_view* lb, const lvx_view* o, const lvx_view* l, void* stream) {
  for (const lvx_view* v : {oa, la, ob, lb, o, l})
    if (!valid_view(v)) return LVX_EINVAL;
  if (!same_hr(oa, ob) || oa->d != ob->d || !same_hr(oa, o) || o->d != oa->d ||
      !same_hr(la, oa) || !same_hr(lb, oa) || !same_hr(l, oa))
    return LVX_EINVAL;
  for (const lvx_view* v : {oa, la, ob, lb, l})
    if (v->dtype != o->dtype) return LVX_EDTYPE;
  return merge(oa, la, ob, lb, o, l, static_cast<cudaStream_t>(stream));
}

int lvx_row_stats(const lvx_view* o, const lvx_view* d_o, const lvx_view* dd, void* stream) {
  if (!valid_view(o) || !valid_view(d_o) || !valid_view(dd)) return LVX_EINVAL;
  if (!same_hr(o, d_o) || o->d != d_o->d || !same_hr(dd, o)) return LVX_EINVAL;
  if (dd->dtype != o->dtype) return LVX_EDTYPE;
  return row_stats(o, d_o, dd, static_cast<cudaStream_t>(stream));
}

static size_t simt_bwd_ws(const lvx_view* q) {
  const size_t e = q->dtype == LVX_F64 ? 8 : 4;
  return ((size_t)q->heads * q->rows * q->d * e + 255) / 256 * 256 + 256;
}

static lvx_view simt_dq_view(const lvx_view* q, void* ws) {
  return lvx_view{ws, q->heads, q->rows, q->d, q->rows * q->d, q->d, state_dtype(q->dtype), 0};
}

static bool use_tc_bwd(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                       const lvx_view* dO, const lvx_view* a, const lvx_view* b) {
  return tc_bwd_eligible(q, k, v) && tc_bwd_outputs_ok(dO, a, b);
}

size_t lvx_bwd_workspace(const lvx_view* q, const lvx_view* k) {
  if (!q || !k) return 0;
  return tc_bwd_eligible(q, k, k) ? tc_bwd_workspace(q, k) : simt_bwd_ws(q);
}

size_t lvx_blockwise_bwd_workspace(const lvx_view* q, const lvx_view* k) {
  return lvx_bwd_workspace(q, k);
}

static int check_bwd_inputs(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                            const lvx_view* L, const lvx_view* D, const lvx_view* dO) {
  int s = check_qkv(q, k, v);
  if (s) return s;
  if (!valid_view(L) || !valid_view(D) || !valid_view(dO)) return LVX_EINVAL;
  const int sd = state_dtype(q->dtype);
  if (dO->dtype != q->dtype || L->dtype != sd || D->dtype != sd) return LVX_EDTYPE;
  if (!same_hr(dO, q) || dO->d != q->d || !same_hr(L, q) || !same_hr(D, q)) return LVX_EINVAL;
  return LVX_OK;
}

static int check_acc(const lvx_view* a, const lvx_view* like, int sd) {
  if (!valid_view(a)) return LVX_EINVAL;
  if (a->dtype != sd) return LVX_EDTYPE;
  if (!same_hr(a, like) || a->d != like->d) return LVX_EINVAL;
  return LVX_OK;
}

int lvx_bwd_dq_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                       const lvx_view* L, const lvx_view* D, const lvx_view* dO, double scale,
                       void* ws, size_t ws_bytes, void* stream) {
  int s = check_bwd_inputs(q, k, v, L, D, dO);
  if (s) return s;
  if (ws_bytes < lvx_bwd_workspace(q, k)) return LVX_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q->heads * q->rows == 0) return LVX_OK;
  // the tensor-core choice depends on (q, k) only, so _finish makes the same one
  if (tc_bwd_eligible(q, k, v)) {
    if (!tc_bwd_outputs_ok(dO, nullptr, nullptr)) return LVX_EINVAL;  // dO must align like q
    return tc_bwd_dq_partial(q, k, v, L, D, dO, scale, ws, ws_bytes, st);
  }
  lvx_view w = simt_dq_view(q, ws);
  if (k->rows == 0) return fill_empty_zero(&w, st);
  return simt_bwd(q, k, v, L, D, dO, scale, &w, nullptr, nullptr, 0, st);
}

int lvx_bwd_dq_finish(const lvx_view* q, const lvx_view* k, const lvx_view* dq, int accumulate,
                      void* ws, size_t ws_bytes, void* stream) {
  if (!valid_view(q) || !valid_view(k) || !dtype_ok(q->dtype)) return LVX_EINVAL;
  int s = check_acc(dq, q, state_dtype(q->dtype));
  if (s) return s;
  if (ws_bytes < lvx_bwd_workspace(q, k)) return LVX_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q->heads * q->rows == 0) return LVX_OK;
  if (tc_bwd_eligible(q, k, k))
    return tc_bwd_dq_finish(q, k, dq, accumulate, ws, ws_bytes, st);
  lvx_view w = simt_dq_view(q, ws);
  return accumulate_into(&w, dq, accumulate, st);
}

int lvx_bwd_dkv(const lvx_view* q, const lvx_view* k, const lvx_view* v, const lvx_view* L,
                const lvx_view* D, const lvx_view* dO, double scale, const lvx_view* dk,
                const lvx_view* dv, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  int s = check_bwd_inputs(q, k, v, L, D, dO);
  if (s) return s;
  // dK / dV in the state dtype (any mode) or, overwriting, in the bf16 input
  // dtype straight from the tensor-core epilogue
  const bool in_dtype = q->dtype == LVX_BF16 && dk && dv && dk->dtype == LVX_BF16 &&
                        dv->dtype == LVX_BF16;
  const int sd = in_dtype ? LVX_BF16 : state_dtype(q->dtype);
  if ((s = check_acc(dk, k, sd)) || (s = check_acc(dv, k, sd))) return s;
  if (in_dtype && accumulate) return LVX_EDTYPE;
  if (ws_bytes < lvx_bwd_workspace(q, k)) return LVX_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k->heads * k->rows == 0) return LVX_OK;
  if (in_dtype && !use_tc_bwd(q, k, v, dO, dk, dv)) return LVX_EUNSUPPORTED;
  if (use_tc_bwd(q, k, v, dO, dk, dv))
    return tc_bwd_dkv(q, k, v, L, D, dO, scale, dk, dv, accumulate, ws, ws_bytes, st);
  if (q->heads * q->rows == 0) {
    if (accumulate) return LVX_OK;
    if ((s = fill_empty_zero(dk, st))) return s;
    return fill_empty_zero(dv, st);
  }
  return simt_bwd(q, k, v, L, D, dO, scale, nullptr, dk, dv, accumulate, st);
}

int lvx_blockwise_bwd(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                      const lvx_view* L, const lvx_view* D, const lvx_view* dO, double scale,
                      const lvx_view* dq, const lvx_view* dk, const lvx_view* dv,
                      int accumulate, void* ws, size_t ws_bytes, void* stream) {
  int s = lvx_bwd_dkv(q, k, v, L, D, dO, scale, dk, dv, accumulate, ws, ws_bytes, stream);
  if (s) return s;
  if ((s = lvx_bwd_dq_partial(q, k, v, L, D, dO, scale, ws, ws_bytes, stream))) return s;
  return lvx_bwd_dq_finish(q, k, dq, accumulate, ws, ws_bytes, stream);
}

int lvx_fill_empty_state(const lvx_view* o, const lvx_view* l, void* stream) {
  if (!valid_view(o) || !valid_view(l) || !same_hr(o, l)) return LVX_EINVAL;
  if (o->dtype != l->dtype) return LVX_EDTYPE;
  return fill_empty(o, l, static_cast<cudaStream_t>(stream));
}

int lvx_accumulate(const lvx_view* src, const lvx_view* dst, void* stream) {
  if (!valid_view(src) || !valid_view(dst) || !same_hr(src, dst) || src->d != dst->d)
    return LVX_EINVAL;
  if (src->dtype != dst->dtype || src->dtype == LVX_BF16) return LVX_EDTYPE;
  return accumulate_into(src, dst, 1, static_cast<cudaStream_t>(stream));
}

int lvx_convert(const lvx_view* src, const lvx_view* dst, void* stream) {
  if (!valid_view(src) || !valid_view(dst) || !same_hr(src, dst) || src->d != dst->d)
    return LVX_EINVAL;
  if (!dtype_ok(src->dtype) || !dtype_ok(dst->dtype)) return LVX_EDTYPE;
  return convert(src, dst, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
