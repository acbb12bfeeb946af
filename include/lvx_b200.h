/*
 * lvx_b200.h — C ABI of the B200-native LV-XAttn hot path.
 *
 * One shared library (paper_2502_02406_b200/liblvx_b200.so) exports the
 * kernels that replace the numpy kernels of the reference package
 * `lvxattn` (reference: /root/reference/pkg/src/lvxattn/kernels.py).  The
 * ring-exchange scheduler that calls them (lvx_forward / lvx_backward /
 * ring_forward / ring_backward / run_distributed) lives in the Python host
 * layer `paper_2502_02406_b200.strategies`, one process per GPU; the ring
 * hops run on the copy engines through the lvx_peer_* transport below.
 *
 * Conventions:
 *   - Tensors are strided [heads, rows, d] views with the last dim
 *     contiguous; strides are in ELEMENTS.  Rank shards are views
 *     (Q[:, qa:qb]) so a view never needs a copy.
 *   - L is the natural-log log-sum-exp of the *scaled* scores; an empty row
 *     is (O = 0, L = -inf), the identity of lvx_merge_states.
 *   - GQA: q head a reads k/v head a / (q->heads / k->heads).  MHA (the
 *     reference's only layout) is heads equal.
 *   - Input dtypes: F32, F64 (exact-parity SIMT kernels) and BF16
 *     (tcgen05/TMEM tensor-core kernels for d in {64,128}; SIMT otherwise).
 *     Softmax state (O partial, L, D) and gradient accumulators are F32 for
 *     F32/BF16 inputs and F64 for F64 inputs.
 *   - Every call is asynchronous on the caller's cudaStream_t, never
 *     synchronises the host, allocates nothing (scratch comes from the
 *     caller's workspace; the transport's arena from lvx_peer_create) and
 *     keeps no global mutable state beyond the launch counter.
 *   - Return value: LVX_OK (0) or a negative lvx_status.  The Python shim
 *     maps LVX_EINVAL/LVX_EDTYPE to ValueError with the reference messages
 *     (kernels.py:62-73) and LVX_ECUDA to RuntimeError.
 */
#ifndef LVX_B200_H
#define LVX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LVX_ABI_VERSION 1

typedef enum lvx_status {
  LVX_OK = 0,
  LVX_EINVAL = -1,      /* shape / stride / argument error            */
  LVX_EDTYPE = -2,      /* unsupported or mismatched dtype             */
  LVX_ECUDA = -3,       /* CUDA launch / runtime error                 */
  LVX_EUNSUPPORTED = -4,/* valid request, no kernel for it (e.g. d>256) */
  LVX_EWORKSPACE = -5   /* caller workspace smaller than required      */
} lvx_status;

typedef enum lvx_dtype {
  LVX_F32 = 0,
  LVX_F64 = 1,
  LVX_BF16 = 2
} lvx_dtype;

/* A strided [heads, rows, d] view.  For row statistics (L, D) d == 1 and
 * row_stride == 1.  Strides in elements. */
typedef struct lvx_view {
  void* data;
  int64_t heads;
  int64_t rows;
  int64_t d;
  int64_t head_stride;
  int64_t row_stride;
  int32_t dtype; /* lvx_dtype */
  int32_t _pad;
} lvx_view;

/* ---- introspection ---------------------------------------------------- */
int lvx_abi_version(void);
const char* lvx_strerror(int status);
/* Number of kernels this library has launched in this process (a
 * diagnostic counter; the only process-wide state, updated atomically). */
unsigned long long lvx_kernel_launches(void);
/* 1 when the tcgen05 path would serve (q, k) on the current device. */
int lvx_tc_eligible(const lvx_view* q, const lvx_view* k);

/* ---- K1: blockwise forward -------------------------------------------
 * Replaces kernels.py:105 blockwise_attention(Q, K, V, scale, tile_rows).
 * (o_out, l_out) <- partial state of q against this KV block; if `prior_o`
 * and `prior_l` are non-NULL the result is merged with that state
 * (fused kernels.py:144 merge_states(prior, delta), as lvx_forward does at
 * strategies.py:213).  prior may alias out.  `workspace` must hold
 * lvx_blockwise_fwd_workspace(q, k) bytes.  k->rows == 0 yields the
 * empty state (kernels.py:119-120) merged with prior.
 * tile_rows is semantically a no-op (tests/test_kernels.py:99-103) and is
 * not part of the ABI. */
size_t lvx_blockwise_fwd_workspace(const lvx_view* q, const lvx_view* k);
int lvx_blockwise_fwd(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                      double scale,
                      const lvx_view* prior_o, const lvx_view* prior_l,
                      const lvx_view* o_out, const lvx_view* l_out,
                      void* workspace, size_t workspace_bytes, void* stream);
/* The same operation in two launches so a ring scheduler can start the
 * attention before the prior state has arrived over NVLink: _partial runs
 * the tensor-core main loop into `workspace` (per-split partial states),
 * _finish combines the splits and merges the prior (strategies.py:207-213
 * blockwise_attention + merge_states).  Same (q, k) shapes and workspace in
 * both calls. */
int lvx_fwd_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v, double scale,
                    void* workspace, size_t workspace_bytes, void* stream);
int lvx_fwd_finish(const lvx_view* q, const lvx_view* k,
                   const lvx_view* prior_o, const lvx_view* prior_l,
                   const lvx_view* o_out, const lvx_view* l_out,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ---- K2: LSE merge ------------------------------------------------------
 * Replaces kernels.py:144 merge_states(a, b).  out may alias a or b. */
int lvx_merge_states(const lvx_view* oa, const lvx_view* la,
                     const lvx_view* ob, const lvx_view* lb,
                     const lvx_view* o_out, const lvx_view* l_out, void* stream);

/* ---- K3: backward row statistic ----------------------------------------
 * Replaces kernels.py:164 attention_row_stats(state, dO): D = rowsum(dO*O). */
int lvx_row_stats(const lvx_view* o, const lvx_view* d_o, const lvx_view* d_out,
                  void* stream);

/* ---- K4: blockwise backward ---------------------------------------------
 * Replaces kernels.py:192 blockwise_attention_backward(Q, K, V, L, D, dO).
 * Adds (accumulate=1) or writes (accumulate=0) the contributions into the
 * F32/F64 accumulators dq_acc [hq, rows_q, d], dk_acc / dv_acc
 * [hkv, rows_kv, d] (GQA: dK/dV summed over the query-head group). */
size_t lvx_blockwise_bwd_workspace(const lvx_view* q, const lvx_view* k);
int lvx_blockwise_bwd(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                      const lvx_view* l, const lvx_view* dd, const lvx_view* d_o,
                      double scale,
                      const lvx_view* dq_acc, const lvx_view* dk_acc,
                      const lvx_view* dv_acc, int accumulate,
                      void* workspace, size_t workspace_bytes, void* stream);

/* The backward in its two independent halves, so the ring scheduler can
 * compute dQ per round (it travels with the query block, strategies.py:
 * 258-268) and dK/dV once over every query block that passed through
 * (strategies.py:261-262 sums them over the rounds).
 *   _dq_partial: dQ contribution of this (Q block, KV block) into `workspace`
 *   _dq_finish:  dq_acc (+)= that contribution (after the travelling dQ has
 *                arrived; same q/k shapes and workspace)
 *   _dkv:        dk_acc / dv_acc (+)= contributions of every row of q.
 * lvx_bwd_workspace(q, k) bytes serve any of the three for these shapes. */
size_t lvx_bwd_workspace(const lvx_view* q, const lvx_view* k);
int lvx_bwd_dq_partial(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                       const lvx_view* l, const lvx_view* dd, const lvx_view* d_o,
                       double scale, void* workspace, size_t workspace_bytes, void* stream);
int lvx_bwd_dq_finish(const lvx_view* q, const lvx_view* k, const lvx_view* dq_acc,
                      int accumulate, void* workspace, size_t workspace_bytes, void* stream);
/* lvx_bwd_dkv: dk_acc / dv_acc in the state dtype (accumulate 0 or 1), or -- for
 * BF16 inputs with accumulate == 0 -- in BF16, written straight from the
 * tensor-core epilogue (the reference's output-dtype convention); BF16 outputs
 * on shapes the tensor-core kernel does not take return LVX_EUNSUPPORTED. */
int lvx_bwd_dkv(const lvx_view* q, const lvx_view* k, const lvx_view* v,
                const lvx_view* l, const lvx_view* dd, const lvx_view* d_o, double scale,
                const lvx_view* dk_acc, const lvx_view* dv_acc, int accumulate,
                void* workspace, size_t workspace_bytes, void* stream);

/* ---- utilities ---------------------------------------------------------
 * empty_state (kernels.py:48-53): O = 0, L = -inf. */
int lvx_fill_empty_state(const lvx_view* o, const lvx_view* l, void* stream);
/* dst += src for F32/F64 state tensors of one shape (the Ring baseline adds
 * a round's dK/dV contribution to the partial that arrived over the ring,
 * strategies.py:330-350). */
int lvx_accumulate(const lvx_view* src, const lvx_view* dst, void* stream);
/* dst = src converted (F32/F64/BF16 <-> F32/F64/BF16), strided views. */
int lvx_convert(const lvx_view* src, const lvx_view* dst, void* stream);

/* ---- projections (SURVEY.md §8(b) lvx_kv_recompute / lvx_project_bwd) --
 * GEMMs on the library's own tcgen05 kernel (bf16 in, fp32 accumulate, bf16
 * out; row strides multiple of 8 elements, 16-byte aligned bases) or its
 * exact SIMT kernel (f32 / f64, and bf16 views TMA cannot describe).
 * Row-major matrices; strides in elements; all operands one dtype.  Tall-K
 * products with few output tiles split K across the SMs and reduce in fp32
 * scratch from the stream-ordered allocator (cudaMallocAsync on `stream`);
 * the first such call raises the release threshold of the device's default
 * memory pool so that scratch is not unmapped at every synchronisation. */
typedef struct lvx_matrix {
  void* data;
  int64_t rows, cols, row_stride;
  int32_t dtype, _pad;
} lvx_matrix;

/* General GEMM of the layer's projections: c (+)= op(a) op(b), row-major
 * matrices, op = transpose when ta / tb.  bf16 runs on the tcgen05 kernel
 * (fp32 accumulate), f32 / f64 on an exact SIMT kernel.  With bf16 a / b, c
 * may be F32: the result is stored or (accumulate) reduce-added in fp32 in
 * the epilogue — the CA layers' shared visual-token gradient
 * (mllm.py:368 d_y +=) accumulates this way.  Used for the output
 * projection W_O of the cross-attention block (mllm.py:297-301 forward,
 * :343-351 backward); the three calls below are special cases of it. */
int lvx_gemm(const lvx_matrix* a, int ta, const lvx_matrix* b, int tb, const lvx_matrix* c,
             int accumulate, void* stream);
/* project (kernels.py:227-235): out[h] = x [S, e] @ w[:, h*d:(h+1)*d] for every
 * head of the [heads, S, d] view out.  out->head_stride == d (heads are column
 * blocks of one [S, heads*d] matrix) is one GEMM; any other head stride one
 * strided-batched GEMM. */
int lvx_project(const lvx_matrix* x, const lvx_matrix* w, const lvx_view* out, void* stream);
/* project_backward (kernels.py:238-254): dx = dout_flat w^T, dw = x^T dout_flat
 * for dout a [heads, S, d] view (the flat [S, heads*d] matrix is never copied). */
int lvx_project_bwd(const lvx_matrix* x, const lvx_matrix* w, const lvx_view* dout,
                    const lvx_matrix* dx, const lvx_matrix* dw, void* stream);
/* The MLLM K/V recompute from the shared visual tokens (mllm.py:296-300,
 * :358-360): k = project(y, w_k), v = project(y, w_v).  When w_v follows w_k in
 * one [e, 2*hkv*d] weight and v_out follows k_out in one [S, 2*hkv*d] output
 * (head_stride == d) it is ONE GEMM y @ [W_K | W_V]. */
int lvx_kv_recompute(const lvx_matrix* y, const lvx_matrix* w_k, const lvx_matrix* w_v,
                     const lvx_view* k_out, const lvx_view* v_out, void* stream);

/* ---- ring transport (copy engines over NVLink, no SMs) -----------------
 * Replaces the reference's in-process mailboxes: Cluster.send / recv
 * (cluster.py:173-220) and WorkerContext.send / recv / ring_shift
 * (cluster.py:227-272).  Each rank owns an "arena" (device memory allocated
 * and zeroed by _create) laid out identically on every rank; a message is
 * copied by the sender's copy engine into the same offset of the receiver's
 * arena, followed by a 32-bit flag write the receiver's stream waits on.
 * All calls are asynchronous on the given stream and never block the host.
 *   _create / _destroy   per-rank arena of `bytes` + peer map (rank in
 *                        [0, n), n <= LVX_MAX_PEERS); _base is its address
 *   _export / _open      CUDA IPC mapping of a peer process's arena
 *                        (handle of lvx_peer_handle_bytes() bytes)
 *   _attach              a peer arena in the same process (thread ranks)
 *   _put                 2-D copy (height rows of width bytes) from local
 *                        memory into peer's arena at dst_off
 *   _signal              peer's u32 at flag_off <- value, after prior work
 *                        on the stream (fenced)
 *   _wait                stream waits until (int32)(own u32 at flag_off -
 *                        value) >= 0
 */
#define LVX_MAX_PEERS 16
typedef struct lvx_peer_map lvx_peer_map;
int lvx_peer_create(uint64_t bytes, int rank, int n, lvx_peer_map** out);
int lvx_peer_destroy(lvx_peer_map* m);
void* lvx_peer_base(const lvx_peer_map* m);
uint64_t lvx_peer_handle_bytes(void);
int lvx_peer_export(const lvx_peer_map* m, void* handle);
int lvx_peer_open(lvx_peer_map* m, int peer, const void* handle);
int lvx_peer_attach(lvx_peer_map* m, int peer, const lvx_peer_map* other);
int lvx_peer_put(const lvx_peer_map* m, int peer, uint64_t dst_off, uint64_t dst_pitch,
                 const void* src, uint64_t src_pitch, uint64_t width, uint64_t height,
                 void* stream);
int lvx_peer_signal(const lvx_peer_map* m, int peer, uint64_t flag_off, uint32_t value,
                    void* stream);
int lvx_peer_wait(const lvx_peer_map* m, uint64_t flag_off, uint32_t value, void* stream);
/* A dedicated non-blocking CUDA stream (a rank's compute / copy stream; thread
 * ranks sharing one GPU must not share streams). */
int lvx_stream_create(void** out);
int lvx_stream_destroy(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LVX_B200_H */
