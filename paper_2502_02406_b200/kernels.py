"""Attention kernels of the LV-XAttn path on B200 — drop-in for
``lvxattn.kernels`` (reference ``pkg/src/lvxattn/kernels.py``).

Same names, argument meaning, layout ``[heads, rows, d]`` and error
messages as the reference.  Arrays may be numpy (copied to the current CUDA
device and back — the reference-facing host-buffer path) or torch tensors
(CUDA tensors stay on the device).  Every computation runs in the CUDA
library ``liblvx_b200.so``; there is no CPU fallback: without a CUDA device
the calls raise.

Precision: float32/float64 inputs go to exact SIMT kernels that compute in
float64 like the reference (kernels.py:3-8).  bfloat16 inputs with d in
{64, 128} go to the tcgen05/TMEM tensor-core kernels; their softmax state
(O partial, L, D) and gradient accumulators are float32.

GQA extension: K/V may have fewer heads than Q (hq a multiple of hkv); query
head a reads key/value head a // (hq // hkv).  The reference is MHA-only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

DEFAULT_TILE_ROWS = 64


# ---------------------------------------------------------------------------
# tensor plumbing
# ---------------------------------------------------------------------------

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2502_02406_b200 kernels need a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x):
    """Returns (tensor on the CUDA device, how to give results back)."""
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)).to(_device()), "numpy"
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return x, "cuda"
        return x.to(_device()), "cpu"
    raise TypeError(f"expected numpy array or torch tensor, got {type(x).__name__}")


def _back(t: torch.Tensor, kind: str):
    if kind == "numpy":
        return t.cpu().numpy()
    if kind == "cpu":
        return t.cpu()
    return t


def state_dtype(dt: torch.dtype) -> torch.dtype:
    return torch.float64 if dt == torch.float64 else torch.float32


_WS: dict = {}


def workspace(nbytes: int, device: torch.device | None = None, slot: int = 0) -> torch.Tensor:
    """Per (device, stream, slot) scratch buffer, grown on demand."""
    device = device or _device()
    key = (device.index, torch.cuda.current_stream(device).cuda_stream, slot)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


# ---------------------------------------------------------------------------
# types — kernels.py:20-55
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class AttentionState:
    """Partial attention output O [h, rows, d] plus row logsumexp L [h, rows]."""

    O: object
    L: object

    def __post_init__(self):
        if len(self.O.shape) != 3 or len(self.L.shape) != 2:
            raise ValueError(f"state shapes must be [h,rows,d] and [h,rows], "
                             f"got {tuple(self.O.shape)} and {tuple(self.L.shape)}")
        if tuple(self.O.shape[:2]) != tuple(self.L.shape):
            raise ValueError(f"O {tuple(self.O.shape)} and L {tuple(self.L.shape)} "
                             f"disagree on heads/rows")

    @property
    def heads(self) -> int:
        return self.O.shape[0]

    @property
    def rows(self) -> int:
        return self.O.shape[1]


@dataclass(frozen=True)
class GradientBundle:
    dQ: object
    dK: object
    dV: object


def empty_state(heads: int, rows: int, d: int, dtype=torch.float32, device=None) -> AttentionState:
    """The merge identity O = 0, L = -inf (kernels.py:48-53), on the device."""
    if isinstance(dtype, np.dtype) or dtype in (np.float32, np.float64):
        dtype = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    device = device or _device()
    O = torch.empty((heads, rows, d), dtype=dtype, device=device)
    L = torch.empty((heads, rows), dtype=dtype, device=device)
    if O.numel() or L.numel():
        _lib.check("lvx_fill_empty_state",
                   _lib.load().lvx_fill_empty_state(_lib.view(O), _lib.view(L),
                                                    _lib.stream_ptr(device)))
    return AttentionState(O=O, L=L)


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)


def validate_qkv(Q, K, V) -> None:
    """kernels.py:62-73 with the reference's messages; GQA allowed."""
    for name, t in (("Q", Q), ("K", K), ("V", V)):
        if len(t.shape) != 3:
            raise ValueError(f"{name} must be [heads, rows, d], got shape {tuple(t.shape)}")
    if not (K.shape[0] == V.shape[0]) or K.shape[0] == 0 or Q.shape[0] % K.shape[0]:
        raise ValueError(f"head counts differ: Q {Q.shape[0]}, K {K.shape[0]}, V {V.shape[0]}")
    if K.shape[1] != V.shape[1]:
        raise ValueError(f"K rows {K.shape[1]} != V rows {V.shape[1]}")
    if Q.shape[2] != K.shape[2]:
        raise ValueError(f"Q cols {Q.shape[2]} != K cols {K.shape[2]}")
    if V.shape[2] != Q.shape[2]:
        raise ValueError(f"V cols {V.shape[2]} != Q cols {Q.shape[2]}")


def _common_dtype(*ts) -> torch.dtype:
    dts = {t.dtype for t in ts}
    if len(dts) == 1:
        return dts.pop()
    return torch.promote_types(*sorted(dts, key=str)[:2]) if len(dts) == 2 else torch.float64


def _prep_qkv(Q, K, V):
    validate_qkv(Q, K, V)
    (q, kind), (k, _), (v, _) = _to_dev(Q), _to_dev(K), _to_dev(V)
    dt = _common_dtype(q, k, v)
    q, k, v = (t if t.dtype == dt else t.to(dt) for t in (q, k, v))
    q, k, v = (_lastdim_contig(t) for t in (q, k, v))
    return q, k, v, kind


def _lastdim_contig(t: torch.Tensor) -> torch.Tensor:
    return t if t.shape[-1] <= 1 or t.stride(-1) == 1 else t.contiguous()


# ---------------------------------------------------------------------------
# K1 forward — kernels.py:105-141 (and the fused merge of strategies.py:213)
# ---------------------------------------------------------------------------

def fwd_workspace_bytes(q: torch.Tensor, k: torch.Tensor) -> int:
    return int(_lib.load().lvx_blockwise_fwd_workspace(_lib.view(q), _lib.view(k)))


def fwd_partial(q, k, v, scale: float, ws: torch.Tensor) -> None:
    """Launch the attention main loop of q against this KV block into ``ws``."""
    _lib.check("lvx_fwd_partial", _lib.load().lvx_fwd_partial(
        _lib.view(q), _lib.view(k), _lib.view(v), float(scale), ws.data_ptr(), ws.numel(),
        _lib.stream_ptr(q.device)))


def fwd_finish(q, k, ws: torch.Tensor, out_o, out_l, prior_o=None, prior_l=None) -> None:
    """Combine the splits in ``ws`` and merge with (prior_o, prior_l) into out."""
    _lib.check("lvx_fwd_finish", _lib.load().lvx_fwd_finish(
        _lib.view(q), _lib.view(k), _lib.view(prior_o), _lib.view(prior_l),
        _lib.view(out_o), _lib.view(out_l), ws.data_ptr(), ws.numel(),
        _lib.stream_ptr(q.device)))


def blockwise_attention(Q, K, V, scale: float | None = None,
                        tile_rows: int = DEFAULT_TILE_ROWS) -> AttentionState:
    """Partial state (O, L) of Q against one KV block (kernels.py:105-141).
    ``tile_rows`` is validated like the reference but is semantically a
    no-op (tests/test_kernels.py:99-103); the kernels pick their own tiles."""
    if tile_rows < 1:
        raise ValueError(f"tile_rows must be >= 1, got {tile_rows}")
    q, k, v, kind = _prep_qkv(Q, K, V)
    scale = default_scale(q.shape[2]) if scale is None else scale
    sd = state_dtype(q.dtype)
    O = torch.empty(q.shape, dtype=sd, device=q.device)
    L = torch.empty(q.shape[:2], dtype=sd, device=q.device)
    if q.numel():
        ws = workspace(fwd_workspace_bytes(q, k), q.device)
        fwd_partial(q, k, v, scale, ws)
        fwd_finish(q, k, ws, O, L)
    out_dt = q.dtype if q.dtype != torch.bfloat16 else torch.float32
    return AttentionState(O=_back(O.to(out_dt), kind), L=_back(L.to(out_dt), kind))


def dense_attention(Q, K, V, scale: float | None = None) -> AttentionState:
    """The n=1 attention (kernels.py:80-102).  On the GPU the dense oracle and
    the blockwise kernel are the same computation; the materialised-S oracle
    stays on the CPU in ``oracle/``."""
    return blockwise_attention(Q, K, V, scale)


# ---------------------------------------------------------------------------
# K2 merge — kernels.py:144-161
# ---------------------------------------------------------------------------

def merge_into(a_o, a_l, b_o, b_l, out_o, out_l) -> None:
    _lib.check("lvx_merge_states", _lib.load().lvx_merge_states(
        _lib.view(a_o), _lib.view(a_l), _lib.view(b_o), _lib.view(b_l), _lib.view(out_o),
        _lib.view(out_l), _lib.stream_ptr(a_o.device)))


def merge_states(a: AttentionState, b: AttentionState) -> AttentionState:
    """L = logaddexp(La, Lb); O = e^(La-L) Oa + e^(Lb-L) Ob; empty rows stay empty."""
    if tuple(a.O.shape) != tuple(b.O.shape):
        raise ValueError(f"state shape mismatch: {tuple(a.O.shape)} vs {tuple(b.O.shape)}")
    (ao, kind), (al, _), (bo, _), (bl, _) = (_to_dev(t) for t in (a.O, a.L, b.O, b.L))
    dt = _common_dtype(ao, bo)
    ao, al, bo, bl = (t.to(dt) for t in (ao, al, bo, bl))
    O = torch.empty_like(ao)
    L = torch.empty_like(al)
    if O.numel():
        merge_into(ao, al, bo, bl, O, L)
    return AttentionState(O=_back(O, kind), L=_back(L, kind))


# ---------------------------------------------------------------------------
# K3 row statistic — kernels.py:164-169
# ---------------------------------------------------------------------------

def row_stats_into(o, d_o, out) -> None:
    _lib.check("lvx_row_stats", _lib.load().lvx_row_stats(
        _lib.view(o), _lib.view(d_o), _lib.view(out), _lib.stream_ptr(o.device)))


def attention_row_stats(state: AttentionState, dO):
    """D = rowsum(dO * O)."""
    if tuple(dO.shape) != tuple(state.O.shape):
        raise ValueError(f"dO shape {tuple(dO.shape)} != O shape {tuple(state.O.shape)}")
    (o, kind), (g, _) = _to_dev(state.O), _to_dev(dO)
    sd = state_dtype(g.dtype)
    o = o.to(sd)
    D = torch.empty(o.shape[:2], dtype=sd, device=o.device)
    if D.numel():
        row_stats_into(o, _lastdim_contig(g), D)
    return _back(D, kind)


# ---------------------------------------------------------------------------
# K4 backward — kernels.py:192-224
# ---------------------------------------------------------------------------

def bwd_workspace_bytes(q, k) -> int:
    return int(_lib.load().lvx_blockwise_bwd_workspace(_lib.view(q), _lib.view(k)))


def bwd_accumulate(q, k, v, L, D, d_o, scale: float, dq, dk, dv, accumulate: bool = True):
    """dq/dk/dv (state dtype) += contributions of this (Q block, KV block)."""
    ws = workspace(bwd_workspace_bytes(q, k), q.device, slot=1)
    _lib.check("lvx_blockwise_bwd", _lib.load().lvx_blockwise_bwd(
        _lib.view(q), _lib.view(k), _lib.view(v), _lib.view(L), _lib.view(D), _lib.view(d_o),
        float(scale), _lib.view(dq), _lib.view(dk), _lib.view(dv), int(bool(accumulate)),
        ws.data_ptr(), ws.numel(), _lib.stream_ptr(q.device)))


def bwd_dq_partial(q, k, v, L, D, d_o, scale: float, ws: torch.Tensor) -> None:
    """dQ contribution of (q block, this KV block) into ``ws``."""
    _lib.check("lvx_bwd_dq_partial", _lib.load().lvx_bwd_dq_partial(
        _lib.view(q), _lib.view(k), _lib.view(v), _lib.view(L), _lib.view(D), _lib.view(d_o),
        float(scale), ws.data_ptr(), ws.numel(), _lib.stream_ptr(q.device)))


def bwd_dq_finish(q, k, ws: torch.Tensor, dq, accumulate: bool = True) -> None:
    """dq (+)= the contribution held in ``ws``."""
    _lib.check("lvx_bwd_dq_finish", _lib.load().lvx_bwd_dq_finish(
        _lib.view(q), _lib.view(k), _lib.view(dq), int(bool(accumulate)), ws.data_ptr(),
        ws.numel(), _lib.stream_ptr(q.device)))


def bwd_dkv(q, k, v, L, D, d_o, scale: float, dk, dv, accumulate: bool = True,
            ws: torch.Tensor | None = None) -> None:
    """dk/dv (+)= contributions of every query row in q."""
    if ws is None:
        ws = workspace(bwd_ws_bytes(q, k), q.device, slot=2)
    st = _lib.load().lvx_bwd_dkv(
        _lib.view(q), _lib.view(k), _lib.view(v), _lib.view(L), _lib.view(D), _lib.view(d_o),
        float(scale), _lib.view(dk), _lib.view(dv), int(bool(accumulate)), ws.data_ptr(),
        ws.numel(), _lib.stream_ptr(q.device))
    sd = state_dtype(q.dtype)
    if st == -4 and dk.dtype != sd and not accumulate:
        # bf16 outputs on a shape the tensor-core kernel does not take: the
        # exact SIMT kernels write the state dtype, converted on the device
        tk, tv = torch.empty(dk.shape, dtype=sd, device=dk.device), \
            torch.empty(dv.shape, dtype=sd, device=dv.device)
        bwd_dkv(q, k, v, L, D, d_o, scale, tk, tv, False, ws)
        dk.copy_(tk)
        dv.copy_(tv)
        return
    _lib.check("lvx_bwd_dkv", st)


def bwd_ws_bytes(q, k) -> int:
    return int(_lib.load().lvx_bwd_workspace(_lib.view(q), _lib.view(k)))


def blockwise_attention_backward(Q_block, K_block, V_block, L_full, D_full, dO_block,
                                 scale: float | None = None):
    """Additive (dQ+, dK+, dV+) of one (Q block, KV block) pair given the final
    forward statistics; summing over KV blocks gives the dense backward."""
    validate_qkv(Q_block, K_block, V_block)
    if tuple(dO_block.shape) != tuple(Q_block.shape):
        raise ValueError(f"dO shape {tuple(dO_block.shape)} != Q shape {tuple(Q_block.shape)}")
    if tuple(L_full.shape) != tuple(Q_block.shape[:2]) or \
            tuple(D_full.shape) != tuple(Q_block.shape[:2]):
        raise ValueError(f"L/D shapes {tuple(L_full.shape)}/{tuple(D_full.shape)} != "
                         f"{tuple(Q_block.shape[:2])}")
    q, k, v, kind = _prep_qkv(Q_block, K_block, V_block)
    scale = default_scale(q.shape[2]) if scale is None else scale
    sd = state_dtype(q.dtype)
    L, D = (_to_dev(t)[0].to(sd) for t in (L_full, D_full))
    g = _lastdim_contig(_to_dev(dO_block)[0].to(q.dtype))
    dq = torch.zeros(q.shape, dtype=sd, device=q.device)
    dk = torch.zeros(k.shape, dtype=sd, device=q.device)
    dv = torch.zeros(v.shape, dtype=sd, device=q.device)
    if q.numel() and k.numel():
        bwd_accumulate(q, k, v, L, D, g, scale, dq, dk, dv, accumulate=False)
    out_dt = q.dtype
    return tuple(_back(t.to(out_dt), kind) for t in (dq, dk, dv))


def dense_attention_backward(Q, K, V, O, L, dO, scale: float | None = None) -> GradientBundle:
    """Full backward from saved (O, L) (kernels.py:172-189)."""
    validate_qkv(Q, K, V)
    if tuple(O.shape) != tuple(Q.shape) or tuple(dO.shape) != tuple(Q.shape):
        raise ValueError(f"O/dO must match Q shape {tuple(Q.shape)}, got "
                         f"{tuple(O.shape)}/{tuple(dO.shape)}")
    if tuple(L.shape) != tuple(Q.shape[:2]):
        raise ValueError(f"L shape {tuple(L.shape)} != {tuple(Q.shape[:2])}")
    D = attention_row_stats(AttentionState(O=O, L=L), dO)
    dq, dk, dv = blockwise_attention_backward(Q, K, V, L, D, dO, scale)
    return GradientBundle(dQ=dq, dK=dk, dV=dv)


# ---------------------------------------------------------------------------
# projections — kernels.py:227-254 (the library's tcgen05 GEMM, lvx_gemm_sm100.cu)
# ---------------------------------------------------------------------------

def project(x, W, heads: int):
    """x [S, e] @ W [e, h*d] -> [h, S, d]; head k owns cols [kd, (k+1)d)."""
    if len(x.shape) != 2 or len(W.shape) != 2:
        raise ValueError(f"expected 2-D input and weight, got {tuple(x.shape)} and "
                         f"{tuple(W.shape)}")
    if x.shape[1] != W.shape[0]:
        raise ValueError(f"inner dims disagree: input {x.shape[1]} vs weight {W.shape[0]}")
    if W.shape[1] % heads != 0:
        raise ValueError(f"weight cols {W.shape[1]} not divisible by heads {heads}")
    (xt, kind), (wt, _) = _to_dev(x), _to_dev(W)
    dt = _common_dtype(xt, wt)
    xt, wt = _rows_contig(xt.to(dt)), _rows_contig(wt.to(dt))
    out = torch.empty((heads, xt.shape[0], wt.shape[1] // heads), dtype=dt, device=xt.device)
    project_into(xt, wt, out)
    return _back(out, kind)


def _rows_contig(t: torch.Tensor) -> torch.Tensor:
    return t if (t.dim() != 2 or t.numel() == 0 or t.shape[1] <= 1 or t.stride(1) == 1) \
        else t.contiguous()


def project_into(x: torch.Tensor, W: torch.Tensor, out: torch.Tensor) -> None:
    """out[h] = x @ W[:, h*d:(h+1)*d] for a [heads, S, d] device view (lvx_project;
    one GEMM when the heads are column blocks of one [S, heads*d] matrix)."""
    _lib.check("lvx_project", _lib.load().lvx_project(
        _lib.matrix(x), _lib.matrix(W), _lib.view(out), _lib.stream_ptr(x.device)))


def kv_recompute(y: torch.Tensor, w_k: torch.Tensor, w_v: torch.Tensor, k_out: torch.Tensor,
                 v_out: torch.Tensor) -> None:
    """K, V of the MLLM recompute from the shared visual tokens (mllm.py:296-300,
    :358-360) into [hkv, S, d] device views (lvx_kv_recompute)."""
    _lib.check("lvx_kv_recompute", _lib.load().lvx_kv_recompute(
        _lib.matrix(y), _lib.matrix(w_k), _lib.matrix(w_v), _lib.view(k_out), _lib.view(v_out),
        _lib.stream_ptr(y.device)))


def project_backward_into(x: torch.Tensor, W: torch.Tensor, d_out: torch.Tensor,
                          dx: torch.Tensor, dw: torch.Tensor) -> None:
    """dx = dOut_flat W^T, dw = x^T dOut_flat for a [heads, S, d] device view
    d_out (lvx_project_bwd, no flattening copy)."""
    _lib.check("lvx_project_bwd", _lib.load().lvx_project_bwd(
        _lib.matrix(x), _lib.matrix(W), _lib.view(d_out), _lib.matrix(dx), _lib.matrix(dw),
        _lib.stream_ptr(x.device)))


def gemm_into(a: torch.Tensor, ta: bool, b: torch.Tensor, tb: bool, c: torch.Tensor,
              accumulate: bool = False) -> None:
    """c (+)= op(a) op(b) for row-major device matrices (lvx_gemm)."""
    L = _lib.load()
    _lib.check("lvx_gemm", L.lvx_gemm(_lib.matrix(a), int(ta), _lib.matrix(b), int(tb),
                                      _lib.matrix(c), int(accumulate), _lib.stream_ptr(c.device)))


def project_backward(x, W, dOut):
    """(dInput = dOut_flat W^T, dW = x^T dOut_flat)."""
    heads = dOut.shape[0]
    if len(dOut.shape) != 3 or dOut.shape[1] != x.shape[0] or \
            heads * dOut.shape[2] != W.shape[1]:
        raise ValueError(f"dOut shape {tuple(dOut.shape)} inconsistent with input "
                         f"{tuple(x.shape)} and weight {tuple(W.shape)}")
    (xt, kind), (wt, _), (gt, _) = _to_dev(x), _to_dev(W), _to_dev(dOut)
    dt = _common_dtype(xt, wt)
    xt, wt, gt = _rows_contig(xt.to(dt)), _rows_contig(wt.to(dt)), gt.to(dt)
    if gt.numel() and gt.shape[2] > 1 and gt.stride(2) != 1:
        gt = gt.contiguous()
    dx = torch.empty(xt.shape, dtype=dt, device=xt.device)
    dw = torch.empty(wt.shape, dtype=dt, device=xt.device)
    project_backward_into(xt, wt, gt, dx, dw)
    return _back(dx, kind), _back(dw, kind)
