"""The kernel set the ring schedulers call: the CUDA library, nothing else.

``CudaOps`` is the only implementation shipped with the product.  The
schedulers in ``strategies.py`` take it from ``DeviceContext.ops`` so the
protocol logic (rounds, block indices, buffers, byte counts) is written once;
the CPU protocol tests substitute the oracle there (tests/ only).
"""
from __future__ import annotations

import torch

from . import kernels as K


class CudaOps:
    """liblvx_b200.so kernels on the current CUDA stream."""

    name = "cuda"

    @staticmethod
    def state_dtype(dt: torch.dtype) -> torch.dtype:
        return K.state_dtype(dt)

    @staticmethod
    def grad_dtype(dt: torch.dtype) -> torch.dtype:
        """Gradients come back in the input dtype (the reference's convention);
        dK/dV are written in it directly by the tensor-core epilogue."""
        return dt

    def fwd_workspace(self, q: torch.Tensor, k: torch.Tensor) -> torch.Tensor:
        return K.workspace(K.fwd_workspace_bytes(q, k), q.device, slot=0)

    def fwd_partial(self, q, k, v, scale, ws) -> None:
        if q.numel() and k.shape[1]:
            K.fwd_partial(q, k, v, scale, ws)

    def fwd_finish(self, q, k, ws, out_o, out_l, prior_o=None, prior_l=None) -> None:
        if q.numel():
            K.fwd_finish(q, k, ws, out_o, out_l, prior_o, prior_l)

    def fill_empty(self, o, l) -> None:
        if o.numel():
            K._lib.check("lvx_fill_empty_state", K._lib.load().lvx_fill_empty_state(
                K._lib.view(o), K._lib.view(l), K._lib.stream_ptr(o.device)))

    def row_stats(self, o, d_o, out) -> None:
        if out.numel():
            K.row_stats_into(o, d_o, out)

    def bwd_accumulate(self, q, k, v, L, D, d_o, scale, dq, dk, dv) -> None:
        if q.numel() and k.shape[1]:
            K.bwd_accumulate(q, k, v, L, D, d_o, scale, dq, dk, dv, accumulate=True)

    # split backward used by the LV-XAttn ring (dQ travels, dK/dV once)
    def bwd_workspace(self, q, k, slot: int = 1) -> torch.Tensor:
        return K.workspace(K.bwd_ws_bytes(q, k), q.device, slot=slot)

    def bwd_dq_partial(self, q, k, v, L, D, d_o, scale, ws) -> None:
        if q.numel():
            K.bwd_dq_partial(q, k, v, L, D, d_o, scale, ws)

    def bwd_dq_finish(self, q, k, ws, dq, accumulate: bool) -> None:
        if q.numel():
            K.bwd_dq_finish(q, k, ws, dq, accumulate)

    def bwd_dkv(self, q, k, v, L, D, d_o, scale, dk, dv, accumulate: bool) -> None:
        if k.numel():
            K.bwd_dkv(q, k, v, L, D, d_o, scale, dk, dv, accumulate,
                      ws=self.bwd_workspace(q, k, slot=2))

    def accumulate(self, src, dst) -> None:
        """dst += src (state dtype; the Ring baseline's dK/dV partials)."""
        if dst.numel():
            K._lib.check("lvx_accumulate", K._lib.load().lvx_accumulate(
                K._lib.view(src), K._lib.view(dst), K._lib.stream_ptr(dst.device)))

    def gemm(self, a, ta, b, tb, out, accumulate=False) -> None:
        """out (+)= op(a) op(b) (lvx_gemm)."""
        if out.numel():
            K.gemm_into(a, ta, b, tb, out, accumulate)

    def kv_recompute(self, y, w_k, w_v, k_out, v_out) -> None:
        """k_out / v_out ([hkv, S, d] views) = project(y, W_K / W_V) (lvx_kv_recompute)."""
        if y.shape[0]:
            K.kv_recompute(y, w_k, w_v, k_out, v_out)
        else:
            k_out.zero_()
            v_out.zero_()

    def project_backward(self, x, W, d_out, dx, dw) -> None:
        """dx = dOut_flat W^T, dw = x^T dOut_flat for a [heads, S, d] view (lvx_project_bwd)."""
        K.project_backward_into(x, W, d_out, dx, dw)

    # -- device timing (CUDA events on the compute stream) -----------------
    @staticmethod
    def event():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    @staticmethod
    def elapsed(a, b) -> float:
        return a.elapsed_time(b) / 1e3
