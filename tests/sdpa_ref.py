"""torch SDPA in bf16 as the yardstick of the bf16 gate — TESTS ONLY.

SURVEY.md §8(c): the bf16 results must be "no worse than 2x torch's bf16
SDPA error on the same inputs", both measured against the f64 oracle.  SDPA
(flash / cuDNN backend, fp32 accumulation, bf16 P and outputs) runs forward
and backward on the same bf16-rounded tensors; its max-normalised errors per
output at the same sampled rows are the reference error level."""
import numpy as np
import torch

from oracle import lvx_oracle as orc

GATE = 2.0          # ours <= GATE x SDPA's error ...
FLOOR = 5e-4        # ... or below this absolute floor (a few bf16 ulps at |x| ~ 1)
L_TOL = 1e-3        # L has no SDPA counterpart: f32 LSE of bf16 scores


def sdpa_grads(q, k, v, do, scale):
    """O, dQ, dK, dV of torch SDPA bf16 (flash backend).  GQA: K/V heads are
    expanded to the query heads and dK / dV summed back per group in fp32."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    grp = q.shape[0] // k.shape[0]
    qq, kk, vv = (t.detach().clone().unsqueeze(0).requires_grad_(True) for t in (q, k, v))
    with sdpa_kernel([SDPBackend.FLASH_ATTENTION, SDPBackend.CUDNN_ATTENTION,
                      SDPBackend.EFFICIENT_ATTENTION]):
        o = torch.nn.functional.scaled_dot_product_attention(
            qq, kk.repeat_interleave(grp, dim=1), vv.repeat_interleave(grp, dim=1), scale=scale)
        o.backward(do.unsqueeze(0))
    return o[0].detach(), qq.grad[0], kk.grad[0], vv.grad[0]


def gate(ours: dict, sdpa: dict) -> list:
    """Names whose error breaks the gate (empty list = pass)."""
    bad = []
    for k, e in ours.items():
        lim = L_TOL if k == "L" else max(GATE * sdpa[k], FLOOR)
        if not e <= lim:
            bad.append((k, e, lim))
    return bad


def errors(got: dict, want: dict) -> dict:
    return {k: orc.max_norm_error(np.asarray(got[k], dtype=np.float64), want[k]) for k in want
            if k in got}
