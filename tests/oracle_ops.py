"""Kernel set backed by the CPU oracle — TESTS ONLY.

Lets the CPU test-suite drive the product's ring schedulers
(paper_2502_02406_b200.strategies) over a gloo process group with the
oracle doing the arithmetic, so the protocol logic (rounds, block indices,
buffers, byte counts) is checked without a GPU.  The product never imports
this module; its only kernel set is ops.CudaOps.
"""
import time

import numpy as np
import torch

from oracle import lvx_oracle as orc


def _np(t):
    return t.detach().cpu().numpy()


class OracleOps:
    name = "oracle"
    device = "cpu"

    @staticmethod
    def state_dtype(dt):
        return torch.float64 if dt == torch.float64 else torch.float32

    @staticmethod
    def grad_dtype(dt):
        return OracleOps.state_dtype(dt)

    def fwd_workspace(self, q, k):
        return {}

    def fwd_partial(self, q, k, v, scale, ws):
        if q.numel() and k.shape[1]:
            o, l = orc.blockwise_attention(_np(q), _np(k), _np(v), scale)
            ws["delta"] = (o, l)

    def fwd_finish(self, q, k, ws, out_o, out_l, prior_o=None, prior_l=None):
        if not q.numel():
            return
        sd = out_o.dtype
        if "delta" in ws:
            o, l = ws.pop("delta")
        else:
            h, r, d = q.shape
            o, l = np.zeros((h, r, d)), np.full((h, r), -np.inf)
        o = torch.from_numpy(np.asarray(o)).to(sd)
        l = torch.from_numpy(np.asarray(l)).to(sd)
        if prior_o is not None:
            mo, ml = orc.merge_states(_np(prior_o), _np(prior_l), _np(o), _np(l))
            o, l = torch.from_numpy(mo).to(sd), torch.from_numpy(ml).to(sd)
        out_o.copy_(o)
        out_l.copy_(l)

    def fill_empty(self, o, l):
        o.zero_()
        l.fill_(-np.inf)

    def row_stats(self, o, d_o, out):
        out.copy_(torch.from_numpy(orc.attention_row_stats(_np(o), _np(d_o))).to(out.dtype))

    def bwd_accumulate(self, q, k, v, L, D, d_o, scale, dq, dk, dv):
        if not (q.numel() and k.shape[1]):
            return
        gq, gk, gv = orc.blockwise_attention_backward(_np(q), _np(k), _np(v), _np(L), _np(D),
                                                      _np(d_o), scale)
        dq += torch.from_numpy(gq).to(dq.dtype)
        dk += torch.from_numpy(gk).to(dk.dtype)
        dv += torch.from_numpy(gv).to(dv.dtype)

    def bwd_workspace(self, q, k, slot=1):
        return {}

    def bwd_dq_partial(self, q, k, v, L, D, d_o, scale, ws):
        if q.numel() and k.shape[1]:
            gq, _, _ = orc.blockwise_attention_backward(_np(q), _np(k), _np(v), _np(L), _np(D),
                                                        _np(d_o), scale)
            ws["dq"] = gq
        else:
            ws["dq"] = np.zeros(tuple(q.shape))

    def bwd_dq_finish(self, q, k, ws, dq, accumulate):
        if not q.numel():
            return
        g = torch.from_numpy(np.asarray(ws.pop("dq"))).to(dq.dtype)
        if accumulate:
            dq += g
        else:
            dq.copy_(g)

    def bwd_dkv(self, q, k, v, L, D, d_o, scale, dk, dv, accumulate):
        if not k.numel():
            return
        if q.numel():
            _, gk, gv = orc.blockwise_attention_backward(_np(q), _np(k), _np(v), _np(L),
                                                         _np(D), _np(d_o), scale)
        else:
            gk, gv = np.zeros(tuple(k.shape)), np.zeros(tuple(v.shape))
        gk = torch.from_numpy(gk).to(dk.dtype)
        gv = torch.from_numpy(gv).to(dv.dtype)
        if accumulate:
            dk += gk
            dv += gv
        else:
            dk.copy_(gk)
            dv.copy_(gv)

    def accumulate(self, src, dst):
        dst += src

    def gemm(self, a, ta, b, tb, out, accumulate=False):
        r = (a.T if ta else a).double() @ (b.T if tb else b).double()
        if accumulate:
            r = r + out.double()
        out.copy_(r.to(out.dtype))

    def kv_recompute(self, y, w_k, w_v, k_out, v_out):
        h = k_out.shape[0]
        for w, out in ((w_k, k_out), (w_v, v_out)):
            out.copy_(torch.from_numpy(orc.project(_np(y), _np(w), h)).to(out.dtype))

    def project_backward(self, x, W, d_out, dx, dw):
        gx, gw = orc.project_backward(_np(x), _np(W), _np(d_out))
        dx.copy_(torch.from_numpy(np.asarray(gx)).to(dx.dtype))
        dw.copy_(torch.from_numpy(np.asarray(gw)).to(dw.dtype))

    @staticmethod
    def event():
        return time.perf_counter()

    @staticmethod
    def elapsed(a, b):
        return b - a
