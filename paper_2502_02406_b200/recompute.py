"""Cross-attention layer with the MLLM-specific K/V activation recompute
(§3.2; reference ``src/mllm.py:290-301`` forward CA block and
``:343-370`` backward CA branch), distributed over the LV-XAttn ring.

Each rank keeps its shard of the text tokens ``x_i`` (rows of the query
block) and of the visual tokens ``y_i`` (rows of the KV block) resident;
the weights are replicated.  Every projection is row-local, so:

  forward   q_i = x_i W_Q;  [k_i | v_i] = y_i [W_K | W_V]  (one GEMM);
            (O_i, L_i) = lvx_forward(...);  out_i = x_i + flat(O_i) W_O.
            RECOMPUTE_KV saves only (x_i, O_i, L_i) — K/V are dropped
            (``src/mllm.py:296-300``); STORE_KV also keeps k_i, v_i.
  backward  d_o = g W_O^T; q_i re-projected from x_i (both policies,
            ``:352``); k_i, v_i re-projected from the shared y_i under
            RECOMPUTE (``:358-360``); lvx_backward; d_x = g + dQ W_Q^T;
            d_y_i = dK W_K^T + dV W_V^T (``:365-368``); weight gradients are
            partial sums over the rank's rows and are all-reduced (the
            reference is single-worker, so this collective is new).

Every projection GEMM runs on the library's own tcgen05 GEMM behind the C ABI
(``lvx_kv_recompute``, ``lvx_project_bwd``, and ``lvx_gemm`` for W_Q / W_O;
heads folded into the GEMM strides, no copies); why the K/V recompute is not
fused into the attention kernels is measured in DESIGN.md §4.  Across layers
that share y, ``VisualGradSink`` turns the per-layer ``d_y +=`` into one GEMM.
``OpCounter`` counts forward-direction projection FLOP
done inside the backward, like ``src/mllm.py:242-253``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import torch
import torch.distributed as dist

from .comm import DeviceContext
from .kernels import AttentionState, default_scale
from .strategies import (ShardSpec, lvx_backward, lvx_forward, ring_backward, ring_forward)


class ActivationPolicy(str, Enum):
    STORE_KV = "store"
    RECOMPUTE_KV = "recompute"


@dataclass
class CrossAttentionWeights:
    """W_Q [e, hq*d], W_K / W_V [e, hkv*d], W_O [hq*d, e] (head k owns
    columns [k*d, (k+1)*d), ``src/kernels.py:228-229``)."""

    w_q: torch.Tensor
    w_k: torch.Tensor
    w_v: torch.Tensor
    w_o: torch.Tensor
    hq: int
    hkv: int

    @property
    def d(self) -> int:
        return self.w_q.shape[1] // self.hq

    def kv_weight(self) -> torch.Tensor:
        """[W_K | W_V] as one [e, 2*hkv*d] matrix (one GEMM for K and V),
        built once and rebuilt only when either weight changes (in place or
        by reassignment)."""
        key = (self.w_k.data_ptr(), self.w_k._version, self.w_v.data_ptr(), self.w_v._version)
        cached = getattr(self, "_wkv", None)
        if cached is None or cached[0] != key:
            cached = (key, torch.cat([self.w_k, self.w_v], dim=1))
            object.__setattr__(self, "_wkv", cached)
        return cached[1]


@dataclass
class CrossAttentionGrads:
    d_x: torch.Tensor
    d_y: torch.Tensor
    w_q: torch.Tensor
    w_k: torch.Tensor
    w_v: torch.Tensor
    w_o: torch.Tensor


@dataclass
class OpCounter:
    """Forward-direction projection FLOP performed inside the backward."""

    projection_flops: int = 0

    def add(self, rows: int, d_in: int, d_out: int) -> None:
        self.projection_flops += 2 * rows * d_in * d_out


@dataclass
class SavedCA:
    policy: ActivationPolicy
    x: torch.Tensor
    state: AttentionState
    kv: tuple | None = None
    extras: dict = field(default_factory=dict)


class VisualGradSink:
    """The visual tokens' gradient over the CA layers that share y
    (``src/mllm.py:368``: ``d_y += dK-part + dV-part`` per layer) as ONE GEMM.

    Each layer's backward writes its [dK | dV] into its own column block of
    one [S, sum(widths)] buffer (``slot``) instead of multiplying it out; at
    the end ``finish`` computes dY = [dKV_1 | dKV_2 | ...] [W_1 | W_2 | ...]^T,
    i.e. sum_l dKV_l W_l^T with the layer sum inside the GEMM's K loop (fp32
    in TMEM) and the [S, e] result written once.  Per-layer accumulation
    instead reads and writes the fp32 [S, e] accumulator once per layer
    (C4 at n = 1: 4.3 GB each way per layer).  ``widths`` are the layers'
    2 hkv d in the order their backward runs."""

    def __init__(self, y: torch.Tensor, widths):
        self.rows, self.e = y.shape
        self.widths = [int(w) for w in widths]
        self.offs = [0]
        for w in self.widths:
            self.offs.append(self.offs[-1] + w)
        self.dkv = torch.empty((self.rows, self.offs[-1]), dtype=y.dtype, device=y.device)
        self.acc_dtype = torch.float64 if y.dtype == torch.float64 else torch.float32
        self.weights: list = []

    def slot(self, wkv: torch.Tensor) -> torch.Tensor:
        """The next layer's [S, 2 hkv d] dKV block (a strided view); ``wkv``
        is that layer's [W_K | W_V]."""
        i = len(self.weights)
        if i >= len(self.widths):
            raise ValueError(f"sink holds {len(self.widths)} layers; a layer more was added")
        if wkv.shape != (self.e, self.widths[i]):
            raise ValueError(f"layer {i}: [W_K|W_V] is {tuple(wkv.shape)}, expected "
                             f"({self.e}, {self.widths[i]})")
        self.weights.append(wkv)
        return self.dkv[:, self.offs[i]:self.offs[i + 1]]

    def finish(self, ctx: DeviceContext, out: torch.Tensor | None = None,
               dtype: torch.dtype | None = None) -> torch.Tensor:
        """dY [S, e] = sum over the slots of dKV W^T, accumulated in fp32 (f64
        for f64 y) and written once in ``dtype`` (default: that accumulator
        dtype; y's bf16 rounds the fp32 sum once in the GEMM epilogue)."""
        if len(self.weights) != len(self.widths):
            raise ValueError(f"{len(self.weights)} of {len(self.widths)} layers added")
        if out is None:
            out = torch.empty((self.rows, self.e), dtype=dtype or self.acc_dtype,
                              device=self.dkv.device)
        w = torch.cat(self.weights, dim=1) if len(self.weights) > 1 else self.weights[0]
        ctx.ops.gemm(self.dkv, False, w, True, out)
        return out


def _heads(flat: torch.Tensor, heads: int) -> torch.Tensor:
    """[S, heads*d] -> [heads, S, d] as a zero-copy strided view
    (``src/kernels.py:236-240`` reshapes and copies): the tensor-core kernels
    take any 16-byte-multiple head/row strides through their TMA maps."""
    s = flat.shape[0]
    return flat.view(s, heads, -1).transpose(0, 1)


def _flat(t: torch.Tensor) -> torch.Tensor:
    """[heads, S, d] -> [S, heads*d] (``src/mllm.py:256-258``)."""
    h, s, d = t.shape
    return t.transpose(0, 1).reshape(s, h * d)


def _mm(ctx: DeviceContext, a: torch.Tensor, b: torch.Tensor, ta: bool = False,
        tb: bool = False, out: torch.Tensor | None = None, accumulate: bool = False):
    """op(a) op(b) (+ out) through the kernel set's GEMM (lvx_gemm)."""
    m = a.shape[1] if ta else a.shape[0]
    n = b.shape[0] if tb else b.shape[1]
    if out is None:
        out = torch.empty((m, n), dtype=a.dtype, device=a.device)
    ctx.ops.gemm(a, ta, b, tb, out, accumulate)
    return out


def _out_proj(ctx: DeviceContext, x_i: torch.Tensor, st: AttentionState,
              w: CrossAttentionWeights) -> torch.Tensor:
    """x_i + flat(O_i) W_O (``src/mllm.py:297-301``): the residual is the GEMM's
    accumulator."""
    out = x_i.clone()
    return _mm(ctx, _flat(st.O.to(x_i.dtype)), w.w_o, out=out, accumulate=True)


def project_kv(ctx: DeviceContext, y: torch.Tensor, w: CrossAttentionWeights):
    """K/V from the visual tokens with ONE GEMM y [S, e] @ [W_K | W_V]
    (``lvx_kv_recompute``); K and V are zero-copy head views of its output."""
    hkd = w.hkv * w.d
    wkv = w.kv_weight()
    kv = torch.empty((y.shape[0], 2 * hkd), dtype=y.dtype, device=y.device)
    k, v = _heads(kv[:, :hkd], w.hkv), _heads(kv[:, hkd:], w.hkv)
    ctx.ops.kv_recompute(y, wkv[:, :hkd], wkv[:, hkd:], k, v)
    return k, v


# RECOMPUTE_KV at n = 1 projects, attends and merges K/V in chunks of this many
# visual rows, so the layer never holds more than one chunk's K/V (the
# reference materialises the whole layer's K/V, mllm.py:294-295, :358-360).
KV_CHUNK_ROWS = 1 << 17


def _row_chunks(rows: int, chunk: int):
    return [(a, min(a + chunk, rows)) for a in range(0, rows, chunk)]


def _chunked(ctx: DeviceContext, policy: ActivationPolicy, strategy: str, y_rows: int,
             kv_chunk_rows: int | None) -> bool:
    return (kv_chunk_rows is not None and ctx.n == 1 and strategy == "lvx" and
            policy is ActivationPolicy.RECOMPUTE_KV and y_rows > kv_chunk_rows)


def _attend_chunked(ctx: DeviceContext, q, y, w: CrossAttentionWeights, scale: float,
                    chunk: int) -> AttentionState:
    """n = 1 forward over K/V chunks: partial + fused LSE merge per chunk."""
    ops = ctx.ops
    sd = ops.state_dtype(q.dtype)
    O = torch.empty(q.shape, dtype=sd, device=q.device)
    L = torch.empty(q.shape[:2], dtype=sd, device=q.device)
    ops.fill_empty(O, L)
    for a, b in _row_chunks(y.shape[0], chunk):
        k, v = project_kv(ctx, y[a:b], w)
        ws = ops.fwd_workspace(q, k)
        ops.fwd_partial(q, k, v, scale, ws)
        ops.fwd_finish(q, k, ws, O, L, O, L)
        del k, v      # the allocator hands the chunk buffer to the next chunk
    return AttentionState(O=O, L=L)


def ca_forward(ctx: DeviceContext, shards: ShardSpec, x_i: torch.Tensor, y_i: torch.Tensor,
               w: CrossAttentionWeights, policy: ActivationPolicy = ActivationPolicy.RECOMPUTE_KV,
               scale: float | None = None, strategy: str = "lvx",
               kv_chunk_rows: int | None = KV_CHUNK_ROWS):
    """Returns (out_i = x_i + flat(O_i) W_O, saved)."""
    policy = ActivationPolicy(policy)
    scale = default_scale(w.d) if scale is None else scale
    q = _heads(_mm(ctx, x_i, w.w_q), w.hq)
    if _chunked(ctx, policy, strategy, y_i.shape[0], kv_chunk_rows):
        st = _attend_chunked(ctx, q, y_i, w, scale, kv_chunk_rows)
        saved = SavedCA(policy=policy, x=x_i, state=st, kv=None)
        saved.extras["kv_chunk_rows"] = kv_chunk_rows
        return _out_proj(ctx, x_i, st, w), saved
    k, v = project_kv(ctx, y_i, w)
    fwd = lvx_forward if strategy == "lvx" else ring_forward
    st = fwd(ctx, shards, q, k, v, scale)
    saved = SavedCA(policy=policy, x=x_i, state=st,
                    kv=(k, v) if policy is ActivationPolicy.STORE_KV else None)
    del q, k, v   # under RECOMPUTE nothing but y_i remains for the visual side
    return _out_proj(ctx, x_i, st, w), saved


def ca_backward(ctx: DeviceContext, shards: ShardSpec, g_i: torch.Tensor, saved: SavedCA,
                y_i: torch.Tensor, w: CrossAttentionWeights, scale: float | None = None,
                strategy: str = "lvx", counter: OpCounter | None = None,
                group=None, d_y_acc: torch.Tensor | None = None,
                dy_sink: VisualGradSink | None = None) -> CrossAttentionGrads:
    """Backward of ``ca_forward`` (``src/mllm.py:343-370``).  Weight gradients
    are all-reduced over the process group when n > 1.

    ``d_y_acc``: an fp32 [S_kv, e] accumulator of the visual tokens' gradient
    over the CA layers that share y (``src/mllm.py:368`` ``d_y +=``).  Given,
    this layer's dY = [dK|dV] [W_K|W_V]^T is reduce-added into it inside the
    GEMM's epilogue (no bf16 dY, no separate add pass) and returned as
    ``d_y``; else a fresh dY in y's dtype is returned.

    ``dy_sink``: the layer's [dK | dV] goes into the sink's next slot and the
    dY GEMM is left to ``VisualGradSink.finish`` (one GEMM over all layers);
    ``d_y`` is then None."""
    if dy_sink is not None and d_y_acc is not None:
        raise ValueError("give d_y_acc or dy_sink, not both")
    scale = default_scale(w.d) if scale is None else scale
    dt = g_i.dtype
    # n > 1: the weight gradients are partial sums over the rank's rows; they
    # come out of their GEMMs in the fp32 (f64) state dtype, packed in one
    # buffer, are summed over the ranks in ONE all-reduce at that precision
    # and rounded to the weights' dtype once
    wbuf = None
    if ctx.n > 1:
        shapes = (tuple(w.w_q.shape), (w.w_k.shape[0], w.w_k.shape[1] + w.w_v.shape[1]),
                  tuple(w.w_o.shape))
        sizes = [a * b for a, b in shapes]
        flat = torch.empty(sum(sizes), dtype=ctx.ops.state_dtype(dt), device=g_i.device)
        wbuf = [t.view(sh) for t, sh in zip(torch.split(flat, sizes), shapes)]
    d_o = _heads(_mm(ctx, g_i, w.w_o, tb=True), w.hq)                  # g W_O^T
    g_wo = _mm(ctx, _flat(saved.state.O.to(dt)), g_i, ta=True,         # flat(O)^T g
               out=wbuf[2] if wbuf else None)
    q = _heads(_mm(ctx, saved.x, w.w_q), w.hq)
    if counter is not None:
        counter.add(saved.x.shape[0], w.w_q.shape[0], w.w_q.shape[1])
    hkd = w.hkv * w.d
    wkv = w.kv_weight()
    chunk = saved.extras.get("kv_chunk_rows")
    if chunk:   # n = 1 RECOMPUTE in K/V chunks (see _attend_chunked)
        if counter is not None:
            counter.add(y_i.shape[0], w.w_k.shape[0], w.w_k.shape[1])
            counter.add(y_i.shape[0], w.w_v.shape[0], w.w_v.shape[1])
        dq, d_y, g_wkv = _backward_chunked(ctx, q, y_i, w, wkv, saved.state,
                                           d_o.to(q.dtype), scale, chunk, d_y_acc,
                                           dy_sink.slot(wkv) if dy_sink is not None else None)
        dq = _flat(dq.to(dt))
    else:
        if saved.policy is ActivationPolicy.STORE_KV:
            k, v = saved.kv
        else:   # the MLLM-specific recompute from the one shared y
            k, v = project_kv(ctx, y_i, w)
            if counter is not None:
                counter.add(y_i.shape[0], w.w_k.shape[0], w.w_k.shape[1])
                counter.add(y_i.shape[0], w.w_v.shape[0], w.w_v.shape[1])
        if strategy == "lvx":   # dK / dV written straight into the [S, 2 hkv d] GEMM operand
            dkv = dy_sink.slot(wkv) if dy_sink is not None else \
                torch.empty((y_i.shape[0], 2 * hkd), dtype=dt, device=y_i.device)
            dq, _, _ = lvx_backward(ctx, shards, q, k, v, saved.state, d_o.to(q.dtype), scale,
                                    dk_out=_heads(dkv[:, :hkd], w.hkv),
                                    dv_out=_heads(dkv[:, hkd:], w.hkv))
            dq = _flat(dq.to(dt))
        else:
            dq, dk, dv = ring_backward(ctx, shards, q, k, v, saved.state, d_o.to(q.dtype), scale)
            dq, dk, dv = _flat(dq.to(dt)), _flat(dk.to(dt)), _flat(dv.to(dt))
            if dy_sink is not None:
                dkv = dy_sink.slot(wkv)
                dkv[:, :hkd], dkv[:, hkd:] = dk, dv
            else:
                dkv = torch.cat([dk, dv], dim=1)
        del k, v
        g_wkv = wbuf[1] if wbuf else torch.empty_like(wkv)
        if dy_sink is not None:   # dY comes from the sink's one GEMM over all layers
            ctx.ops.gemm(y_i, True, dkv, False, g_wkv)                      # y^T dKV
            d_y = None
        elif d_y_acc is not None:
            ctx.ops.gemm(dkv, False, wkv, True, d_y_acc, accumulate=True)   # += dKV W^T
            ctx.ops.gemm(y_i, True, dkv, False, g_wkv)                      # y^T dKV
            d_y = d_y_acc
        elif wbuf:
            d_y = torch.empty_like(y_i)
            ctx.ops.gemm(dkv, False, wkv, True, d_y)                        # dKV W^T
            ctx.ops.gemm(y_i, True, dkv, False, g_wkv)                      # y^T dKV
        else:
            d_y = torch.empty_like(y_i)
            ctx.ops.project_backward(y_i, wkv, _heads(dkv, 2 * w.hkv), d_y, g_wkv)
    d_x = torch.empty_like(g_i)
    if wbuf:
        g_wq = wbuf[0]
        ctx.ops.gemm(dq, False, w.w_q, True, d_x)                           # d_x = dq W_Q^T
        ctx.ops.gemm(saved.x, True, dq, False, g_wq)                        # x^T dq
    else:
        g_wq = torch.empty_like(w.w_q)
        ctx.ops.project_backward(saved.x, w.w_q, _heads(dq, w.hq), d_x, g_wq)   # d_x = dq W_Q^T
    d_x += g_i
    if wbuf:   # one all-reduce of the layer's weight gradients, packed, at fp32
        if group is not None:
            dist.all_reduce(flat, group=group)
        else:
            ctx.all_reduce_sum_(flat)
        wd = w.w_q.dtype
        g_wq, g_wkv, g_wo = (t.to(wd) for t in wbuf)
    g_wk, g_wv = g_wkv[:, :hkd].contiguous(), g_wkv[:, hkd:].contiguous()
    return CrossAttentionGrads(d_x=d_x, d_y=d_y, w_q=g_wq, w_k=g_wk, w_v=g_wv, w_o=g_wo)


def _backward_chunked(ctx: DeviceContext, q, y, w: CrossAttentionWeights, wkv, state,
                      d_o, scale: float, chunk: int, d_y_acc=None, dkv_slot=None):
    """n = 1 backward over K/V chunks: per chunk re-project K/V, add its dQ
    contribution (fp32, in place), compute its dK/dV and fold them into the
    chunk's d_y rows (or reduce-add them into ``d_y_acc``; or, given a sink
    slot ``dkv_slot``, leave them there for the sink's GEMM) and into the fp32
    K/V weight gradient (the GEMM accumulates across chunks in its epilogue).
    Returns (dQ, d_y or None, g_wkv)."""
    ops = ctx.ops
    sd = ops.state_dtype(q.dtype)
    D = torch.empty(state.L.shape, dtype=sd, device=q.device)
    ops.row_stats(state.O, d_o, D)
    dq = torch.empty(q.shape, dtype=sd, device=q.device)
    d_y = None if dkv_slot is not None else d_y_acc if d_y_acc is not None else \
        torch.empty_like(y)
    g_wkv = torch.empty(wkv.shape, dtype=ops.state_dtype(wkv.dtype), device=y.device)
    hkd = w.hkv * w.d
    for c, (a, b) in enumerate(_row_chunks(y.shape[0], chunk)):
        k, v = project_kv(ctx, y[a:b], w)
        ws = ops.bwd_workspace(q, k)
        ops.bwd_dq_partial(q, k, v, state.L, D, d_o, scale, ws)
        ops.bwd_dq_finish(q, k, ws, dq, accumulate=c > 0)
        dkv = dkv_slot[a:b] if dkv_slot is not None else \
            torch.empty((b - a, 2 * hkd), dtype=y.dtype, device=y.device)
        ops.bwd_dkv(q, k, v, state.L, D, d_o, scale, _heads(dkv[:, :hkd], w.hkv),
                    _heads(dkv[:, hkd:], w.hkv), accumulate=False)
        del k, v
        if d_y is not None:
            ops.gemm(dkv, False, wkv, True, d_y[a:b], accumulate=d_y_acc is not None)  # dKV W^T
        ops.gemm(y[a:b], True, dkv, False, g_wkv, accumulate=c > 0)                # y^T dKV
    return dq, d_y, g_wkv.to(wkv.dtype)


def activation_bytes(saved: SavedCA) -> int:
    """Bytes this layer keeps alive between forward and backward (the
    per-layer categories of ``src/mllm.py:190-209``): x, O, L (+ K, V)."""
    n = saved.x.numel() * saved.x.element_size()
    n += saved.state.O.numel() * saved.state.O.element_size()
    n += saved.state.L.numel() * saved.state.L.element_size()
    if saved.kv is not None:
        n += sum(t.numel() * t.element_size() for t in saved.kv)
    return n
