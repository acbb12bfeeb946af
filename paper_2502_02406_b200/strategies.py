"""Distributed cross-attention schedulers on B200 — drop-in for
``lvxattn.strategies`` (reference ``pkg/src/lvxattn/strategies.py``).

One process per GPU.  Each rank keeps its KV shard resident in HBM; the
schedulers move the rotating blocks with grouped NCCL send/recv (``comm``)
on NCCL's stream while the attention kernels run on the compute stream.

  lvx   query rotation (strategies.py:175-276, Algorithm 1): the
        (O, L, Q) blocks travel, the fused split-combine+merge kernel folds
        the received state into the new partial.
  ring  KV rotation baseline (strategies.py:279-361).

Round structure, block indices, epilogues, per-message metadata checks and
byte accounting follow the reference exactly, so byte counters equal the
closed forms of ``volumes`` (GQA-aware).  Deviations, all documented in
DESIGN.md: partial states (O, L, D, dQ, dK/dV accumulators) travel in
float32 when the inputs are bfloat16; the receive buffers are preallocated
and double-buffered instead of freshly allocated per message.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch
import torch.distributed as dist

from .comm import ClusterError, ClusterSpec, DeviceContext, TransportStats
from .kernels import (DEFAULT_TILE_ROWS, AttentionState, GradientBundle, default_scale,
                      state_dtype, validate_qkv)


class StrategyKind(str, Enum):
    LVX = "lvx"
    RING = "ring"
    HEAD_PARALLEL = "head"
    SINGLE = "single"


def partition_rows(total: int, n: int) -> list[tuple[int, int]]:
    """Balanced contiguous ranges; the first (total mod n) ranks get one extra
    row (strategies.py:47-61)."""
    if n < 1:
        raise ValueError(f"worker count must be >= 1, got {n}")
    if total < 0:
        raise ValueError(f"row count must be >= 0, got {total}")
    base, extra = divmod(total, n)
    out, lo = [], 0
    for i in range(n):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


@dataclass(frozen=True)
class ShardSpec:
    """Per-rank row ranges over [0, S_Q) and [0, S_KV) (strategies.py:64-99)."""

    q_ranges: tuple
    kv_ranges: tuple

    def __post_init__(self):
        if len(self.q_ranges) != len(self.kv_ranges):
            raise ValueError("q_ranges and kv_ranges must have one entry per worker")
        for name, ranges in (("q", self.q_ranges), ("kv", self.kv_ranges)):
            pos = 0
            for a, b in ranges:
                if a != pos or b < a:
                    raise ValueError(f"{name} ranges must be contiguous ascending, got {ranges}")
                pos = b
            sizes = [b - a for a, b in ranges]
            if sizes and max(sizes) - min(sizes) > 1:
                raise ValueError(f"{name} shard sizes differ by more than 1: {sizes}")

    @classmethod
    def balanced(cls, s_q: int, s_kv: int, n: int) -> "ShardSpec":
        return cls(q_ranges=tuple(partition_rows(s_q, n)),
                   kv_ranges=tuple(partition_rows(s_kv, n)))

    @property
    def n(self) -> int:
        return len(self.q_ranges)

    @property
    def q_sizes(self) -> list[int]:
        return [b - a for a, b in self.q_ranges]

    @property
    def kv_sizes(self) -> list[int]:
        return [b - a for a, b in self.kv_ranges]


@dataclass
class RoundRecord:
    index: int
    compute_seconds: float          # measured on the device (CUDA events)
    comm_seconds: float             # measured exposed wait for this round's hop
    sent_bytes_by_class: dict

    @property
    def sent_bytes(self) -> int:
        return sum(self.sent_bytes_by_class.values())


@dataclass
class RoundTrace:
    """Per-round record (strategies.py:102-159).  ``comm_seconds`` is the
    MEASURED time the compute stream waited on the hop (0 when fully
    overlapped), not a modeled time."""

    strategy: str
    phase: str
    rounds: list = field(default_factory=list)
    epilogue_bytes_by_class: dict = field(default_factory=dict)
    epilogue_comm_seconds: float = 0.0
    sections: dict = field(default_factory=dict)   # named device-timed phases (seconds)
    _pending: list = field(default_factory=list, repr=False)
    _pending_sec: list = field(default_factory=list, repr=False)

    def add_round(self, compute_seconds, comm_seconds, sent_bytes_by_class) -> None:
        self.rounds.append(RoundRecord(len(self.rounds), compute_seconds, comm_seconds,
                                       dict(sent_bytes_by_class)))

    def _add_timed(self, ops, t0, t1, t2, sent) -> None:
        self.add_round(0.0, 0.0, sent)
        self._pending.append((len(self.rounds) - 1, ops, t0, t1, t2))

    def section(self, name: str, ops, a, b) -> None:
        """Accumulate the device time between events a and b under ``name``."""
        self._pending_sec.append((name, ops, a, b))

    def resolve(self) -> None:
        """Convert device events into seconds (call after a synchronize)."""
        for name, ops, a, b in self._pending_sec:
            self.sections[name] = self.sections.get(name, 0.0) + ops.elapsed(a, b)
        self._pending_sec = []
        for idx, ops, t0, t1, t2 in self._pending:
            rec = self.rounds[idx]
            rec.compute_seconds = ops.elapsed(t0, t1)
            rec.comm_seconds = ops.elapsed(t1, t2) if t2 is not None else 0.0
        self._pending = []

    @property
    def num_rounds(self) -> int:
        return len(self.rounds)

    @property
    def num_shifts(self) -> int:
        return sum(1 for r in self.rounds if r.sent_bytes > 0)

    def total_sent_bytes(self) -> int:
        return sum(r.sent_bytes for r in self.rounds) + sum(self.epilogue_bytes_by_class.values())

    def compute_only_seconds(self) -> float:
        return sum(r.compute_seconds for r in self.rounds)

    def modeled_overlapped_seconds(self) -> float:
        return sum(max(r.compute_seconds, r.comm_seconds) for r in self.rounds)

    def as_dict(self) -> dict:
        return {"strategy": self.strategy, "phase": self.phase,
                "rounds": [{"index": r.index, "compute_seconds": r.compute_seconds,
                            "comm_seconds": r.comm_seconds, "sent_bytes": r.sent_bytes_by_class}
                           for r in self.rounds],
                "epilogue_sent_bytes": self.epilogue_bytes_by_class,
                "epilogue_comm_seconds": self.epilogue_comm_seconds}


def _expect(got, want, what: str) -> None:
    """Per-message block check (strategies.py:169-172), done on the host
    schedule: the block a rank holds each round is a pure function of
    (rank, round), so a mismatch is a protocol bug."""
    if got != want:
        raise ClusterError(f"{what}: expected block {want}, got {got}")


class _Flat:
    """Double-buffered contiguous storage for rotating blocks of varying rows."""

    def __init__(self, heads: int, max_rows: int, d: int | None, dtype, device, count: int = 2):
        # d=None: a row statistic [heads, rows] (L, D)
        self.h, self.d = heads, d
        self.bufs = [torch.empty(max(heads * max_rows * (d or 1), 1), dtype=dtype, device=device)
                     for _ in range(count)]

    def view(self, idx: int, rows: int) -> torch.Tensor:
        t = self.bufs[idx][:self.h * rows * (self.d or 1)]
        return t.view(self.h, rows) if self.d is None else t.view(self.h, rows, self.d)


def _dev_copy(t: torch.Tensor, buf: torch.Tensor) -> torch.Tensor:
    buf.copy_(t)
    return buf


# ---------------------------------------------------------------------------
# LV-XAttn query rotation
# ---------------------------------------------------------------------------

@dataclass
class KVStream:
    """K/V rows of the local block arriving / leaving in chunks (the host
    pipeline, ``host_pipeline.py``).  ``bounds`` are row ranges covering the
    block.  ``wait_chunk(c)`` makes the compute stream wait until chunk c is
    resident (forward round 0 consumes chunks as they land; later rounds and
    the backward find the whole block resident).  ``dkv_done(c, dk, dv)`` is
    called once chunk c's dK / dV are final (the batched dK/dV pass runs per
    chunk), so they can leave while the next chunk computes."""

    bounds: list
    wait_chunk: object = None
    dkv_done: object = None


def lvx_forward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                scale: float, tile_rows: int = DEFAULT_TILE_ROWS,
                trace: RoundTrace | None = None,
                kv_stream: KVStream | None = None) -> AttentionState:
    """Query-rotation forward for one rank; collective over all n
    (strategies.py:175-231).  Round r: ship the state finished last round
    (block i-r+1; round 0 ships the empty state) plus Q of block i-r to the
    successor, run block i-r's attention against the resident K/V, receive
    the predecessor's state and Q, merge.  After n rounds an epilogue hop
    sends each completed state home."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, _, d = q_block.shape
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    qs = shards.q_sizes
    mq = max(qs) if qs else 0
    O = _Flat(h, mq, d, sd, dev)
    Lb = _Flat(h, mq, None, sd, dev)
    Qb = _Flat(h, mq, d, q_block.dtype, dev)

    cur = 0
    send_block = (i + 1) % n
    o_s, l_s = O.view(cur, qs[send_block]), Lb.view(cur, qs[send_block])
    ops.fill_empty(o_s, l_s)
    q_cur = _dev_copy(q_block, Qb.view(cur, qs[i]))
    q_block_id = i
    for r in range(n):
        j, j_next = (i - r) % n, (i - r - 1) % n
        _expect(q_block_id, j, f"worker {i} round {r} query")
        _expect(send_block, (j + 1) % n, f"worker {i} round {r} state")
        o_r, l_r = O.view(1 - cur, qs[j]), Lb.view(1 - cur, qs[j])
        q_r = Qb.view(1 - cur, qs[j_next])
        if n == 1:  # loopback (cluster.py:178-180): the sent state comes straight back
            o_r, l_r, q_r = o_s, l_s, q_cur
        t0 = ops.event() if trace is not None else None
        hop, sent = ctx.shift([o_s, l_s, q_cur], [o_r, l_r, q_r], ["O", "L", "Q"])
        if r == 0 and kv_stream is not None and len(kv_stream.bounds) > 1:
            # K/V still streaming in: one partial + merge per resident chunk
            for c, (a, b) in enumerate(kv_stream.bounds):
                if kv_stream.wait_chunk is not None:
                    kv_stream.wait_chunk(c)
                kc, vc = k_block[:, a:b], v_block[:, a:b]
                ws = ops.fwd_workspace(q_cur, kc)
                ops.fwd_partial(q_cur, kc, vc, scale, ws)
                if c == 0:
                    t1 = ops.event() if trace is not None else None
                    hop.wait()
                    t2 = ops.event() if trace is not None else None
                ops.fwd_finish(q_cur, kc, ws, o_r, l_r, o_r, l_r)
        else:
            if kv_stream is not None and kv_stream.wait_chunk is not None:
                for c in range(len(kv_stream.bounds)):
                    kv_stream.wait_chunk(c)
            ws = ops.fwd_workspace(q_cur, k_block)
            ops.fwd_partial(q_cur, k_block, v_block, scale, ws)
            t1 = ops.event() if trace is not None else None
            hop.wait()
            t2 = ops.event() if trace is not None else None
            ops.fwd_finish(q_cur, k_block, ws, o_r, l_r, o_r, l_r)   # merge(recv, delta)
        if trace is not None:
            t3 = ops.event()
            trace._add_timed(ops, t0, t1, t2, sent)
            trace.section("fwd_kernel", ops, t0, t1)
            trace.section("fwd_finish", ops, t2, t3)
            trace.section("wait", ops, t1, t2)
        o_s, l_s, q_cur = o_r, l_r, q_r
        send_block, q_block_id, cur = j, j_next, 1 - cur

    # epilogue: the completed state of block i+1 goes home (strategies.py:220-231)
    out_o = torch.empty((h, qs[i], d), dtype=sd, device=dev)
    out_l = torch.empty((h, qs[i]), dtype=sd, device=dev)
    if n == 1:
        out_o.copy_(o_s)
        out_l.copy_(l_s)
        epi = {"O": 0, "L": 0}
    else:
        hop, epi = ctx.shift([o_s, l_s], [out_o, out_l], ["O", "L"])
        hop.wait()
    _expect(send_block, (i + 1) % n, f"worker {i} epilogue")
    if trace is not None:
        trace.epilogue_bytes_by_class = epi
    return AttentionState(O=out_o, L=out_l)


def lvx_backward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                 state: AttentionState, do_block, scale: float,
                 trace: RoundTrace | None = None, kv_stream: KVStream | None = None):
    """Query-rotation backward (strategies.py:234-276): the tuple
    (Q, dO, L, D, dQ) of every block travels once around the ring and every
    rank adds its K/V block's contribution; the last dQ hop is the
    homecoming.  Returns (dQ_i, dK_i, dV_i) in the input dtype (the
    reference's convention): everything is computed and carried in the fp32
    state dtype and the batched dK/dV pass writes bf16 gradients directly.

    B200 schedule (same messages and bytes per rank as the reference; see
    DESIGN.md §5):
      * the immutable part (Q, dO, L, D) of block j is sent at the START of
        round r, overlapping this round's dQ kernel, instead of after it;
      * dQ lags one hop: round r sends the dQ of block j+1 finished in round
        r-1, and the received dQ of block j is folded in by the dQ finish
        kernel after the local contribution is computed;
      * every block's (Q, dO, L, D) passes through every rank anyway, so dK_i
        and dV_i (the sum over rounds at strategies.py:261-262) are computed
        ONCE after the ring over all gathered query rows — one tensor-core
        pass with dK/dV in TMEM and a single write, instead of n passes with
        an fp32 read-modify-write each.
    """
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, _, d = q_block.shape
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    qs, qr = shards.q_sizes, shards.q_ranges
    mq = max(qs) if qs else 0
    Qb = _Flat(h, mq, d, q_block.dtype, dev)
    Gb = _Flat(h, mq, d, q_block.dtype, dev)
    Lb = _Flat(h, mq, None, sd, dev)
    Db = _Flat(h, mq, None, sd, dev)
    dQb = _Flat(h, mq, d, sd, dev)
    if n > 1:   # gather of every block's immutable rows for the batched dK/dV
        s_tot = sum(qs)
        Qg = torch.empty((h, s_tot, d), dtype=q_block.dtype, device=dev)
        Gg = torch.empty((h, s_tot, d), dtype=q_block.dtype, device=dev)
        Lg = torch.empty((h, s_tot), dtype=sd, device=dev)
        Dg = torch.empty((h, s_tot), dtype=sd, device=dev)

    cur = 0
    q_j = _dev_copy(q_block, Qb.view(cur, qs[i]))
    do_j = _dev_copy(do_block, Gb.view(cur, qs[i]))
    l_j = _dev_copy(state.L, Lb.view(cur, qs[i]))
    d_j = Db.view(cur, qs[i])
    ops.row_stats(state.O, do_block, d_j)             # strategies.py:247
    gd = _grad_dtype(ops, q_block.dtype)
    dk = torch.empty(k_block.shape, dtype=gd, device=dev)   # written once, in gd
    dv = torch.empty(v_block.shape, dtype=gd, device=dev)
    early_dkv = n == 1 and kv_stream is not None and kv_stream.dkv_done is not None
    if early_dkv:   # n = 1: the rows are all local, so dK/dV first and their chunks
        # leave the GPU while the dQ kernel runs
        t4 = ops.event() if trace is not None else None
        _dkv_chunks(ops, kv_stream, q_j, k_block, v_block, l_j, d_j, do_j, scale, dk, dv)
        if trace is not None:
            trace.section("dkv_kernel", ops, t4, ops.event())
    dq_prev = None
    blk = i
    for r in range(n):
        j, nxt = (i - r) % n, (i - r - 1) % n
        _expect(blk, j, f"worker {i} backward round {r}")
        send = [q_j, do_j, l_j, d_j]
        recv = [Qb.view(1 - cur, qs[nxt]), Gb.view(1 - cur, qs[nxt]),
                Lb.view(1 - cur, qs[nxt]), Db.view(1 - cur, qs[nxt])]
        classes = ["Q", "dO", "L", "D"]
        dq_in = None
        if r >= 1:   # dQ of block j+1 (finished last round) out, dQ of block j in
            dq_in = dQb.view(r % 2, qs[j])
            send.append(dq_prev)
            recv.append(dq_in)
            classes.append("dQ")
        if n == 1:
            recv = send
        t0 = ops.event() if trace is not None else None
        hop, sent = ctx.shift(send, recv, classes)
        ws = ops.bwd_workspace(q_j, k_block)
        ops.bwd_dq_partial(q_j, k_block, v_block, l_j, d_j, do_j, scale, ws)
        t1 = ops.event() if trace is not None else None
        if n > 1:
            a, b = qr[j]
            Qg[:, a:b].copy_(q_j)
            Gg[:, a:b].copy_(do_j)
            Lg[:, a:b].copy_(l_j)
            Dg[:, a:b].copy_(d_j)
        else:
            Qg, Gg, Lg, Dg = q_j, do_j, l_j, d_j
        hop.wait()
        t2 = ops.event() if trace is not None else None
        if dq_in is None:
            dq_acc = dQb.view(0, qs[j])
            ops.bwd_dq_finish(q_j, k_block, ws, dq_acc, accumulate=False)
        else:
            ops.bwd_dq_finish(q_j, k_block, ws, dq_in, accumulate=True)
            dq_acc = dq_in
        if trace is not None:
            t3 = ops.event()
            trace._add_timed(ops, t0, t1, t2, sent)
            trace.section("dq_kernel", ops, t0, t1)
            trace.section("gather+wait", ops, t1, t2)
            trace.section("dq_finish", ops, t2, t3)
        dq_prev = dq_acc
        if n > 1:
            q_j, do_j, l_j, d_j = recv[:4]
        blk, cur = nxt, 1 - cur
    _expect(blk, i, f"worker {i} backward homecoming")
    # the dQ of block i+1 goes home; this rank's own dQ_i arrives
    dq_out = torch.empty((h, qs[i], d), dtype=sd, device=dev)
    if n == 1:
        dq_out.copy_(dq_prev)
    else:
        hop, epi = ctx.shift([dq_prev], [dq_out], ["dQ"])
        hop.wait()
        if trace is not None:
            trace.epilogue_bytes_by_class = epi
    if not early_dkv:
        t4 = ops.event() if trace is not None else None
        if kv_stream is not None and kv_stream.dkv_done is not None:
            _dkv_chunks(ops, kv_stream, Qg, k_block, v_block, Lg, Dg, Gg, scale, dk, dv)
        else:
            ops.bwd_dkv(Qg, k_block, v_block, Lg, Dg, Gg, scale, dk, dv, accumulate=False)
        if trace is not None:
            trace.section("dkv_kernel", ops, t4, ops.event())
    return dq_out.to(gd), dk, dv


def _grad_dtype(ops, dt):
    return ops.grad_dtype(dt) if hasattr(ops, "grad_dtype") else ops.state_dtype(dt)


def _dkv_chunks(ops, kv_stream: KVStream, q, k_block, v_block, L, D, g, scale, dk, dv):
    """The batched dK/dV pass per KV chunk (each chunk's rows are independent)."""
    for c, (a, b) in enumerate(kv_stream.bounds):
        dkc, dvc = dk[:, a:b], dv[:, a:b]
        ops.bwd_dkv(q, k_block[:, a:b], v_block[:, a:b], L, D, g, scale, dkc, dvc,
                    accumulate=False)
        kv_stream.dkv_done(c, dkc, dvc)


# ---------------------------------------------------------------------------
# Ring Attention KV rotation (the baseline)
# ---------------------------------------------------------------------------

def ring_forward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                 scale: float, tile_rows: int = DEFAULT_TILE_ROWS,
                 trace: RoundTrace | None = None) -> AttentionState:
    """KV-rotation forward (strategies.py:279-311): Q/O/L stay resident and
    (K, V) shift n-1 times, each shift overlapping the attention on the block
    in hand."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, rows, d = q_block.shape
    hk = k_block.shape[0]
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    ks = shards.kv_sizes
    mk = max(ks) if ks else 0
    O = torch.empty((h, rows, d), dtype=sd, device=dev)
    L = torch.empty((h, rows), dtype=sd, device=dev)
    ops.fill_empty(O, L)
    if n > 1:
        Kb = _Flat(hk, mk, d, k_block.dtype, dev)
        Vb = _Flat(hk, mk, d, v_block.dtype, dev)
        k_cur = _dev_copy(k_block, Kb.view(0, ks[i]))
        v_cur = _dev_copy(v_block, Vb.view(0, ks[i]))
    else:
        k_cur, v_cur = k_block, v_block
    cur, blk = 0, i
    for r in range(n):
        hop, sent = None, {}
        nxt = (i - r - 1) % n
        if r < n - 1:
            hop, sent = ctx.shift([k_cur, v_cur], [Kb.view(1 - cur, ks[nxt]),
                                                   Vb.view(1 - cur, ks[nxt])], ["K", "V"])
        t0 = ops.event() if trace is not None else None
        ws = ops.fwd_workspace(q_block, k_cur)
        ops.fwd_partial(q_block, k_cur, v_cur, scale, ws)
        ops.fwd_finish(q_block, k_cur, ws, O, L, O, L)       # merge(state, delta)
        t1 = ops.event() if trace is not None else None
        if trace is not None:
            trace.section("fwd_kernel", ops, t0, t1)
        if hop is not None:
            hop.wait()
            k_cur, v_cur = Kb.view(1 - cur, ks[nxt]), Vb.view(1 - cur, ks[nxt])
            blk, cur = nxt, 1 - cur
        t2 = ops.event() if trace is not None else None
        if trace is not None:
            trace._add_timed(ops, t0, t1, t2, sent)
    return AttentionState(O=O, L=L)


def ring_backward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                  state: AttentionState, do_block, scale: float,
                  trace: RoundTrace | None = None):
    """KV-rotation backward (strategies.py:314-361): (K, V, dK, dV) rotate
    n-1 times while dQ accumulates locally; an epilogue hop returns each
    (dK, dV) pair to its owner."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, rows, d = q_block.shape
    hk = k_block.shape[0]
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    ks = shards.kv_sizes
    mk = max(ks) if ks else 0
    D = torch.empty((h, rows), dtype=sd, device=dev)
    ops.row_stats(state.O, do_block, D)
    L = state.L
    dq = torch.zeros((h, rows, d), dtype=sd, device=dev)
    Kb = _Flat(hk, mk, d, k_block.dtype, dev)
    Vb = _Flat(hk, mk, d, v_block.dtype, dev)
    dKb = _Flat(hk, mk, d, sd, dev)
    dVb = _Flat(hk, mk, d, sd, dev)
    cur = 0
    k_cur = _dev_copy(k_block, Kb.view(0, ks[i]))
    v_cur = _dev_copy(v_block, Vb.view(0, ks[i]))
    dk_cur, dv_cur = dKb.view(0, ks[i]), dVb.view(0, ks[i])
    dk_cur.zero_()
    dv_cur.zero_()
    blk = i
    for r in range(n):
        t0 = ops.event() if trace is not None else None
        ops.bwd_accumulate(q_block, k_cur, v_cur, L, D, do_block, scale, dq, dk_cur, dv_cur)
        t1 = ops.event() if trace is not None else None
        sent = {}
        if r < n - 1:
            nxt = (i - r - 1) % n
            recv = [Kb.view(1 - cur, ks[nxt]), Vb.view(1 - cur, ks[nxt]),
                    dKb.view(1 - cur, ks[nxt]), dVb.view(1 - cur, ks[nxt])]
            hop, sent = ctx.shift([k_cur, v_cur, dk_cur, dv_cur], recv, ["K", "V", "dK", "dV"])
            hop.wait()
            k_cur, v_cur, dk_cur, dv_cur = recv
            blk, cur = nxt, 1 - cur
        t2 = ops.event() if trace is not None else None
        if trace is not None:
            trace._add_timed(ops, t0, t1, t2, sent)
    # dk_cur / dv_cur now belong to block i+1: send them home
    dk = torch.empty((hk, ks[i], d), dtype=sd, device=dev)
    dv = torch.empty((hk, ks[i], d), dtype=sd, device=dev)
    if n == 1:
        dk.copy_(dk_cur)
        dv.copy_(dv_cur)
        epi = {"dK": 0, "dV": 0}
    else:
        hop, epi = ctx.shift([dk_cur, dv_cur], [dk, dv], ["dK", "dV"])
        hop.wait()
    _expect(blk, (i + 1) % n, f"worker {i} backward epilogue")
    if trace is not None:
        trace.epilogue_bytes_by_class = epi
    gd = _grad_dtype(ctx.ops, q_block.dtype)
    return dq.to(gd), dk.to(gd), dv.to(gd)


# ---------------------------------------------------------------------------
# Head parallelism (DeepSpeed-Ulysses style), the reference's third strategy
# ---------------------------------------------------------------------------

def _check_heads(h: int, hk: int, n: int) -> None:
    if h % n != 0:
        raise ValueError(f"head count {h} not divisible by workers {n}")
    if hk % n != 0:
        raise ValueError(f"kv head count {hk} not divisible by workers {n}")


def head_parallel_forward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                          scale: float, tile_rows: int = DEFAULT_TILE_ROWS,
                          trace: RoundTrace | None = None):
    """All-to-all from sequence sharding to head sharding, local attention on
    the owned heads over the full sequence, all-to-all back
    (strategies.py:364-400).  Requires hq and hkv divisible by n (GQA keeps
    whole groups together).  Returns (own state, saved for backward)."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, _, d = q_block.shape
    hk = k_block.shape[0]
    _check_heads(h, hk, n)
    hpw, kpw = h // n, hk // n
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    qs, ks = shards.q_sizes, shards.kv_sizes
    s_q, s_kv = sum(qs), sum(ks)
    q_full = torch.empty((hpw, s_q, d), dtype=q_block.dtype, device=dev)
    k_full = torch.empty((kpw, s_kv, d), dtype=k_block.dtype, device=dev)
    v_full = torch.empty((kpw, s_kv, d), dtype=v_block.dtype, device=dev)
    chunks = [[q_block[w * hpw:(w + 1) * hpw].contiguous(),
               k_block[w * kpw:(w + 1) * kpw].contiguous(),
               v_block[w * kpw:(w + 1) * kpw].contiguous()] for w in range(n)]
    recv = [[torch.empty((hpw, qs[w], d), dtype=q_block.dtype, device=dev),
             torch.empty((kpw, ks[w], d), dtype=k_block.dtype, device=dev),
             torch.empty((kpw, ks[w], d), dtype=v_block.dtype, device=dev)] for w in range(n)]
    t0 = ops.event() if trace is not None else None
    hop, g_sent = ctx.all_to_all(chunks, recv, ["Q", "K", "V"])
    hop.wait()
    for w in range(n):
        (qa, qb), (ka, kb) = shards.q_ranges[w], shards.kv_ranges[w]
        q_full[:, qa:qb].copy_(recv[w][0])
        k_full[:, ka:kb].copy_(recv[w][1])
        v_full[:, ka:kb].copy_(recv[w][2])
    t1 = ops.event() if trace is not None else None
    O = torch.empty((hpw, s_q, d), dtype=sd, device=dev)
    L = torch.empty((hpw, s_q), dtype=sd, device=dev)
    if s_kv == 0:
        ops.fill_empty(O, L)
    else:
        ws = ops.fwd_workspace(q_full, k_full)
        ops.fwd_partial(q_full, k_full, v_full, scale, ws)
        ops.fwd_finish(q_full, k_full, ws, O, L)
    t2 = ops.event() if trace is not None else None
    out_chunks = [[O[:, qa:qb].contiguous(), L[:, qa:qb].contiguous()]
                  for qa, qb in shards.q_ranges]
    back = [[torch.empty((hpw, qs[i], d), dtype=sd, device=dev),
             torch.empty((hpw, qs[i]), dtype=sd, device=dev)] for _ in range(n)]
    hop, s_sent = ctx.all_to_all(out_chunks, back, ["O", "L"])
    hop.wait()
    o_i = torch.cat([b[0] for b in back], dim=0)
    l_i = torch.cat([b[1] for b in back], dim=0)
    if trace is not None:
        t3 = ops.event()
        trace._add_timed(ops, t1, t2, t3, {"QKV_gather": sum(g_sent.values()),
                                           "OL_scatter": sum(s_sent.values())})
        trace.section("fwd_kernel", ops, t1, t2)
        trace.section("all_to_all", ops, t0, t1)
    return AttentionState(O=o_i, L=l_i), (q_full, k_full, v_full, AttentionState(O=O, L=L))


def head_parallel_backward(ctx: DeviceContext, shards: ShardSpec, saved, do_block, scale: float,
                           trace: RoundTrace | None = None):
    """Mirror of the forward: all-to-all dO to head sharding, local backward on
    the owned heads, all-to-all dQ/dK/dV back (strategies.py:403-432)."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    q_full, k_full, v_full, st = saved
    hpw, s_q, d = q_full.shape
    kpw, s_kv, _ = k_full.shape
    dev = q_full.device
    sd = ops.state_dtype(q_full.dtype)
    qs, ks = shards.q_sizes, shards.kv_sizes
    chunks = [[do_block[w * hpw:(w + 1) * hpw].contiguous()] for w in range(n)]
    recv = [[torch.empty((hpw, qs[w], d), dtype=do_block.dtype, device=dev)] for w in range(n)]
    t0 = ops.event() if trace is not None else None
    hop, g_sent = ctx.all_to_all(chunks, recv, ["dO"])
    hop.wait()
    do_full = torch.empty((hpw, s_q, d), dtype=do_block.dtype, device=dev)
    for w in range(n):
        qa, qb = shards.q_ranges[w]
        do_full[:, qa:qb].copy_(recv[w][0])
    t1 = ops.event() if trace is not None else None
    D = torch.empty((hpw, s_q), dtype=sd, device=dev)
    ops.row_stats(st.O, do_full, D)
    dq = torch.empty((hpw, s_q, d), dtype=sd, device=dev)
    dk = torch.empty((kpw, s_kv, d), dtype=sd, device=dev)
    dv = torch.empty((kpw, s_kv, d), dtype=sd, device=dev)
    ws = ops.bwd_workspace(q_full, k_full)
    ops.bwd_dq_partial(q_full, k_full, v_full, st.L, D, do_full, scale, ws)
    ops.bwd_dq_finish(q_full, k_full, ws, dq, accumulate=False)
    ops.bwd_dkv(q_full, k_full, v_full, st.L, D, do_full, scale, dk, dv, accumulate=False)
    t2 = ops.event() if trace is not None else None
    out = [[dq[:, qa:qb].contiguous(), dk[:, ka:kb].contiguous(), dv[:, ka:kb].contiguous()]
           for (qa, qb), (ka, kb) in zip(shards.q_ranges, shards.kv_ranges)]
    back = [[torch.empty((hpw, qs[i], d), dtype=sd, device=dev),
             torch.empty((kpw, ks[i], d), dtype=sd, device=dev),
             torch.empty((kpw, ks[i], d), dtype=sd, device=dev)] for _ in range(n)]
    hop, s_sent = ctx.all_to_all(out, back, ["dQ", "dK", "dV"])
    hop.wait()
    if trace is not None:
        t3 = ops.event()
        trace._add_timed(ops, t1, t2, t3, {"dO_gather": sum(g_sent.values()),
                                           "grad_scatter": sum(s_sent.values())})
        trace.section("bwd_kernel", ops, t1, t2)
        trace.section("all_to_all", ops, t0, t1)
    gd = _grad_dtype(ops, do_block.dtype)
    return (torch.cat([b[0] for b in back], dim=0).to(gd),
            torch.cat([b[1] for b in back], dim=0).to(gd),
            torch.cat([b[2] for b in back], dim=0).to(gd))


# ---------------------------------------------------------------------------
# driver — strategies.py:435-551
# ---------------------------------------------------------------------------

@dataclass
class RunResult:
    O: object
    L: object
    grads: GradientBundle | None
    stats: TransportStats
    traces_forward: list
    traces_backward: list | None
    shards: ShardSpec


def _np_dtype_to_torch(dt) -> torch.dtype:
    return {np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64}[np.dtype(dt)]


def run_rank(strategy: str, ctx: DeviceContext, shards: ShardSpec, q_i, k_i, v_i, do_i=None,
             scale: float | None = None, tile_rows: int = DEFAULT_TILE_ROWS, trace: bool = True):
    """One rank's forward (+ backward when ``do_i`` is given) on device
    tensors — the body of run_distributed (strategies.py:477-512).
    Returns (state, grads or None, trace_fwd, trace_bwd)."""
    strategy = StrategyKind(strategy)
    scale = default_scale(q_i.shape[2]) if scale is None else scale
    tf = RoundTrace(strategy=strategy.value, phase="forward") if trace else None
    tb = RoundTrace(strategy=strategy.value, phase="backward") if (trace and do_i is not None) \
        else None
    saved = None
    if strategy in (StrategyKind.LVX, StrategyKind.SINGLE):
        st = lvx_forward(ctx, shards, q_i, k_i, v_i, scale, tile_rows, tf)
    elif strategy is StrategyKind.RING:
        st = ring_forward(ctx, shards, q_i, k_i, v_i, scale, tile_rows, tf)
    else:
        st, saved = head_parallel_forward(ctx, shards, q_i, k_i, v_i, scale, tile_rows, tf)
    grads = None
    if do_i is not None:
        if strategy in (StrategyKind.LVX, StrategyKind.SINGLE):
            grads = lvx_backward(ctx, shards, q_i, k_i, v_i, st, do_i, scale, tb)
        elif strategy is StrategyKind.RING:
            grads = ring_backward(ctx, shards, q_i, k_i, v_i, st, do_i, scale, tb)
        else:
            grads = head_parallel_backward(ctx, shards, saved, do_i, scale, tb)
    return st, grads, tf, tb


def _to_torch(x) -> tuple[torch.Tensor, str]:
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)), "numpy"
    if isinstance(x, torch.Tensor):
        return x, ("cuda" if x.is_cuda else "cpu")
    raise TypeError(f"expected numpy array or torch tensor, got {type(x).__name__}")


def run_distributed(strategy, Q, K, V, dO=None, spec: ClusterSpec | None = None,
                    scale: float | None = None, tile_rows: int = DEFAULT_TILE_ROWS,
                    timeout: float | None = None, *, group=None, ops=None) -> RunResult:
    """Scatter Q/K/V by rows, run the strategy collectively, gather the full
    O, L (and gradients when dO is given) with transport stats and traces
    (strategies.py:454-551).

    Process model: under an initialised ``torch.distributed`` group of n
    ranks (torchrun, one GPU each) every rank calls this with the same full
    inputs, uploads only its own shard, and all ranks return the gathered
    result.  Without a process group, n = 1 runs on the current GPU and
    n > 1 spawns n processes on n local GPUs (``launch.spawn_run``).
    Output dtype = input dtype (O, L, grads), as the reference."""
    strategy = StrategyKind(strategy)
    validate_qkv(Q, K, V)
    h, s_q, d = Q.shape
    s_kv = K.shape[1]
    if dO is not None and tuple(dO.shape) != tuple(Q.shape):
        raise ValueError(f"dO shape {tuple(dO.shape)} != Q shape {tuple(Q.shape)}")
    scale = default_scale(d) if scale is None else scale
    n_req = spec.n if spec is not None else None
    if dist.is_initialized() and (group is not None or n_req is None or n_req > 1 or
                                  dist.get_world_size(group) == 1):
        n = dist.get_world_size(group)
        rank = dist.get_rank(group)
        if n_req is not None and n_req != n:
            raise ValueError(f"spec.n={n_req} but the process group has {n} ranks")
    else:
        n = n_req or 1
        rank = 0
        if n > 1:
            from .launch import spawn_run
            return spawn_run(strategy.value, Q, K, V, dO, n, scale, tile_rows)
    if strategy is StrategyKind.SINGLE and n != 1:
        raise ValueError("single-worker strategy requires n=1")
    if strategy is StrategyKind.HEAD_PARALLEL:
        _check_heads(h, K.shape[0], n)
    shards = ShardSpec.balanced(s_q, s_kv, n)

    (Qt, kind), (Kt, _), (Vt, _) = _to_torch(Q), _to_torch(K), _to_torch(V)
    dt = torch.promote_types(torch.promote_types(Qt.dtype, Kt.dtype), Vt.dtype)
    if ops is None:
        if not torch.cuda.is_available():
            raise RuntimeError("run_distributed needs a CUDA device (no CPU fallback)")
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device(getattr(ops, "device", "cuda"))
    ctx = DeviceContext(rank, n, group=group if n > 1 else None, device=dev, ops=ops)
    qa, qb = shards.q_ranges[rank]
    ka, kb = shards.kv_ranges[rank]
    q_i = Qt[:, qa:qb].to(dev).to(dt).contiguous()
    k_i = Kt[:, ka:kb].to(dev).to(dt).contiguous()
    v_i = Vt[:, ka:kb].to(dev).to(dt).contiguous()
    do_i = None
    if dO is not None:
        do_i = _to_torch(dO)[0][:, qa:qb].to(dev).to(dt).contiguous()
    st, grads, tf, tb = run_rank(strategy, ctx, shards, q_i, k_i, v_i, do_i, scale, tile_rows)
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    tf.resolve()
    if tb is not None:
        tb.resolve()

    out_dt = dt if dt in (torch.float32, torch.float64) else torch.bfloat16
    sd = state_dtype(dt)

    def gather(local, full_shape, rng, dtype):
        # disjoint row ranges: the sum of zero-padded shards is an exact
        # gather (x + 0 == x, -inf + 0 == -inf)
        full = torch.zeros(full_shape, dtype=dtype, device=dev)
        if local.numel():
            full[:, rng[0]:rng[1]] = local.to(dtype)
        if n > 1:
            dist.all_reduce(full, group=group)
        return full

    O = gather(st.O, (h, s_q, d), shards.q_ranges[rank], out_dt)
    L = gather(st.L, (h, s_q), shards.q_ranges[rank], sd if dt == torch.bfloat16 else out_dt)
    gb = None
    if grads is not None:
        gb = GradientBundle(dQ=gather(grads[0], (h, s_q, d), shards.q_ranges[rank], out_dt),
                            dK=gather(grads[1], tuple(Kt.shape), shards.kv_ranges[rank], out_dt),
                            dV=gather(grads[2], tuple(Vt.shape), shards.kv_ranges[rank], out_dt))
    stats = ctx.stats
    traces_f, traces_b = [tf], [tb] if tb is not None else None
    if n > 1:
        objs = [None] * n
        dist.all_gather_object(objs, (ctx.stats, tf, tb), group=group)
        stats = TransportStats()
        for s, _, _ in objs:
            stats.merge(s)
        traces_f = [o[1] for o in objs]
        traces_b = [o[2] for o in objs] if tb is not None else None

    def back(t):
        if t is None:
            return None
        if kind == "numpy":
            return t.cpu().numpy()
        return t.cpu() if kind == "cpu" else t

    grads_out = None if gb is None else GradientBundle(dQ=back(gb.dQ), dK=back(gb.dK),
                                                       dV=back(gb.dV))
    return RunResult(O=back(O), L=back(L), grads=grads_out, stats=stats,
                     traces_forward=traces_f, traces_backward=traces_b, shards=shards)
