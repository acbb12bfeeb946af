"""Distributed cross-attention schedulers on B200 — drop-in for
``lvxattn.strategies`` (reference ``pkg/src/lvxattn/strategies.py``).

One rank per GPU (or thread ranks sharing one GPU).  Each rank keeps its KV
shard resident in HBM; the schedulers move the rotating blocks with
copy-engine puts into the successor's arena (``comm.PeerTransport``) on a
side stream while the attention kernels run on the compute stream, which
waits on a stream-side flag only right before the kernel that consumes a hop.

  lvx   query rotation (strategies.py:175-276, Algorithm 1): the
        (O, L, Q) blocks travel, the fused split-combine+merge kernel folds
        the received state into the new partial.
  ring  KV rotation baseline (strategies.py:279-361).

Round structure, block indices, epilogues, per-message metadata checks and
byte accounting follow the reference exactly, so byte counters equal the
closed forms of ``volumes`` (GQA-aware).  Deviations, all documented in
DESIGN.md: partial states (O, L, D, dQ, dK/dV accumulators) travel in
float32 when the inputs are bfloat16; the receive buffers live in the
rank's arena, laid out per call identically on every rank, instead of being
allocated per message; the backward schedules send their immutable blocks
first and let dQ (LV-XAttn) or the dK/dV partials (Ring) lag one hop, so
message counts differ from the reference's (``volumes.messages_per_rank``)
while byte totals per rank are identical.
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


def _shaped(flat: torch.Tensor, h: int, rows: int, d: int | None = None) -> torch.Tensor:
    """[h, rows, d] (or [h, rows] for d=None) view of the prefix of a flat
    buffer: a block of any row count has the same layout on every rank, so a
    record sent as a whole lands exactly where the receiver reads it."""
    cache = getattr(flat, "_lvx_shaped", None)
    if cache is None:
        cache = {}
        try:
            flat._lvx_shaped = cache    # arena views live across calls (comm._Call.alloc)
        except (AttributeError, RuntimeError):
            pass
    key = (h, rows, d)
    v = cache.get(key)
    if v is None:
        t = flat[:h * rows * (d or 1)]
        v = t.view(h, rows) if d is None else t.view(h, rows, d)
        cache[key] = v
    return v


def _after(ctx: DeviceContext, chan: int, m: int, slots: int):
    """Message m of channel ``chan`` reuses slot m % slots: it waits until the
    receiver released message m - slots (one FREE word per message, so every
    word is written and consumed once per call)."""
    if m < slots:
        return None
    return (chan * 256 + (m - slots), 0)


def _release(ctx: DeviceContext, chan: int, m: int, slots: int) -> None:
    ctx.release(chan * 256 + m, 0)


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


def _attend_merge(ops, q, k_block, v_block, scale, o, l, hop, kv_stream, first, prior):
    """One round's attention of q against the resident KV block merged into
    (o, l): the main loop runs before the hop is waited on, the split combine
    + merge after it.  ``prior``: (o, l) hold a state to merge with (the
    received one) — else they are overwritten.  Round 0 of a streamed block
    consumes K/V chunk by chunk.  Returns the events (t1, t2) around the wait."""
    t1 = t2 = None
    if first and kv_stream is not None and len(kv_stream.bounds) > 1:
        for c, (a, b) in enumerate(kv_stream.bounds):
            if kv_stream.wait_chunk is not None:
                kv_stream.wait_chunk(c)
            kc, vc = k_block[:, a:b], v_block[:, a:b]
            ws = ops.fwd_workspace(q, kc)
            ops.fwd_partial(q, kc, vc, scale, ws)
            if c == 0:
                t1 = ops.event()
                if hop is not None:
                    hop.wait()
                t2 = ops.event()
            merge = prior or c > 0
            ops.fwd_finish(q, kc, ws, o, l, o if merge else None, l if merge else None)
        return t1, t2
    if kv_stream is not None and kv_stream.wait_chunk is not None:
        for c in range(len(kv_stream.bounds)):
            kv_stream.wait_chunk(c)
    ws = ops.fwd_workspace(q, k_block)
    ops.fwd_partial(q, k_block, v_block, scale, ws)
    t1 = ops.event()
    if hop is not None:
        hop.wait()
    t2 = ops.event()
    ops.fwd_finish(q, k_block, ws, o, l, o if prior else None, l if prior else None)
    return t1, t2


# ---------------------------------------------------------------------------
# LV-XAttn query rotation
# ---------------------------------------------------------------------------

def lvx_forward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                scale: float, tile_rows: int = DEFAULT_TILE_ROWS,
                trace: RoundTrace | None = None,
                kv_stream: KVStream | None = None) -> AttentionState:
    """Query-rotation forward for one rank; collective over all n
    (strategies.py:175-231).  Round r: ship the state finished last round
    (block i-r+1; round 0 ships the empty state) plus Q of block i-r to the
    successor, run block i-r's attention against the resident K/V, receive
    the predecessor's state and Q, merge.  After n rounds an epilogue hop
    sends each completed state home.

    Buffers: round r's message lands in record r of the call's arena
    ([O | L | Q], one record per round, so no slot is ever reused inside the
    call); from round 1 on the record received last round is forwarded whole
    — one copy-engine transfer per hop."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, _, d = q_block.shape
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    qs = shards.q_sizes
    mq = max(qs) if qs else 0
    with ctx.call() as call:
        if n == 1:   # loopback (cluster.py:178-180): the empty state merges to nothing
            out_o = torch.empty((h, qs[0], d), dtype=sd, device=dev)
            out_l = torch.empty((h, qs[0]), dtype=sd, device=dev)
            t0 = ops.event() if trace is not None else None
            t1, t2 = _attend_merge(ops, q_block, k_block, v_block, scale, out_o, out_l, None,
                                   kv_stream, True, False)
            if trace is not None:
                t3 = ops.event()
                trace._add_timed(ops, t0, t1, t2, {"O": 0, "L": 0, "Q": 0})
                trace.section("fwd_kernel", ops, t0, t1)
                trace.section("fwd_finish", ops, t2, t3)
                trace.section("wait", ops, t1, t2)
                trace.epilogue_bytes_by_class = {"O": 0, "L": 0}
            return AttentionState(O=out_o, L=out_l)
        buf = call.alloc({"rec": (n, [("O", h * mq * d, sd), ("L", h * mq, sd),
                                      ("Q", h * mq * d, q_block.dtype)]),
                          "home": (1, [("O", h * mq * d, sd), ("L", h * mq, sd)])})
        R, home = buf["rec"], buf["home"][0]
        send_block, q_block_id = (i + 1) % n, i
        o_s = torch.empty((h, qs[send_block], d), dtype=sd, device=dev)
        l_s = torch.empty((h, qs[send_block]), dtype=sd, device=dev)
        ops.fill_empty(o_s, l_s)
        send = [o_s, l_s, q_block]
        q_cur = q_block
        for r in range(n):
            j, j_next = (i - r) % n, (i - r - 1) % n
            _expect(q_block_id, j, f"worker {i} round {r} query")
            _expect(send_block, (j + 1) % n, f"worker {i} round {r} state")
            rec = R[r]
            recv = [_shaped(rec["O"], h, qs[j], d), _shaped(rec["L"], h, qs[j]),
                    _shaped(rec["Q"], h, qs[j_next], d)]
            dst = [_shaped(rec["O"], h, qs[send_block], d), _shaped(rec["L"], h, qs[send_block]),
                   _shaped(rec["Q"], h, qs[j], d)]
            t0 = ops.event() if trace is not None else None
            hop, sent = ctx.shift(send, recv, ["O", "L", "Q"], dst=dst)
            t1, t2 = _attend_merge(ops, q_cur, k_block, v_block, scale, recv[0], recv[1], hop,
                                   kv_stream, r == 0, True)      # merge(recv, delta)
            if trace is not None:
                t3 = ops.event()
                trace._add_timed(ops, t0, t1, t2, sent)
                trace.section("fwd_kernel", ops, t0, t1)
                trace.section("fwd_finish", ops, t2, t3)
                trace.section("wait", ops, t1, t2)
            send, q_cur = recv, recv[2]
            send_block, q_block_id = j, j_next

        # epilogue: the completed state of block i+1 goes home (strategies.py:220-231)
        _expect(send_block, (i + 1) % n, f"worker {i} epilogue")
        recv = [_shaped(home["O"], h, qs[i], d), _shaped(home["L"], h, qs[i])]
        dst = [_shaped(home["O"], h, qs[send_block], d), _shaped(home["L"], h, qs[send_block])]
        hop, epi = ctx.shift(send[:2], recv, ["O", "L"], dst=dst)
        hop.wait()
        out_o, out_l = recv[0].clone(), recv[1].clone()
    if trace is not None:
        trace.epilogue_bytes_by_class = epi
    return AttentionState(O=out_o, L=out_l)


def lvx_backward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                 state: AttentionState, do_block, scale: float,
                 trace: RoundTrace | None = None, kv_stream: KVStream | None = None,
                 dk_out=None, dv_out=None):
    """Query-rotation backward (strategies.py:234-276): the tuple
    (Q, dO, L, D, dQ) of every block travels once around the ring and every
    rank adds its K/V block's contribution; the last dQ hop is the
    homecoming.  Returns (dQ_i, dK_i, dV_i) in the input dtype (the
    reference's convention): everything is computed and carried in the fp32
    state dtype and the batched dK/dV pass writes bf16 gradients directly.

    B200 schedule (same bytes per rank as the reference):
      * the immutable part (Q, dO, L, D) of block j is sent at the START of
        round r, overlapping this round's dQ kernel, instead of after it; it
        lands at block j's rows of the receiver's gather buffers, so every
        rank ends the ring holding every block's rows with no extra copy;
      * dQ lags one hop: round r sends the dQ of block j+1 finished in round
        r-1, and the received dQ of block j is folded in by the dQ finish
        kernel after the local contribution is computed; the epilogue hop
        takes the last one home;
      * dK_i and dV_i (the sum over rounds at strategies.py:261-262) are
        computed ONCE after the ring over the gathered query rows — one
        tensor-core pass with dK/dV in TMEM and a single write, instead of n
        passes with an fp32 read-modify-write each.
    """
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, _, d = q_block.shape
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    gd = _grad_dtype(ops, q_block.dtype)
    qs, qr = shards.q_sizes, shards.q_ranges
    mq = max(qs) if qs else 0
    # written once, in gd; ``dk_out`` / ``dv_out`` let the caller choose the
    # layout (e.g. head views of one [rows, 2 hkv d] matrix the next GEMM reads)
    dk = dk_out if dk_out is not None else torch.empty(k_block.shape, dtype=gd, device=dev)
    dv = dv_out if dv_out is not None else torch.empty(v_block.shape, dtype=gd, device=dev)
    with ctx.call() as call:
        if n == 1:
            return _lvx_backward_local(ops, q_block, k_block, v_block, state, do_block, scale,
                                       trace, kv_stream, dk, dv, sd, gd)
        s_tot = sum(qs)
        buf = call.alloc({"Qg": (h * s_tot * d, q_block.dtype), "Gg": (h * s_tot * d, q_block.dtype),
                          "Lg": (h * s_tot, sd), "Dg": (h * s_tot, sd),
                          "dq": (n, [("dQ", h * mq * d, sd)]),
                          "home": (1, [("dQ", h * mq * d, sd)])})
        Qg, Gg = buf["Qg"].view(h, s_tot, d), buf["Gg"].view(h, s_tot, d)
        Lg, Dg = buf["Lg"].view(h, s_tot), buf["Dg"].view(h, s_tot)
        DQ = [rec["dQ"] for rec in buf["dq"]]
        a, b = qr[i]
        Qg[:, a:b].copy_(q_block)
        Gg[:, a:b].copy_(do_block)
        Lg[:, a:b].copy_(state.L)
        ops.row_stats(state.O, do_block, Dg[:, a:b])          # strategies.py:247
        dq_prev, blk = None, i
        for r in range(n):
            j, nxt = (i - r) % n, (i - r - 1) % n
            _expect(blk, j, f"worker {i} backward round {r}")
            (a, b), (an, bn) = qr[j], qr[nxt]
            q_j, do_j, l_j, d_j = Qg[:, a:b], Gg[:, a:b], Lg[:, a:b], Dg[:, a:b]
            send = [q_j, do_j, l_j, d_j]
            dst = list(send)        # block j's rows: the same offsets on the successor
            recv = [Qg[:, an:bn], Gg[:, an:bn], Lg[:, an:bn], Dg[:, an:bn]]
            classes = ["Q", "dO", "L", "D"]
            dq_in = None
            if r >= 1:   # dQ of block j+1 (finished last round) out, dQ of block j in
                dq_in = _shaped(DQ[r], h, qs[j], d)
                send.append(dq_prev)
                dst.append(_shaped(DQ[r], h, qs[(j + 1) % n], d))
                recv.append(dq_in)
                classes.append("dQ")
            t0 = ops.event() if trace is not None else None
            hop, sent = ctx.shift(send, recv, classes, dst=dst)
            ws = ops.bwd_workspace(q_j, k_block)
            ops.bwd_dq_partial(q_j, k_block, v_block, l_j, d_j, do_j, scale, ws)
            t1 = ops.event() if trace is not None else None
            hop.wait()
            t2 = ops.event() if trace is not None else None
            if dq_in is None:
                dq_acc = _shaped(DQ[0], h, qs[j], d)
                ops.bwd_dq_finish(q_j, k_block, ws, dq_acc, accumulate=False)
            else:
                ops.bwd_dq_finish(q_j, k_block, ws, dq_in, accumulate=True)
                dq_acc = dq_in
            if trace is not None:
                t3 = ops.event()
                trace._add_timed(ops, t0, t1, t2, sent)
                trace.section("dq_kernel", ops, t0, t1)
                trace.section("wait", ops, t1, t2)
                trace.section("dq_finish", ops, t2, t3)
            dq_prev, blk = dq_acc, nxt
        _expect(blk, i, f"worker {i} backward homecoming")
        # the dQ of block i+1 goes home; this rank's own dQ_i arrives
        home = buf["home"][0]["dQ"]
        dq_home = _shaped(home, h, qs[i], d)
        hop, epi = ctx.shift([dq_prev], [dq_home], ["dQ"],
                             dst=[_shaped(home, h, qs[(i + 1) % n], d)])
        if trace is not None:
            trace.epilogue_bytes_by_class = epi
        t4 = ops.event() if trace is not None else None
        if kv_stream is not None and kv_stream.dkv_done is not None:
            _dkv_chunks(ops, kv_stream, Qg, k_block, v_block, Lg, Dg, Gg, scale, dk, dv)
        else:
            ops.bwd_dkv(Qg, k_block, v_block, Lg, Dg, Gg, scale, dk, dv, accumulate=False)
        if trace is not None:
            trace.section("dkv_kernel", ops, t4, ops.event())
        hop.wait()
        dq_out = dq_home.to(gd, copy=True)
    return dq_out, dk, dv


def _lvx_backward_local(ops, q_block, k_block, v_block, state, do_block, scale, trace,
                        kv_stream, dk, dv, sd, gd):
    """n = 1: the one round of lvx_backward on the resident block (loopback
    hops are free and carry nothing)."""
    h, rows, d = q_block.shape
    dev = q_block.device
    D = torch.empty((h, rows), dtype=sd, device=dev)
    ops.row_stats(state.O, do_block, D)                      # strategies.py:247
    streamed = kv_stream is not None and kv_stream.dkv_done is not None
    if streamed:   # dK/dV first, so their chunks leave the GPU while dQ runs
        t4 = ops.event() if trace is not None else None
        _dkv_chunks(ops, kv_stream, q_block, k_block, v_block, state.L, D, do_block, scale,
                    dk, dv)
        if trace is not None:
            trace.section("dkv_kernel", ops, t4, ops.event())
    dq = torch.empty((h, rows, d), dtype=sd, device=dev)
    t0 = ops.event() if trace is not None else None
    ws = ops.bwd_workspace(q_block, k_block)
    ops.bwd_dq_partial(q_block, k_block, v_block, state.L, D, do_block, scale, ws)
    t1 = ops.event() if trace is not None else None
    ops.bwd_dq_finish(q_block, k_block, ws, dq, accumulate=False)
    if trace is not None:
        t3 = ops.event()
        trace._add_timed(ops, t0, t1, t1, {"Q": 0, "dO": 0, "L": 0, "D": 0})
        trace.section("dq_kernel", ops, t0, t1)
        trace.section("wait", ops, t1, t1)
        trace.section("dq_finish", ops, t1, t3)
        trace.epilogue_bytes_by_class = {"dQ": 0}
    if not streamed:
        t4 = ops.event() if trace is not None else None
        ops.bwd_dkv(q_block, k_block, v_block, state.L, D, do_block, scale, dk, dv,
                    accumulate=False)
        if trace is not None:
            trace.section("dkv_kernel", ops, t4, ops.event())
    return (dq if gd == sd else dq.to(gd)), dk, dv


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

RING_SLOTS = 3   # receive slots per rotating class (K/V, dK/dV partials)


def ring_forward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                 scale: float, tile_rows: int = DEFAULT_TILE_ROWS,
                 trace: RoundTrace | None = None) -> AttentionState:
    """KV-rotation forward (strategies.py:279-311): Q/O/L stay resident and
    (K, V) shift n-1 times, each shift (sent at the start of the round)
    overlapping the attention on the block in hand.  Blocks land in
    RING_SLOTS reusable slots; a slot is released to the sender once the
    round that computed on it (and forwarded it) is done."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, rows, d = q_block.shape
    hk = k_block.shape[0]
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    ks = shards.kv_sizes
    mk = max(ks) if ks else 0
    S = max(1, min(RING_SLOTS, n - 1))
    O = torch.empty((h, rows, d), dtype=sd, device=dev)
    L = torch.empty((h, rows), dtype=sd, device=dev)
    with ctx.call() as call:
        R = call.alloc({"kv": (S, [("K", hk * mk * d, k_block.dtype),
                                   ("V", hk * mk * d, v_block.dtype)])})["kv"] if n > 1 else None
        k_cur, v_cur, blk = k_block, v_block, i
        for r in range(n):
            _expect(blk, (i - r) % n, f"worker {i} ring round {r}")
            hop, sent = None, {}
            nxt = (i - r - 1) % n
            if r < n - 1:
                s = R[r % S]
                recv = [_shaped(s["K"], hk, ks[nxt], d), _shaped(s["V"], hk, ks[nxt], d)]
                dst = [_shaped(s["K"], hk, ks[blk], d), _shaped(s["V"], hk, ks[blk], d)]
                hop, sent = ctx.shift([k_cur, v_cur], recv, ["K", "V"], dst=dst,
                                      after=_after(ctx, 0, r, S))
            t0 = ops.event() if trace is not None else None
            if ks[blk]:
                ws = ops.fwd_workspace(q_block, k_cur)
                ops.fwd_partial(q_block, k_cur, v_cur, scale, ws)
                ops.fwd_finish(q_block, k_cur, ws, O, L, O if r else None, L if r else None)
            elif r == 0:
                ops.fill_empty(O, L)
            t1 = ops.event() if trace is not None else None
            if trace is not None:
                trace.section("fwd_kernel", ops, t0, t1)
            if r >= 1:   # the slot this round computed on (message r-1) is free
                _release(ctx, 0, r - 1, S)
            if hop is not None:
                hop.wait()
                k_cur, v_cur, blk = recv[0], recv[1], nxt
            t2 = ops.event() if trace is not None else None
            if trace is not None:
                trace._add_timed(ops, t0, t1, t2, sent)
    return AttentionState(O=O, L=L)


def ring_backward(ctx: DeviceContext, shards: ShardSpec, q_block, k_block, v_block,
                  state: AttentionState, do_block, scale: float,
                  trace: RoundTrace | None = None):
    """KV-rotation backward (strategies.py:314-361): (K, V) rotate n-1 times
    while dQ accumulates locally, and each block's dK/dV partial follows its
    K/V around the ring; an epilogue hop returns each (dK, dV) to its owner.

    Overlapped schedule (same bytes per rank as the reference, K/V and dK/dV
    as separate messages): K/V of the next round are sent at the START of the
    round; this round's dK/dV contribution is computed into a local fp32
    buffer while the partial of the same block is still in flight from the
    predecessor, then added to it (``accumulate``) and forwarded — the
    partials lag one hop behind the K/V they belong to."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, rows, d = q_block.shape
    hk = k_block.shape[0]
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    gd = _grad_dtype(ops, q_block.dtype)
    ks = shards.kv_sizes
    mk = max(ks) if ks else 0
    S = max(1, min(RING_SLOTS, n - 1))
    D = torch.empty((h, rows), dtype=sd, device=dev)
    ops.row_stats(state.O, do_block, D)
    L = state.L
    dq = torch.zeros((h, rows, d), dtype=sd, device=dev)
    with ctx.call() as call:
        if n == 1:
            dk = torch.empty(k_block.shape, dtype=sd, device=dev)
            dv = torch.empty(v_block.shape, dtype=sd, device=dev)
            t0 = ops.event() if trace is not None else None
            ws = ops.bwd_workspace(q_block, k_block)
            ops.bwd_dq_partial(q_block, k_block, v_block, L, D, do_block, scale, ws)
            ops.bwd_dq_finish(q_block, k_block, ws, dq, accumulate=False)
            ops.bwd_dkv(q_block, k_block, v_block, L, D, do_block, scale, dk, dv, accumulate=False)
            if trace is not None:
                t1 = ops.event()
                trace._add_timed(ops, t0, t1, t1, {})
                trace.epilogue_bytes_by_class = {"dK": 0, "dV": 0}
            return _cast(dq, gd), _cast(dk, gd), _cast(dv, gd)
        buf = call.alloc({"kv": (S, [("K", hk * mk * d, k_block.dtype),
                                     ("V", hk * mk * d, v_block.dtype)]),
                          "part": (S, [("dK", hk * mk * d, sd), ("dV", hk * mk * d, sd)]),
                          "home": (1, [("dK", hk * mk * d, sd), ("dV", hk * mk * d, sd)])})
        R, P, home = buf["kv"], buf["part"], buf["home"][0]
        own_k = torch.empty((hk, ks[i], d), dtype=sd, device=dev)   # round 0's partial
        own_v = torch.empty((hk, ks[i], d), dtype=sd, device=dev)
        tmp_k = torch.empty((hk * mk * d,), dtype=sd, device=dev)
        tmp_v = torch.empty((hk * mk * d,), dtype=sd, device=dev)
        k_cur, v_cur, blk = k_block, v_block, i
        hop_p = recv_p = None
        for r in range(n):
            _expect(blk, (i - r) % n, f"worker {i} ring backward round {r}")
            nxt = (i - r - 1) % n
            hop_kv, sent = None, {}
            if r < n - 1:
                s = R[r % S]
                recv_kv = [_shaped(s["K"], hk, ks[nxt], d), _shaped(s["V"], hk, ks[nxt], d)]
                dst = [_shaped(s["K"], hk, ks[blk], d), _shaped(s["V"], hk, ks[blk], d)]
                hop_kv, sent = ctx.shift([k_cur, v_cur], recv_kv, ["K", "V"], dst=dst,
                                         after=_after(ctx, 0, r, S))
            t0 = ops.event() if trace is not None else None
            ws = ops.bwd_workspace(q_block, k_cur)
            ops.bwd_dq_partial(q_block, k_cur, v_cur, L, D, do_block, scale, ws)
            ops.bwd_dq_finish(q_block, k_cur, ws, dq, accumulate=True)
            if r == 0:
                acc_k, acc_v = own_k, own_v
                ops.bwd_dkv(q_block, k_cur, v_cur, L, D, do_block, scale, acc_k, acc_v,
                            accumulate=False)
            else:
                tk, tv = _shaped(tmp_k, hk, ks[blk], d), _shaped(tmp_v, hk, ks[blk], d)
                ops.bwd_dkv(q_block, k_cur, v_cur, L, D, do_block, scale, tk, tv,
                            accumulate=False)
                hop_p.wait()                 # the partial of this block from upstream
                acc_k, acc_v = recv_p
                ops.accumulate(tk, acc_k)
                ops.accumulate(tv, acc_v)
            t1 = ops.event() if trace is not None else None
            if r >= 1:
                _release(ctx, 0, r - 1, S)   # K/V slot computed on this round
            if r < n - 1:                    # the partial follows its block downstream
                s = P[r % S]
                recv_p = [_shaped(s["dK"], hk, ks[nxt], d), _shaped(s["dV"], hk, ks[nxt], d)]
                dst = [_shaped(s["dK"], hk, ks[blk], d), _shaped(s["dV"], hk, ks[blk], d)]
                hop_p, sent_p = ctx.shift([acc_k, acc_v], recv_p, ["dK", "dV"], dst=dst,
                                          after=_after(ctx, 1, r, S))
                sent = {**sent, **sent_p}
            else:                            # block i+1 is complete: send it home
                _expect(blk, (i + 1) % n, f"worker {i} backward epilogue")
                recv_h = [_shaped(home["dK"], hk, ks[i], d), _shaped(home["dV"], hk, ks[i], d)]
                dst = [_shaped(home["dK"], hk, ks[blk], d), _shaped(home["dV"], hk, ks[blk], d)]
                hop_h, epi = ctx.shift([acc_k, acc_v], recv_h, ["dK", "dV"], dst=dst)
            if r >= 1:
                _release(ctx, 1, r - 1, S)   # partial slot added into and forwarded
            if hop_kv is not None:
                hop_kv.wait()
                k_cur, v_cur, blk = recv_kv[0], recv_kv[1], nxt
            t2 = ops.event() if trace is not None else None
            if trace is not None:
                trace._add_timed(ops, t0, t1, t2, sent)
        hop_h.wait()
        dk, dv = recv_h[0].to(gd, copy=True), recv_h[1].to(gd, copy=True)
    if trace is not None:
        trace.epilogue_bytes_by_class = epi
    return _cast(dq, gd), dk, dv


def ring_backward_reference_schedule(ctx: DeviceContext, shards: ShardSpec, q_block, k_block,
                                     v_block, state: AttentionState, do_block, scale: float,
                                     trace: RoundTrace | None = None):
    """The Ring backward in the reference's own order (strategies.py:314-361):
    each round computes on the block in hand, THEN ships (K, V, dK, dV)
    together and waits for the predecessor's — no overlap of the hop with
    compute.  Same results and bytes as ``ring_backward``; kept as the
    reference-faithful Ring baseline beside the overlapped one."""
    n, i, ops = ctx.n, ctx.rank, ctx.ops
    h, rows, d = q_block.shape
    hk = k_block.shape[0]
    dev = q_block.device
    sd = ops.state_dtype(q_block.dtype)
    gd = _grad_dtype(ops, q_block.dtype)
    ks = shards.kv_sizes
    mk = max(ks) if ks else 0
    if n == 1:
        return ring_backward(ctx, shards, q_block, k_block, v_block, state, do_block, scale,
                             trace)
    D = torch.empty((h, rows), dtype=sd, device=dev)
    ops.row_stats(state.O, do_block, D)
    L = state.L
    dq = torch.zeros((h, rows, d), dtype=sd, device=dev)
    with ctx.call() as call:
        buf = call.alloc({"rec": (2, [("K", hk * mk * d, k_block.dtype),
                                      ("V", hk * mk * d, v_block.dtype),
                                      ("dK", hk * mk * d, sd), ("dV", hk * mk * d, sd)]),
                          "home": (1, [("dK", hk * mk * d, sd), ("dV", hk * mk * d, sd)])})
        R, home = buf["rec"], buf["home"][0]
        acc_k = torch.empty((hk, ks[i], d), dtype=sd, device=dev)   # round 0's partial
        acc_v = torch.empty((hk, ks[i], d), dtype=sd, device=dev)
        tmp_k = torch.empty((hk * mk * d,), dtype=sd, device=dev)
        tmp_v = torch.empty((hk * mk * d,), dtype=sd, device=dev)
        k_cur, v_cur, blk = k_block, v_block, i
        for r in range(n):
            _expect(blk, (i - r) % n, f"worker {i} ring backward round {r}")
            t0 = ops.event() if trace is not None else None
            ws = ops.bwd_workspace(q_block, k_cur)
            ops.bwd_dq_partial(q_block, k_cur, v_cur, L, D, do_block, scale, ws)
            ops.bwd_dq_finish(q_block, k_cur, ws, dq, accumulate=True)
            if r == 0:
                ops.bwd_dkv(q_block, k_cur, v_cur, L, D, do_block, scale, acc_k, acc_v,
                            accumulate=False)
            else:
                tk, tv = _shaped(tmp_k, hk, ks[blk], d), _shaped(tmp_v, hk, ks[blk], d)
                ops.bwd_dkv(q_block, k_cur, v_cur, L, D, do_block, scale, tk, tv,
                            accumulate=False)
                ops.accumulate(tk, acc_k)
                ops.accumulate(tv, acc_v)
            t1 = ops.event() if trace is not None else None
            sent = {}
            nxt = (i - r - 1) % n
            if r < n - 1:   # compute, then shift (K, V, dK, dV) and wait
                s = R[r % 2]
                recv = [_shaped(s["K"], hk, ks[nxt], d), _shaped(s["V"], hk, ks[nxt], d),
                        _shaped(s["dK"], hk, ks[nxt], d), _shaped(s["dV"], hk, ks[nxt], d)]
                dst = [_shaped(s["K"], hk, ks[blk], d), _shaped(s["V"], hk, ks[blk], d),
                       _shaped(s["dK"], hk, ks[blk], d), _shaped(s["dV"], hk, ks[blk], d)]
                # a slot is rewritten two rounds later, after its reader has
                # finished with it (this wait chain orders the whole ring)
                hop, sent = ctx.shift([k_cur, v_cur, acc_k, acc_v], recv,
                                      ["K", "V", "dK", "dV"], dst=dst,
                                      after=_after(ctx, 0, r, 2))
                hop.wait()
                if r >= 1:
                    _release(ctx, 0, r - 1, 2)
                k_cur, v_cur, acc_k, acc_v = recv
                blk = nxt
            t2 = ops.event() if trace is not None else None
            if trace is not None:
                trace._add_timed(ops, t0, t1, t2, sent)
        _expect(blk, (i + 1) % n, f"worker {i} backward epilogue")
        recv_h = [_shaped(home["dK"], hk, ks[i], d), _shaped(home["dV"], hk, ks[i], d)]
        dst = [_shaped(home["dK"], hk, ks[blk], d), _shaped(home["dV"], hk, ks[blk], d)]
        hop_h, epi = ctx.shift([acc_k, acc_v], recv_h, ["dK", "dV"], dst=dst)
        hop_h.wait()
        _release(ctx, 0, n - 2, 2)
        dk, dv = recv_h[0].to(gd, copy=True), recv_h[1].to(gd, copy=True)
    if trace is not None:
        trace.epilogue_bytes_by_class = epi
    return _cast(dq, gd), dk, dv


def _cast(t: torch.Tensor, dt) -> torch.Tensor:
    return t if t.dtype == dt else t.to(dt)


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
    mq, mk = max(qs), max(ks)
    s_q, s_kv = sum(qs), sum(ks)
    q_full = torch.empty((hpw, s_q, d), dtype=q_block.dtype, device=dev)
    k_full = torch.empty((kpw, s_kv, d), dtype=k_block.dtype, device=dev)
    v_full = torch.empty((kpw, s_kv, d), dtype=v_block.dtype, device=dev)
    O = torch.empty((hpw, s_q, d), dtype=sd, device=dev)
    L = torch.empty((hpw, s_q), dtype=sd, device=dev)
    with ctx.call() as call:
        buf = call.alloc({"g": (n, [("Q", hpw * mq * d, q_block.dtype),
                                    ("K", kpw * mk * d, k_block.dtype),
                                    ("V", kpw * mk * d, v_block.dtype)]),
                          "s": (n, [("O", hpw * mq * d, sd), ("L", hpw * mq, sd)])})
        G, Sc = buf["g"], buf["s"]
        chunks = [[q_block[w * hpw:(w + 1) * hpw], k_block[w * kpw:(w + 1) * kpw],
                   v_block[w * kpw:(w + 1) * kpw]] for w in range(n)]
        recv = [[_shaped(G[w]["Q"], hpw, qs[w], d), _shaped(G[w]["K"], kpw, ks[w], d),
                 _shaped(G[w]["V"], kpw, ks[w], d)] for w in range(n)]
        t0 = ops.event() if trace is not None else None
        hop, g_sent = ctx.all_to_all(chunks, recv, ["Q", "K", "V"])
        hop.wait()
        for w in range(n):
            (qa, qb), (ka, kb) = shards.q_ranges[w], shards.kv_ranges[w]
            q_full[:, qa:qb].copy_(recv[w][0])
            k_full[:, ka:kb].copy_(recv[w][1])
            v_full[:, ka:kb].copy_(recv[w][2])
        t1 = ops.event() if trace is not None else None
        if s_kv == 0:
            ops.fill_empty(O, L)
        else:
            ws = ops.fwd_workspace(q_full, k_full)
            ops.fwd_partial(q_full, k_full, v_full, scale, ws)
            ops.fwd_finish(q_full, k_full, ws, O, L)
        t2 = ops.event() if trace is not None else None
        out_chunks = [[O[:, qa:qb], L[:, qa:qb]] for qa, qb in shards.q_ranges]
        back = [[_shaped(Sc[w]["O"], hpw, qs[i], d), _shaped(Sc[w]["L"], hpw, qs[i])]
                for w in range(n)]
        # rank w keeps our block in its record i, sized by ITS rows
        dst = [[_shaped(Sc[i]["O"], hpw, qs[w], d), _shaped(Sc[i]["L"], hpw, qs[w])]
               for w in range(n)]
        hop, s_sent = ctx.all_to_all(out_chunks, back, ["O", "L"], dst=dst)
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
    mq, mk = max(qs), max(ks)
    do_full = torch.empty((hpw, s_q, d), dtype=do_block.dtype, device=dev)
    D = torch.empty((hpw, s_q), dtype=sd, device=dev)
    dq = torch.empty((hpw, s_q, d), dtype=sd, device=dev)
    dk = torch.empty((kpw, s_kv, d), dtype=sd, device=dev)
    dv = torch.empty((kpw, s_kv, d), dtype=sd, device=dev)
    gd = _grad_dtype(ops, do_block.dtype)
    with ctx.call() as call:
        buf = call.alloc({"g": (n, [("dO", hpw * mq * d, do_block.dtype)]),
                          "s": (n, [("dQ", hpw * mq * d, sd), ("dK", kpw * mk * d, sd),
                                    ("dV", kpw * mk * d, sd)])})
        G, Sc = buf["g"], buf["s"]
        chunks = [[do_block[w * hpw:(w + 1) * hpw]] for w in range(n)]
        recv = [[_shaped(G[w]["dO"], hpw, qs[w], d)] for w in range(n)]
        t0 = ops.event() if trace is not None else None
        hop, g_sent = ctx.all_to_all(chunks, recv, ["dO"])
        hop.wait()
        for w in range(n):
            qa, qb = shards.q_ranges[w]
            do_full[:, qa:qb].copy_(recv[w][0])
        t1 = ops.event() if trace is not None else None
        ops.row_stats(st.O, do_full, D)
        ws = ops.bwd_workspace(q_full, k_full)
        ops.bwd_dq_partial(q_full, k_full, v_full, st.L, D, do_full, scale, ws)
        ops.bwd_dq_finish(q_full, k_full, ws, dq, accumulate=False)
        ops.bwd_dkv(q_full, k_full, v_full, st.L, D, do_full, scale, dk, dv, accumulate=False)
        t2 = ops.event() if trace is not None else None
        out = [[dq[:, qa:qb], dk[:, ka:kb], dv[:, ka:kb]]
               for (qa, qb), (ka, kb) in zip(shards.q_ranges, shards.kv_ranges)]
        back = [[_shaped(Sc[w]["dQ"], hpw, qs[i], d), _shaped(Sc[w]["dK"], kpw, ks[i], d),
                 _shaped(Sc[w]["dV"], kpw, ks[i], d)] for w in range(n)]
        dst = [[_shaped(Sc[i]["dQ"], hpw, qs[w], d), _shaped(Sc[i]["dK"], kpw, ks[w], d),
                _shaped(Sc[i]["dV"], kpw, ks[w], d)] for w in range(n)]
        hop, s_sent = ctx.all_to_all(out, back, ["dQ", "dK", "dV"], dst=dst)
        hop.wait()
        res = (torch.cat([b[0] for b in back], dim=0).to(gd),
               torch.cat([b[1] for b in back], dim=0).to(gd),
               torch.cat([b[2] for b in back], dim=0).to(gd))
    if trace is not None:
        t3 = ops.event()
        trace._add_timed(ops, t1, t2, t3, {"dO_gather": sum(g_sent.values()),
                                           "grad_scatter": sum(s_sent.values())})
        trace.section("bwd_kernel", ops, t1, t2)
        trace.section("all_to_all", ops, t0, t1)
    return res


# ---------------------------------------------------------------------------
# one rank's step as a CUDA graph
# ---------------------------------------------------------------------------

class StepGraph:
    """One rank's step — e.g. ``lvx_forward`` + ``lvx_backward`` of a layer on
    fixed device buffers — recorded once as a CUDA graph and replayed.

    The schedulers issue ~10 kernel launches, ~10 copies and ~20 stream-side
    flag operations per ring round from Python; at small shards (C4 at n = 8,
    Lkv 64K at n >= 4) that host time is as long as the device work.  A replay
    is one host call.  Everything the schedulers do is capturable: kernels,
    copy-engine puts into peer arenas, one-shot flag writes / waits with
    constant values (comm.PeerTransport), and the side stream's fork / join
    through events.  Collective: every rank records (the flags pair up at
    capture like at run time) and every rank replays the same number of times.
    ``fn`` must not need tracing, host sync or new arena space after
    ``warmup`` eager runs (which size the arena and the workspaces)."""

    def __init__(self, ctx: DeviceContext, fn, warmup: int = 2):
        self.ctx = ctx
        for _ in range(warmup):
            fn()
        ctx.synchronize()
        ctx.barrier()
        from . import _lib
        self.graph = torch.cuda.CUDAGraph()
        # a capture stream of its own (torch's default one comes from the
        # shared pool, and thread ranks record concurrently)
        self._stream = _lib.OwnStream(ctx.device)
        with torch.cuda.graph(self.graph, stream=self._stream.stream,
                              capture_error_mode="thread_local"):
            self.outputs = fn()
        ctx.barrier()

    def replay(self):
        """Runs the recorded step on the current stream; returns the outputs
        of the recorded call (overwritten by every replay)."""
        self.graph.replay()
        return self.outputs


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
                    timeout: float | None = None, *, group=None, ops=None,
                    ranks: str = "auto") -> RunResult:
    """Scatter Q/K/V by rows, run the strategy collectively, gather the full
    O, L (and gradients when dO is given) with transport stats and traces
    (strategies.py:454-551).

    Process model: under an initialised ``torch.distributed`` group of n
    ranks (torchrun, one GPU each) every rank calls this with the same full
    inputs, uploads only its own shard, and all ranks return the gathered
    result.  Without a process group, n = 1 runs on the current GPU and
    n > 1 runs ``ranks``: "processes" (n processes on n local GPUs,
    ``launch.spawn_run``), "threads" (n thread ranks sharing the current
    device, the reference's own worker model, ``launch.spawn_ranks``), or
    "auto" (processes when n GPUs are visible, else threads).  ``timeout``
    (else $LVX_TIMEOUT_SECS, else 30 s) bounds every wait on a peer; the
    first failing rank is raised as ``WorkerFailed`` (cluster.py:300-335).
    Output dtype = input dtype (O, L, grads), as the reference."""
    strategy = StrategyKind(strategy)
    validate_qkv(Q, K, V)
    h, s_q, d = Q.shape
    s_kv = K.shape[1]
    if dO is not None and tuple(dO.shape) != tuple(Q.shape):
        raise ValueError(f"dO shape {tuple(dO.shape)} != Q shape {tuple(Q.shape)}")
    scale = default_scale(d) if scale is None else scale
    n_req = spec.n if spec is not None else None
    if strategy is StrategyKind.SINGLE and (n_req or 1) != 1:
        raise ValueError("single-worker strategy requires n=1")
    if strategy is StrategyKind.HEAD_PARALLEL and n_req:
        _check_heads(h, K.shape[0], n_req)
    if dist.is_initialized() and (group is not None or n_req is None or n_req > 1 or
                                  dist.get_world_size(group) == 1) and ranks != "threads":
        n = dist.get_world_size(group)
        rank = dist.get_rank(group)
        if n_req is not None and n_req != n:
            raise ValueError(f"spec.n={n_req} but the process group has {n} ranks")
        if strategy is StrategyKind.SINGLE and n != 1:
            raise ValueError("single-worker strategy requires n=1")
        if strategy is StrategyKind.HEAD_PARALLEL:
            _check_heads(h, K.shape[0], n)
        dev = _device_for(ops)
        ctx = DeviceContext(rank, n, group=group if n > 1 else None, device=dev, ops=ops,
                            timeout=timeout)
        try:
            return rank_body(strategy, ctx, Q, K, V, dO, scale, tile_rows)
        finally:
            ctx.close()
    n = n_req or 1
    if n == 1:
        ctx = DeviceContext(0, 1, device=_device_for(ops), ops=ops, timeout=timeout)
        return rank_body(strategy, ctx, Q, K, V, dO, scale, tile_rows)
    from . import launch
    if ranks not in ("auto", "threads", "processes"):
        raise ValueError(f"ranks must be 'auto', 'threads' or 'processes', got {ranks!r}")
    gpus = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ranks == "processes" or (ranks == "auto" and ops is None and gpus >= n):
        return launch.spawn_run(strategy.value, Q, K, V, dO, n, scale, tile_rows, timeout)
    dev = _device_for(ops)

    def body(ctx):
        return rank_body(strategy, ctx, Q, K, V, dO, scale, tile_rows)
    res = launch.spawn_ranks(ClusterSpec(n), body, timeout=timeout, device=dev,
                             ops_factory=(type(ops) if ops is not None else None))
    return res.results[0]


def _device_for(ops) -> torch.device:
    if ops is None:
        if not torch.cuda.is_available():
            raise RuntimeError("run_distributed needs a CUDA device (no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(getattr(ops, "device", "cuda"))


def rank_body(strategy, ctx: DeviceContext, Q, K, V, dO, scale: float,
              tile_rows: int = DEFAULT_TILE_ROWS) -> RunResult:
    """One rank of run_distributed on full host (or device) inputs: upload
    this rank's shard, run the strategy, wait with the context's deadline,
    gather O / L / grads by row range and the stats / traces of every rank
    (strategies.py:475-551).  Every rank returns the same RunResult."""
    strategy = StrategyKind(strategy)
    n, rank, dev = ctx.n, ctx.rank, ctx.device
    h, s_q, d = Q.shape
    s_kv = K.shape[1]
    shards = ShardSpec.balanced(s_q, s_kv, n)
    (Qt, kind), (Kt, _), (Vt, _) = _to_torch(Q), _to_torch(K), _to_torch(V)
    dt = torch.promote_types(torch.promote_types(Qt.dtype, Kt.dtype), Vt.dtype)
    qa, qb = shards.q_ranges[rank]
    ka, kb = shards.kv_ranges[rank]
    q_i = Qt[:, qa:qb].to(dev).to(dt).contiguous()
    k_i = Kt[:, ka:kb].to(dev).to(dt).contiguous()
    v_i = Vt[:, ka:kb].to(dev).to(dt).contiguous()
    do_i = None
    if dO is not None:
        do_i = _to_torch(dO)[0][:, qa:qb].to(dev).to(dt).contiguous()
    st, grads, tf, tb = run_rank(strategy, ctx, shards, q_i, k_i, v_i, do_i, scale, tile_rows)
    ctx.synchronize()          # CollectiveTimeout if a hop never arrives
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
        ctx.all_reduce_sum_(full)
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
        objs = ctx.all_gather_object((ctx.stats, tf, tb))
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
