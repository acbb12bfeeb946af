"""LV-XAttn layers on HOST-resident inputs, streamed over PCIe.

The reference runs on device tensors only (``pkg/src/lvxattn/strategies.py``
takes blocks that already live on the worker).  In an MLLM the visual tokens
of a long video are often produced or kept off-GPU; this is the path that
takes pinned host buffers, and it is what ``bench.py`` times as ``e2e``.

A step is one layer forward + backward: Q, K, V, dO of this rank's shard in,
O, L, dQ, dK, dV out (bf16, L fp32), every byte crossing PCIe inside the step.
Three streams per rank:

  h2d      K/V rows in ``chunks`` row ranges (one contiguous copy per head and
           chunk), each chunk followed by an event.  The forward's round 0
           consumes chunks as they land (``strategies.KVStream``); later
           rounds and the backward find the block resident.
  compute  the LV-XAttn forward / backward of ``strategies`` (the ring hops
           on the transport's copy stream as usual).
  d2h      dK/dV leave per chunk as soon as the batched dK/dV pass has
           finished that chunk (at n = 1 that pass runs before dQ, so dQ
           hides the tail); O, L, dQ leave at the end.

With ``prefetch`` (default) the device inputs are double-buffered: step s+1's
H2D is queued right behind step s's and runs while step s computes, since
PCIe carries H2D and D2H concurrently.  Step s+1's copies only start once step
s-1 has released the slot, and nothing of step s+1 is read before its own
events, so results are identical to running the steps one by one.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .comm import DeviceContext
from .strategies import KVStream, ShardSpec, lvx_backward, lvx_forward, partition_rows


@dataclass
class HostStep:
    """Pinned host buffers of one step: inputs q [hq, sq, d], k / v [hkv, skv, d],
    do [hq, sq, d] (bf16); outputs o, dq [hq, sq, d], dk, dv [hkv, skv, d] (bf16)
    and l [hq, sq] (fp32), written when the step's events complete."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    do: torch.Tensor
    o: torch.Tensor
    l: torch.Tensor
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor

    @classmethod
    def allocate(cls, q, k, v, do) -> "HostStep":
        """Output buffers (pinned) shaped like the inputs."""
        def pin(shape, dtype):
            return torch.empty(shape, dtype=dtype, pin_memory=True)
        return cls(q, k, v, do, o=pin(q.shape, torch.bfloat16),
                   l=pin(q.shape[:2], torch.float32), dq=pin(q.shape, torch.bfloat16),
                   dk=pin(k.shape, torch.bfloat16), dv=pin(v.shape, torch.bfloat16))

    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.q, self.k, self.v, self.do))

    def d2h_bytes(self) -> int:
        return sum(t.numel() * t.element_size()
                   for t in (self.o, self.l, self.dq, self.dk, self.dv))


class _Slot:
    def __init__(self, q, k, do, dev):
        self.q = torch.empty(q.shape, dtype=q.dtype, device=dev)
        self.do = torch.empty(do.shape, dtype=do.dtype, device=dev)
        self.k = torch.empty(k.shape, dtype=k.dtype, device=dev)
        self.v = torch.empty(k.shape, dtype=k.dtype, device=dev)
        self.free = None   # event: the last step using this slot has finished


class HostLayerPipeline:
    """Streams LV-XAttn fwd+bwd steps whose inputs and outputs live in pinned
    host memory (one instance per rank; collective like the strategies)."""

    def __init__(self, ctx: DeviceContext, shards: ShardSpec, scale: float,
                 chunks: int = 8, prefetch: bool = True):
        if not torch.cuda.is_available():
            raise RuntimeError("HostLayerPipeline needs a CUDA device (there is no CPU path)")
        self.ctx, self.shards, self.scale = ctx, shards, scale
        self.chunks, self.prefetch = max(1, chunks), prefetch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        self._slots: list[_Slot] = []

    # ------------------------------------------------------------- copies
    def _issue_h2d(self, st: HostStep, slot: _Slot, bounds) -> list:
        """Queue one step's inputs on the h2d stream; returns per-chunk events."""
        evs = []
        with torch.cuda.stream(self.h2d):
            if slot.free is not None:
                self.h2d.wait_event(slot.free)
            slot.q.copy_(st.q, non_blocking=True)
            slot.do.copy_(st.do, non_blocking=True)
            for a, b in bounds:
                for h in range(st.k.shape[0]):   # contiguous per head
                    slot.k[h, a:b].copy_(st.k[h, a:b], non_blocking=True)
                    slot.v[h, a:b].copy_(st.v[h, a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(self.h2d)
                evs.append(e)
        return evs

    def _d2h(self, dst: torch.Tensor, src: torch.Tensor, rows: tuple | None = None) -> None:
        """src (device, any float dtype) -> dst (pinned host, its dtype), after
        the compute stream's current position."""
        cur = torch.cuda.current_stream(self.dev)
        tmp = src if src.dtype == dst.dtype else src.to(dst.dtype)
        ev = torch.cuda.Event()
        ev.record(cur)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(ev)
            if rows is None:
                dst.copy_(tmp, non_blocking=True)
            else:
                a, b = rows
                for h in range(dst.shape[0]):
                    dst[h, a:b].copy_(tmp[h], non_blocking=True)
            tmp.record_stream(self.d2h)

    # ---------------------------------------------------------------- run
    def run(self, steps: list[HostStep]) -> None:
        """Runs every step; returns once all outputs are in host memory."""
        if not steps:
            return
        k0 = steps[0].k
        bounds = [r for r in partition_rows(k0.shape[1], min(self.chunks, max(1, k0.shape[1])))
                  if r[1] > r[0]]
        nslots = 2 if (self.prefetch and len(steps) > 1) else 1
        if len(self._slots) != nslots or self._slots[0].k.shape != k0.shape:
            self._slots = [_Slot(steps[0].q, k0, steps[0].do, self.dev) for _ in range(nslots)]
        cur = torch.cuda.current_stream(self.dev)
        pending = {0: self._issue_h2d(steps[0], self._slots[0], bounds)}
        for s, st in enumerate(steps):
            slot = self._slots[s % nslots]
            if s not in pending:   # one slot: this step's copies wait for the last step's release
                pending[s] = self._issue_h2d(st, slot, bounds)
            evs = pending.pop(s)
            if nslots == 2 and s + 1 < len(steps):   # prefetch behind this step's copies
                pending[s + 1] = self._issue_h2d(steps[s + 1], self._slots[(s + 1) % 2], bounds)
            stream = KVStream(bounds=bounds,
                              wait_chunk=lambda c, evs=evs: cur.wait_event(evs[c]),
                              dkv_done=lambda c, dk, dv, st=st: (
                                  self._d2h(st.dk, dk, bounds[c]),
                                  self._d2h(st.dv, dv, bounds[c])))
            # Q / dO are the first copies of the step: chunk 0's event covers them
            cur.wait_event(evs[0])
            state = lvx_forward(self.ctx, self.shards, slot.q, slot.k, slot.v, self.scale,
                                kv_stream=stream)
            self._d2h(st.o, state.O)
            self._d2h(st.l, state.L)
            dq, _, _ = lvx_backward(self.ctx, self.shards, slot.q, slot.k, slot.v, state,
                                    slot.do, self.scale, kv_stream=stream)
            self._d2h(st.dq, dq)
            # the next copies into this slot (step s+1 with one slot, s+2 with
            # two) wait until this step's kernels have read it
            slot.free = torch.cuda.Event()
            slot.free.record(cur)
        self.d2h.synchronize()
        cur.synchronize()
