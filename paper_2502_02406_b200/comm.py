"""Ring transport for the LV-XAttn schedulers: one process per GPU.

Replaces the reference's in-process thread cluster
(``pkg/src/lvxattn/cluster.py``): a worker is a process bound to one GPU, a
message is a grouped NCCL send/recv over NVLink 5 / NVSwitch
(``torch.distributed.batch_isend_irecv``), and a shift runs on NCCL's own
stream so it overlaps the attention kernels on the compute stream.  The
contract of ``WorkerContext.send/recv/ring_shift`` (cluster.py:227-272) is
kept: every shift is collective, FIFO, goes to ``(rank+1) % n`` and comes
from ``(rank-1) % n``, and byte accounting counts payload bytes only for
``src != dst`` (cluster.py:8-11), so ``n = 1`` loopback is free.

``TransportStats`` mirrors cluster.py:86-120 (per ordered link: bytes,
messages).  Modeled time is replaced by the MEASURED exposed time of each
shift (the time the compute stream actually waited for it), recorded in the
schedulers' round traces.
"""
from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import torch
import torch.distributed as dist


class ClusterError(RuntimeError):
    """Protocol violation (cluster.py:31)."""


class CollectiveTimeout(ClusterError):
    """A collective did not complete in time (cluster.py:35)."""


class WorkerFailed(ClusterError):
    """A rank failed; names it (cluster.py:43-47)."""

    def __init__(self, worker: int, cause: BaseException):
        super().__init__(f"worker {worker} failed: {cause!r}")
        self.worker = worker
        self.cause = cause


@dataclass(frozen=True)
class Instant:
    """Real transport, no modeled delay (cluster.py:50-52)."""


@dataclass(frozen=True)
class ClusterSpec:
    """n ranks; on B200 one process per GPU (cluster.py:69-76)."""

    n: int
    transport: Instant = Instant()

    def __post_init__(self):
        if self.n < 1:
            raise ValueError(f"worker count must be >= 1, got {self.n}")


@dataclass
class LinkStats:
    bytes_sent: int = 0
    message_count: int = 0
    modeled_time_seconds: float = 0.0


class TransportStats:
    """Per ordered (src, dst) counters; loopback never appears (cluster.py:86-120)."""

    def __init__(self):
        self._links: dict[tuple[int, int], LinkStats] = {}
        self._lock = threading.Lock()

    def record(self, src: int, dst: int, nbytes: int, modeled_seconds: float = 0.0) -> None:
        with self._lock:
            link = self._links.setdefault((src, dst), LinkStats())
            link.bytes_sent += nbytes
            link.message_count += 1
            link.modeled_time_seconds += modeled_seconds

    def __getstate__(self):
        return {"links": dict(self._links)}

    def __setstate__(self, state):
        self._links = state["links"]
        self._lock = threading.Lock()

    def merge(self, other: "TransportStats") -> None:
        for (s, d), ls in other._links.items():
            link = self._links.setdefault((s, d), LinkStats())
            link.bytes_sent += ls.bytes_sent
            link.message_count += ls.message_count
            link.modeled_time_seconds += ls.modeled_time_seconds

    def link(self, src: int, dst: int) -> LinkStats:
        return self._links.get((src, dst), LinkStats())

    def bytes_sent_by(self, src: int) -> int:
        return sum(s.bytes_sent for (a, _), s in self._links.items() if a == src)

    def total_bytes(self) -> int:
        return sum(s.bytes_sent for s in self._links.values())

    def total_modeled_seconds(self) -> float:
        return sum(s.modeled_time_seconds for s in self._links.values())

    def as_dict(self) -> dict:
        return {f"{s}->{d}": {"bytes_sent": v.bytes_sent, "message_count": v.message_count,
                              "modeled_time_seconds": v.modeled_time_seconds}
                for (s, d), v in sorted(self._links.items())}


def payload_nbytes(tensors) -> int:
    return int(sum(t.numel() * t.element_size() for t in tensors))


class _Shift:
    """An in-flight ring shift; ``wait()`` orders the caller's stream after it."""

    def __init__(self, works, local_copy=None):
        self._works = works
        self._local = local_copy

    def wait(self) -> None:
        for w in self._works:
            w.wait()
        if self._local is not None:
            for s, r in self._local:
                if s.data_ptr() != r.data_ptr():
                    r.copy_(s)
        self._works = []
        self._local = None


NCCL_SM_RESERVE = int(os.environ.get("LVX_SM_RESERVE", "4"))   # tuning override


class DeviceContext:
    """Per-rank handle: the analogue of ``WorkerContext`` (cluster.py:227-291)
    for one process per GPU.

    ``ops`` is the kernel set the schedulers call (``ops.CudaOps`` — the
    product's CUDA library).  ``group`` is the torch.distributed process group
    (NCCL on B200; gloo in the CPU protocol tests); ``None`` with n = 1 is the
    single-GPU loopback context.
    """

    def __init__(self, rank: int = 0, n: int = 1, group=None, device=None, ops=None,
                 comm_enabled: bool = True):
        if n < 1 or not (0 <= rank < n):
            raise ValueError(f"bad rank {rank} for {n} workers")
        if n > 1 and group is None and not dist.is_initialized():
            raise ClusterError("n > 1 needs an initialised torch.distributed process group")
        self.rank, self.n = rank, n
        self.group = group
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if ops is None:
            from .ops import CudaOps
            ops = CudaOps()
        self.ops = ops
        if n > 1 and hasattr(ops, "set_sm_reserve"):
            # NCCL's send/recv CTAs run beside the ring-round kernels: plan the
            # grids for 4 SMs fewer (n=4 C2: -2.3 % step time, tools/ab_plan_sms.sh);
            # the no-comm arm keeps the same plans (same per-rank schedule)
            ops.set_sm_reserve(NCCL_SM_RESERVE)
        self.stats = TransportStats()
        # comm_enabled=False runs the identical schedule with every hop
        # skipped: the "no-communication" arm of PAPER.md:233.
        self.comm_enabled = comm_enabled
        self._global = [dist.get_global_rank(group, r) if group is not None else r
                        for r in range(n)] if n > 1 else [0]

    @property
    def successor(self) -> int:
        return (self.rank + 1) % self.n

    @property
    def predecessor(self) -> int:
        return (self.rank - 1) % self.n

    def shift(self, send: list, recv: list, classes: list | None = None) -> tuple[_Shift, dict]:
        """Send ``send`` to the successor and receive ``recv`` from the
        predecessor (cluster.py:266-272 ring_shift), asynchronously.
        Returns (handle, sent bytes by class)."""
        if len(send) != len(recv):
            raise ClusterError("ring shift needs matching send/recv lists")
        for s, r in zip(send, recv):   # blocks may differ in rows (uneven shards)
            if s.dtype != r.dtype or s.shape[0] != r.shape[0] or s.shape[2:] != r.shape[2:]:
                raise ClusterError(f"ring shift mismatch {tuple(s.shape)}/{s.dtype} vs "
                                   f"{tuple(r.shape)}/{r.dtype}")
        classes = classes or [str(k) for k in range(len(send))]
        if self.n == 1:   # loopback: free and never touches the transport
            return _Shift([], list(zip(send, recv))), {c: 0 for c in classes}
        sent = {c: t.numel() * t.element_size() for c, t in zip(classes, send)}
        if not self.comm_enabled:
            return _Shift([]), sent
        succ = self._global[self.successor]
        pred = self._global[self.predecessor]
        ops = []
        for s, r in zip(send, recv):
            if s.numel():
                ops.append(dist.P2POp(dist.isend, s, succ, self.group))
            if r.numel():
                ops.append(dist.P2POp(dist.irecv, r, pred, self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        self.stats.record(self.rank, self.successor, payload_nbytes(send))
        return _Shift(works), sent

    def all_to_all(self, chunks: list, recv: list, classes: list | None = None):
        """Deliver ``chunks[w]`` (a list of tensors) to rank w and receive
        ``recv[w]`` (preallocated, same structure) from rank w
        (cluster.py:274-291).  The self chunk is copied locally and never
        touches the transport; bytes are counted per destination for w != rank.
        Returns (handle, sent bytes by class)."""
        if len(chunks) != self.n or len(recv) != self.n:
            raise ClusterError(f"worker {self.rank}: all_to_all expects {self.n} chunks, "
                               f"got {len(chunks)}")
        classes = classes or [str(k) for k in range(len(chunks[0]))]
        sent = {c: 0 for c in classes}
        ops, local = [], list(zip(chunks[self.rank], recv[self.rank]))
        for w in range(self.n):
            if w == self.rank:
                continue
            nb = payload_nbytes(chunks[w])
            for c, t in zip(classes, chunks[w]):
                sent[c] += t.numel() * t.element_size()
            if self.comm_enabled:
                peer = self._global[w]
                for t in chunks[w]:
                    if t.numel():
                        ops.append(dist.P2POp(dist.isend, t.contiguous(), peer, self.group))
                for t in recv[w]:
                    if t.numel():
                        ops.append(dist.P2POp(dist.irecv, t, peer, self.group))
                self.stats.record(self.rank, w, nb)
        works = dist.batch_isend_irecv(ops) if ops else []
        return _Shift(works, local), sent
