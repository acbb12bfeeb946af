"""Ring transport for the LV-XAttn schedulers.

Replaces the reference's in-process thread cluster (``pkg/src/lvxattn/
cluster.py``).  The contract of ``WorkerContext.send/recv/ring_shift``
(cluster.py:227-272) is kept: every shift is collective, FIFO, goes to
``(rank+1) % n`` and comes from ``(rank-1) % n``; byte accounting counts
payload bytes only for ``src != dst`` (cluster.py:8-11), so ``n = 1``
loopback is free; the first failing rank is reported as ``WorkerFailed``
and a collective that does not complete within the timeout raises
``CollectiveTimeout`` (cluster.py:35-47, :149-220, :300-335).

Two transports carry the hops:

``PeerTransport`` (the product path on GPUs)
    Every rank owns an *arena* (``lvx_peer_*`` in the C ABI): one device
    allocation laid out identically on all ranks.  A hop is a few 2-D
    ``cudaMemcpyAsync`` from local memory into the same offset of the
    successor's arena, issued on a side stream so the GPU's copy engines push
    it over NVLink 5 / NVSwitch while the attention kernels keep every SM,
    followed by a stream-ordered flag write (``cuStreamWriteValue32``) that
    the successor's compute stream waits on (``cuStreamWaitValue32``).  No
    host thread ever blocks on a hop.  Peers are mapped with CUDA IPC (one
    process per GPU) or by pointer (``ThreadGroup``: n ranks as threads of one
    process on one GPU — the reference's own worker model, used to run the
    n-rank protocols on a single device).

``ProcessGroupTransport``
    Grouped ``torch.distributed`` isend/irecv (NCCL, or gloo for the CPU
    protocol tests that plug the oracle into the schedulers).  Kept as the
    A/B baseline of the copy-engine path.

``TransportStats`` mirrors cluster.py:86-120 (per ordered link: bytes,
messages).  Modeled time is replaced by the MEASURED exposed time of each
shift (the time the compute stream waited for it), recorded in the
schedulers' round traces.
"""
from __future__ import annotations

import ctypes
import os
import threading
import time
from contextlib import contextmanager
from dataclasses import dataclass

import torch
import torch.distributed as dist

DEFAULT_TIMEOUT_SECONDS = 30.0          # cluster.py:25
TIMEOUT_ENV_VAR = "LVX_TIMEOUT_SECS"    # cluster.py:26


class ClusterError(RuntimeError):
    """Protocol violation (cluster.py:31)."""


class CollectiveTimeout(ClusterError):
    """A collective did not complete in time (cluster.py:35)."""


class ClusterAborted(ClusterError):
    """Another rank failed while this one was communicating (cluster.py:39)."""


class WorkerFailed(ClusterError):
    """A rank failed; names it (cluster.py:43-47)."""

    def __init__(self, worker: int, cause: BaseException):
        super().__init__(f"worker {worker} failed: {cause!r}")
        self.worker = worker
        self.cause = cause


def resolve_timeout(timeout: float | None) -> float:
    """Explicit value, else $LVX_TIMEOUT_SECS, else 30 s (cluster.py:293-300)."""
    if timeout is not None:
        return float(timeout)
    env = os.environ.get(TIMEOUT_ENV_VAR)
    return float(env) if env else DEFAULT_TIMEOUT_SECONDS


@dataclass(frozen=True)
class Instant:
    """Real transport, no modeled delay (cluster.py:50-52)."""


@dataclass(frozen=True)
class ClusterSpec:
    """n ranks; on B200 one process per GPU, or n thread ranks sharing one GPU
    when fewer GPUs than ranks are visible (cluster.py:69-76)."""

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


# ---------------------------------------------------------------------------
# collectives used outside the hot path (setup, gathers, barriers)
# ---------------------------------------------------------------------------

class ThreadGroup:
    """n ranks as threads of one process — the reference's worker model
    (cluster.py:300-335) — sharing one GPU, each on its own CUDA stream.
    Provides the few collectives the schedulers need outside the hops.  The
    first failure aborts the group: every blocked or later collective raises
    ``ClusterAborted``."""

    def __init__(self, n: int, timeout: float | None = None):
        self.n = n
        self.timeout = resolve_timeout(timeout)
        self._barrier = threading.Barrier(n)
        self._slots: list = [None] * n
        self._lock = threading.Lock()
        self.first_failure: tuple[int, BaseException] | None = None
        self.transports: list = [None] * n    # per-rank transport (for abort)
        # mailboxes of the host transport (cluster.py:133-145): per receiving
        # rank, FIFO queues keyed by (src, message index)
        self.cond = threading.Condition()
        self.boxes: list = [dict() for _ in range(n)]
        # copy-engine transport between thread ranks: per rank r and flag word
        # w, how many stream-side writes into it have been ENQUEUED, and how
        # many of them r's waits have consumed
        self.marks: list = [dict() for _ in range(n)]
        self.consumed: list = [dict() for _ in range(n)]

    def fail(self, rank: int, exc: BaseException) -> None:
        with self._lock:
            if self.first_failure is None:
                self.first_failure = (rank, exc)
        self._barrier.abort()
        with self.cond:
            self.cond.notify_all()
        for t in self.transports:
            if t is not None:
                t.abort()

    @property
    def aborted(self) -> bool:
        return self.first_failure is not None

    def mark(self, rank: int, word: int) -> None:
        """One more write into rank's flag word has been enqueued."""
        with self.cond:
            m = self.marks[rank]
            m[word] = m.get(word, 0) + 1
            self.cond.notify_all()

    def await_mark(self, rank: int, word: int) -> None:
        """Block the host until a write into rank's flag word that this wait
        has not consumed yet has been enqueued (on any stream), and consume
        it.  Thread ranks share one CUDA context: a device-side wait enqueued
        before its write could deadlock against any device-synchronising call
        (allocator growth, free) another rank's thread makes meanwhile, so a
        wait is only ever enqueued behind its signal."""
        deadline = time.monotonic() + self.timeout
        with self.cond:
            c = self.consumed[rank]
            while self.marks[rank].get(word, 0) <= c.get(word, 0):
                if self.aborted:
                    raise ClusterAborted(f"worker {rank}: cluster aborted while waiting for a hop")
                now = time.monotonic()
                if now >= deadline:
                    raise CollectiveTimeout(f"worker {rank}: hop (flag {word}) did not arrive "
                                            f"within {self.timeout}s")
                self.cond.wait(timeout=deadline - now)
            c[word] = c.get(word, 0) + 1

    def reset_marks(self, rank: int) -> None:
        """rank's flag words were re-created at zero (a new arena)."""
        with self.cond:
            self.marks[rank] = {}
            self.consumed[rank] = {}

    def put(self, dst: int, key, payload) -> None:
        with self.cond:
            self.boxes[dst].setdefault(key, []).append(payload)
            self.cond.notify_all()

    def get(self, rank: int, key):
        """Blocking FIFO receive with the group deadline (cluster.py:197-220)."""
        deadline = time.monotonic() + self.timeout
        with self.cond:
            while True:
                if self.aborted:
                    raise ClusterAborted(f"worker {rank}: cluster aborted while receiving "
                                         f"(src={key[0]}, msg={key[1]})")
                q = self.boxes[rank].get(key)
                if q:
                    return q.pop(0)
                now = time.monotonic()
                if now >= deadline:
                    raise CollectiveTimeout(f"worker {rank}: recv(src={key[0]}, msg={key[1]}) "
                                            f"timed out after {self.timeout}s")
                self.cond.wait(timeout=deadline - now)

    def rank(self, r: int) -> "ThreadRank":
        return ThreadRank(self, r)

    def _wait(self, rank: int, timeout: float | None = None) -> None:
        if self.first_failure is not None:
            raise ClusterAborted(f"worker {rank}: group aborted")
        try:
            self._barrier.wait(timeout=self.timeout if timeout is None else timeout)
        except threading.BrokenBarrierError:
            if self.first_failure is not None:
                raise ClusterAborted(f"worker {rank}: group aborted") from None
            raise CollectiveTimeout(f"worker {rank}: barrier timed out after "
                                    f"{self.timeout}s") from None


@dataclass(frozen=True)
class ThreadRank:
    """Handle of one thread rank (what a torch.distributed group is to a process)."""

    group: ThreadGroup
    rank: int

    @property
    def n(self) -> int:
        return self.group.n


class _Coll:
    """barrier / all_gather_object / all_reduce over a torch.distributed group
    or a ThreadGroup."""

    def __init__(self, group, rank: int, n: int):
        self.group, self.rank, self.n = group, rank, n

    @property
    def threaded(self) -> bool:
        return isinstance(self.group, ThreadRank)

    def barrier(self, timeout: float | None = None) -> None:
        if self.n == 1:
            return
        if self.threaded:
            self.group.group._wait(self.rank, timeout)
        else:
            dist.barrier(group=self.group)

    def all_gather_object(self, obj) -> list:
        if self.n == 1:
            return [obj]
        if self.threaded:
            g = self.group.group
            g._slots[self.rank] = obj
            g._wait(self.rank)
            out = list(g._slots)
            g._wait(self.rank)
            return out
        out = [None] * self.n
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def all_reduce_sum_(self, t: torch.Tensor) -> None:
        if self.n == 1:
            return
        if self.threaded:
            torch.cuda.current_stream(t.device).synchronize() if t.is_cuda else None
            parts = self.all_gather_object(t)
            acc = parts[0].clone()
            for p in parts[1:]:
                acc += p
            if t.is_cuda:
                torch.cuda.current_stream(t.device).synchronize()
            self.barrier()         # every rank has read every part before any is reused
            t.copy_(acc)
            return
        dist.all_reduce(t, group=self.group)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

def _as_rows(t: torch.Tensor, split: bool = False) -> tuple[int, int, int, int]:
    """(ptr, pitch, width, height) bytes of a [h, rows, d] or [h, rows] view
    whose rows are contiguous within each head: one span when the view is
    contiguous (unless ``split``), else one row of ``width`` bytes per head."""
    es = t.element_size()
    if t.numel() == 0:
        return t.data_ptr(), 0, 0, 0
    if t.is_contiguous() and (not split or t.shape[0] == 1):
        return t.data_ptr(), t.numel() * es, t.numel() * es, 1
    inner = t[0]
    if not inner.is_contiguous():
        raise ClusterError(f"transport view {tuple(t.shape)} stride {t.stride()} has "
                           "non-contiguous rows")
    if t.shape[0] == 1:
        return t.data_ptr(), inner.numel() * es, inner.numel() * es, 1
    return t.data_ptr(), t.stride(0) * es, inner.numel() * es, t.shape[0]


def _copy_overlap(src: torch.Tensor, dst: torch.Tensor) -> None:
    """dst <- src over the rows both have (blocks of uneven shards differ by
    one row); same-shape blocks are a plain copy."""
    if src.numel() == 0 or dst.numel() == 0 or src.data_ptr() == dst.data_ptr():
        return
    if src.shape == dst.shape:
        dst.copy_(src)
        return
    m = min(src.shape[1], dst.shape[1])
    dst[:, :m].copy_(src[:, :m])


def _rows_packed(t: torch.Tensor) -> bool:
    """Rows contiguous within each head (any head stride)."""
    return t.numel() == 0 or t[0].is_contiguous()


class _Hop:
    """An in-flight shift; ``wait()`` orders the caller's stream after it."""

    def __init__(self, fn=None):
        self._fn = fn

    def wait(self) -> None:
        if self._fn is not None:
            self._fn()
            self._fn = None


class ProcessGroupTransport:
    """Grouped isend/irecv on a torch.distributed group (NCCL or gloo)."""

    kind = "process-group"

    def __init__(self, coll: _Coll):
        if coll.threaded:
            raise ClusterError("the process-group transport needs a torch.distributed group")
        self.coll = coll
        self._global = [dist.get_global_rank(coll.group, r) if coll.group is not None else r
                        for r in range(coll.n)]

    def alloc(self, nbytes: int, device) -> torch.Tensor:
        return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)

    def begin(self, handshake: bool = True):
        pass

    def end(self, handshake: bool = True):
        pass

    def shift(self, send, dst, recv, to: int, frm: int, k: int, after=None):
        ops, staged = [], []
        for s, r in zip(send, recv):
            if s.numel():
                ops.append(dist.P2POp(dist.isend, s.contiguous(), self._global[to],
                                      self.coll.group))
            if r.numel():
                t = r if r.is_contiguous() else torch.empty(r.shape, dtype=r.dtype,
                                                            device=r.device)
                if t is not r:
                    staged.append((t, r))
                ops.append(dist.P2POp(dist.irecv, t, self._global[frm], self.coll.group))
        works = dist.batch_isend_irecv(ops) if ops else []

        def wait():
            for w in works:
                w.wait()
            for t, r in staged:
                r.copy_(t)
        return _Hop(wait)

    def release(self, flag: int, value: int, peer: int) -> None:
        pass

    def all_to_all(self, chunks, recv, dst, rank: int, k: int):
        ops, staged = [], []
        for w in range(self.coll.n):
            if w == rank:
                continue
            for t in chunks[w]:
                if t.numel():
                    ops.append(dist.P2POp(dist.isend, t.contiguous(), self._global[w],
                                          self.coll.group))
            for r in recv[w]:
                if r.numel():
                    t = r if r.is_contiguous() else torch.empty(r.shape, dtype=r.dtype,
                                                                device=r.device)
                    if t is not r:
                        staged.append((t, r))
                    ops.append(dist.P2POp(dist.irecv, t, self._global[w], self.coll.group))
        works = dist.batch_isend_irecv(ops) if ops else []

        def wait():
            for w in works:
                w.wait()
            for t, r in staged:
                r.copy_(t)
        return _Hop(wait)

    def abort(self) -> None:
        pass

    def close(self) -> None:
        pass


class MailboxTransport:
    """Thread ranks on a host device (the CPU protocol tests): the reference's
    buffered send / blocking FIFO recv (cluster.py:173-220) on the
    ThreadGroup's mailboxes.  A message is a list of tensor copies."""

    kind = "mailbox"

    def __init__(self, coll: _Coll):
        if not coll.threaded:
            raise ClusterError("the mailbox transport runs thread ranks")
        self.group = coll.group.group
        self.rank = coll.rank
        self.group.transports[self.rank] = self

    def alloc(self, nbytes: int, device) -> torch.Tensor:
        return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)

    def begin(self, handshake: bool = True):
        if self.group.aborted:
            raise ClusterAborted(f"worker {self.rank}: group aborted")

    def end(self, handshake: bool = True):
        pass

    def _recv_into(self, frm: int, k: int, recv) -> None:
        msg = self.group.get(self.rank, (frm, k))
        for m, r in zip(msg, recv):
            if r.numel():
                r.copy_(m.reshape(r.shape))

    def shift(self, send, dst, recv, to: int, frm: int, k: int, after=None):
        self.group.put(to, (self.rank, k), [t.clone() for t in send])
        return _Hop(lambda: self._recv_into(frm, k, recv))

    def release(self, word: int, value: int, peer: int) -> None:
        pass

    def all_to_all(self, chunks, recv, dst, rank: int, k: int):
        for w in range(self.group.n):
            if w != rank:
                self.group.put(w, (rank, k), [t.clone() for t in chunks[w]])

        def wait():
            for w in range(self.group.n):
                if w != rank:
                    self._recv_into(w, k, recv[w])
        return _Hop(wait)

    def abort(self) -> None:
        pass

    def close(self) -> None:
        pass


class PeerTransport:
    """Copy-engine hops into symmetric arenas (see the module docstring).

    Arena = data region (laid out per scheduler call by ``DeviceContext.call``)
    + a flag region of u32 words at the end.  Flags are one-shot: the writer
    sets a word to 1 (fenced behind its copies), its single consumer waits for
    >= 1 and resets it to 0 on the same stream, and every word is written and
    consumed at most once per call:
      READY[k * 16 + src]  message k of this call from rank src has landed
      FREE[c * 256 + m]    the receiver is done with message m of channel c
                           (the sender may rewrite that slot)
      EPOCH[src]           rank src finished its previous call (its arena and
                           its reads of ours are done); consumed by begin()
    The values never change, so a recorded step replays as a CUDA graph
    (``strategies.StepGraph``), and no host exchange is needed per call.
    One-shot EPOCH words stay unambiguous because a peer's next end-of-call
    write cannot come before this rank consumed the previous one: in every
    schedule here (ring shifts, all-to-all) a rank's call finishes only after
    receiving data that transitively left every peer after that peer's
    begin(); calls that send nothing skip the handshake (``handshake``)."""

    kind = "copy-engine"
    MAXN = 16
    READY, NREADY = 0, 768 * 16
    FREE = READY + NREADY
    FREE_PER_CHANNEL = 256
    EPOCH = FREE + 2 * FREE_PER_CHANNEL
    FLAG_WORDS = 16384
    FLAG_BYTES = FLAG_WORDS * 4

    def __init__(self, coll: _Coll, device: torch.device):
        from . import _lib
        self.lib = _lib.load()
        self.coll = coll
        self.rank, self.n = coll.rank, coll.n
        if self.n > self.MAXN:
            raise ClusterError(f"copy-engine transport supports at most {self.MAXN} ranks")
        self.device = torch.device(device)
        self._copy_own = _lib.OwnStream(self.device)    # never a pooled stream another rank holds
        self.copy = self._copy_own.stream
        self.map = None
        self.capacity = 0
        self.base = 0
        self.arena: torch.Tensor | None = None
        self.epoch = 0
        self._aborted = False
        self.tg = coll.group.group if coll.threaded else None
        if coll.threaded:
            coll.group.group.transports[self.rank] = self

    # -- arena --------------------------------------------------------------
    def _wrap(self, ptr: int, nbytes: int) -> torch.Tensor:
        class _Iface:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                        "data": (ptr, False), "version": 2, "strides": None}
        return torch.as_tensor(_Iface(), device=self.device)

    def reserve(self, data_bytes: int) -> None:
        """Collective: make the arena's data region at least ``data_bytes``."""
        if data_bytes <= self.capacity:
            return
        from . import _lib
        # exact need rounded to 2 MiB (HBM is the Ring baseline's limit at
        # multi-million-row shards); calls of one schedule repeat their sizes
        cap = max(data_bytes, 1 << 20)
        cap = (cap + (2 << 20) - 1) // (2 << 20) * (2 << 20)
        # every rank asks for the same layout; agree on the largest request
        cap = max(self.coll.all_gather_object(cap))
        torch.cuda.synchronize(self.device)
        self.coll.barrier()            # no peer is still writing into the old arenas
        self._free_map()
        self.coll.barrier()
        m = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check("lvx_peer_create", self.lib.lvx_peer_create(
                cap + self.FLAG_BYTES, self.rank, self.n, ctypes.byref(m)))
        self.map = m
        self.base = int(self.lib.lvx_peer_base(m))
        self.capacity = cap
        self.arena = self._wrap(self.base, cap + self.FLAG_BYTES)
        # the new arena's flags are zero (lvx_peer_create): this call's EPOCH
        # handshake was consumed in the old one by begin()
        torch.cuda.synchronize(self.device)
        if self.tg is not None:
            self.tg.reset_marks(self.rank)
        if self.coll.threaded:
            maps = self.coll.all_gather_object(m.value)
            for p in range(self.n):
                if p != self.rank:
                    _lib.check("lvx_peer_attach", self.lib.lvx_peer_attach(
                        m, p, ctypes.c_void_p(maps[p])))
        else:
            hb = int(self.lib.lvx_peer_handle_bytes())
            buf = (ctypes.c_char * hb)()
            _lib.check("lvx_peer_export", self.lib.lvx_peer_export(m, buf))
            handles = self.coll.all_gather_object(bytes(buf))
            for p in range(self.n):
                if p != self.rank:
                    hbuf = (ctypes.c_char * hb).from_buffer_copy(handles[p])
                    with torch.cuda.device(self.device):
                        _lib.check("lvx_peer_open", self.lib.lvx_peer_open(m, p, hbuf))
        self.coll.barrier()

    def alloc(self, nbytes: int, device) -> torch.Tensor:
        self.reserve(nbytes)
        return self.arena[:max(nbytes, 1)]

    def release_arena(self) -> None:
        """Collective, between calls: free the arena (the next call maps a new
        one of the size it needs) — after a schedule with big slots (the Ring
        baseline's K/V) when later calls need far less."""
        torch.cuda.synchronize(self.device)
        self.coll.barrier()
        self._free_map()
        self.coll.barrier()

    def _flag(self, word: int) -> int:
        return self.capacity + 4 * word

    def _signal(self, peer: int, word: int, stream) -> None:
        """peer's flag word <- 1, stream-ordered after prior work."""
        self._check("lvx_peer_signal", self.lib.lvx_peer_signal(
            self.map, peer, self._flag(word), 1, stream))
        if self.tg is not None:
            self.tg.mark(peer, word)

    def _wait(self, word: int, stream) -> None:
        """stream waits until this rank's flag word is set, then clears it."""
        if self.tg is not None:
            self.tg.await_mark(self.rank, word)
        self._check("lvx_peer_wait", self.lib.lvx_peer_wait(
            self.map, self._flag(word), 1, stream))
        self._check("lvx_peer_signal", self.lib.lvx_peer_signal(
            self.map, self.rank, self._flag(word), 0, stream))

    def _check(self, fn: str, st: int) -> None:
        if st != 0:
            from . import _lib
            _lib.check(fn, st)

    # -- calls and hops -----------------------------------------------------
    def begin(self, handshake: bool = True):
        """A call starts: the copy stream waits until every peer finished its
        previous call (so it is no longer reading our arena or writing into
        the slots this call will reuse).  ``handshake=False``: a call that
        never writes into peers (the no-communication arm) skips the flags,
        so a context of its own never races the ring's one-shot EPOCH words."""
        if self._aborted:
            raise ClusterAborted(f"worker {self.rank}: transport aborted")
        self.epoch += 1
        if self.map is not None and handshake:
            cs = self.copy.cuda_stream
            for p in range(self.n):
                if p != self.rank:
                    self._wait(self.EPOCH + p, cs)

    def end(self, handshake: bool = True):
        """The caller's arena is free once its compute stream gets here; tell
        every peer (they may write into it in the next call), then join the
        copy stream back so nothing outlives the call."""
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        self.copy.wait_event(ev)
        cs = self.copy.cuda_stream
        for p in range(self.n if handshake else 0):
            if p != self.rank:
                self._signal(p, self.EPOCH + self.rank, cs)
        done = torch.cuda.Event()
        done.record(self.copy)
        cur.wait_event(done)

    def _put_many(self, peer: int, send, recv) -> None:
        """Copy each ``send`` tensor into ``peer``'s arena at the offset of the
        matching ``recv`` view of this rank's arena (identical layouts).  A
        contiguous block and a strided one (per-head rows) go as a 2-D copy
        with their own pitches.  Pieces that are exactly adjacent on both
        sides and both inside this rank's arena (a record forwarded whole)
        coalesce into one copy; nothing else does, since a gap between two
        pieces may hold rows the receiver already has."""
        cs = self.copy.cuda_stream
        runs = []   # [dst_off, dst_pitch, src_ptr, src_pitch, width, height]
        for s, r in zip(send, recv):
            if s.numel() == 0:
                continue
            if s.numel() != r.numel() or s.dtype != r.dtype:
                raise ClusterError(f"shift mismatch {tuple(s.shape)} vs {tuple(r.shape)}")
            if not (_rows_packed(s) and _rows_packed(r)):
                # rows strided inside a head (heads interleaved in the rows of a
                # projection output): one 2-D copy of the head's rows per head
                es = s.element_size()
                for hh in range(s.shape[0]):
                    sh, rh = s[hh], r[hh]
                    off = rh.data_ptr() - self.base
                    rows = sh.shape[0]
                    w = (sh.shape[1] if sh.dim() > 1 else 1) * es
                    if off < 0 or off + (rows - 1) * rh.stride(0) * es + w > self.capacity:
                        raise ClusterError("receive buffer is not in the transport arena")
                    runs.append([off, rh.stride(0) * es, sh.data_ptr(), sh.stride(0) * es, w, rows,
                                 False])
                continue
            sp, spitch, w, h = _as_rows(s)
            rp, rpitch, w2, h2 = _as_rows(r)
            if (w, h) != (w2, h2):       # one side strided: copy per head on both
                sp, spitch, w, h = _as_rows(s, split=True)
                rp, rpitch, w2, h2 = _as_rows(r, split=True)
                if (w, h) != (w2, h2):
                    raise ClusterError(f"shift layout mismatch {tuple(s.shape)}/{s.stride()} "
                                       f"vs {tuple(r.shape)}/{r.stride()}")
            off = rp - self.base
            if off < 0 or off + (h - 1) * rpitch + w > self.capacity:
                raise ClusterError("receive buffer is not in the transport arena")
            src_in_arena = self.base <= sp and sp + (h - 1) * spitch + w <= self.base + \
                self.capacity
            if runs and h == 1 and runs[-1][5] == 1 and src_in_arena and runs[-1][6]:
                o0, _, s0, _, w0, _, _ = runs[-1]
                if off == o0 + w0 and sp == s0 + w0:
                    runs[-1][4] = w0 + w
                    continue
            runs.append([off, rpitch, sp, spitch, w, h, src_in_arena])
        for off, rpitch, sp, spitch, w, h, _ in runs:
            self._check("lvx_peer_put", self.lib.lvx_peer_put(
                self.map, peer, off, rpitch, ctypes.c_void_p(sp), spitch, w, h, cs))

    def shift(self, send, dst, recv, to: int, frm: int, k: int, after=None):
        """Message k of this call: send -> successor (into its copy of the
        arena at ``dst``'s offsets); the returned hop makes the compute stream
        wait for the predecessor's message k (landed in ``recv``)."""
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        self.copy.wait_event(ev)
        cs = self.copy.cuda_stream
        if after is not None:           # the successor released the slot
            self._wait(self.FREE + after[0], cs)
        self._put_many(to, send, dst)
        self._signal(to, self.READY + k * self.MAXN + self.rank, cs)

        def wait():
            self._wait(self.READY + k * self.MAXN + frm,
                       torch.cuda.current_stream(self.device).cuda_stream)
        return _Hop(wait)

    def release(self, word: int, value: int, peer: int) -> None:
        """Tell ``peer`` (the sender) that the message behind FREE word
        ``word`` is consumed, once the compute stream gets here (and our own
        sends from that slot, earlier on the copy stream, are done)."""
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        self.copy.wait_event(ev)
        self._signal(peer, self.FREE + word, self.copy.cuda_stream)

    def all_to_all(self, chunks, recv, dst, rank: int, k: int):
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        self.copy.wait_event(ev)
        cs = self.copy.cuda_stream
        for w in range(self.n):
            if w == rank:
                continue
            self._put_many(w, chunks[w], dst[w])
            self._signal(w, self.READY + k * self.MAXN + rank, cs)

        def wait():
            st = torch.cuda.current_stream(self.device).cuda_stream
            for w in range(self.n):
                if w != rank:
                    self._wait(self.READY + k * self.MAXN + w, st)
        return _Hop(wait)

    def abort(self) -> None:
        """Release every stream-side wait of this rank (after a failure), so the
        device can drain and the process can exit."""
        self._aborted = True
        if self.arena is None:
            return
        s = torch.cuda.Stream(self.device)
        with torch.cuda.stream(s):   # every pending one-shot wait passes
            self.arena[self.capacity:].view(torch.int32).fill_(1)

    def _free_map(self) -> None:
        if self.map is not None:
            self.arena = None
            self.lib.lvx_peer_destroy(self.map)
            self.map = None
            self.capacity = 0

    def close(self) -> None:
        try:
            self.copy.synchronize()
            torch.cuda.current_stream(self.device).synchronize()
        finally:
            self._free_map()
            self._copy_own.close()


# ---------------------------------------------------------------------------
# the per-rank context the schedulers use
# ---------------------------------------------------------------------------

_ALIGN = 256


class _Layout:
    """Bump allocator for one scheduler call (identical on every rank).
    Buffers start on 256-byte boundaries; the fields of one record on 16-byte
    boundaries, so a record whose fields are all full is one adjacent span."""

    def __init__(self):
        self.items = []
        self.size = 0

    def add(self, shape, dtype, align: int = _ALIGN) -> int:
        if isinstance(shape, int):
            shape = (shape,)
        nbytes = 1
        for s in shape:
            nbytes *= int(s)
        nbytes *= torch.empty((), dtype=dtype).element_size()
        off = (self.size + align - 1) // align * align
        self.size = off + nbytes
        self.items.append((off, tuple(int(s) for s in shape), dtype))
        return len(self.items) - 1


class _Call:
    def __init__(self, ctx: "DeviceContext"):
        self.ctx = ctx
        self.k = 0

    def alloc(self, spec: dict) -> dict:
        """One allocation for the whole call.  ``spec`` maps a name to
        (shape, dtype) — a plain buffer — or to (count, [(field, shape, dtype),
        ...]) — ``count`` records, each a packed run of fields (a record sent
        as a whole is one copy).  Buffers live in the transport arena when the
        transport has one (so peers can write into them)."""
        # a schedule repeats its calls with the same shapes: the views are
        # built once per (layout, arena) and reused (host time per step)
        key = tuple((name, a, tuple(map(tuple, b)) if isinstance(b, list) else b)
                    for name, (a, b) in spec.items())
        memo = self.ctx._views
        hit = memo.get(key)
        if hit is not None:
            size, out, base_ptr = hit
            base = self.ctx._raw(size)
            if base.data_ptr() == base_ptr:
                return out
        lay = _Layout()
        plan = {}
        for name, (a, b) in spec.items():
            if isinstance(b, list):
                plan[name] = [{f: lay.add(shape, dt, align=_ALIGN if j == 0 else 16)
                               for j, (f, shape, dt) in enumerate(b)} for _ in range(a)]
            else:
                plan[name] = lay.add(a, b)
        base = self.ctx._raw(lay.size)

        def view(idx):
            off, shape, dt = lay.items[idx]
            es = torch.empty((), dtype=dt).element_size()
            n = 1
            for s in shape:
                n *= s
            return base[off:off + n * es].view(dt).view(shape)
        out = {}
        for name, p in plan.items():
            out[name] = [{f: view(i) for f, i in rec.items()} for rec in p] \
                if isinstance(p, list) else view(p)
        if self.ctx.transport is not None and isinstance(self.ctx.transport, PeerTransport):
            if len(memo) > 64:
                memo.clear()
            memo[key] = (lay.size, out, base.data_ptr())
        return out

    def next_msg(self) -> int:
        k = self.k
        self.k += 1
        return k


class DeviceContext:
    """Per-rank handle: the analogue of ``WorkerContext`` (cluster.py:227-291).

    ``ops`` is the kernel set the schedulers call (``ops.CudaOps`` — the
    product's CUDA library).  ``group`` is a torch.distributed process group
    (one process per GPU; gloo in the CPU protocol tests), a ``ThreadRank``
    (thread ranks sharing one GPU), or ``None`` with n = 1.  ``transport``:
    "ce" (copy-engine arenas, the default on CUDA) or "pg" (torch.distributed
    send/recv: NCCL or gloo), or another context's transport object.
    ``comm_enabled=False`` runs the identical schedule with every hop skipped
    — the no-communication arm of PAPER.md:233.  Its receive slots hold
    zeros (a fresh arena) or, sharing the comm arm's transport, the data of
    the last real hop, so every kernel reads the same kind of values."""

    def __init__(self, rank: int = 0, n: int = 1, group=None, device=None, ops=None,
                 comm_enabled: bool = True, transport: str | None = None,
                 timeout: float | None = None):
        if n < 1 or not (0 <= rank < n):
            raise ValueError(f"bad rank {rank} for {n} workers")
        if isinstance(group, ThreadRank):
            if group.rank != rank or group.n != n:
                raise ValueError(f"thread rank {group.rank}/{group.n} != {rank}/{n}")
        elif n > 1 and group is None and not dist.is_initialized():
            raise ClusterError("n > 1 needs an initialised torch.distributed process group "
                               "or a ThreadGroup")
        self.rank, self.n = rank, n
        self.group = group
        self.timeout = resolve_timeout(timeout)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if ops is None:
            from .ops import CudaOps
            ops = CudaOps()
        self.ops = ops
        self.stats = TransportStats()
        self.comm_enabled = comm_enabled
        self.coll = _Coll(group if n > 1 else None, rank, n)
        if transport is None:
            transport = "ce" if self.device.type == "cuda" else \
                ("mailbox" if isinstance(group, ThreadRank) else "pg")
        if n == 1:
            self.transport = None
        elif isinstance(transport, (PeerTransport, ProcessGroupTransport, MailboxTransport)):
            # another context's transport: the no-comm arm shares the comm
            # arm's arena, so its receive slots hold the last real hop's data
            self.transport = transport
        elif transport == "mailbox":
            self.transport = MailboxTransport(self.coll)
        elif transport == "ce":
            self.transport = PeerTransport(self.coll, self.device)
        elif transport in ("pg", "nccl"):
            self.transport = ProcessGroupTransport(self.coll)
        else:
            raise ValueError(f"unknown transport {transport!r}")
        self._call: _Call | None = None
        self._views: dict = {}      # call layout -> views into the arena (see _Call.alloc)

    @property
    def transport_kind(self) -> str:
        return self.transport.kind if self.transport is not None else "loopback"

    @property
    def successor(self) -> int:
        return (self.rank + 1) % self.n

    @property
    def predecessor(self) -> int:
        return (self.rank - 1) % self.n

    @property
    def epoch(self) -> int:
        return getattr(self.transport, "epoch", 0)

    # -- one scheduler call -------------------------------------------------
    @contextmanager
    def call(self):
        """Brackets one collective scheduler call (lvx_forward, ring_backward,
        ...): buffers from ``alloc`` are valid inside it only."""
        if self._call is not None:
            raise ClusterError("scheduler calls do not nest")
        self._call = _Call(self)
        if self.transport is not None:
            self.transport.begin(handshake=self.comm_enabled)
        try:
            yield self._call
        finally:
            if self.transport is not None:
                self.transport.end(handshake=self.comm_enabled)
            self._call = None

    def release_arena(self) -> None:
        """Collective: drop the transport's arena (see PeerTransport)."""
        if isinstance(self.transport, PeerTransport):
            self.transport.release_arena()
            self._views.clear()

    def _raw(self, nbytes: int) -> torch.Tensor:
        if self.transport is not None and isinstance(self.transport, PeerTransport):
            return self.transport.alloc(nbytes, self.device)
        return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device)

    def _msg(self) -> int:
        if self._call is None:
            raise ClusterError("hops must run inside ctx.call()")
        return self._call.next_msg()

    # -- hops -----------------------------------------------------------------
    def shift(self, send: list, recv: list, classes: list | None = None, dst: list | None = None,
              after=None):
        """Send ``send`` to the successor and receive ``recv`` from the
        predecessor (cluster.py:266-272 ring_shift), asynchronously.  ``recv``
        and ``dst`` are views from ``call().alloc``: ``dst[k]`` is where, in
        the successor's copy of the layout, ``send[k]`` lands (default
        ``recv``, right when both blocks have the same shape).  ``after=(word,
        value)`` makes the send wait until the successor released that slot.
        Returns (handle, sent bytes by class)."""
        if len(send) != len(recv):
            raise ClusterError("ring shift needs matching send/recv lists")
        for s, r in zip(send, recv):   # blocks may differ in rows (uneven shards)
            if s.dtype != r.dtype or s.shape[0] != r.shape[0] or s.shape[2:] != r.shape[2:]:
                raise ClusterError(f"ring shift mismatch {tuple(s.shape)}/{s.dtype} vs "
                                   f"{tuple(r.shape)}/{r.dtype}")
        classes = classes or [str(k) for k in range(len(send))]
        if self.n == 1:   # loopback: free and never touches the transport

            def local():
                for s, r in zip(send, recv):
                    if s.data_ptr() != r.data_ptr() and s.numel():
                        r.copy_(s)
            return _Hop(local), {c: 0 for c in classes}
        k = self._msg()
        sent = {c: t.numel() * t.element_size() for c, t in zip(classes, send)}
        if not self.comm_enabled:
            return self._local_hop(list(zip(send, recv))), sent
        hop = self.transport.shift(send, recv if dst is None else dst, recv, self.successor,
                                   self.predecessor, k, after)
        self.stats.record(self.rank, self.successor, payload_nbytes(send))
        return hop, sent

    def _local_hop(self, pairs):
        """No-communication arm: instead of the hop, each receive slot gets a
        local copy of the matching send block (the overlapping rows when
        uneven shards make them differ), on the transport's side stream like
        a real hop.  The kernels then read the same kind of values as with
        communication (a stale or recycled slot can hold anything, and the
        attention kernels' speed depends on the score range)."""
        if not pairs:
            return _Hop()
        side = getattr(self.transport, "copy", None) if self.device.type == "cuda" else None
        if side is None:
            def copy_now():
                for s_, r_ in pairs:
                    _copy_overlap(s_, r_)
            return _Hop(copy_now)
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            for s_, r_ in pairs:
                _copy_overlap(s_, r_)
        done = torch.cuda.Event()
        done.record(side)
        return _Hop(lambda: torch.cuda.current_stream(self.device).wait_event(done))

    def release(self, word: int, value: int) -> None:
        """The slot the predecessor filled may be reused (see ``shift(after=)``)."""
        if self.n > 1 and self.comm_enabled:
            self.transport.release(word, value, self.predecessor)

    def all_to_all(self, chunks: list, recv: list, classes: list | None = None,
                   dst: list | None = None):
        """Deliver ``chunks[w]`` (a list of tensors) to rank w and receive
        ``recv[w]`` from rank w (cluster.py:274-291).  ``recv[w]`` views come
        from ``call().alloc`` and are laid out so that the block rank w sends
        to rank v sits at the same offset on every rank (index by source).
        The self chunk is copied locally and never touches the transport;
        bytes are counted per destination for w != rank.  Returns (handle,
        sent bytes by class)."""
        if len(chunks) != self.n or len(recv) != self.n:
            raise ClusterError(f"worker {self.rank}: all_to_all expects {self.n} chunks, "
                               f"got {len(chunks)}")
        classes = classes or [str(k) for k in range(len(chunks[0]))]
        sent = {c: 0 for c in classes}
        for w in range(self.n):
            if w == self.rank:
                continue
            for c, t in zip(classes, chunks[w]):
                sent[c] += t.numel() * t.element_size()
        local = list(zip(chunks[self.rank], recv[self.rank]))

        def copy_local():
            for s, r in local:
                if s.numel() and s.data_ptr() != r.data_ptr():
                    r.copy_(s)
        if self.n == 1:
            return _Hop(copy_local), sent
        k = self._msg()
        if not self.comm_enabled:
            hop = self._local_hop([(c, r) for w in range(self.n) if w != self.rank
                                   for c, r in zip(chunks[w], recv[w])])

            def wait_nc():
                copy_local()
                hop.wait()
            return _Hop(wait_nc), sent
        for w in range(self.n):
            if w != self.rank:
                self.stats.record(self.rank, w, payload_nbytes(chunks[w]))
        if dst is None:
            dst = [recv[self.rank]] * self.n
        hop = self.transport.all_to_all(chunks, recv, dst, self.rank, k)

        def wait():
            copy_local()
            hop.wait()
        return _Hop(wait), sent

    # -- collectives outside the hot path ----------------------------------
    def barrier(self) -> None:
        self.coll.barrier()

    def all_gather_object(self, obj) -> list:
        return self.coll.all_gather_object(obj)

    def all_reduce_sum_(self, t: torch.Tensor) -> None:
        self.coll.all_reduce_sum_(t)

    def synchronize(self, timeout: float | None = None) -> None:
        """Wait for this rank's device work with a deadline: a hop that never
        arrives (a failed peer) raises ``CollectiveTimeout`` instead of
        hanging (cluster.py:149-171 recv deadline)."""
        if self.device.type != "cuda":
            return
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        deadline = time.monotonic() + (self.timeout if timeout is None else timeout)
        while not ev.query():
            if isinstance(self.group, ThreadRank) and self.group.group.first_failure:
                raise ClusterAborted(f"worker {self.rank}: group aborted")
            if time.monotonic() > deadline:
                if self.transport is not None:
                    self.transport.abort()
                raise CollectiveTimeout(f"worker {self.rank}: device work did not complete "
                                        f"within {self.timeout}s (a hop never arrived)")
            time.sleep(2e-4)

    def close(self) -> None:
        if self.transport is not None:
            self.transport.close()
