"""Rank launch for run_distributed without torchrun.

``spawn_run`` is the single-call form of the reference's
``run_distributed(..., spec=ClusterSpec(n))`` (strategies.py:454-551) with
one process per GPU: n processes on n local GPUs, rendezvous on 127.0.0.1,
copy-engine ring hops between them, rank 0's gathered result returned.

``spawn_ranks`` is the reference's ``spawn_cluster`` (cluster.py:300-335):
``body(ctx)`` runs on n thread ranks of this process that share one device,
each on its own CUDA stream (copy-engine hops into each other's arenas on a
GPU; mailboxes on a host device).  It is how the n-rank protocols run on a
single GPU.

Both honour the timeout contract (cluster.py:25-26, :149-220): every wait on
a peer is bounded by ``timeout`` (else $LVX_TIMEOUT_SECS, else 30 s); the
first failing rank aborts the others and is raised as ``WorkerFailed``
naming it, with the rank's exception (``CollectiveTimeout`` for a hop that
never arrived) as the cause.
"""
from __future__ import annotations

import datetime
import os
import queue as _queue
import shutil
import socket
import tempfile
import threading
import time
import traceback
from dataclasses import dataclass

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from . import _lib
from .comm import (ClusterAborted, ClusterSpec, CollectiveTimeout, DeviceContext, PeerTransport,
                   ThreadGroup, TransportStats, WorkerFailed, resolve_timeout)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---------------------------------------------------------------------------
# thread ranks (cluster.py:300-335)
# ---------------------------------------------------------------------------

@dataclass
class RanksResult:
    results: list
    stats: TransportStats


def spawn_ranks(spec: ClusterSpec, body, timeout: float | None = None, device=None,
                ops_factory=None) -> RanksResult:
    """Run ``body(ctx)`` on ``spec.n`` thread ranks sharing ``device``
    (default: the current GPU); block until all finish; return their results
    in rank order and the merged transport counters.  The first failure
    aborts the group (blocked waits on the host and on the device are
    released) and is re-raised as ``WorkerFailed(rank, exc)``."""
    n = spec.n
    tmo = resolve_timeout(timeout)
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("spawn_ranks needs a CUDA device or an explicit host device")
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    group = ThreadGroup(n, tmo)
    results: list = [None] * n
    ctxs: list = [None] * n

    def run(rank: int) -> None:
        own = None
        try:
            ops = ops_factory() if ops_factory is not None else None
            if device.type == "cuda":
                torch.cuda.set_device(device)
                # a stream of its own: torch's pooled streams repeat after 32,
                # and two ranks on one stream would share its workspaces
                own = _lib.OwnStream(device)
                with torch.cuda.stream(own.stream):
                    _run_one(rank, ops, own.stream)
            else:
                _run_one(rank, ops, None)
        except BaseException as exc:   # surfaced as WorkerFailed below
            group.fail(rank, exc)      # releases every rank's stream-side waits
        finally:
            if own is not None:
                try:
                    own.close()
                except Exception:      # noqa: BLE001 - a failed rank's stream
                    pass

    def _run_one(rank, ops, stream):
        ctx = DeviceContext(rank, n, group=group.rank(rank) if n > 1 else None, device=device,
                            ops=ops, timeout=tmo)
        ctxs[rank] = ctx
        results[rank] = body(ctx)
        ctx.synchronize()
        if isinstance(ctx.transport, PeerTransport):
            # no rank frees its arena while a peer may still write into it; the
            # deadline is longer than a hop's so a peer's own timeout (the
            # root cause) is the failure reported
            ctx.coll.barrier(timeout=2 * tmo + 5)
        ctx.close()

    if n == 1:
        run(0)
    else:
        threads = [threading.Thread(target=run, args=(r,), name=f"lvx-rank-{r}", daemon=True)
                   for r in range(n)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if group.first_failure is not None:
        rank, exc = group.first_failure
        if device.type == "cuda":
            _drain(device)
        raise WorkerFailed(rank, exc) from exc
    stats = TransportStats()
    for c in ctxs:
        if c is not None:
            stats.merge(c.stats)
    return RanksResult(results=results, stats=stats)


def _drain(device) -> None:
    """After an abort every stream-side wait has been released (the flags
    were overwritten), so the device drains; a kernel error surfaces here."""
    try:
        torch.cuda.synchronize(device)
    except RuntimeError:
        pass


# ---------------------------------------------------------------------------
# one process per GPU
# ---------------------------------------------------------------------------

def _worker(rank, n, store_path, args, q):
    try:
        torch.cuda.set_device(rank)
        strategy, Q, K, V, dO, scale, tile_rows, timeout = args
        # file rendezvous: no TCP port to collide with another run's
        dist.init_process_group("nccl", init_method=f"file://{store_path}", rank=rank,
                                world_size=n,
                                device_id=torch.device("cuda", rank),
                                timeout=datetime.timedelta(seconds=max(timeout, 1.0)))
        from .strategies import run_distributed
        res = run_distributed(strategy, Q, K, V, dO, ClusterSpec(n), scale, tile_rows,
                              timeout, group=dist.group.WORLD)
        if rank == 0:
            q.put(("ok", rank, res))
        else:
            q.put(("done", rank, None))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # noqa: BLE001 - reported to the parent
        q.put(("err", rank, (type(exc).__name__, str(exc), traceback.format_exc())))


_KNOWN = {c.__name__: c for c in (CollectiveTimeout, ClusterAborted, ValueError, RuntimeError,
                                   TypeError)}


def _rebuild(name: str, msg: str, tb: str) -> BaseException:
    """A rank's exception as seen by the parent: same class when it is one of
    the protocol / argument errors, its traceback attached."""
    exc = _KNOWN.get(name, RuntimeError)(msg if name in _KNOWN else f"{name}: {msg}")
    exc.remote_traceback = tb
    return exc


def spawn_run(strategy, Q, K, V, dO, n, scale, tile_rows, timeout: float | None = None):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        raise RuntimeError(f"run_distributed with n={n} processes needs {n} local GPUs "
                           f"(found {have}); use ranks='threads' or torchrun")
    tmo = resolve_timeout(timeout)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    rdzv_dir = tempfile.mkdtemp(prefix="lvx_rdzv_")
    store = os.path.join(rdzv_dir, "store")
    procs = [ctx.Process(target=_worker, args=(r, n, store, (strategy, Q, K, V, dO, scale,
                                                             tile_rows, tmo), q))
             for r in range(n)]
    try:
        return _collect(procs, q, n, tmo)
    finally:
        shutil.rmtree(rdzv_dir, ignore_errors=True)


def _collect(procs, q, n, tmo):
    for p in procs:
        p.start()
    # process start-up + CUDA init + the run itself: the per-wait timeout
    # bounds each hop inside the ranks; the parent only needs to notice a
    # rank that died without reporting
    result, failure, pending = None, None, set(range(n))
    while pending and failure is None:
        try:
            kind, rank, payload = q.get(timeout=1.0)
        except _queue.Empty:
            dead = [r for r in pending if not procs[r].is_alive() and procs[r].exitcode]
            if dead:
                failure = (dead[0], RuntimeError(f"exit code {procs[dead[0]].exitcode}"))
            continue
        pending.discard(rank)
        if kind == "err":
            failure = (rank, _rebuild(*payload))
        elif kind == "ok":
            result = payload
    if failure is not None:
        for p in procs:                # abort the survivors (cluster.py:160-166)
            if p.is_alive():
                p.terminate()
        for p in procs:
            p.join(timeout=10)
        raise WorkerFailed(failure[0], failure[1]) from failure[1]
    for p in procs:
        p.join(timeout=tmo + 30)
        if p.is_alive():
            p.terminate()
    return result


__all__ = ["spawn_ranks", "spawn_run", "RanksResult", "free_port", "CollectiveTimeout",
           "ClusterAborted"]
