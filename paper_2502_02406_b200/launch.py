"""Process launch for run_distributed without torchrun: one process per GPU.

``spawn_run`` is the single-call form of the reference's
``run_distributed(..., spec=ClusterSpec(n))`` (strategies.py:454-551), where
the reference spawned n threads (cluster.py:309-335).  Here it spawns n
processes on n local GPUs, rendezvous on 127.0.0.1, NCCL, and returns rank
0's gathered result.  A failing rank surfaces as ``WorkerFailed`` naming it.
"""
from __future__ import annotations

import os
import socket
import traceback

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from .comm import ClusterSpec, WorkerFailed


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, n, port, args, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        os.environ.setdefault("TORCH_NCCL_HIGH_PRIORITY", "1")
        dist.init_process_group("nccl", rank=rank, world_size=n,
                                device_id=torch.device("cuda", rank))
        from .strategies import run_distributed
        strategy, Q, K, V, dO, scale, tile_rows = args
        res = run_distributed(strategy, Q, K, V, dO, ClusterSpec(n), scale, tile_rows)
        if rank == 0:
            q.put(("ok", res))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # noqa: BLE001 - reported to the parent
        q.put(("err", rank, f"{exc!r}\n{traceback.format_exc()}"))


def spawn_run(strategy, Q, K, V, dO, n, scale, tile_rows):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        raise RuntimeError(f"run_distributed with n={n} needs {n} local GPUs (found {have}); "
                           "or launch one process per GPU with torchrun")
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, n, port, (strategy, Q, K, V, dO, scale,
                                                            tile_rows), q))
             for r in range(n)]
    for p in procs:
        p.start()
    msg = q.get()
    for p in procs:
        p.join()
    if msg[0] == "err":
        raise WorkerFailed(msg[1], RuntimeError(msg[2]))
    return msg[1]
