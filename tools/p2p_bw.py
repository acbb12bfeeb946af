"""Achieved ring-shift bandwidth over NVLink (the transport the schedulers use:
``DeviceContext.shift`` = grouped NCCL send to (r+1)%n / recv from (r-1)%n).

    torchrun --nproc-per-node N tools/p2p_bw.py

Every rank sends and receives one message per shift, concurrently; reports
per-rank bytes / s per direction for message sizes 1 MiB .. 1 GiB (max over
ranks of the CUDA-event time of 10 shifts after warm-up)."""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    os.environ.setdefault("TORCH_NCCL_HIGH_PRIORITY", "1")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    from paper_2502_02406_b200.comm import DeviceContext
    ctx = DeviceContext(rank, world, group=dist.group.WORLD)
    out = {}
    for mib in (1, 4, 16, 64, 256, 1024):
        n = mib * (1 << 20) // 2
        a = torch.empty(n, dtype=torch.bfloat16, device="cuda").fill_(1)
        b = torch.empty_like(a)
        for _ in range(3):
            ctx.shift([a], [b], ["K"])[0].wait()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        iters = 10
        for _ in range(iters):
            ctx.shift([a], [b], ["K"])[0].wait()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3 / iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[f"{mib}MiB"] = {"s_per_shift": t.item(), "GBps_per_direction": 2 * n / t.item() / 1e9}
    if rank == 0:
        print(json.dumps({"world": world, "shift": out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
