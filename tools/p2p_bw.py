"""Achieved ring-shift bandwidth over NVLink through the transport the
schedulers use: ``DeviceContext.shift`` = a copy-engine put into the
successor's arena + a stream-ordered flag (comm.PeerTransport).

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
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    from paper_2502_02406_b200.comm import DeviceContext
    ctx = DeviceContext(rank, world, group=dist.group.WORLD)
    out = {}
    for mib in (1, 4, 16, 64, 256, 1024):
        n = mib * (1 << 20) // 2
        a = torch.empty((1, n, 1), dtype=torch.bfloat16, device="cuda").fill_(1)
        iters = 10

        def shifts(k):
            # one scheduler call = k shifts into k receive slots of the arena
            with ctx.call() as call:
                slots = call.alloc({"r": (k, [("K", n, torch.bfloat16)])})["r"]
                for j in range(k):
                    hop, _ = ctx.shift([a], [slots[j]["K"].view(1, n, 1)], ["K"])
                    hop.wait()
        shifts(iters)   # warm-up with the timed call's layout (the arena is sized once)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        shifts(iters)
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
