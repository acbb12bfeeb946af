"""Per-call timing of the ring schedulers (torchrun, C2 shapes at N ranks):
lvx fwd / bwd, ring fwd / bwd (overlapped) / bwd (reference order)."""
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.strategies import (ring_backward, ring_backward_reference_schedule,
                                                  ring_forward, lvx_forward, lvx_backward)
    skv = int(os.environ.get("SKV", 1 << 20))
    hq, hkv, sq, d = 32, 8, 2048, 128
    sh = lvx.ShardSpec.balanced(sq, skv, world)
    (qa, qb), (ka, kb) = sh.q_ranges[rank], sh.kv_ranges[rank]
    g = torch.Generator(device=dev).manual_seed(rank)
    r = lambda *s: (torch.rand(*s, device=dev, generator=g) - 0.5).bfloat16()  # noqa: E731
    q, k, v, do = r(hq, qb - qa, d), r(hkv, kb - ka, d), r(hkv, kb - ka, d), r(hq, qb - qa, d)
    ctx = lvx.DeviceContext(rank, world, group=dist.group.WORLD, device=dev)
    scale = d ** -0.5

    def t(fn, reps=3):
        out = []
        for _ in range(reps):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            res = fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(round(e0.elapsed_time(e1), 2))
        return out, res

    for name, f, b in (("lvx", lvx_forward, lvx_backward), ("ring", ring_forward, ring_backward),
                       ("ring_ref", ring_forward, ring_backward_reference_schedule)):
        for _ in range(2):
            st = f(ctx, sh, q, k, v, scale)
            b(ctx, sh, q, k, v, st, do, scale)
        tf, st = t(lambda: f(ctx, sh, q, k, v, scale))
        tb, _ = t(lambda: b(ctx, sh, q, k, v, st, do, scale))
        if rank == 0:
            print(name, "fwd ms", tf, "bwd ms", tb, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
