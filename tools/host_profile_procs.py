"""Host-side cost of one LV-XAttn layer step over PROCESS ranks (one per GPU,
copy-engine transport), the bench's setting: cProfile of rank 0 at a small
shard where the device work is short.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/host_profile_procs.py [--skv 262144]
"""
import argparse
import cProfile
import io
import os
import pstats
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skv", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.strategies import lvx_backward, lvx_forward
    hq, hkv, sq, d = 32, 8, 2048, 128
    sh = lvx.ShardSpec.balanced(sq, a.skv, n)
    (qa, qb), (ka, kb) = sh.q_ranges[rank], sh.kv_ranges[rank]
    g = torch.Generator(device=dev).manual_seed(rank)
    r = lambda *s: (torch.rand(*s, device=dev, generator=g) - 0.5).bfloat16()  # noqa: E731
    q, k, v, do = r(hq, qb - qa, d), r(hkv, kb - ka, d), r(hkv, kb - ka, d), r(hq, qb - qa, d)
    ctx = lvx.DeviceContext(rank, n, group=dist.group.WORLD, device=dev)

    def step():
        st = lvx_forward(ctx, sh, q, k, v, d ** -0.5)
        lvx_backward(ctx, sh, q, k, v, st, do, d ** -0.5)
    for _ in range(3):
        step()
    ctx.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    ctx.synchronize()
    dev_ms = e0.elapsed_time(e1) / a.steps
    dist.barrier()
    prof = cProfile.Profile() if rank == 0 else None
    t0 = time.perf_counter()
    if prof:
        prof.enable()
    for _ in range(a.steps):
        step()
    if prof:
        prof.disable()
    host_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    ctx.synchronize()
    dist.barrier()
    if rank == 0:
        s = io.StringIO()
        pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(30)
        print(f"n {n}, Lkv {a.skv}: device ms per step {dev_ms:.3f}; host ms per step "
              f"(profiled) {host_ms:.3f}")
        print(s.getvalue())
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
