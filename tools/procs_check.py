"""n PROCESS ranks over the copy-engine transport when there are fewer GPUs
than ranks (e.g. the 8-rank path on a 1- or 4-GPU box): rank r runs on GPU
r % ngpus, the ring hops go through CUDA IPC into the peers' arenas (same
device or not), and a gloo group carries only setup and barriers (NCCL
refuses two ranks on one GPU).  Each strategy's gathered O, L, dQ, dK, dV are
compared with the single-rank run of the same inputs on rank 0.

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/procs_check.py
Prints one JSON line (rank 0); exit code 1 on a mismatch.
"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)) % ngpu)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.strategies import run_rank
    hq, hkv, sq, skv, d = 32, 8, 1000, 40_000, 128      # ragged shards on purpose
    g = torch.Generator(device=dev).manual_seed(8)
    r = lambda *s: (torch.rand(*s, device=dev, generator=g) * 2 - 1).bfloat16()  # noqa: E731
    Q, K, V, dO = r(hq, sq, d), r(hkv, skv, d), r(hkv, skv, d), r(hq, sq, d)   # same on every rank
    sh = lvx.ShardSpec.balanced(sq, skv, n)
    (qa, qb), (ka, kb) = sh.q_ranges[rank], sh.kv_ranges[rank]
    ctx = lvx.DeviceContext(rank, n, group=dist.group.WORLD, device=dev)
    out = {"n": n, "gpus": ngpu, "errors": {}}
    ok = True
    ref = None
    if rank == 0:
        c1 = lvx.DeviceContext(0, 1, device=dev)
        st, gr, _, _ = run_rank("lvx", c1, lvx.ShardSpec.balanced(sq, skv, 1), Q, K, V, dO)
        ref = {"O": st.O, "L": st.L, "dQ": gr[0], "dK": gr[1], "dV": gr[2]}
    for strategy in ("lvx", "ring", "head"):
        if strategy == "head" and hq % n:
            continue
        st, gr, _, _ = run_rank(strategy, ctx, sh, Q[:, qa:qb], K[:, ka:kb], V[:, ka:kb],
                                dO[:, qa:qb])
        ctx.synchronize()
        parts = [None] * n
        dist.all_gather_object(parts, {k: t.float().cpu() for k, t in
                                       (("O", st.O), ("L", st.L), ("dQ", gr[0]), ("dK", gr[1]),
                                        ("dV", gr[2]))})
        if rank == 0:
            errs = {}
            for key, dim in (("O", 1), ("L", 1), ("dQ", 1), ("dK", 1), ("dV", 1)):
                got = torch.cat([p[key] for p in parts], dim=dim)
                want = ref[key].float().cpu()
                errs[key] = float((got - want).abs().max() / want.abs().max().clamp_min(1e-30))
            out["errors"][strategy] = errs
            # same bf16 kernels, different split / merge order: within bf16 rounding
            ok &= max(errs.values()) <= 1e-2
        dist.barrier()
    if rank == 0:
        out["pass"] = bool(ok)
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if (rank != 0 or ok) else 1)


if __name__ == "__main__":
    main()
