"""Full-scale multi-GPU parity (SURVEY.md §8(c) iii): the C2 workload (Lq 2048,
hq 32 / hkv 8, d 128, Lkv 1,048,576, bf16) through the n-way LV-XAttn ring vs
the single-GPU computation on the SAME inputs.

    torchrun --nproc-per-node N tools/fullscale_multi_check.py

Every rank draws the full inputs from one seed on its own GPU, runs the n-way
ring on its shard AND the n = 1 layer on the full inputs, and compares its own
query rows (O, L, dQ) and KV rows (dK, dV); rank 0 prints the max-normalised
differences over ranks as JSON.  Both sides are bf16 tensor-core results that
differ only in split / merge order, so they agree to bf16 rounding."""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

HQ, HKV, SQ, SKV, D = 32, 8, 2048, 1 << 20, 128


def max_norm(a: torch.Tensor, b: torch.Tensor) -> float:
    a, b = a.double(), b.double()
    den = b.abs().max().item()
    return (a - b).abs().max().item() / (den if den > 0 else 1.0)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    from paper_2502_02406_b200.comm import DeviceContext
    from paper_2502_02406_b200.kernels import default_scale
    from paper_2502_02406_b200.strategies import ShardSpec, lvx_backward, lvx_forward
    g = torch.Generator(device="cuda").manual_seed(2502)

    def u(*shape):
        return (torch.rand(*shape, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    q, k, v, do = u(HQ, SQ, D), u(HKV, SKV, D), u(HKV, SKV, D), u(HQ, SQ, D)
    scale = default_scale(D)
    # n-way ring on this rank's shard
    shards = ShardSpec.balanced(SQ, SKV, world)
    (qa, qb), (ka, kb) = shards.q_ranges[rank], shards.kv_ranges[rank]
    ctx = DeviceContext(rank, world, group=dist.group.WORLD)
    st = lvx_forward(ctx, shards, q[:, qa:qb], k[:, ka:kb], v[:, ka:kb], scale)
    dq, dk, dv = lvx_backward(ctx, shards, q[:, qa:qb], k[:, ka:kb], v[:, ka:kb], st,
                              do[:, qa:qb], scale)
    torch.cuda.synchronize()
    # the single-GPU layer on the full inputs
    one = ShardSpec.balanced(SQ, SKV, 1)
    ctx1 = DeviceContext(0, 1)
    st1 = lvx_forward(ctx1, one, q, k, v, scale)
    dq1, dk1, dv1 = lvx_backward(ctx1, one, q, k, v, st1, do, scale)
    torch.cuda.synchronize()
    errs = torch.tensor([max_norm(st.O, st1.O[:, qa:qb]), max_norm(st.L, st1.L[:, qa:qb]),
                         max_norm(dq, dq1[:, qa:qb]), max_norm(dk, dk1[:, ka:kb]),
                         max_norm(dv, dv1[:, ka:kb])], device="cuda", dtype=torch.float64)
    dist.all_reduce(errs, op=dist.ReduceOp.MAX)
    if rank == 0:
        e = dict(zip(("O", "L", "dQ", "dK", "dV"), errs.tolist()))
        print(json.dumps({"check": "C2 full scale, n-way ring vs n=1, same inputs", "n": world,
                          "max_norm_error": e, "tolerance": 1e-2,
                          "pass": max(e.values()) <= 1e-2}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
