"""NVLink hardware counters vs the host byte counters.

    torchrun --nproc-per-node N tools/nvlink_counters.py [--skv 1048576] [--steps 3]

Each rank runs LV-XAttn layer steps (lvx_forward + lvx_backward) on its C2
shard and reads its GPU's NVLink counters through NVML around them, summed
over links: NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / RX (payload, KiB) and
NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / RCV_BYTES.  Rank 0 prints, per rank and
step, the hardware bytes next to the host counter (DeviceContext.stats, the
reference's TransportStats contract) and the GQA closed form
(volumes.bytes_by_worker, as bench.py).
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

DATA_TX, DATA_RX, XMIT, RCV = 138, 139, 202, 204
HQ, HKV, SQ, D = 32, 8, 2048, 128


def nvlink_bytes(handle, links=18):
    import pynvml as n
    out = {}
    for name, fid, unit in (("data_tx", DATA_TX, 1024), ("data_rx", DATA_RX, 1024),
                            ("xmit", XMIT, 1), ("rcv", RCV, 1)):
        vals = n.nvmlDeviceGetFieldValues(handle, [(fid, l) for l in range(links)])
        tot, ok = 0, 0
        for v in vals:
            if v.nvmlReturn == 0:
                tot += int(v.value.ullVal) * unit
                ok += 1
        out[name] = tot if ok else None
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skv", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    import pynvml
    pynvml.nvmlInit()
    idx = torch.cuda.current_device()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = int(vis.split(",")[idx]) if vis else idx
    handle = pynvml.nvmlDeviceGetHandleByIndex(phys)
    from paper_2502_02406_b200 import volumes
    from paper_2502_02406_b200.comm import DeviceContext
    from paper_2502_02406_b200.kernels import default_scale
    from paper_2502_02406_b200.strategies import ShardSpec, lvx_backward, lvx_forward
    shards = ShardSpec.balanced(SQ, a.skv, world)
    (qa, qb), (ka, kb) = shards.q_ranges[rank], shards.kv_ranges[rank]
    g = torch.Generator(device="cuda").manual_seed(100 + rank)

    def u(*shape):
        return (torch.rand(*shape, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    q, do = u(HQ, qb - qa, D), u(HQ, qb - qa, D)
    k, v = u(HKV, kb - ka, D), u(HKV, kb - ka, D)
    ctx = DeviceContext(rank, world, group=dist.group.WORLD)
    scale = default_scale(D)

    def step():
        st = lvx_forward(ctx, shards, q, k, v, scale)
        lvx_backward(ctx, shards, q, k, v, st, do, scale)

    step()   # warm-up (arena mapping)
    torch.cuda.synchronize()
    dist.barrier()
    h0, c0 = nvlink_bytes(handle), ctx.stats.bytes_sent_by(rank)
    for _ in range(a.steps):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    h1, c1 = nvlink_bytes(handle), ctx.stats.bytes_sent_by(rank)
    per = {k2: (None if h0[k2] is None or h1[k2] is None else (h1[k2] - h0[k2]) / a.steps)
           for k2 in h0}
    host = (c1 - c0) / a.steps
    rec = torch.tensor([host] + [per[k2] if per[k2] is not None else -1.0
                                 for k2 in ("data_tx", "data_rx", "xmit", "rcv")],
                       dtype=torch.float64, device="cuda")
    allrec = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(allrec, rec)
    if rank == 0:
        w = volumes.Wire.b200(HQ, HKV, D, 2)
        closed = [volumes.bytes_by_worker("lvx", "forward", shards.q_sizes, shards.kv_sizes, w)[r]
                  + volumes.bytes_by_worker("lvx", "backward", shards.q_sizes, shards.kv_sizes, w)[r]
                  for r in range(world)]
        rows = []
        for r, t in enumerate(allrec):
            hst, tx, rx, xm, rc = t.tolist()
            rows.append({"rank": r, "host_bytes_sent_per_step": hst,
                         "nvlink_data_tx_per_step": tx, "nvlink_data_rx_per_step": rx,
                         "nvlink_xmit_bytes_per_step": xm, "nvlink_rcv_bytes_per_step": rc,
                         "data_tx_over_host": tx / hst if hst > 0 and tx >= 0 else None})
        print(json.dumps({"n": world, "s_kv": a.skv, "steps": a.steps, "per_rank": rows,
                          "closed_form": closed}, indent=1))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
