"""Copy-engine transport probe (2 ranks, torchrun): what one hop of the
ring costs on this box, by message size.

    torchrun --nproc-per-node 2 tools/ce_probe.py

* ping-pong latency of a flag-only hop (cuStreamWriteValue32 into the peer's
  arena, cuStreamWaitValue32 on the own one), rank 0 <-> rank 1;
* one-way bandwidth of a put of S bytes + flag, the data split over k copy
  streams (k = 1, 2, 4, 8), each stream its own cudaMemcpyAsync of S/k;
* the same put issued as ONE cudaMemcpyAsync after the peer's buffer was
  touched (warm mapping).
Each timing is the CUDA-event time on rank 0 of `iters` back-to-back
transfers (the receiver acknowledges each, so they do not pile up), median
of 3 repeats.  JSON on rank 0.
"""
import ctypes
import json
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 2
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2502_02406_b200 import _lib
    lib = _lib.load()
    peer = 1 - rank
    cap = 256 << 20
    flag_bytes = 4096
    m = ctypes.c_void_p()
    _lib.check("create", lib.lvx_peer_create(cap + flag_bytes, rank, 2, ctypes.byref(m)))
    hb = int(lib.lvx_peer_handle_bytes())
    buf = (ctypes.c_char * hb)()
    _lib.check("export", lib.lvx_peer_export(m, buf))
    objs = [None, None]
    dist.all_gather_object(objs, bytes(buf))
    _lib.check("open", lib.lvx_peer_open(m, peer, (ctypes.c_char * hb).from_buffer_copy(objs[peer])))
    src = torch.ones(cap // 2, dtype=torch.bfloat16, device=dev)
    streams = [_lib.OwnStream(dev) for _ in range(8)]
    main_s = streams[0].stream
    FLAG_DATA, FLAG_ACK = cap, cap + 64
    seq = [0]

    def hop(nbytes, k):
        """rank 0 -> rank 1: nbytes in k chunks on k streams, then a flag;
        rank 1 waits, acknowledges with a flag back; rank 0 waits for it."""
        seq[0] += 1
        v = seq[0]
        if rank == 0:
            ev = torch.cuda.Event()
            ev.record(main_s)
            chunk = (nbytes + k - 1) // k
            done = []
            for j in range(k):
                a, b = j * chunk, min(nbytes, (j + 1) * chunk)
                if b <= a:
                    continue
                s = streams[j].stream
                s.wait_event(ev)
                _lib.check("put", lib.lvx_peer_put(m, peer, a, 0, ctypes.c_void_p(src.data_ptr() + a),
                                                   0, b - a, 1, ctypes.c_void_p(s.cuda_stream)))
                e = torch.cuda.Event()
                e.record(s)
                done.append(e)
            for e in done:
                main_s.wait_event(e)
            _lib.check("signal", lib.lvx_peer_signal(m, peer, FLAG_DATA, v, ctypes.c_void_p(main_s.cuda_stream)))
            _lib.check("wait", lib.lvx_peer_wait(m, FLAG_ACK, v, ctypes.c_void_p(main_s.cuda_stream)))
        else:
            _lib.check("wait", lib.lvx_peer_wait(m, FLAG_DATA, v, ctypes.c_void_p(main_s.cuda_stream)))
            _lib.check("signal", lib.lvx_peer_signal(m, peer, FLAG_ACK, v, ctypes.c_void_p(main_s.cuda_stream)))

    def timed(nbytes, k, iters):
        res = []
        for _ in range(3):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            for _ in range(iters):
                hop(nbytes, k)
            e1.record(main_s)
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / iters * 1e-3)
        return statistics.median(res)

    out = {"flag_roundtrip_us": timed(0, 1, 200) * 1e6}
    for size in (64 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20):
        row = {}
        for k in (1, 2, 4, 8):
            t = timed(size, k, 20 if size >= (64 << 20) else 50)
            row[f"k{k}"] = {"us": t * 1e6, "GBps": size / t / 1e9}
        out[f"{size >> 10}KiB"] = row
    if rank == 0:
        print(json.dumps(out), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    lib.lvx_peer_destroy(m)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
