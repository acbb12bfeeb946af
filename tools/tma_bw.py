"""L2 -> SMEM TMA throughput, unicast vs cluster-2 multicast (tools/tma_bw.cu).

    nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC \\
         -o build/tma_bw.so tools/tma_bw.cu -cudart static
    python tools/tma_bw.py
"""
import ctypes
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent


def main():
    lib = ctypes.CDLL(str(ROOT / "build" / "tma_bw.so"))
    ntiles = 8192   # 512 MB of (tile A | tile B) pairs; 8 CTA groups stream distinct sequences
    buf = torch.empty(ntiles * 256, 128, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    clk = torch.zeros(1, dtype=torch.int64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {}
    for mode, name in ((0, "unicast"), (1, "multicast_pair")):
        for steps in (200, 2000):
            args = (ctypes.c_void_p(buf.data_ptr()), ntiles, sms, steps, mode,
                    ctypes.c_void_p(clk.data_ptr()), ctypes.c_void_p(0))
            for _ in range(2):
                assert lib.tma_bw_run(*args) == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.tma_bw_run(*args) == 0
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            landed = sms * steps * 65536   # bytes landed in SMEM (all CTAs)
            out[f"{name}_steps{steps}"] = {
                "ms": ms, "smem_TBps": landed / ms / 1e9,
                "bytes_per_sm_per_clk": 65536 * steps / int(clk.item()),
                "l2_read_TBps": landed / (2 if mode else 1) / ms / 1e9}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
