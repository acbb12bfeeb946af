"""HBM-bound kernels of the path: achieved GB/s vs the measured
copy bandwidth (MEASURED_PEAKS.json hbm_gbs).

    python tools/bench_hbm_kernels.py

Each launch is timed alone with CUDA events after a 512 MB READ that flushes
L2 with clean lines (a write flush would leave ~126 MB of dirty lines for the
timed kernel to write back), so the inputs come from HBM.  Algorithmic bytes per §8(d):
  merge_states   rows*h*(3d+3)*4   (read O_a, O_b, L_a, L_b; write O, L; fp32)
  row_stats      rows*h*(d*4 + d*2 + 4)   (O fp32, dO bf16, D fp32)
  fwd_finish     splits*rows*h*(d+1)*4 + prior rows*h*(d+1)*4 + out rows*h*(d+1)*4
  dq_finish      splits*rows*h*d*4 + dQ read+write rows*h*d*4*2 (accumulate)
Shapes: C2 per GPU at n=1 (hq 32 x 2048 rows, d 128) and C3 (hq 28 x 5514 rows).
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    from paper_2502_02406_b200 import kernels as K
    dev = torch.device("cuda")
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)   # 512 MB
    sink = torch.empty((), device=dev)

    def timed(fn, iters=20):
        fn()
        ts = []
        for _ in range(iters):
            torch.sum(flush, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]   # median, ms

    out = {"peak_hbm_GBps": peak,
           "method": "median of 20 single launches, L2 flushed by a 512 MB read before each"}
    for name, (h, rows, d) in {"C2_n1": (32, 2048, 128), "C3": (28, 5514, 128)}.items():
        r = {}
        f32 = dict(device=dev, dtype=torch.float32)
        oa, ob = torch.randn(h, rows, d, **f32), torch.randn(h, rows, d, **f32)
        la, lb = torch.randn(h, rows, **f32), torch.randn(h, rows, **f32)
        o, l = torch.empty_like(oa), torch.empty_like(la)
        ms = timed(lambda: K.merge_into(oa, la, ob, lb, o, l))
        b = rows * h * (3 * d + 3) * 4
        r["merge_states"] = {"ms": ms, "bytes": b, "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / peak}
        g = torch.randn(h, rows, d, device=dev).bfloat16()
        D = torch.empty(h, rows, **f32)
        ms = timed(lambda: K.row_stats_into(oa, g, D))
        b = rows * h * (d * 4 + d * 2 + 4)
        r["row_stats"] = {"ms": ms, "bytes": b, "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / peak}
        # split combine + prior merge (fwd_finish) and the dQ split sum, at the
        # launch shapes the bench uses (Lkv = 1M rows of K/V for C2)
        q = torch.randn(h, rows, d, device=dev).bfloat16()
        kv_rows = (1 << 20) if name == "C2_n1" else (1 << 18)
        k = torch.empty(h // (4 if name == "C2_n1" else 7), kv_rows, d, device=dev,
                        dtype=torch.bfloat16).uniform_(-1, 1)
        ws = K.workspace(K.fwd_workspace_bytes(q, k))
        K.fwd_partial(q, k, k, d ** -0.5, ws)
        # splits from the REQUESTED workspace (the cached buffer may be larger)
        splits = (K.fwd_workspace_bytes(q, k) // (rows * h * 4)) // (d + 1)
        ms = timed(lambda: K.fwd_finish(q, k, ws, o, l, ob, lb))
        b = (splits + 2) * rows * h * (d + 1) * 4
        r["fwd_finish"] = {"ms": ms, "splits": splits, "bytes": b, "GBps": b / ms / 1e6,
                           "frac": b / ms / 1e6 / peak}
        wsb = K.workspace(K.bwd_ws_bytes(q, k), dev, slot=3)
        Lq = torch.zeros(h, rows, **f32)
        K.bwd_dq_partial(q, k, k, Lq, D, q, d ** -0.5, wsb)
        dq = torch.zeros(h, rows, d, **f32)
        dq_splits = max(1, (K.bwd_ws_bytes(q, k) // 4) // (rows * h * d))   # upper bound
        ms = timed(lambda: K.bwd_dq_finish(q, k, wsb, dq, True))
        b = (dq_splits + 2) * rows * h * d * 4
        r["dq_finish"] = {"ms": ms, "splits_upper_bound": dq_splits, "bytes": b,
                          "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / peak}
        out[name] = r
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
