"""The CPU path at BASELINE configs[0] (C1: Lq 128, Lkv 4096, h 8, d 64, fp32,
world 2): LV-XAttn fwd+bwd through the oracle port of the
reference (numpy; the reference itself is pure Python + numpy, so the port runs
the same BLAS calls) with 1 BLAS thread and with all host threads, best of 5,
next to the GPU path on the same inputs (exact f32 SIMT kernels, n = 1 layer;
run with a GPU for that column).

    python tools/cpu_c1.py
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import lvx_oracle as orc
    Q, K, V, dO = orc.make_inputs(128, 4096, 8, 64, 2502)
    Q, K, V, dO = (t.astype(np.float32) for t in (Q, K, V, dO))
    out = {"config": "C1: Lq 128, Lkv 4096, h 8, d 64, fp32, world 2", "cpu_count": os.cpu_count()}
    for threads in (1, os.cpu_count()):
        with threadpool_limits(limits=threads, user_api="blas"):
            orc.simulate("lvx", Q, K, V, dO, n=2)   # warm
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                orc.simulate("lvx", Q, K, V, dO, n=2)
                ts.append(time.perf_counter() - t0)
        out[f"cpu_lvx_fwd_bwd_ms_{threads}_threads"] = 1e3 * min(ts)
    out["cpu_best_ms"] = min(v for k, v in out.items() if k.startswith("cpu_lvx"))
    try:
        import torch
        if torch.cuda.is_available():
            import paper_2502_02406_b200 as lvx
            q, k, v, g = (torch.from_numpy(t).cuda() for t in (Q, K, V, dO))

            def layer():
                st = lvx.blockwise_attention(q, k, v)
                D = lvx.attention_row_stats(st, g)
                lvx.blockwise_attention_backward(q, k, v, st.L, D, g)
            for _ in range(3):
                layer()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                layer()
            e1.record()
            torch.cuda.synchronize()
            out["gpu_layer_fwd_bwd_ms_n1_f32"] = e0.elapsed_time(e1) / 20
    except Exception as e:   # CPU-only host
        out["gpu"] = f"not run: {e}"
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
