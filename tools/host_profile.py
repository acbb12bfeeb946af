"""Host-side cost of one LV-XAttn layer step (Python schedulers + C ABI calls),
thread ranks on one GPU: cProfile of rank 0's thread over a few steps at a
small shape where the device work is short.

    python tools/host_profile.py [--n 4] [--skv 65536]
"""
import argparse
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--skv", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.comm import ClusterSpec
    from paper_2502_02406_b200.launch import spawn_ranks
    from paper_2502_02406_b200.strategies import ShardSpec, lvx_backward, lvx_forward
    hq, hkv, sq, d = 32, 8, 2048, 128
    sh = ShardSpec.balanced(sq, a.skv, a.n)
    out = {}

    def body(ctx):
        (qa, qb), (ka, kb) = sh.q_ranges[ctx.rank], sh.kv_ranges[ctx.rank]
        g = torch.Generator(device="cuda").manual_seed(ctx.rank)
        r = lambda *s: (torch.rand(*s, device="cuda", generator=g) - 0.5).bfloat16()  # noqa: E731
        q, k, v, do = r(hq, qb - qa, d), r(hkv, kb - ka, d), r(hkv, kb - ka, d), r(hq, qb - qa, d)

        def step():
            st = lvx_forward(ctx, sh, q, k, v, d ** -0.5)
            lvx_backward(ctx, sh, q, k, v, st, do, d ** -0.5)
        for _ in range(3):
            step()
        ctx.synchronize()
        prof = cProfile.Profile() if ctx.rank == 0 else None
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        for _ in range(a.steps):
            step()
        if prof:
            prof.disable()
        host = (time.perf_counter() - t0) / a.steps
        ctx.synchronize()
        if ctx.rank == 0:
            s = io.StringIO()
            pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(25)
            out["profile"] = s.getvalue()
            out["host_ms_per_step"] = host * 1e3
    spawn_ranks(ClusterSpec(a.n), body, timeout=120)
    print(f"host ms per step (rank 0, profiled): {out['host_ms_per_step']:.3f}")
    print(out["profile"])


if __name__ == "__main__":
    main()
