"""K/V recompute overhead of one cross-attention layer (§3.2, the
"< 8 %" claim) on one B200: ca_forward + ca_backward under STORE_KV vs
RECOMPUTE_KV, bf16, CUDA-event timed in 5 interleaved rounds (median; clocks
drift under the power cap), and the activation bytes each keeps.

    python tools/bench_recompute.py [--preset flamingo|llama] [--iters N]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

PRESETS = {  # e, hq, hkv, d, s_q, s_kv   (one rank's shard of the visual tokens)
    "flamingo": (2048, 8, 8, 64, 1024, 65536),      # OpenFlamingo-3b-like, 512K / 8 ranks
    "llama": (4096, 32, 8, 128, 2048, 131072),      # Llama-3-V, 1M / 8 ranks
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="flamingo")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import (ActivationPolicy, CrossAttentionWeights,
                                                 activation_bytes, ca_backward, ca_forward)
    e, hq, hkv, d, sq, skv = PRESETS[a.preset]
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    r = lambda *s, sc=1.0: ((torch.rand(*s, device=dev, generator=g) * 2 - 1) * sc).bfloat16()  # noqa: E731
    ws = 0.5 / e ** 0.5
    w = CrossAttentionWeights(r(e, hq * d, sc=ws), r(e, hkv * d, sc=ws), r(e, hkv * d, sc=ws),
                              r(hq * d, e, sc=ws), hq, hkv)
    x, y, go = r(sq, e), r(skv, e), r(sq, e)
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(sq, skv, 1)
    out = {"preset": a.preset, "dims": [e, hq, hkv, d, sq, skv]}
    pols = (ActivationPolicy.STORE_KV, ActivationPolicy.RECOMPUTE_KV)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    times = {p: {"fwd": [], "bwd": [], "step": []} for p in pols}
    saved_of = {}
    for p in pols:   # warm-up both
        for _ in range(2):
            o, sv = ca_forward(ctx, sh, x, y, w, p)
            ca_backward(ctx, sh, go, sv, y, w)
    torch.cuda.synchronize()
    # interleaved rounds (clocks drift under the power cap): median per policy
    for _ in range(5):
        for p in pols:
            tf = tb = 0.0
            for _ in range(a.iters):
                e0, e1, e2 = ev(), ev(), ev()
                e0.record()
                o, sv = ca_forward(ctx, sh, x, y, w, p)
                e1.record()
                ca_backward(ctx, sh, go, sv, y, w)
                e2.record()
                torch.cuda.synchronize()
                tf += e0.elapsed_time(e1)
                tb += e1.elapsed_time(e2)
                saved_of[p] = sv
            times[p]["fwd"].append(tf / a.iters)
            times[p]["bwd"].append(tb / a.iters)
            times[p]["step"].append((tf + tb) / a.iters)
    med = lambda xs: sorted(xs)[len(xs) // 2]  # noqa: E731
    for p in pols:
        out[p.value] = {"ms": med(times[p]["step"]), "fwd_ms": med(times[p]["fwd"]),
                        "bwd_ms": med(times[p]["bwd"]),
                        "activation_bytes": activation_bytes(saved_of[p])}
    out["recompute_overhead"] = out["recompute"]["ms"] / out["store"]["ms"] - 1.0
    out["activation_saving_bytes"] = out["store"]["activation_bytes"] - \
        out["recompute"]["activation_bytes"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
