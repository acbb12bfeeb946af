"""Host-side cost of the C4 layer-stack step (ca_forward / ca_backward over
4 layers sharing y, K/V recompute) on one GPU at a small visual-token count,
where the device work is short: cProfile of a few eager steps.

    python tools/host_profile_layers.py [--skv 65536] [--steps 5]
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
    ap.add_argument("--skv", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import (ActivationPolicy, CrossAttentionWeights,
                                                 VisualGradSink, ca_backward, ca_forward)
    dev = torch.device("cuda")
    sq, hq, hkv, d, e, nl = 1024, 8, 8, 64, 2048, 4
    g = torch.Generator(device=dev).manual_seed(1)

    def r(*s, sc=1.0):
        return ((torch.rand(*s, device=dev, generator=g) * 2 - 1) * sc).bfloat16()
    ws = 0.5 / e ** 0.5
    layers = [CrossAttentionWeights(r(e, hq * d, sc=ws), r(e, hkv * d, sc=ws), r(e, hkv * d, sc=ws),
                                    r(hq * d, e, sc=ws), hq, hkv) for _ in range(nl)]
    x0, y, go = r(sq, e), r(a.skv, e), r(sq, e)
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(sq, a.skv, 1)

    def step():
        x, saved = x0, []
        for w in layers:
            x, sv = ca_forward(ctx, sh, x, y, w, ActivationPolicy.RECOMPUTE_KV)
            saved.append(sv)
        sink, gx = VisualGradSink(y, [w.kv_weight().shape[1] for w in layers]), go
        for w, sv in zip(reversed(layers), reversed(saved)):
            gx = ca_backward(ctx, sh, gx, sv, y, w, dy_sink=sink).d_x
        return gx, sink.finish(ctx, dtype=y.dtype)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / a.steps
    prof = cProfile.Profile()
    t0 = time.perf_counter()
    prof.enable()
    for _ in range(a.steps):
        step()
    prof.disable()
    host_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    torch.cuda.synchronize()
    s = io.StringIO()
    pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(30)
    print(f"device ms per step {dev_ms:.3f}; host ms per step (profiled) {host_ms:.3f}")
    print(s.getvalue())


if __name__ == "__main__":
    main()
