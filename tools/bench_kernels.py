"""Kernel-level timing of the tcgen05 forward/backward on one B200 (dev tool).

    python tools/bench_kernels.py [--shape c2round|c2full|c4round] [--iters N]

Times fwd_partial, fwd_finish and bwd with CUDA events on the launching
stream after warm-up and prints TFLOP/s against MEASURED_PEAKS.json."""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SHAPES = {  # hq, hkv, rows_q, rows_kv, d
    "c2round": (32, 8, 256, 131072, 128),     # Llama-3-V, one rank-round at n=8
    "c2full": (32, 8, 2048, 1 << 20, 128),    # Llama-3-V, n=1
    "c4round": (8, 8, 128, 65536, 64),        # OpenFlamingo, n=8
    "c3round": (28, 4, 690, 65536, 128),      # Owl3 256K, n=4 (ragged rows)
    "c2gath": (32, 8, 2048, 131072, 128),     # Llama-3-V n=8: batched dK/dV over all blocks
    "c2gath_q2": (32, 8, 4096, 65536, 128),   # same work, 2x query steps per dK/dV CTA
    "c4gath": (8, 8, 1024, 65536, 64),        # OpenFlamingo n=8: the batched dK/dV launch
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="c2round")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--bf16-grads", action="store_true", help="dK/dV in bf16 (the lvx path)")
    a = ap.parse_args()
    from paper_2502_02406_b200 import kernels as K
    hq, hkv, sq, skv, d = SHAPES[a.shape]
    dev = torch.device("cuda")
    q = (torch.rand(hq, sq, d, device=dev) * 2 - 1).bfloat16()
    k = (torch.rand(hkv, skv, d, device=dev) * 2 - 1).bfloat16()
    v = (torch.rand(hkv, skv, d, device=dev) * 2 - 1).bfloat16()
    g = (torch.rand(hq, sq, d, device=dev) * 2 - 1).bfloat16()
    O = torch.empty(hq, sq, d, device=dev)
    L = torch.empty(hq, sq, device=dev)
    ws = K.workspace(K.fwd_workspace_bytes(q, k))
    scale = d ** -0.5
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {"bf16_tflops": 1590, "hbm_gbs": 6650}

    def t(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters

    res = {"shape": a.shape, "dims": [hq, hkv, sq, skv, d]}
    ff = 4.0 * sq * skv * hq * d
    ms = t(lambda: K.fwd_partial(q, k, v, scale, ws))
    res["fwd_partial_ms"] = ms
    res["fwd_tflops"] = ff / ms / 1e9
    res["fwd_frac_of_peak"] = res["fwd_tflops"] / peaks["bf16_tflops"]
    ms2 = t(lambda: K.fwd_finish(q, k, ws, O, L, O, L))
    res["fwd_finish_ms"] = ms2
    if a.bwd:
        D = torch.zeros(hq, sq, device=dev)
        dq = torch.zeros(hq, sq, d, device=dev)
        dk = torch.zeros(hkv, skv, d, device=dev)
        dv = torch.zeros(hkv, skv, d, device=dev)
        gdt = torch.bfloat16 if a.bf16_grads else torch.float32
        dkg = torch.zeros(hkv, skv, d, device=dev, dtype=gdt)
        dvg = torch.zeros(hkv, skv, d, device=dev, dtype=gdt)
        bf = 10.0 * sq * skv * hq * d
        ms3 = t(lambda: K.bwd_accumulate(q, k, v, L, D, g, scale, dq, dk, dv))
        res["bwd_ms"] = ms3
        res["bwd_tflops"] = bf / ms3 / 1e9
        res["bwd_frac_of_peak"] = res["bwd_tflops"] / peaks["bf16_tflops"]
        wsb = K.workspace(K.bwd_ws_bytes(q, k), dev, slot=3)
        res["bwd_dkv_ms"] = t(lambda: K.bwd_dkv(q, k, v, L, D, g, scale, dkg, dvg, False, ws=wsb))
        res["bwd_dq_ms"] = t(lambda: (K.bwd_dq_partial(q, k, v, L, D, g, scale, wsb),
                                      K.bwd_dq_finish(q, k, wsb, dq, True)))
        # tensor work actually issued: dkv 4 GEMMs, dq 3 GEMMs of 2*sq*skv*hq*d each
        res["dkv_tensor_tflops"] = 8.0 * sq * skv * hq * d / res["bwd_dkv_ms"] / 1e9
        res["dq_tensor_tflops"] = 6.0 * sq * skv * hq * d / res["bwd_dq_ms"] / 1e9
    # HBM roofline of the K/V stream (the bound when few query rows meet many
    # KV rows, e.g. c4round: 128 FLOP / byte in the forward): K and V read once
    kv_bytes = 2 * skv * hkv * d * 2
    hbm = peaks.get("hbm_gbs", 6500.0)
    res["kv_bytes"] = kv_bytes
    res["fwd_kv_GBps"] = kv_bytes / res["fwd_partial_ms"] / 1e6
    res["fwd_hbm_frac"] = res["fwd_kv_GBps"] / hbm
    res["fwd_hbm_roofline_tflops"] = ff / (kv_bytes / (hbm * 1e9)) / 1e12
    if a.bwd:
        res["dq_kv_GBps"] = kv_bytes / res["bwd_dq_ms"] / 1e6
        res["dkv_bytes"] = 2 * kv_bytes if a.bf16_grads else 3 * kv_bytes   # + dK, dV written
        res["dkv_GBps"] = res["dkv_bytes"] / res["bwd_dkv_ms"] / 1e6
    print(json.dumps(res))


if __name__ == "__main__":
    main()
