"""The recompute layer's GEMMs on one B200: the library's tcgen05 GEMM
(lvx_gemm / lvx_kv_recompute) against torch.mm (cuBLAS) at the same shapes,
CUDA-event timed, interleaved (the power cap moves clocks), median of 5.

    python tools/gemm_probe.py [--preset llama|flamingo]
Prints one JSON line per GEMM: ms and TFLOP/s of both, and the ratio.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_02406_b200 import kernels as K  # noqa: E402

PRESETS = {  # S (visual rows per rank), e, hkv * d
    "llama": (131072, 4096, 1024),
    "flamingo": (65536, 2048, 512),
}


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="llama")
    args = ap.parse_args()
    S, e, hkd = PRESETS[args.preset]
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: (torch.rand(*s, device="cuda", generator=g) - 0.5).bfloat16()  # noqa: E731
    y, w, dkv = r(S, e), r(e, 2 * hkd), r(S, 2 * hkd)
    out_kv = torch.empty(S, 2 * hkd, device="cuda", dtype=torch.bfloat16)
    out_dy = torch.empty(S, e, device="cuda", dtype=torch.bfloat16)
    out_dw = torch.empty(e, 2 * hkd, device="cuda", dtype=torch.bfloat16)
    cases = {
        # name: (flops, ours, torch)
        "kv_recompute y@[Wk|Wv]": (2 * S * e * 2 * hkd,
                                   lambda: K.gemm_into(y, False, w, False, out_kv),
                                   lambda: torch.mm(y, w, out=out_kv)),
        "dY = dKV @ W^T": (2 * S * e * 2 * hkd,
                           lambda: K.gemm_into(dkv, False, w, True, out_dy),
                           lambda: torch.mm(dkv, w.T, out=out_dy)),
        "dW = y^T @ dKV": (2 * S * e * 2 * hkd,
                           lambda: K.gemm_into(y, True, dkv, False, out_dw),
                           lambda: torch.mm(y.T, dkv, out=out_dw)),
    }
    for name, (fl, ours, ref) in cases.items():
        a_ms, b_ms = [], []
        for _ in range(5):
            a_ms.append(timeit(ours))
            b_ms.append(timeit(ref))
        ms_a, ms_b = statistics.median(a_ms), statistics.median(b_ms)
        # correctness at this shape against cuBLAS's output
        ours()
        mine = {"kv_recompute y@[Wk|Wv]": out_kv, "dY = dKV @ W^T": out_dy,
                "dW = y^T @ dKV": out_dw}[name].float().clone()
        ref()
        theirs = {"kv_recompute y@[Wk|Wv]": out_kv, "dY = dKV @ W^T": out_dy,
                  "dW = y^T @ dKV": out_dw}[name].float()
        err = ((mine - theirs).abs().max() / theirs.abs().max()).item()
        print(json.dumps({"preset": args.preset, "gemm": name, "M_N_K": None,
                          "lvx_ms": ms_a, "lvx_tflops": fl / ms_a / 1e9,
                          "cublas_ms": ms_b, "cublas_tflops": fl / ms_b / 1e9,
                          "lvx_over_cublas": ms_b / ms_a, "max_norm_diff_vs_cublas": err}),
              flush=True)


if __name__ == "__main__":
    main()
