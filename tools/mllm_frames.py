"""How many video frames fit under a memory budget, STORE_KV vs RECOMPUTE_KV
(reference mllm.py:374-397, PAPER.md "1.5x / 1.6x more frames"), and a GPU
check that the analytic answer really fits.

    python tools/mllm_frames.py [--budget-gib 180] [--check-gib 16]

Analytic part: ``max_frames_under_budget`` per preset (B200 layout: bf16 x/y/K/V,
fp32 O/L) at n = 1 and n = 8.  Check part (needs a GPU): a stack at the frame
count the ledger allows under --check-gib runs its forward under each policy;
the peak ``torch.cuda.max_memory_allocated`` of the pass is compared with the
budget and the ledger's peak (the ledger, like the reference's, is what lives
through the forward; the backward's transients come on top).  Prints one JSON document."""
import argparse
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

PRESETS = {
    # reference toy preset (mllm.py:110-111) in bf16
    "toy": dict(num_lm_blocks=8, ca_positions=(1, 3, 5, 7), d_embed=128, h=2, d=64, frames=16,
                tokens_per_frame=729, s_q=64),
    # OpenFlamingo-like: CA every 4th of 32 blocks, 64 visual tokens per frame (C4 heads)
    "flamingo": dict(num_lm_blocks=32, ca_positions=tuple(range(3, 32, 4)), d_embed=512, h=8,
                     d=64, frames=1, tokens_per_frame=64, s_q=1024),
    # Llama-3-V-like: 8 CA layers over 40 blocks, GQA 32/8, 1601 tokens per frame (C2 heads)
    "llama3v": dict(num_lm_blocks=40, ca_positions=(3, 8, 13, 18, 23, 28, 33, 38), d_embed=4096,
                    h=32, hkv=8, d=128, frames=1, tokens_per_frame=1601, s_q=2048),
}


def analytic(budget: int) -> dict:
    from paper_2502_02406_b200.mllm import ToyMllmConfig, max_frames_under_budget
    out = {}
    for name, kw in PRESETS.items():
        cfg = ToyMllmConfig(dtype="bf16", **kw)
        row = {}
        for n in (1, 8):
            fs = max_frames_under_budget(cfg, "store", budget, n)
            fr = max_frames_under_budget(cfg, "recompute", budget, n)
            row[f"n{n}"] = {"store": fs, "recompute": fr, "ratio": fr / fs if fs else None}
        out[name] = row
    return out


def check(budget: int) -> dict:
    import torch
    from paper_2502_02406_b200.mllm import (ModelParams, ToyMllmConfig,
                                            max_frames_under_budget, mllm_forward)
    base = ToyMllmConfig(num_lm_blocks=8, ca_positions=(1, 3, 5, 7), d_embed=1024, h=8, hkv=8,
                         d=128, frames=1, tokens_per_frame=256, s_q=512, dtype="bf16")
    res = {"budget_bytes": budget, "config": base.as_dict()}
    frames = {p: max_frames_under_budget(base, p, budget) for p in ("store", "recompute")}
    res["max_frames"] = frames
    for pol in ("store", "recompute"):
        cfg = replace(base, frames=frames[pol])
        params = ModelParams.init_random(cfg, seed=0)
        gen = torch.Generator(device="cuda").manual_seed(1)
        x0 = (torch.rand(cfg.s_q, cfg.d_embed, device="cuda", generator=gen) * 2 - 1).bfloat16()
        y = (torch.rand(cfg.s_kv, cfg.d_embed, device="cuda", generator=gen) * 2 - 1).bfloat16()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        t0 = time.perf_counter()
        out, saved, ledger = mllm_forward(x0, y, params, cfg, pol)
        torch.cuda.synchronize()
        held, peak = torch.cuda.memory_allocated(), torch.cuda.max_memory_allocated()
        res[pol] = {"frames": frames[pol], "ledger_peak": ledger.peak_total,
                    "held_after_forward": held, "held_minus_ledger": held - ledger.peak_total,
                    "measured_forward_peak": peak, "transient_over_held": peak - held,
                    "held_fits_budget": held <= budget, "peak_fits_budget": peak <= budget,
                    "forward_s": time.perf_counter() - t0}
        del out, saved, params, x0, y
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget-gib", type=float, default=180.0)
    ap.add_argument("--check-gib", type=float, default=16.0)
    ap.add_argument("--no-check", action="store_true")
    a = ap.parse_args()
    out = {"analytic": analytic(int(a.budget_gib * 2 ** 30)), "budget_gib": a.budget_gib}
    if not a.no_check:
        out["check"] = check(int(a.check_gib * 2 ** 30))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
