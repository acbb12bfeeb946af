"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes ``tests/golden/golden_kernels.npz``, ``golden_strategies.npz``,
``golden_c1.npz``, ``golden_mllm_ca.npz`` and ``golden_mllm_stack.npz``
and ``golden_analytics.json`` (``--only mllm`` / ``--only analytics``: one of them).  The GPU box never reads ``/root/reference``; it only
reads these committed fixtures.  Inputs come from the reference's own
``seeded_random_tensor`` (Philox) and are stored alongside the outputs.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    from lvxattn import kernels as K
    from lvxattn.cluster import ClusterSpec
    from lvxattn.strategies import run_distributed
    from lvxattn.tensorio import seeded_random_tensor as srt

    def qkv(h, sq, skv, d, seed):
        return (srt(seed, (h, sq, d)), srt(seed, (h, skv, d), stream=1),
                srt(seed, (h, skv, d), stream=2), srt(seed, (h, sq, d), stream=3))

    # ---------------- per-kernel vectors --------------------------------
    kern = {}
    cases = [(2, 5, 9, 4, 3, 11), (1, 4, 6, 3, 64, 12), (3, 7, 33, 5, 8, 13),
             (2, 16, 70, 8, 16, 14), (1, 3, 1, 2, 64, 15)]
    for ci, (h, sq, skv, d, tile, seed) in enumerate(cases):
        Q, Kt, V, dO = qkv(h, sq, skv, d, seed)
        for dt in (np.float64, np.float32):
            tag = f"c{ci}_{np.dtype(dt).name}"
            q, k, v, g = (t.astype(dt) for t in (Q, Kt, V, dO))
            st = K.blockwise_attention(q, k, v, tile_rows=tile)
            dn = K.dense_attention(q, k, v)
            D = K.attention_row_stats(dn, g).astype(dt)
            dq, dk, dv = K.blockwise_attention_backward(q, k, v, dn.L, D, g)
            kern.update({f"{tag}_Q": q, f"{tag}_K": k, f"{tag}_V": v, f"{tag}_dO": g,
                         f"{tag}_blockO": st.O, f"{tag}_blockL": st.L,
                         f"{tag}_denseO": dn.O, f"{tag}_denseL": dn.L, f"{tag}_D": D,
                         f"{tag}_dQ": dq, f"{tag}_dK": dk, f"{tag}_dV": dv,
                         f"{tag}_tile": np.array(tile)})
            # split into two KV blocks and merge (merge_states vector)
            cut = skv // 2
            a = K.blockwise_attention(q, k[:, :cut], v[:, :cut])
            b = K.blockwise_attention(q, k[:, cut:], v[:, cut:])
            m = K.merge_states(a, b)
            kern.update({f"{tag}_mAO": a.O, f"{tag}_mAL": a.L, f"{tag}_mBO": b.O,
                         f"{tag}_mBL": b.L, f"{tag}_mO": m.O, f"{tag}_mL": m.L})
    # projection
    x = srt(26, (5, 6))
    W = srt(27, (6, 8))
    g = srt(28, (2, 5, 4))
    kern["proj_x"], kern["proj_W"], kern["proj_g"] = x, W, g
    kern["proj_out"] = K.project(x, W, 2)
    kern["proj_dX"], kern["proj_dW"] = K.project_backward(x, W, g)
    np.savez_compressed(OUT / "golden_kernels.npz", **kern)

    # ---------------- distributed protocol vectors ----------------------
    strat = {}
    scases = [(1, 5, 7, 3, 1, 1), (2, 5, 7, 4, 3, 2), (2, 8, 8, 4, 4, 3),
              (1, 2, 9, 3, 4, 4),     # empty Q shards
              (1, 9, 2, 3, 4, 5),     # empty KV shards
              (4, 16, 3, 5, 6, 6), (2, 7, 9, 4, 2, 7)]
    for ci, (h, sq, skv, d, n, seed) in enumerate(scases):
        Q, Kt, V, dO = qkv(h, sq, skv, d, seed)
        for dt in (np.float64, np.float32):
            q, k, v, g = (t.astype(dt) for t in (Q, Kt, V, dO))
            for s in ("lvx", "ring", "head"):
                if s == "head" and h % n:
                    continue
                tag = f"s{ci}_{s}_{np.dtype(dt).name}"
                res = run_distributed(s, q, k, v, dO=g, spec=ClusterSpec(n))
                strat.update({
                    f"{tag}_Q": q, f"{tag}_K": k, f"{tag}_V": v, f"{tag}_dO": g,
                    f"{tag}_n": np.array(n), f"{tag}_O": res.O, f"{tag}_L": res.L,
                    f"{tag}_dQ": res.grads.dQ, f"{tag}_dK": res.grads.dK,
                    f"{tag}_dV": res.grads.dV,
                    f"{tag}_fwd_bytes": np.array([t.total_sent_bytes() for t in res.traces_forward]),
                    f"{tag}_bwd_bytes": np.array([t.total_sent_bytes() for t in res.traces_backward]),
                    f"{tag}_fwd_rounds": np.array([t.num_rounds for t in res.traces_forward]),
                })
    np.savez_compressed(OUT / "golden_strategies.npz", **strat)

    # ---------------- BASELINE configs[0] (C1) --------------------------
    # Lq=128, Lkv=4096, 8 heads, d=64, fp32, world_size=2 ring.  Inputs are
    # NOT stored (regenerated bit-exactly from the seed); O, L and dQ are
    # stored whole, dK/dV on a row sample plus per-head sums.
    h, sq, skv, d, n, seed = 8, 128, 4096, 64, 2, 2024
    Q, Kt, V, dO = (t.astype(np.float32) for t in qkv(h, sq, skv, d, seed))
    res = run_distributed("lvx", Q, Kt, V, dO=dO, spec=ClusterSpec(n))
    rows = np.arange(0, skv, 61)
    c1 = {"seed": np.array(seed), "shape": np.array([h, sq, skv, d, n]),
          "Q_head": Q[:, :2].copy(), "O": res.O, "L": res.L, "dQ": res.grads.dQ,
          "dK_rows": rows, "dK_sample": res.grads.dK[:, rows], "dV_sample": res.grads.dV[:, rows],
          "dK_sum": res.grads.dK.astype(np.float64).sum(axis=(1, 2)),
          "dV_sum": res.grads.dV.astype(np.float64).sum(axis=(1, 2)),
          "fwd_bytes": np.array([t.total_sent_bytes() for t in res.traces_forward]),
          "bwd_bytes": np.array([t.total_sent_bytes() for t in res.traces_backward])}
    np.savez_compressed(OUT / "golden_c1.npz", **c1)
    # ---------------- MLLM cross-attention block (recompute) -------------
    # one block, CA at position 0, MLP weights zeroed so the block is exactly
    # the CA layer (x + tanh(x*0)*0 = x): pins the CA math incl. K/V recompute
    from dataclasses import replace as _replace
    from lvxattn.mllm import (ActivationPolicy, ModelParams, ToyMllmConfig, mllm_backward,
                              mllm_forward, OpCounter)
    cfg = ToyMllmConfig(num_lm_blocks=1, ca_positions=(0,), d_embed=12, h=2, d=6, frames=3,
                        tokens_per_frame=7, s_q=9, dtype="f64")
    params = ModelParams.init_random(cfg, seed=3)
    for blk in params.lm:
        blk.w1[...] = 0.0
        blk.w2[...] = 0.0
    x0 = srt(61, (cfg.s_q, cfg.d_embed))
    y = srt(62, (cfg.s_kv, cfg.d_embed))
    gout = srt(63, (cfg.s_q, cfg.d_embed))
    ca = {}
    for pol in (ActivationPolicy.STORE_KV, ActivationPolicy.RECOMPUTE_KV):
        out, saved, ledger = mllm_forward(x0, y, params, cfg, pol)
        cnt = OpCounter()
        gr = mllm_backward(gout, saved, y, params, cfg, pol, counter=cnt)
        p0 = params.ca[0]
        ca.update({f"{pol.value}_out": out, f"{pol.value}_dx": gr.d_x0, f"{pol.value}_dy": gr.d_y,
                   f"{pol.value}_gwq": gr.ca[0].w_q, f"{pol.value}_gwk": gr.ca[0].w_k,
                   f"{pol.value}_gwv": gr.ca[0].w_v, f"{pol.value}_gwo": gr.ca[0].w_o,
                   f"{pol.value}_flops": np.array(cnt.projection_flops)})
    ca.update({"x": x0, "y": y, "g": gout, "w_q": params.ca[0].w_q, "w_k": params.ca[0].w_k,
               "w_v": params.ca[0].w_v, "w_o": params.ca[0].w_o,
               "dims": np.array([cfg.h, cfg.d, cfg.d_embed])})
    np.savez_compressed(OUT / "golden_mllm_ca.npz", **ca)

    for f in ("golden_kernels.npz", "golden_strategies.npz", "golden_c1.npz",
              "golden_mllm_ca.npz"):
        print(f, (OUT / f).stat().st_size, "bytes")


def make_mllm_stack() -> None:
    """Full toy-MLLM stack: several LM blocks with CA
    layers sharing one y, both policies, ledgers, measured activation bytes
    and max_frames_under_budget answers -> golden_mllm_stack.npz."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import json
    from dataclasses import replace as _replace
    from lvxattn.mllm import (TOY_CONFIG, ActivationPolicy, ModelParams, OpCounter,
                              ToyMllmConfig, analytic_ledger, max_frames_under_budget,
                              measured_activation_bytes, mllm_backward, mllm_forward)
    from lvxattn.tensorio import seeded_random_tensor as srt
    cfg = ToyMllmConfig(num_lm_blocks=5, ca_positions=(0, 2, 3), d_embed=16, h=2, d=8,
                        frames=3, tokens_per_frame=11, s_q=10, dtype="f64")
    params = ModelParams.init_random(cfg, seed=5)
    x0 = srt(71, (cfg.s_q, cfg.d_embed))
    y = srt(72, (cfg.s_kv, cfg.d_embed))
    gout = srt(73, (cfg.s_q, cfg.d_embed))
    out = {"config": np.array(json.dumps(cfg.as_dict())), "x0": x0, "y": y, "g": gout}
    for pos, p in params.ca.items():
        for n in ("w_q", "w_k", "w_v", "w_o"):
            out[f"p_ca{pos}_{n}"] = getattr(p, n)
    for i, p in enumerate(params.lm):
        out[f"p_lm{i}_w1"], out[f"p_lm{i}_w2"] = p.w1, p.w2
    for pol in (ActivationPolicy.STORE_KV, ActivationPolicy.RECOMPUTE_KV):
        o, saved, ledger = mllm_forward(x0, y, params, cfg, pol)
        cnt = OpCounter()
        gr = mllm_backward(gout, saved, y, params, cfg, pol, counter=cnt)
        t = pol.value
        out[f"{t}_out"], out[f"{t}_dx0"], out[f"{t}_dy"] = o, gr.d_x0, gr.d_y
        for pos, gp in gr.ca.items():
            for n in ("w_q", "w_k", "w_v", "w_o"):
                out[f"{t}_g_ca{pos}_{n}"] = getattr(gp, n)
        for i, gp in enumerate(gr.lm):
            out[f"{t}_g_lm{i}_w1"], out[f"{t}_g_lm{i}_w2"] = gp.w1, gp.w2
        out[f"{t}_flops"] = np.array(cnt.projection_flops)
        out[f"{t}_ledger"] = np.array(json.dumps(ledger.as_dict()))
        out[f"{t}_measured"] = np.array(json.dumps(measured_activation_bytes(saved)))
    # ledgers and frame budgets of the shipped TOY_CONFIG and a bf16-sized variant
    budgets = [1 << 20, 5 << 20, 64 << 20, 1 << 30]
    for name, c in (("toy", TOY_CONFIG), ("toy_f32_many", _replace(TOY_CONFIG, frames=256))):
        for pol in (ActivationPolicy.STORE_KV, ActivationPolicy.RECOMPUTE_KV):
            out[f"{name}_{pol.value}_ledger"] = np.array(json.dumps(analytic_ledger(c, pol).as_dict()))
            out[f"{name}_{pol.value}_frames"] = np.array(
                [max_frames_under_budget(c, pol, b) for b in budgets])
    out["budgets"] = np.array(budgets)
    np.savez_compressed(OUT / "golden_mllm_stack.npz", **out)
    print("golden_mllm_stack.npz", (OUT / "golden_mllm_stack.npz").stat().st_size, "bytes")


def make_analytics() -> None:
    """The reference's cost model (analytics.py) on a grid of workloads and the
    shipped presets -> golden_analytics.json (§8(f) next 3)."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import json
    from lvxattn import analytics as A
    hw = A.HardwareSpec(1665.5e12, 900e9)
    cases = [(2048, 1 << 20, 32, 128, 8, 2), (5514, 1 << 18, 28, 128, 4, 2), (1024, 524288, 8, 64, 8, 2),
             (128, 4096, 8, 64, 2, 4), (7, 0, 2, 4, 3, 8), (1000, 1000, 4, 16, 1, 4)]
    out = {"hw": [hw.gpu_flops, hw.net_bandwidth], "cases": []}
    for (sq, skv, h, d, n, b) in cases:
        w = A.WorkloadSpec(s_q=sq, s_kv=skv, h=h, d=d, n=n, elem_bytes=b)
        out["cases"].append({
            "w": [sq, skv, h, d, n, b],
            "round_times": {k: v.as_dict() for k, v in A.round_times(w, hw).items()},
            "speedup": A.speedup(w, hw), "closed_form": A.speedup_closed_form(w, hw),
            "regime": A.classify_regime(w, hw).as_dict(),
            "volume_report": A.volume_report(w) if sq and skv else None})
    out["memory"] = A.memory_cross_attention(2048, 1 << 20, 4096, 2)
    out["video"] = [vars(A.workload_from_video(m, 600, 1, 512, 8)) for m in sorted(A.TOKENS_PER_FRAME)]
    out["presets"] = {k: {"w": vars(p.workload), "d_model": p.d_model}
                      for k, p in A.PRESETS.items()}
    grid = A.grid_values(256, 65536, 5)
    out["grid"] = grid
    out["sweep_csv"] = A.format_sweep_csv(A.sweep(grid, A.grid_values(1 << 16, 1 << 24, 4), hw,
                                                  32, 128, 8, 2))
    (OUT / "golden_analytics.json").write_text(json.dumps(out, indent=0, sort_keys=True))
    print("golden_analytics.json", (OUT / "golden_analytics.json").stat().st_size, "bytes")


def make_lvxt() -> None:
    """LVXT files written by the reference (tensorio.py:85-130) plus a numeric
    run (the data path of cli.cmd_run, cli.py:96-177) -> tests/golden/lvxt/."""
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import json
    from lvxattn.cluster import ClusterSpec
    from lvxattn.strategies import run_distributed
    from lvxattn.tensorio import seeded_random_tensor as srt, store_tensor
    out = OUT / "lvxt"
    out.mkdir(exist_ok=True)
    store_tensor(srt(5, (3, 4, 2), np.float32), out / "f32_3d.lvxt")
    store_tensor(srt(6, (7,), np.float64, scale=2.0, stream=3), out / "f64_1d.lvxt")
    store_tensor(srt(7, (2, 5), np.float32, stream=9), out / "f32_2d.lvxt")
    # inputs + outputs of one numeric run: lvx, n = 3, f64, with backward
    h, sq, skv, d, seed = 2, 7, 11, 4, 17
    Q = srt(seed, (h, sq, d), np.float64, stream=0)
    K = srt(seed, (h, skv, d), np.float64, stream=1)
    V = srt(seed, (h, skv, d), np.float64, stream=2)
    dO = srt(seed, (h, sq, d), np.float64, stream=3)
    for name, t in (("q", Q), ("k", K), ("v", V), ("do", dO)):
        store_tensor(t, out / f"run_in_{name}.lvxt")
    res = run_distributed("lvx", Q, K, V, dO=dO, spec=ClusterSpec(3))
    for name, t in (("o", res.O), ("l", res.L), ("dq", res.grads.dQ), ("dk", res.grads.dK),
                    ("dv", res.grads.dV)):
        store_tensor(t, out / f"run_out_{name}.lvxt")
    (out / "run_stats.json").write_text(json.dumps({
        "total_bytes": res.stats.total_bytes(),
        "per_worker_bytes_sent": [res.stats.bytes_sent_by(i) for i in range(3)],
        "rounds_forward": res.traces_forward[0].num_rounds}))
    print("lvxt goldens:", sorted(p.name for p in out.iterdir()))


if __name__ == "__main__":
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    if only == "mllm":
        make_mllm_stack()
    elif only == "analytics":
        make_analytics()
    elif only == "lvxt":
        make_lvxt()
    else:
        main()
        make_mllm_stack()
        make_analytics()
        make_lvxt()
