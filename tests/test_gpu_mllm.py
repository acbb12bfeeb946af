"""Toy MLLM stack on the GPU vs the reference.

* f64: the whole 5-block / 3-CA-layer stack, both policies, against the
  reference's own outputs and gradients (tests/golden/golden_mllm_stack.npz),
  1e-10 max-normalised (exact SIMT attention + the library's exact f64 GEMM).
* ledgers and frame budgets: identical to the reference's numbers when the
  layout matches (f32 / f64: one element size everywhere).
* bf16: measured live bytes == the ledger categories, and the allocator agrees.
"""
import json

import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_02406_b200 import build
    build.build()


@pytest.fixture(scope="module")
def stack():
    from tests.conftest import GOLDEN
    return dict(np.load(GOLDEN / "golden_mllm_stack.npz"))


def _model(g):
    from paper_2502_02406_b200.mllm import ModelParams, ToyMllmConfig
    from paper_2502_02406_b200.recompute import CrossAttentionWeights
    cfg = ToyMllmConfig.from_dict(json.loads(str(g["config"])))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ca = {p: CrossAttentionWeights(*(t(g[f"p_ca{p}_{n}"]) for n in ("w_q", "w_k", "w_v", "w_o")),
                                   cfg.h, cfg.h) for p in cfg.ca_positions}
    lm = [(t(g[f"p_lm{i}_w1"]), t(g[f"p_lm{i}_w2"])) for i in range(cfg.num_lm_blocks)]
    return cfg, ModelParams(ca=ca, lm=lm), t


@pytest.mark.parametrize("policy", ["store", "recompute"])
def test_mllm_stack_f64_vs_reference(stack, policy):
    from paper_2502_02406_b200.mllm import OpCounter, mllm_backward, mllm_forward
    g = stack
    cfg, params, t = _model(g)
    x0, y, gout = t(g["x0"]), t(g["y"]), t(g["g"])
    out, saved, ledger = mllm_forward(x0, y, params, cfg, policy)
    cnt = OpCounter()
    gr = mllm_backward(gout, saved, y, params, cfg, policy, counter=cnt)
    err = lambda a, b: orc.max_norm_error(a.cpu().numpy(), b)  # noqa: E731
    assert err(out, g[f"{policy}_out"]) <= 1e-10
    assert err(gr.d_x0, g[f"{policy}_dx0"]) <= 1e-10
    assert err(gr.d_y, g[f"{policy}_dy"]) <= 1e-10
    for p, cg in gr.ca.items():
        for n in ("w_q", "w_k", "w_v", "w_o"):
            assert err(getattr(cg, n), g[f"{policy}_g_ca{p}_{n}"]) <= 1e-10, (p, n)
    for i, (g1, g2) in enumerate(gr.lm):
        assert err(g1, g[f"{policy}_g_lm{i}_w1"]) <= 1e-10
        assert err(g2, g[f"{policy}_g_lm{i}_w2"]) <= 1e-10
    assert cnt.projection_flops == int(g[f"{policy}_flops"])
    assert ledger.as_dict() == json.loads(str(g[f"{policy}_ledger"]))


def test_ledger_and_frames_match_reference(stack):
    from dataclasses import replace
    from paper_2502_02406_b200.mllm import (TOY_CONFIG, analytic_ledger,
                                            max_frames_under_budget)
    g = stack
    for name, frames in (("toy", 16), ("toy_f32_many", 256)):
        cfg = replace(TOY_CONFIG, dtype="f32", frames=frames)
        for pol in ("store", "recompute"):
            assert analytic_ledger(cfg, pol).as_dict() == \
                json.loads(str(g[f"{name}_{pol}_ledger"])), (name, pol)
            got = [max_frames_under_budget(cfg, pol, int(b)) for b in g["budgets"]]
            assert got == list(g[f"{name}_{pol}_frames"]), (name, pol)


def test_bf16_live_bytes_match_ledger():
    """bf16 stack: the saved tensors are exactly the ledger's categories, the
    allocator's growth over the forward equals them (+ LM inputs, output),
    and RECOMPUTE_KV saves exactly C * 2 * S_kv * hkv * d * 2 bytes."""
    from paper_2502_02406_b200.mllm import (ModelParams, ToyMllmConfig, analytic_ledger,
                                            live_activation_bytes, measured_activation_bytes,
                                            mllm_forward)
    cfg = ToyMllmConfig(num_lm_blocks=6, ca_positions=(1, 3, 5), d_embed=256, h=4, d=64,
                        frames=12, tokens_per_frame=256, s_q=128, dtype="bf16", hkv=2)
    params = ModelParams.init_random(cfg, seed=1)
    gen = torch.Generator(device="cuda").manual_seed(2)
    x0 = (torch.rand(cfg.s_q, cfg.d_embed, device="cuda", generator=gen) * 2 - 1).bfloat16()
    y = (torch.rand(cfg.s_kv, cfg.d_embed, device="cuda", generator=gen) * 2 - 1).bfloat16()
    live = {}
    for pol in ("store", "recompute"):   # warm-up: the cached kernel workspaces exist
        mllm_forward(x0, y, params, cfg, pol)
    for pol in ("store", "recompute"):
        torch.cuda.synchronize()
        before = torch.cuda.memory_allocated()
        out, saved, ledger = mllm_forward(x0, y, params, cfg, pol)
        torch.cuda.synchronize()
        grown = torch.cuda.memory_allocated() - before
        m = measured_activation_bytes(saved)
        c = cfg.num_ca_layers
        assert m["saved_x"] == c * ledger.per_layer_saved_x
        assert m["saved_o_l"] == c * ledger.per_layer_saved_o_l
        assert m["saved_kv"] == c * ledger.per_layer_saved_kv
        assert m["visual_features_y"] == ledger.visual_features_y
        # new allocations only: y and x0 (lm_inputs[0] when block 0 has no CA
        # layer) existed before the forward
        pre = {y.data_ptr(), x0.data_ptr()}
        expect = live_activation_bytes(saved) - m["visual_features_y"] - sum(
            t.numel() * t.element_size() for t in saved.lm_inputs if t.data_ptr() in pre) + \
            out.numel() * out.element_size()
        # caching allocator rounds each block up to 512 B
        nblocks = 4 * c + cfg.num_lm_blocks + 1
        assert expect <= grown <= expect + 512 * nblocks + (1 << 20), (pol, grown, expect)
        live[pol] = expect
        del out, saved
    assert live["store"] - live["recompute"] == \
        cfg.num_ca_layers * 2 * cfg.s_kv * cfg.kv_heads * cfg.d * 2
    assert analytic_ledger(cfg, "store").peak_total > analytic_ledger(cfg, "recompute").peak_total


def test_bf16_stack_vs_oracle():
    """bf16 stack (GQA, recompute) against the oracle's stack on the same
    bf16-rounded inputs and weights: max-normalised <= 3e-2 (bf16 projections
    and attention operands through 4 layers)."""
    from paper_2502_02406_b200.mllm import (ModelParams, ToyMllmConfig, mllm_backward,
                                            mllm_forward)
    cfg = ToyMllmConfig(num_lm_blocks=4, ca_positions=(0, 2), d_embed=128, h=4, d=64,
                        frames=5, tokens_per_frame=129, s_q=96, dtype="bf16", hkv=2)
    params = ModelParams.init_random(cfg, seed=3)
    gen = torch.Generator(device="cuda").manual_seed(4)
    u = lambda *s: (torch.rand(*s, device="cuda", generator=gen) * 2 - 1).bfloat16()  # noqa: E731
    x0, y, gout = u(cfg.s_q, cfg.d_embed), u(cfg.s_kv, cfg.d_embed), u(cfg.s_q, cfg.d_embed)
    out, saved, _ = mllm_forward(x0, y, params, cfg, "recompute")
    gr = mllm_backward(gout, saved, y, params, cfg, "recompute")
    h = lambda t: t.double().cpu().numpy()  # noqa: E731
    ca = {p: tuple(h(getattr(w, n)) for n in ("w_q", "w_k", "w_v", "w_o"))
          for p, w in params.ca.items()}
    lm = [(h(a), h(b)) for a, b in params.lm]
    o_out, o_saved = orc.mllm_stack_forward(h(x0), h(y), ca, lm, cfg.ca_positions, cfg.h, cfg.hkv)
    o_dx, o_dy, _, _ = orc.mllm_stack_backward(h(gout), o_saved, h(y), ca, lm, cfg.ca_positions,
                                               cfg.h, cfg.hkv)
    errs = {"out": orc.max_norm_error(h(out), o_out), "dx0": orc.max_norm_error(h(gr.d_x0), o_dx),
            "dy": orc.max_norm_error(h(gr.d_y), o_dy)}
    print(f"\nbf16 MLLM stack vs oracle: {errs}")
    assert max(errs.values()) <= 3e-2, errs
