"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import lvx_oracle as orc

KCASES = 5
DTS = ("float64", "float32")


def tol(dt):
    return 1e-12 if dt == "float64" else 1e-5


@pytest.mark.parametrize("ci", range(KCASES))
@pytest.mark.parametrize("dt", DTS)
def test_kernels_match_reference(golden_kernels, ci, dt):
    g = golden_kernels
    t = f"c{ci}_{dt}"
    Q, K, V, dO = g[t + "_Q"], g[t + "_K"], g[t + "_V"], g[t + "_dO"]
    O, L = orc.blockwise_attention(Q, K, V, tile_rows=int(g[t + "_tile"]))
    assert O.dtype == np.dtype(dt)
    assert orc.max_norm_error(O, g[t + "_blockO"]) <= tol(dt)
    assert orc.max_norm_error(L, g[t + "_blockL"]) <= tol(dt)
    Od, Ld = orc.dense_attention(Q, K, V)
    assert orc.max_norm_error(Od, g[t + "_denseO"]) <= tol(dt)
    D = orc.attention_row_stats(Od, dO).astype(dt)
    assert orc.max_norm_error(D, g[t + "_D"]) <= tol(dt)
    dq, dk, dv = orc.blockwise_attention_backward(Q, K, V, Ld, D, dO)
    for a, b in ((dq, "_dQ"), (dk, "_dK"), (dv, "_dV")):
        assert orc.max_norm_error(a, g[t + b]) <= tol(dt)
    mo, ml = orc.merge_states(g[t + "_mAO"], g[t + "_mAL"], g[t + "_mBO"], g[t + "_mBL"])
    assert orc.max_norm_error(mo, g[t + "_mO"]) <= tol(dt)
    assert orc.max_norm_error(ml, g[t + "_mL"]) <= tol(dt)


def test_projection_matches_reference(golden_kernels):
    g = golden_kernels
    assert orc.max_norm_error(orc.project(g["proj_x"], g["proj_W"], 2), g["proj_out"]) <= 1e-14
    dx, dw = orc.project_backward(g["proj_x"], g["proj_W"], g["proj_g"])
    assert orc.max_norm_error(dx, g["proj_dX"]) <= 1e-14
    assert orc.max_norm_error(dw, g["proj_dW"]) <= 1e-14


def _scases(g):
    return sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_n")})


def test_simulated_protocols_match_reference(golden_strategies):
    g = golden_strategies
    tags = _scases(g)
    assert len(tags) == 7 * 2 * 2 + 2 * 2   # + head-parallel where h % n == 0
    for t in tags:
        strategy = t.split("_")[1]
        dt = t.split("_")[2]
        n = int(g[t + "_n"])
        res = orc.simulate(strategy, g[t + "_Q"], g[t + "_K"], g[t + "_V"], g[t + "_dO"], n=n)
        for name, arr in (("O", res.O), ("L", res.L), ("dQ", res.dQ), ("dK", res.dK), ("dV", res.dV)):
            assert orc.max_norm_error(arr, g[f"{t}_{name}"]) <= tol(dt), (t, name)
        assert res.fwd_bytes == list(g[t + "_fwd_bytes"]), t
        assert res.bwd_bytes == list(g[t + "_bwd_bytes"]), t


def test_closed_form_volumes_match_reference(golden_strategies):
    g = golden_strategies
    for t in _scases(g):
        strategy, dt = t.split("_")[1], t.split("_")[2]
        n = int(g[t + "_n"])
        h, sq, d = g[t + "_Q"].shape
        skv = g[t + "_K"].shape[1]
        b = np.dtype(dt).itemsize
        qs = [b_ - a for a, b_ in orc.partition_rows(sq, n)]
        ks = [b_ - a for a, b_ in orc.partition_rows(skv, n)]
        if strategy == "head":
            continue   # checked through simulate() above
        if strategy == "lvx":
            f, bw = orc.lvx_forward_bytes(qs, h, d, b), orc.lvx_backward_bytes(qs, h, d, b)
        else:
            f, bw = orc.ring_forward_bytes(ks, h, d, b), orc.ring_backward_bytes(ks, h, d, b)
        assert f == list(g[t + "_fwd_bytes"]) and bw == list(g[t + "_bwd_bytes"]), t


def test_seeded_inputs_bit_exact(golden_c1):
    h, sq, skv, d, n = (int(x) for x in golden_c1["shape"])
    Q = orc.seeded_random_tensor(int(golden_c1["seed"]), (h, sq, d)).astype(np.float32)
    assert np.array_equal(Q[:, :2], golden_c1["Q_head"])


def test_c1_oracle_matches_reference(golden_c1):
    g = golden_c1
    h, sq, skv, d, n = (int(x) for x in g["shape"])
    Q, K, V, dO = (t.astype(np.float32) for t in orc.make_inputs(sq, skv, h, d, int(g["seed"])))
    res = orc.simulate("lvx", Q, K, V, dO, n=n)
    assert orc.max_norm_error(res.O, g["O"]) <= 1e-5
    assert orc.max_norm_error(res.L, g["L"]) <= 1e-5
    assert orc.max_norm_error(res.dQ, g["dQ"]) <= 1e-5
    assert orc.max_norm_error(res.dK[:, g["dK_rows"]], g["dK_sample"]) <= 1e-5
    assert orc.max_norm_error(res.dV[:, g["dK_rows"]], g["dV_sample"]) <= 1e-5
    assert res.fwd_bytes == list(g["fwd_bytes"]) and res.bwd_bytes == list(g["bwd_bytes"])


def test_gqa_adapter_consistent():
    # GQA through the oracle == MHA with explicitly expanded K/V and group-summed grads
    Q, K, V, dO = orc.make_inputs(6, 11, 4, 5, seed=3, hkv=2)
    O, L = orc.dense_attention(Q, K, V)
    Ke, Ve = orc.expand_kv(K, 4), orc.expand_kv(V, 4)
    Om, Lm = orc.dense_attention(Q, Ke, Ve)
    assert orc.max_norm_error(O, Om) <= 1e-14
    dq, dk, dv = orc.dense_attention_backward(Q, K, V, O, L, dO)
    dqm, dkm, dvm = orc.dense_attention_backward(Q, Ke, Ve, Om, Lm, dO)
    assert orc.max_norm_error(dq, dqm) <= 1e-14
    assert orc.max_norm_error(dk, orc.reduce_kv_grad(dkm, 2)) <= 1e-14
    assert orc.max_norm_error(dv, orc.reduce_kv_grad(dvm, 2)) <= 1e-14


def test_ca_block_matches_reference_mllm(golden_mllm_ca):
    g = golden_mllm_ca
    h, d, e = (int(v) for v in g["dims"])
    out, O, L = orc.ca_block_forward(g["x"], g["y"], g["w_q"], g["w_k"], g["w_v"], g["w_o"], h)
    for pol in ("store", "recompute"):
        assert orc.max_norm_error(out, g[f"{pol}_out"]) <= 1e-12
    dx, dy, gq, gk, gv, go = orc.ca_block_backward(g["g"], g["x"], O, L, g["y"], g["w_q"],
                                                   g["w_k"], g["w_v"], g["w_o"], h)
    for pol in ("store", "recompute"):
        for a, b in ((dx, "dx"), (dy, "dy"), (gq, "gwq"), (gk, "gwk"), (gv, "gwv"), (go, "gwo")):
            assert orc.max_norm_error(a, g[f"{pol}_{b}"]) <= 1e-12, (pol, b)
    # the recompute policy does exactly two extra y projections (mllm.py:358-363)
    s_kv = g["y"].shape[0]
    assert int(g["recompute_flops"]) - int(g["store_flops"]) == 2 * 2 * s_kv * e * h * d


def _stack_golden():
    import json
    from tests.conftest import GOLDEN
    g = dict(np.load(GOLDEN / "golden_mllm_stack.npz"))
    cfg = json.loads(str(g["config"]))
    ca = {p: tuple(g[f"p_ca{p}_{n}"] for n in ("w_q", "w_k", "w_v", "w_o"))
          for p in cfg["ca_positions"]}
    lm = [(g[f"p_lm{i}_w1"], g[f"p_lm{i}_w2"]) for i in range(cfg["num_lm_blocks"])]
    return g, cfg, ca, lm


@pytest.mark.parametrize("policy", ["store", "recompute"])
def test_mllm_stack_matches_reference(policy):
    """The oracle's toy-MLLM stack (mllm.py:274-371) vs the reference's own
    forward/backward on a 5-block, 3-CA-layer f64 model."""
    g, cfg, ca, lm = _stack_golden()
    out, saved = orc.mllm_stack_forward(g["x0"], g["y"], ca, lm, cfg["ca_positions"], cfg["h"],
                                        store_kv=policy == "store")
    assert orc.max_norm_error(out, g[f"{policy}_out"]) <= 1e-12
    dx0, dy, cag, lmg = orc.mllm_stack_backward(g["g"], saved, g["y"], ca, lm,
                                                cfg["ca_positions"], cfg["h"])
    assert orc.max_norm_error(dx0, g[f"{policy}_dx0"]) <= 1e-12
    assert orc.max_norm_error(dy, g[f"{policy}_dy"]) <= 1e-12
    for p, gw in cag.items():
        for n, arr in zip(("w_q", "w_k", "w_v", "w_o"), gw):
            assert orc.max_norm_error(arr, g[f"{policy}_g_ca{p}_{n}"]) <= 1e-12
    for i, (g1, g2) in enumerate(lmg):
        assert orc.max_norm_error(g1, g[f"{policy}_g_lm{i}_w1"]) <= 1e-12
        assert orc.max_norm_error(g2, g[f"{policy}_g_lm{i}_w2"]) <= 1e-12


def test_mllm_ledger_and_frames_match_reference():
    import json
    g, cfg, _, _ = _stack_golden()
    toy = dict(num_lm_blocks=8, num_ca_layers=4, d_embed=128, h=2, d=64, s_q=64)   # TOY_CONFIG
    for name, frames in (("toy", 16), ("toy_f32_many", 256)):
        for pol in ("store", "recompute"):
            led = orc.analytic_ledger(**toy, s_kv=frames * 729, store_kv=pol == "store", b=4)
            assert led == json.loads(str(g[f"{name}_{pol}_ledger"])), (name, pol)
            got = [orc.max_frames_under_budget(
                lambda f, p=pol: orc.analytic_ledger(**toy, s_kv=f * 729, store_kv=p == "store",
                                                     b=4)["peak_total"], int(bud))
                   for bud in g["budgets"]]
            assert got == list(g[f"{name}_{pol}_frames"]), (name, pol, got)
    for pol in ("store", "recompute"):
        led = orc.analytic_ledger(cfg["num_lm_blocks"], len(cfg["ca_positions"]), cfg["d_embed"],
                                  cfg["h"], cfg["d"], cfg["s_q"],
                                  cfg["frames"] * cfg["tokens_per_frame"], pol == "store", b=8)
        assert led == json.loads(str(g[f"{pol}_ledger"]))
