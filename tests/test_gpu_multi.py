"""Multi-GPU ring parity (NCCL over NVLink): run_distributed spawning one
process per GPU, against the reference's golden vectors."""
import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.fixture(scope="module", autouse=True)
def _need_gpus():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")


def test_ring_protocols_vs_reference(golden_strategies):
    import paper_2502_02406_b200 as lvx
    g = golden_strategies
    tags = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_n")})
    ran = 0
    for t in tags:
        n = int(g[t + "_n"])
        if n < 2 or n > torch.cuda.device_count():
            continue
        res = lvx.run_distributed(t.split("_")[1], g[t + "_Q"], g[t + "_K"], g[t + "_V"],
                                  dO=g[t + "_dO"], spec=lvx.ClusterSpec(n))
        tol = 1e-12 if t.endswith("float64") else 1e-5
        for name, arr in (("O", res.O), ("L", res.L), ("dQ", res.grads.dQ),
                          ("dK", res.grads.dK), ("dV", res.grads.dV)):
            assert orc.max_norm_error(arr, g[f"{t}_{name}"]) <= tol, (t, name)
        assert [tr.total_sent_bytes() for tr in res.traces_forward] == list(g[t + "_fwd_bytes"])
        assert [tr.total_sent_bytes() for tr in res.traces_backward] == list(g[t + "_bwd_bytes"])
        ran += 1
    assert ran > 0


def test_c1_config_world2_vs_reference(golden_c1):
    import paper_2502_02406_b200 as lvx
    g = golden_c1
    h, sq, skv, d, n = (int(x) for x in g["shape"])
    Q, K, V, dO = (t.astype(np.float32) for t in orc.make_inputs(sq, skv, h, d, int(g["seed"])))
    res = lvx.run_distributed("lvx", Q, K, V, dO=dO, spec=lvx.ClusterSpec(n))
    assert orc.max_norm_error(res.O, g["O"]) <= 1e-4
    assert orc.max_norm_error(res.L, g["L"]) <= 1e-4
    assert orc.max_norm_error(res.grads.dQ, g["dQ"]) <= 1e-4
    assert orc.max_norm_error(res.grads.dK[:, g["dK_rows"]], g["dK_sample"]) <= 1e-4
    assert [tr.total_sent_bytes() for tr in res.traces_forward] == list(g["fwd_bytes"])
    assert [tr.total_sent_bytes() for tr in res.traces_backward] == list(g["bwd_bytes"])


def test_bf16_lvx_and_ring_world2_vs_oracle():
    """bf16 tensor-core path through the NCCL ring (spawned ranks), GQA 8/2."""
    import paper_2502_02406_b200 as lvx
    hq, hkv, sq, skv, d = 8, 2, 300, 5000, 128
    Q, K, V, G = orc.make_inputs(sq, skv, hq, d, seed=44, hkv=hkv)
    q, k, v, g = (torch.from_numpy(t).to(torch.bfloat16) for t in (Q, K, V, G))
    Qr, Kr, Vr, Gr = (t.double().numpy() for t in (q, k, v, g))
    O, L = orc.dense_attention(Qr, Kr, Vr)
    rq, rk, rv = orc.dense_attention_backward(Qr, Kr, Vr, O, L, Gr)
    n = min(torch.cuda.device_count(), 4)
    for strategy in ("lvx", "ring"):
        res = lvx.run_distributed(strategy, q, k, v, dO=g, spec=lvx.ClusterSpec(n))
        errs = {nm: orc.max_norm_error(a.float().numpy(), b) for nm, a, b in
                (("O", res.O, O), ("L", res.L, L), ("dQ", res.grads.dQ, rq),
                 ("dK", res.grads.dK, rk), ("dV", res.grads.dV, rv))}
        print(f"\n{strategy} bf16 n={n}:", errs)
        assert max(errs.values()) <= 1e-2
        w = lvx.volumes.Wire.b200(hq, hkv, d, 2)
        qs, ks = res.shards.q_sizes, res.shards.kv_sizes
        assert [t.total_sent_bytes() for t in res.traces_forward] == \
            lvx.volumes.bytes_by_worker(strategy, "forward", qs, ks, w)
        assert [t.total_sent_bytes() for t in res.traces_backward] == \
            lvx.volumes.bytes_by_worker(strategy, "backward", qs, ks, w)


def test_head_parallel_bf16_world_vs_oracle():
    """Ulysses head parallelism (§8(f) next 1) through NCCL all-to-all."""
    import paper_2502_02406_b200 as lvx
    n = min(torch.cuda.device_count(), 4)
    hq, hkv, sq, skv, d = 8, 4, 200, 3000, 128
    Q, K, V, G = orc.make_inputs(sq, skv, hq, d, seed=52, hkv=hkv)
    q, k, v, g = (torch.from_numpy(t).to(torch.bfloat16) for t in (Q, K, V, G))
    Qr, Kr, Vr, Gr = (t.double().numpy() for t in (q, k, v, g))
    O, L = orc.dense_attention(Qr, Kr, Vr)
    rq, rk, rv = orc.dense_attention_backward(Qr, Kr, Vr, O, L, Gr)
    res = lvx.run_distributed("head", q, k, v, dO=g, spec=lvx.ClusterSpec(n))
    errs = {nm: orc.max_norm_error(a.float().numpy(), b) for nm, a, b in
            (("O", res.O, O), ("L", res.L, L), ("dQ", res.grads.dQ, rq),
             ("dK", res.grads.dK, rk), ("dV", res.grads.dV, rv))}
    print(f"\nhead bf16 n={n}:", errs)
    assert max(errs.values()) <= 1e-2
    w = lvx.volumes.Wire.b200(hq, hkv, d, 2)
    qs, ks = res.shards.q_sizes, res.shards.kv_sizes
    assert [t.total_sent_bytes() for t in res.traces_forward] == \
        lvx.volumes.bytes_by_worker("head", "forward", qs, ks, w)
    assert [t.total_sent_bytes() for t in res.traces_backward] == \
        lvx.volumes.bytes_by_worker("head", "backward", qs, ks, w)
