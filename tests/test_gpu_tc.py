"""bf16 tensor-core (tcgen05/TMEM/TMA) path vs the oracle.

Tolerance (stated): max-normalised error <= 1e-2 against the
f64 oracle evaluated on the SAME bf16-rounded inputs; the dominant error is
P rounded to bf16 before the PV MMA (emulated bound ~2e-3 at C1)."""

import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc

pytestmark = pytest.mark.gpu
TOL_BF16 = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_02406_b200 import build
    build.build()


def bf16_inputs(hq, hkv, sq, skv, d, seed, q_scale=1.0):
    Q, K, V, dO = orc.make_inputs(sq, skv, hq, d, seed, hkv=hkv)
    Q = Q * q_scale
    ts = [torch.from_numpy(t).to("cuda", torch.bfloat16) for t in (Q, K, V, dO)]
    f64 = [t.double().cpu().numpy() for t in ts]
    return ts, f64


SHAPES = [  # hq, hkv, sq, skv, d
    (1, 1, 128, 128, 128), (2, 2, 200, 1000, 128), (8, 2, 77, 515, 64), (4, 1, 256, 4096, 128),
    (8, 8, 128, 4096, 64), (3, 3, 5, 7, 128), (32, 8, 64, 640, 128), (2, 1, 300, 129, 64),
    # one query tile per kv head -> KV-pair mode (even KV tile counts): ragged
    # last tile, one step per tile; and an odd count that stays in normal mode
    (4, 4, 100, 2000, 128), (2, 2, 128, 256, 64), (2, 2, 64, 384, 128)]


@pytest.mark.parametrize("shape", SHAPES)
def test_tc_forward_vs_oracle(shape):
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200 import _lib
    hq, hkv, sq, skv, d = shape
    (q, k, v, _), (Q, K, V, _) = bf16_inputs(hq, hkv, sq, skv, d, seed=hash(shape) % 1000)
    assert _lib.load().lvx_tc_eligible(_lib.view(q), _lib.view(k)) == 1
    st = lvx.blockwise_attention(q, k, v)
    torch.cuda.synchronize()
    O, L = orc.blockwise_attention(Q, K, V)
    eo = orc.max_norm_error(st.O.cpu().numpy(), O)
    el = orc.max_norm_error(st.L.cpu().numpy(), L)
    print(f"\nTC fwd {shape}: O err {eo:.2e}  L err {el:.2e}")
    assert eo <= TOL_BF16 and el <= TOL_BF16


def test_tc_forward_sharp_scores_rescale():
    # Q x 8 makes the running max jump across KV tiles: exercises the lazy O rescale
    import paper_2502_02406_b200 as lvx
    (q, k, v, _), (Q, K, V, _) = bf16_inputs(2, 1, 130, 2000, 128, seed=9, q_scale=8.0)
    st = lvx.blockwise_attention(q, k, v)
    O, L = orc.blockwise_attention(Q, K, V)
    eo = orc.max_norm_error(st.O.cpu().numpy(), O)
    el = orc.max_norm_error(st.L.cpu().numpy(), L)
    print(f"\nTC fwd sharp: O err {eo:.2e}  L err {el:.2e}")
    assert eo <= TOL_BF16 and el <= TOL_BF16


@pytest.mark.parametrize("growth", [0.5, 4.0])
def test_tc_forward_growing_scores_fallback(growth):
    # K rows scaled up tile by tile: the row max rises on every KV tile, so the
    # single-pass softmax must reject its P (row sum over bound) and redo the
    # tile through the two-pass path with an O rescale
    import paper_2502_02406_b200 as lvx
    (q, k, v, _), _ = bf16_inputs(2, 1, 200, 1500, 128, seed=21, q_scale=2.0)
    ramp = 1.0 + growth * torch.arange(1500, device="cuda", dtype=torch.float32) / 128.0
    k = (k.float() * ramp[None, :, None]).to(torch.bfloat16)
    Q, K, V = (t.double().cpu().numpy() for t in (q, k, v))
    st = lvx.blockwise_attention(q, k, v)
    O, L = orc.blockwise_attention(Q, K, V)
    eo = orc.max_norm_error(st.O.cpu().numpy(), O)
    el = orc.max_norm_error(st.L.cpu().numpy(), L)
    assert np.isfinite(st.O.cpu().numpy()).all()
    print(f"\nTC fwd growing x{growth}: O err {eo:.2e}  L err {el:.2e}")
    assert eo <= TOL_BF16 and el <= TOL_BF16


def test_tc_forward_prior_merge_and_split_combine():
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200 import kernels as Kn
    (q, k, v, _), (Q, K, V, _) = bf16_inputs(4, 2, 160, 6000, 128, seed=4)
    half = 2500
    # prior = state of the first KV block, then fused finish merges the second
    a = lvx.blockwise_attention(q, k[:, :half], v[:, :half])
    O = torch.empty(q.shape, dtype=torch.float32, device="cuda")
    L = torch.empty(q.shape[:2], dtype=torch.float32, device="cuda")
    k2, v2 = k[:, half:].contiguous(), v[:, half:].contiguous()
    ws = Kn.workspace(Kn.fwd_workspace_bytes(q, k2))
    Kn.fwd_partial(q, k2, v2, 1 / np.sqrt(128), ws)
    Kn.fwd_finish(q, k2, ws, O, L, a.O, a.L)
    Od, Ld = orc.dense_attention(Q, K, V)
    eo = orc.max_norm_error(O.cpu().numpy(), Od)
    el = orc.max_norm_error(L.cpu().numpy(), Ld)
    print(f"\nTC fwd merge: O err {eo:.2e}  L err {el:.2e}")
    assert eo <= TOL_BF16 and el <= TOL_BF16


def test_tc_matches_simt_fp32_on_same_inputs():
    """The tensor-core bf16 path against the exact SIMT path run in fp32 on
    the same (bf16-rounded) inputs."""
    import paper_2502_02406_b200 as lvx
    (q, k, v, _), _ = bf16_inputs(8, 2, 256, 3000, 128, seed=12)
    tc = lvx.blockwise_attention(q, k, v)
    si = lvx.blockwise_attention(q.float(), k.float(), v.float())
    e = orc.max_norm_error(tc.O.cpu().numpy(), si.O.cpu().numpy())
    print(f"\nTC bf16 vs SIMT fp32: {e:.2e}")
    assert e <= TOL_BF16


def test_tc_forward_large_vs_torch_fp32():
    """Per-GPU round shape of C2 (Llama-3-V, n=8) at 1/8 KV: torch fp32 reference."""
    import paper_2502_02406_b200 as lvx
    torch.manual_seed(0)
    hq, hkv, sq, skv, d = 32, 8, 256, 16384, 128
    q = (torch.rand(hq, sq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(hkv, skv, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(hkv, skv, d, device="cuda") * 2 - 1).bfloat16()
    st = lvx.blockwise_attention(q, k, v)
    ke = k.float().repeat_interleave(hq // hkv, 0)
    ve = v.float().repeat_interleave(hq // hkv, 0)
    s = (q.float() @ ke.transpose(1, 2)) / np.sqrt(d)
    ref_l = torch.logsumexp(s, dim=-1)
    ref_o = torch.softmax(s, dim=-1) @ ve
    eo = ((st.O - ref_o).abs().max() / ref_o.abs().max()).item()
    el = ((st.L - ref_l).abs().max() / ref_l.abs().max()).item()
    print(f"\nTC fwd C2-round: O err {eo:.2e}  L err {el:.2e}")
    assert eo <= TOL_BF16 and el <= TOL_BF16


BWD_SHAPES = [  # hq, hkv, sq, skv, d
    (1, 1, 128, 128, 128), (2, 2, 200, 1000, 128), (8, 2, 77, 515, 64), (4, 1, 256, 2048, 128),
    (3, 3, 5, 7, 128), (32, 8, 64, 640, 128), (2, 1, 300, 129, 64), (4, 4, 128, 3000, 64)]


@pytest.mark.parametrize("shape", BWD_SHAPES)
def test_tc_backward_vs_oracle(shape):
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200 import _lib
    hq, hkv, sq, skv, d = shape
    (q, k, v, g), (Q, K, V, G) = bf16_inputs(hq, hkv, sq, skv, d, seed=17 + sq)
    O, L = orc.dense_attention(Q, K, V)
    D = orc.attention_row_stats(O, G)
    Lt = torch.from_numpy(L).float().cuda()
    Dt = torch.from_numpy(D).float().cuda()
    assert _lib.load().lvx_blockwise_bwd_workspace(_lib.view(q), _lib.view(k)) > 0
    dq, dk, dv = lvx.blockwise_attention_backward(q, k, v, Lt, Dt, g)
    rq, rk, rv = orc.blockwise_attention_backward(Q, K, V, L, D, G)
    errs = [orc.max_norm_error(a.float().cpu().numpy(), b) for a, b in ((dq, rq), (dk, rk), (dv, rv))]
    print(f"\nTC bwd {shape}: dQ {errs[0]:.2e} dK {errs[1]:.2e} dV {errs[2]:.2e}")
    assert max(errs) <= TOL_BF16


def test_tc_backward_accumulates():
    from paper_2502_02406_b200 import kernels as Kn
    (q, k, v, g), (Q, K, V, G) = bf16_inputs(4, 2, 130, 700, 128, seed=3)
    O, L = orc.dense_attention(Q, K, V)
    D = orc.attention_row_stats(O, G)
    Lt, Dt = torch.from_numpy(L).float().cuda(), torch.from_numpy(D).float().cuda()
    dq = torch.ones(q.shape, device="cuda")
    dk = torch.ones(k.shape, device="cuda")
    dv = torch.ones(v.shape, device="cuda")
    Kn.bwd_accumulate(q, k, v, Lt, Dt, g, 1 / np.sqrt(128), dq, dk, dv, accumulate=True)
    rq, rk, rv = orc.blockwise_attention_backward(Q, K, V, L, D, G)
    for a, b in ((dq, rq), (dk, rk), (dv, rv)):
        assert orc.max_norm_error(a.cpu().numpy() - 1.0, b) <= TOL_BF16


def test_tc_lvx_fwd_bwd_single_gpu_vs_oracle():
    """lvx_forward + lvx_backward (n=1 loopback schedule) on bf16 device tensors."""
    import paper_2502_02406_b200 as lvx
    (q, k, v, g), (Q, K, V, G) = bf16_inputs(8, 2, 192, 2500, 128, seed=21)
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(192, 2500, 1)
    st, (dq, dk, dv), _, _ = lvx.run_rank("lvx", ctx, sh, q, k, v, g)
    O, L = orc.dense_attention(Q, K, V)
    rq, rk, rv = orc.dense_attention_backward(Q, K, V, O, L, G)
    errs = {n: orc.max_norm_error(a.float().cpu().numpy(), b) for n, a, b in
            (("O", st.O, O), ("L", st.L, L), ("dQ", dq, rq), ("dK", dk, rk), ("dV", dv, rv))}
    print("\nlvx bf16 n=1 errors:", errs)
    assert max(errs.values()) <= TOL_BF16


def test_tc_backward_large_vs_torch_fp32():
    """C2 per-round shape at 1/16 KV against torch fp32 autograd."""
    import paper_2502_02406_b200 as lvx
    torch.manual_seed(1)
    hq, hkv, sq, skv, d = 32, 8, 256, 8192, 128
    q = (torch.rand(hq, sq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(hkv, skv, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(hkv, skv, d, device="cuda") * 2 - 1).bfloat16()
    g = (torch.rand(hq, sq, d, device="cuda") * 2 - 1).bfloat16()
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    ke, ve = kf.repeat_interleave(hq // hkv, 0), vf.repeat_interleave(hq // hkv, 0)
    s = (qf @ ke.transpose(1, 2)) / np.sqrt(d)
    o = torch.softmax(s, -1) @ ve
    o.backward(g.float())
    L = torch.logsumexp(s, -1).detach()
    D = (o.detach() * g.float()).sum(-1)
    dq, dk, dv = lvx.blockwise_attention_backward(q, k, v, L, D, g)
    errs = [((a.float() - b).abs().max() / b.abs().max()).item()
            for a, b in ((dq, qf.grad), (dk, kf.grad), (dv, vf.grad))]
    print(f"\nTC bwd C2-round/16: dQ {errs[0]:.2e} dK {errs[1]:.2e} dV {errs[2]:.2e}")
    assert max(errs) <= TOL_BF16


@pytest.mark.parametrize("shape", [(2, 2, 200, 1000, 128), (8, 2, 130, 700, 64), (32, 8, 256, 2048, 128)])
def test_tc_kernels_bit_deterministic(shape):
    """No atomics anywhere: repeated launches must be bit-identical.  Doubles
    as a race detector for the warp-specialised pipelines (a TMEM/SMEM hazard
    shows up as run-to-run differences)."""
    import paper_2502_02406_b200 as lvx
    hq, hkv, sq, skv, d = shape
    (q, k, v, g), (Q, K, V, G) = bf16_inputs(hq, hkv, sq, skv, d, seed=77)
    O, L = orc.dense_attention(Q, K, V)
    D = orc.attention_row_stats(O, G)
    Lt, Dt = torch.from_numpy(L).float().cuda(), torch.from_numpy(D).float().cuda()
    base = None
    for _ in range(12):
        st = lvx.blockwise_attention(q, k, v)
        grads = lvx.blockwise_attention_backward(q, k, v, Lt, Dt, g)
        cur = [st.O.clone(), st.L.clone()] + [t.clone() for t in grads]
        if base is None:
            base = cur
        else:
            for a, b in zip(cur, base):
                assert torch.equal(a, b)


def _random_shapes(n=12, seed=2502):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        hkv = int(rng.choice([1, 2, 3, 4, 8]))
        hq = hkv * int(rng.choice([1, 2, 4, 8]))
        out.append((hq, hkv, int(rng.integers(1, 300)), int(rng.integers(1, 2600)),
                    int(rng.choice([64, 128]))))
    return out


@pytest.mark.parametrize("shape", _random_shapes())
def test_tc_random_shapes_fwd_bwd_vs_oracle(shape):
    """Seeded random GQA shapes (ragged rows, tiny and single-row blocks) through
    the bf16 tensor-core path: the full LV-XAttn layer at n = 1 (forward, dQ
    and the batched bf16 dK/dV pass) against the f64 oracle, 1e-2."""
    import paper_2502_02406_b200 as lvx
    hq, hkv, sq, skv, d = shape
    (q, k, v, g), (Q, K, V, G) = bf16_inputs(hq, hkv, sq, skv, d, seed=sum(shape))
    ctx = lvx.DeviceContext(0, 1)
    st, (dq, dk, dv), _, _ = lvx.run_rank("lvx", ctx, lvx.ShardSpec.balanced(sq, skv, 1),
                                          q, k, v, g)
    O, L = orc.dense_attention(Q, K, V)
    dQ, dK, dV = orc.dense_attention_backward(Q, K, V, O, L, G)
    got = {"O": st.O, "L": st.L, "dQ": dq, "dK": dk, "dV": dv}
    errs = {n: orc.max_norm_error(t.double().cpu().numpy(), ref)
            for (n, t), ref in zip(got.items(), (O, L, dQ, dK, dV))}
    assert max(errs.values()) <= TOL_BF16, (shape, errs)


@pytest.mark.parametrize("q_scale", [4.0, 8.0])
def test_tc_forward_second_half_fallback(q_scale):
    # scores jump only in kv rows [64, 128) of every 128-row tile, x3 per tile:
    # the forward publishes P in halves, so the first half of a tile is
    # accepted and already in the PV MMA when the second half fails its bound
    # — the path that waits for that PV, rescales O / l and redoes the half
    # (every KV split sees the jump between its consecutive tiles)
    import paper_2502_02406_b200 as lvx
    (q, k, v, _), _ = bf16_inputs(2, 1, 200, 1536, 128, seed=33, q_scale=q_scale)
    rows = torch.arange(1536, device="cuda")
    scale = torch.where((rows % 128) >= 64, 3.0 ** (rows // 128).float(),
                        torch.ones_like(rows, dtype=torch.float32))
    k = (k.float() * scale[None, :, None]).to(torch.bfloat16)
    Q, K, V = (t.double().cpu().numpy() for t in (q, k, v))
    st = lvx.blockwise_attention(q, k, v)
    O, L = orc.blockwise_attention(Q, K, V)
    eo = orc.max_norm_error(st.O.cpu().numpy(), O)
    el = orc.max_norm_error(st.L.cpu().numpy(), L)
    print(f"\nTC fwd second-half fallback q x{q_scale}: O err {eo:.2e}  L err {el:.2e}")
    assert eo <= TOL_BF16 and el <= TOL_BF16


def test_tc_two_devices_one_process():
    # kernel attributes (227 KB dynamic SMEM) are per device context: one
    # process driving two GPUs must launch on both (skipped on 1-GPU boxes)
    import paper_2502_02406_b200 as lvx
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    (q, k, v, g), (Q, K, V, G) = bf16_inputs(4, 1, 256, 1024, 128, seed=5)
    O, L = orc.blockwise_attention(Q, K, V)
    for dev in (0, 1, 0):
        with torch.cuda.device(dev):
            qd, kd, vd, gd = (t.to(f"cuda:{dev}") for t in (q, k, v, g))
            st = lvx.blockwise_attention(qd, kd, vd)
            D = lvx.attention_row_stats(st, gd)
            grads = lvx.blockwise_attention_backward(qd, kd, vd, st.L, D, gd)
            torch.cuda.synchronize(dev)
            assert orc.max_norm_error(st.O.cpu().numpy(), O) <= TOL_BF16
            assert all(torch.isfinite(t).all() for t in grads)


def _rand_shapes(n, seed):
    """Seeded random bf16 tensor-core shapes: GQA groups 1-4, ragged query and
    KV tails, d in {64, 128}."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        hkv = int(rng.integers(1, 4))
        hq = hkv * int(rng.choice([1, 2, 4]))
        sq = int(rng.integers(1, 400))
        skv = int(rng.integers(1, 3000))
        d = int(rng.choice([64, 128]))
        out.append((hq, hkv, sq, skv, d))
    return out


@pytest.mark.parametrize("shape", _rand_shapes(12, 2026))
def test_tc_random_shapes_fwd_bwd_vs_oracle(shape):
    """Forward + backward (dQ, dK, dV) on seeded random shapes against the f64
    oracle, gated at 2x torch SDPA's bf16 error on the same inputs
    (tests/sdpa_ref.py)."""
    from tests import sdpa_ref
    from paper_2502_02406_b200 import kernels as K
    hq, hkv, sq, skv, d = shape
    (q, k, v, g), (Q, Kr, Vr, G) = bf16_inputs(hq, hkv, sq, skv, d, seed=sum(shape))
    scale = d ** -0.5
    st = K.blockwise_attention(q, k, v)
    D = K.attention_row_stats(st, g)
    dq, dk, dv = K.blockwise_attention_backward(q, k, v, st.L, D, g)
    torch.cuda.synchronize()
    O, L = orc.dense_attention(Q, Kr, Vr)
    rq, rk, rv = orc.dense_attention_backward(Q, Kr, Vr, O, L, G)
    want = {"O": O, "L": L, "dQ": rq, "dK": rk, "dV": rv}
    ours = sdpa_ref.errors({"O": st.O.float().cpu(), "L": st.L.cpu(), "dQ": dq.float().cpu(),
                            "dK": dk.float().cpu(), "dV": dv.float().cpu()}, want)
    so, sq_, sk, sv = (t.float().cpu() for t in sdpa_ref.sdpa_grads(q, k, v, g, scale))
    sdpa = sdpa_ref.errors({"O": so, "dQ": sq_, "dK": sk, "dV": sv}, want)
    print(f"\nrandom {shape}: ours {ours}\n    sdpa {sdpa}")
    assert not sdpa_ref.gate(ours, sdpa), sdpa_ref.gate(ours, sdpa)
