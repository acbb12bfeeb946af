"""K/V recompute cross-attention layer on the GPU (bf16 tensor-core path)."""
import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(e=256, hq=4, hkv=2, d=64, sq=96, skv=700, seed=8):
    from paper_2502_02406_b200.recompute import CrossAttentionWeights
    rnd = lambda s, st, sc=1.0: orc.seeded_random_tensor(seed, s, scale=sc, stream=st)  # noqa: E731
    ws = 0.5 / np.sqrt(e)
    x, y, g = rnd((sq, e), 1), rnd((skv, e), 2), rnd((sq, e), 3)
    wq, wk, wv, wo = rnd((e, hq * d), 4, ws), rnd((e, hkv * d), 5, ws), rnd((e, hkv * d), 6, ws), \
        rnd((hq * d, e), 7, ws)
    bf = lambda a: torch.from_numpy(a).to("cuda", torch.bfloat16)  # noqa: E731
    w = CrossAttentionWeights(bf(wq), bf(wk), bf(wv), bf(wo), hq, hkv)
    host = {k: t.double().cpu().numpy() for k, t in
            dict(x=bf(x), y=bf(y), g=bf(g), wq=w.w_q, wk=w.w_k, wv=w.w_v, wo=w.w_o).items()}
    return w, bf(x), bf(y), bf(g), host


def test_recompute_equals_store_and_saves_kv_memory():
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import (ActivationPolicy, OpCounter, activation_bytes,
                                                 ca_backward, ca_forward)
    w, x, y, g, _ = _setup()
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(x.shape[0], y.shape[0], 1)
    res, mem, ops = {}, {}, {}
    for pol in (ActivationPolicy.STORE_KV, ActivationPolicy.RECOMPUTE_KV):
        out, saved = ca_forward(ctx, sh, x, y, w, pol)
        mem[pol] = activation_bytes(saved)
        cnt = OpCounter()
        gr = ca_backward(ctx, sh, g, saved, y, w, counter=cnt)
        ops[pol] = cnt.projection_flops
        res[pol] = [out, gr.d_x, gr.d_y, gr.w_q, gr.w_k, gr.w_v, gr.w_o]
    for a, b in zip(res[ActivationPolicy.STORE_KV], res[ActivationPolicy.RECOMPUTE_KV]):
        assert torch.equal(a, b)          # the recompute GEMM reproduces K/V bit for bit
    kv_bytes = 2 * y.shape[0] * w.hkv * w.d * 2
    assert mem[ActivationPolicy.STORE_KV] - mem[ActivationPolicy.RECOMPUTE_KV] == kv_bytes
    e = x.shape[1]
    assert ops[ActivationPolicy.RECOMPUTE_KV] - ops[ActivationPolicy.STORE_KV] == \
        2 * 2 * y.shape[0] * e * w.hkv * w.d


def test_recompute_layer_vs_oracle():
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import ActivationPolicy, ca_backward, ca_forward
    w, x, y, g, h = _setup()
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(x.shape[0], y.shape[0], 1)
    out, saved = ca_forward(ctx, sh, x, y, w, ActivationPolicy.RECOMPUTE_KV)
    gr = ca_backward(ctx, sh, g, saved, y, w)
    ro, O, L = orc.ca_block_forward(h["x"], h["y"], h["wq"], h["wk"], h["wv"], h["wo"], w.hq, w.hkv)
    rdx, rdy, rq, rk, rv, rwo = orc.ca_block_backward(h["g"], h["x"], O, L, h["y"], h["wq"],
                                                      h["wk"], h["wv"], h["wo"], w.hq, w.hkv)
    errs = {n: orc.max_norm_error(a.double().cpu().numpy(), b) for n, a, b in
            (("out", out, ro), ("d_x", gr.d_x, rdx), ("d_y", gr.d_y, rdy), ("w_q", gr.w_q, rq),
             ("w_k", gr.w_k, rk), ("w_v", gr.w_v, rv), ("w_o", gr.w_o, rwo))}
    print("\nrecompute CA layer bf16 vs f64 oracle:", errs)
    assert max(errs.values()) <= 3e-2   # bf16 projections + bf16 attention operands


def test_chunked_recompute_matches_unchunked():
    """n = 1 RECOMPUTE_KV in K/V chunks (3 chunks + a ragged tail) vs the
    one-shot layer: same outputs and gradients up to the chunked merge /
    fp32 dQ accumulation order, i.e. bf16 rounding flips (max-normalised
    1e-2 as the other bf16 tests; one bf16 ulp near the max is ~7e-3), same
    recompute FLOP."""
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import ActivationPolicy, OpCounter, ca_backward, ca_forward
    w, x, y, g, _ = _setup()
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(x.shape[0], y.shape[0], 1)
    res, ops = {}, {}
    for chunk in (None, 200):
        out, saved = ca_forward(ctx, sh, x, y, w, ActivationPolicy.RECOMPUTE_KV, kv_chunk_rows=chunk)
        cnt = OpCounter()
        gr = ca_backward(ctx, sh, g, saved, y, w, counter=cnt)
        res[chunk] = [out, gr.d_x, gr.d_y, gr.w_q, gr.w_k, gr.w_v, gr.w_o]
        ops[chunk] = cnt.projection_flops
    for a, b in zip(res[None], res[200]):
        err = orc.max_norm_error(b.double().cpu().numpy(), a.double().cpu().numpy())
        assert err <= 1e-2, err
    assert ops[None] == ops[200]


def test_chunked_recompute_bounds_kv_transient():
    """The forward's peak allocation under chunked recompute stays below the
    one-shot layer's by about the full K/V minus one chunk."""
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import ActivationPolicy, ca_forward
    w, x, _, _, _ = _setup(e=256, hq=4, hkv=2, d=64, sq=128, skv=64)
    y = (torch.rand(65536, 256, device="cuda") * 2 - 1).bfloat16()
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(x.shape[0], y.shape[0], 1)
    peaks = {}
    for chunk in (None, 8192):
        ca_forward(ctx, sh, x, y, w, ActivationPolicy.RECOMPUTE_KV, kv_chunk_rows=chunk)  # warm-up
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        out, saved = ca_forward(ctx, sh, x, y, w, ActivationPolicy.RECOMPUTE_KV, kv_chunk_rows=chunk)
        torch.cuda.synchronize()
        peaks[chunk] = torch.cuda.max_memory_allocated() - base
        del out, saved
    full_kv = 2 * 65536 * w.hkv * w.d * 2
    chunk_kv = 2 * 8192 * w.hkv * w.d * 2
    assert peaks[None] - peaks[8192] >= 0.9 * (full_kv - chunk_kv), (peaks, full_kv)


@pytest.mark.parametrize("chunk,strategy", [(None, "lvx"), (200, "lvx"), (None, "ring")])
def test_visual_grad_sink_equals_per_layer_accumulation(chunk, strategy):
    """dY over three CA layers sharing y (src/mllm.py:368): the sink's ONE GEMM
    over the concatenated [dK|dV] blocks vs per-layer reduce-adds into an fp32
    accumulator.  Same bf16 products summed in fp32 in a different order, so
    1e-5 max-normalised; every other gradient is bit-identical."""
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200.recompute import (ActivationPolicy, CrossAttentionWeights,
                                                 VisualGradSink, ca_backward, ca_forward)
    w0, x, y, g, _ = _setup()
    gen = torch.Generator(device="cuda").manual_seed(5)
    layers = [w0] + [CrossAttentionWeights(
        *(((torch.rand(t.shape, device="cuda", generator=gen) * 2 - 1) * 0.03).bfloat16()
          for t in (w0.w_q, w0.w_k, w0.w_v, w0.w_o)), w0.hq, w0.hkv) for _ in range(2)]
    ctx = lvx.DeviceContext(0, 1)
    sh = lvx.ShardSpec.balanced(x.shape[0], y.shape[0], 1)
    saved = []
    for w in layers:
        _, sv = ca_forward(ctx, sh, x, y, w, ActivationPolicy.RECOMPUTE_KV, strategy=strategy,
                           kv_chunk_rows=chunk)
        saved.append(sv)
    acc = torch.zeros(y.shape, dtype=torch.float32, device="cuda")
    sink = VisualGradSink(y, [w.kv_weight().shape[1] for w in layers])
    ga, gb = [], []
    for w, sv in zip(reversed(layers), reversed(saved)):
        ga.append(ca_backward(ctx, sh, g, sv, y, w, strategy=strategy, d_y_acc=acc))
        gb.append(ca_backward(ctx, sh, g, sv, y, w, strategy=strategy, dy_sink=sink))
    dy = sink.finish(ctx)
    assert dy.dtype == torch.float32 and gb[0].d_y is None
    # y's dtype straight from the GEMM epilogue = the fp32 sum rounded once
    assert torch.equal(sink.finish(ctx, dtype=torch.bfloat16), dy.bfloat16())
    err = orc.max_norm_error(dy.double().cpu().numpy(), acc.double().cpu().numpy())
    assert err <= 1e-5, err
    for a, b in zip(ga, gb):
        for f in ("d_x", "w_q", "w_k", "w_v", "w_o"):
            assert torch.equal(getattr(a, f), getattr(b, f)), f
    with pytest.raises(ValueError):
        sink.slot(layers[0].kv_weight())            # every slot is taken
