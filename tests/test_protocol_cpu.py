"""The product's ring schedulers (lvx / ring, fwd + bwd) driven over a real
multi-process gloo group on CPU, with the oracle as the kernel set.  Checks
outputs and per-rank byte counters against the reference's golden vectors."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lvx_oracle as orc


def _port():
    """A fresh file-rendezvous path for one process group (no TCP port that
    another run could take between the probe and the bind)."""
    return os.path.join(tempfile.mkdtemp(prefix="lvx_gloo_"), "store")


def _worker(rank, n, port, cases, q):
    try:
        dist.init_process_group("gloo", init_method=f"file://{port}", rank=rank, world_size=n)
        from paper_2502_02406_b200.strategies import run_distributed
        from paper_2502_02406_b200.comm import ClusterSpec
        from tests.oracle_ops import OracleOps
        out = []
        for strategy, Q, K, V, dO in cases:
            res = run_distributed(strategy, Q, K, V, dO, ClusterSpec(n), ops=OracleOps())
            out.append((res.O, res.L, res.grads.dQ, res.grads.dK, res.grads.dV,
                        [t.total_sent_bytes() for t in res.traces_forward],
                        [t.total_sent_bytes() for t in res.traces_backward],
                        [res.stats.bytes_sent_by(i) for i in range(n)],
                        [t.num_rounds for t in res.traces_forward]))
        if rank == 0:
            q.put(("ok", out))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # noqa: BLE001
        import traceback
        q.put(("err", rank, traceback.format_exc()))


def run_group(n, cases):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, n, port, cases, q)) for r in range(n)]
    for p in ps:
        p.start()
    msg = q.get()
    for p in ps:
        p.join(timeout=120)
    assert msg[0] == "ok", msg
    return msg[1]


def _golden_cases(g, n):
    tags = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_n")})
    return [t for t in tags if int(g[t + "_n"]) == n]


@pytest.mark.parametrize("n", [2, 3, 4])
def test_gloo_protocols_match_reference(golden_strategies, n):
    g = golden_strategies
    tags = _golden_cases(g, n)
    if not tags:
        pytest.skip(f"no golden case with n={n}")
    cases = [(t.split("_")[1], g[t + "_Q"], g[t + "_K"], g[t + "_V"], g[t + "_dO"]) for t in tags]
    outs = run_group(n, cases)
    for t, (O, L, dQ, dK, dV, fb, bb, sb, rounds) in zip(tags, outs):
        tol = 1e-12 if t.endswith("float64") else 1e-5
        for name, arr in (("O", O), ("L", L), ("dQ", dQ), ("dK", dK), ("dV", dV)):
            assert arr.dtype == g[f"{t}_{name}"].dtype, (t, name)
            assert orc.max_norm_error(arr, g[f"{t}_{name}"]) <= tol, (t, name)
        assert fb == list(g[t + "_fwd_bytes"]), t
        assert bb == list(g[t + "_bwd_bytes"]), t
        assert sb == [a + b for a, b in zip(fb, bb)], t
        assert rounds == list(g[t + "_fwd_rounds"]), t


def test_gloo_gqa_lvx_and_ring_agree_with_oracle():
    # GQA (hq=4, hkv=2) is a B200 extension: pin it against the expanded oracle
    Q, K, V, dO = orc.make_inputs(7, 13, 4, 6, seed=31, hkv=2)
    outs = run_group(2, [("lvx", Q, K, V, dO), ("ring", Q, K, V, dO)])
    Od, Ld = orc.dense_attention(Q, K, V)
    dq, dk, dv = orc.dense_attention_backward(Q, K, V, Od, Ld, dO)
    for O, L, dQ, dK, dV, *_ in outs:
        for a, b in ((O, Od), (L, Ld), (dQ, dq), (dK, dk), (dV, dv)):
            assert orc.max_norm_error(a, b) <= 1e-12


def _ca_worker(rank, n, port, golden, policy, q):
    try:
        dist.init_process_group("gloo", init_method=f"file://{port}", rank=rank, world_size=n)
        from paper_2502_02406_b200.comm import DeviceContext
        from paper_2502_02406_b200.recompute import (CrossAttentionWeights, OpCounter, ca_backward,
                                                     ca_forward)
        from paper_2502_02406_b200.strategies import ShardSpec
        from tests.oracle_ops import OracleOps
        g = golden
        h, d, e = (int(v) for v in g["dims"])
        T = lambda a: torch.from_numpy(a)  # noqa: E731
        w = CrossAttentionWeights(T(g["w_q"]), T(g["w_k"]), T(g["w_v"]), T(g["w_o"]), h, h)
        sh = ShardSpec.balanced(g["x"].shape[0], g["y"].shape[0], n)
        (qa, qb), (ka, kb) = sh.q_ranges[rank], sh.kv_ranges[rank]
        ctx = DeviceContext(rank, n, group=dist.group.WORLD, device="cpu", ops=OracleOps())
        x_i, y_i, g_i = T(g["x"][qa:qb]), T(g["y"][ka:kb]), T(g["g"][qa:qb])
        out, saved = ca_forward(ctx, sh, x_i, y_i, w, policy)
        cnt = OpCounter()
        gr = ca_backward(ctx, sh, g_i, saved, y_i, w, counter=cnt)
        parts = [None] * n
        dist.all_gather_object(parts, (rank, out.numpy(), gr.d_x.numpy(), gr.d_y.numpy(),
                                       cnt.projection_flops))
        if rank == 0:
            parts.sort(key=lambda p: p[0])
            q.put(("ok", np.concatenate([p[1] for p in parts]),
                   np.concatenate([p[2] for p in parts]), np.concatenate([p[3] for p in parts]),
                   gr.w_q.numpy(), gr.w_k.numpy(), gr.w_v.numpy(), gr.w_o.numpy(),
                   sum(p[4] for p in parts)))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        q.put(("err", rank, traceback.format_exc()))


@pytest.mark.parametrize("policy", ["recompute", "store"])
def test_gloo_cross_attention_recompute_matches_reference(golden_mllm_ca, policy):
    n = 3
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    ps = [ctx.Process(target=_ca_worker, args=(r, n, port, golden_mllm_ca, policy, q))
          for r in range(n)]
    for p in ps:
        p.start()
    msg = q.get()
    for p in ps:
        p.join(timeout=120)
    assert msg[0] == "ok", msg
    _, out, dx, dy, gq, gk, gv, go, flops = msg
    g = golden_mllm_ca
    pol = policy
    for a, b in ((out, "out"), (dx, "dx"), (dy, "dy"), (gq, "gwq"), (gk, "gwk"), (gv, "gwv"),
                 (go, "gwo")):
        assert orc.max_norm_error(a, g[f"{pol}_{b}"]) <= 1e-12, b
    assert flops == int(g[f"{pol}_flops"])


def _stream_worker(rank, n, port, q):
    """lvx fwd+bwd with K/V streamed in 3 chunks (KVStream) vs the resident
    call on the same rank: identical up to the chunked merge (f64)."""
    try:
        dist.init_process_group("gloo", init_method=f"file://{port}", rank=rank, world_size=n)
        from paper_2502_02406_b200.comm import DeviceContext
        from paper_2502_02406_b200.strategies import (KVStream, ShardSpec, lvx_backward,
                                                      lvx_forward)
        from tests.oracle_ops import OracleOps
        Q, K, V, dO = (torch.from_numpy(t) for t in orc.make_inputs(96, 301, 4, 16, 5, hkv=2))
        shards = ShardSpec.balanced(96, 301, n)
        ctx = DeviceContext(rank, n, group=dist.group.WORLD, device=torch.device("cpu"),
                            ops=OracleOps())
        (qa, qb), (ka, kb) = shards.q_ranges[rank], shards.kv_ranges[rank]
        q_i, do_i = Q[:, qa:qb].contiguous(), dO[:, qa:qb].contiguous()
        k_i, v_i = K[:, ka:kb].contiguous(), V[:, ka:kb].contiguous()
        scale = 0.25
        st0 = lvx_forward(ctx, shards, q_i, k_i, v_i, scale)
        g0 = lvx_backward(ctx, shards, q_i, k_i, v_i, st0, do_i, scale)
        rows = k_i.shape[1]
        bounds = [(0, rows // 3), (rows // 3, 2 * rows // 3), (2 * rows // 3, rows)]
        waited, done = [], []
        kvs = KVStream(bounds=bounds, wait_chunk=waited.append,
                       dkv_done=lambda c, dk, dv: done.append((c, dk.clone(), dv.clone())))
        st1 = lvx_forward(ctx, shards, q_i, k_i, v_i, scale, kv_stream=kvs)
        g1 = lvx_backward(ctx, shards, q_i, k_i, v_i, st1, do_i, scale, kv_stream=kvs)
        errs = [orc.max_norm_error(a.numpy(), b.numpy())
                for a, b in ((st1.O, st0.O), (st1.L, st0.L), (g1[0], g0[0]), (g1[1], g0[1]),
                             (g1[2], g0[2]))]
        chunks_ok = [c for c, _, _ in done] == [0, 1, 2] and all(
            torch.equal(dk, g1[1][:, a:b]) and torch.equal(dv, g1[2][:, a:b])
            for (c, dk, dv), (a, b) in zip(done, bounds))
        if rank == 0:
            q.put(("ok", errs, waited[:3], chunks_ok))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        import traceback
        q.put(("err", rank, traceback.format_exc()))


@pytest.mark.parametrize("n", [1, 2])
def test_gloo_lvx_kv_stream_chunks(n):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    ps = [ctx.Process(target=_stream_worker, args=(r, n, port, q)) for r in range(n)]
    for p in ps:
        p.start()
    msg = q.get()
    for p in ps:
        p.join(timeout=120)
    assert msg[0] == "ok", msg
    _, errs, waited, chunks_ok = msg
    assert max(errs) <= 1e-12, errs
    assert waited == [0, 1, 2]
    assert chunks_ok


def test_gloo_n8_protocols_vs_oracle_simulation():
    """The rank count of the driver's largest scaling run (n = 8) over gloo:
    lvx / ring / head-parallel forward + backward with uneven shards (13 query
    rows) and empty ones (5 query rows: three ranks hold none) against the
    oracle's rank-by-rank simulation of the reference schedule (f64, 1e-12),
    per-rank byte counters included for the ring protocols."""
    cases = []
    for sq, skv, seed in ((13, 37, 81), (5, 19, 82)):
        Q, K, V, dO = orc.make_inputs(sq, skv, 8, 4, seed)
        for strategy in ("lvx", "ring", "head"):
            cases.append((strategy, Q, K, V, dO))
    outs = run_group(8, cases)
    for (strategy, Q, K, V, dO), (O, L, dQ, dK, dV, fb, bb, sb, rounds) in zip(cases, outs):
        sim = orc.simulate(strategy, Q, K, V, dO, n=8)
        for name, arr in (("O", O), ("L", L), ("dQ", dQ), ("dK", dK), ("dV", dV)):
            assert orc.max_norm_error(arr, getattr(sim, name)) <= 1e-12, (strategy, Q.shape, name)
        if strategy != "head":
            assert fb == list(sim.fwd_bytes), (strategy, fb, sim.fwd_bytes)
            assert bb == list(sim.bwd_bytes), (strategy, bb, sim.bwd_bytes)
