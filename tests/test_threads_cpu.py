"""Thread ranks (launch.spawn_ranks — the reference's spawn_cluster worker
model, cluster.py:300-335) on a host device with the oracle as the kernel
set: the product schedulers against the reference's golden vectors at every
rank count the goldens hold, and the failure semantics of
/root/reference/pkg/tests/test_cluster.py:158-205 (first failure named,
recv deadline, $LVX_TIMEOUT_SECS)."""
import time

import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc


def _tags(g):
    return sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_n")})


def test_thread_ranks_match_reference_goldens(golden_strategies):
    import paper_2502_02406_b200 as lvx
    from tests.oracle_ops import OracleOps
    g = golden_strategies
    for t in _tags(g):
        n = int(g[t + "_n"])
        res = lvx.run_distributed(t.split("_")[1], g[t + "_Q"], g[t + "_K"], g[t + "_V"],
                                  dO=g[t + "_dO"], spec=lvx.ClusterSpec(n), ops=OracleOps(),
                                  ranks="threads")
        tol = 1e-12 if t.endswith("float64") else 1e-5
        for name, arr in (("O", res.O), ("L", res.L), ("dQ", res.grads.dQ),
                          ("dK", res.grads.dK), ("dV", res.grads.dV)):
            assert arr.dtype == g[f"{t}_{name}"].dtype, (t, name)
            assert orc.max_norm_error(arr, g[f"{t}_{name}"]) <= tol, (t, name)
        fb = [tr.total_sent_bytes() for tr in res.traces_forward]
        bb = [tr.total_sent_bytes() for tr in res.traces_backward]
        assert fb == list(g[t + "_fwd_bytes"]), t
        assert bb == list(g[t + "_bwd_bytes"]), t
        assert [res.stats.bytes_sent_by(i) for i in range(n)] == \
            [a + b for a, b in zip(fb, bb)], t


@pytest.mark.parametrize("n", [5, 8])
def test_thread_ranks_uneven_and_empty_shards(n):
    """13 query rows (uneven) and 5 query rows (ranks without queries) at the
    driver's scaling rank counts, against the oracle's rank-by-rank
    simulation of the reference schedule."""
    import paper_2502_02406_b200 as lvx
    from tests.oracle_ops import OracleOps
    for sq, skv, seed in ((13, 37, 81), (5, 19, 82)):
        Q, K, V, dO = orc.make_inputs(sq, skv, 8, 4, seed)
        for strategy in ("lvx", "ring") + (("head",) if 8 % n == 0 else ()):
            res = lvx.run_distributed(strategy, Q, K, V, dO=dO, spec=lvx.ClusterSpec(n),
                                      ops=OracleOps(), ranks="threads")
            sim = orc.simulate(strategy, Q, K, V, dO, n=n)
            for name in ("O", "L", "dQ", "dK", "dV"):
                arr = getattr(res, name) if name in ("O", "L") else getattr(res.grads, name)
                assert orc.max_norm_error(arr, getattr(sim, name)) <= 1e-12, (strategy, name)
            if strategy != "head":
                assert [t.total_sent_bytes() for t in res.traces_forward] == list(sim.fwd_bytes)
                assert [t.total_sent_bytes() for t in res.traces_backward] == list(sim.bwd_bytes)


def _spawn(n, body, **kw):
    from paper_2502_02406_b200.launch import spawn_ranks
    from paper_2502_02406_b200.comm import ClusterSpec
    from tests.oracle_ops import OracleOps
    return spawn_ranks(ClusterSpec(n), body, device="cpu", ops_factory=OracleOps, **kw)


def test_worker_error_names_worker():
    from paper_2502_02406_b200.comm import WorkerFailed

    def body(ctx):
        if ctx.rank == 2:
            raise ValueError("boom")
        with ctx.call():
            t = torch.zeros(1, 1, 4)
            hop, _ = ctx.shift([t], [torch.empty(1, 1, 4)])
            hop.wait()

    with pytest.raises(WorkerFailed, match="worker 2") as ei:
        _spawn(4, body, timeout=5.0)
    assert ei.value.worker == 2
    assert isinstance(ei.value.cause, ValueError)


def test_recv_timeout_raises_collective_timeout():
    from paper_2502_02406_b200.comm import CollectiveTimeout, WorkerFailed

    def body(ctx):
        if ctx.rank == 0:
            with ctx.call():       # rank 1 never sends: the hop never arrives
                hop, _ = ctx.shift([torch.zeros(1, 1, 4)], [torch.empty(1, 1, 4)])
                hop.wait()

    t0 = time.monotonic()
    with pytest.raises(WorkerFailed, match="worker 0") as ei:
        _spawn(2, body, timeout=0.3)
    assert isinstance(ei.value.cause, CollectiveTimeout)
    assert time.monotonic() - t0 < 5.0


def test_timeout_env_override(monkeypatch):
    from paper_2502_02406_b200.comm import WorkerFailed
    monkeypatch.setenv("LVX_TIMEOUT_SECS", "0.2")

    def body(ctx):
        if ctx.rank == 0:
            with ctx.call():
                ctx.shift([torch.zeros(1, 1, 4)], [torch.empty(1, 1, 4)])[0].wait()

    t0 = time.monotonic()
    with pytest.raises(WorkerFailed):
        _spawn(2, body)
    assert time.monotonic() - t0 < 5.0


def test_all_to_all_chunk_count_mismatch():
    from paper_2502_02406_b200.comm import WorkerFailed

    def body(ctx):
        with ctx.call():
            ctx.all_to_all([[torch.zeros(1, 1, 1)]] * 3, [[torch.zeros(1, 1, 1)]] * 3)

    with pytest.raises(WorkerFailed, match="expects 2 chunks"):
        _spawn(2, body)


def test_stats_merge_over_ranks():
    def body(ctx):
        with ctx.call():
            t = torch.full((2, 3, 4), float(ctx.rank))
            r = torch.empty(2, 3, 4)
            ctx.shift([t], [r])[0].wait()
        return float(r[0, 0, 0])

    res = _spawn(3, body)
    assert res.results == [2.0, 0.0, 1.0]        # from the predecessor
    assert res.stats.total_bytes() == 3 * 2 * 3 * 4 * 4
    assert res.stats.link(0, 1).message_count == 1


@pytest.mark.parametrize("n", [2, 3, 5])
def test_message_counts_match_b200_schedule(n):
    """Per-link message counts of the B200 schedules (volumes.messages_per_rank:
    same bytes as the reference, dQ / dK-dV hops on their own messages)."""
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200 import volumes
    from tests.oracle_ops import OracleOps
    Q, K, V, dO = orc.make_inputs(11, 23, 2, 4, seed=3)
    for strategy in ("lvx", "ring"):
        res = lvx.run_distributed(strategy, Q, K, V, dO=dO, spec=lvx.ClusterSpec(n),
                                  ops=OracleOps(), ranks="threads")
        want = volumes.messages_per_rank(strategy, "forward", n) + \
            volumes.messages_per_rank(strategy, "backward", n)
        for i in range(n):
            assert res.stats.link(i, (i + 1) % n).message_count == want, (strategy, i)


@pytest.mark.parametrize("n", [2, 3, 5])
def test_ring_backward_reference_schedule_matches_oracle(n):
    """The Ring backward in the reference's compute-then-shift order gives the
    same gradients and bytes as the reference (oracle simulation)."""
    from paper_2502_02406_b200 import volumes
    from paper_2502_02406_b200.strategies import (RoundTrace, ShardSpec, ring_backward_reference_schedule,
                                                  ring_forward)
    Q, K, V, dO = orc.make_inputs(13, 29, 4, 8, seed=17, hkv=2)
    sim = orc.simulate("ring", Q, K, V, dO, n=n)
    sh = ShardSpec.balanced(13, 29, n)
    T = torch.from_numpy

    def body(ctx):
        (qa, qb), (ka, kb) = sh.q_ranges[ctx.rank], sh.kv_ranges[ctx.rank]
        q, k, v, g = T(Q[:, qa:qb]), T(K[:, ka:kb]), T(V[:, ka:kb]), T(dO[:, qa:qb])
        st = ring_forward(ctx, sh, q, k, v, 8 ** -0.5)
        tb = RoundTrace("ring", "backward")
        dq, dk, dv = ring_backward_reference_schedule(ctx, sh, q, k, v, st, g, 8 ** -0.5, tb)
        return dq.numpy(), dk.numpy(), dv.numpy(), tb.total_sent_bytes()

    res = _spawn(n, body)
    dq = np.concatenate([r[0] for r in res.results], axis=1)
    dk = np.concatenate([r[1] for r in res.results], axis=1)
    dv = np.concatenate([r[2] for r in res.results], axis=1)
    assert orc.max_norm_error(dq, sim.dQ) <= 1e-12
    assert orc.max_norm_error(dk, sim.dK) <= 1e-12
    assert orc.max_norm_error(dv, sim.dV) <= 1e-12
    assert [r[3] for r in res.results] == list(sim.bwd_bytes)
