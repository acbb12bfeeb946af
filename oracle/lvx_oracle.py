"""CPU restatement of the LV-XAttn reference path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 product in
``paper_2502_02406_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it, and
only as the thing the GPU result is compared against (or as the timed CPU
baseline).  The product path never routes through here.

Parity is PINNED: ``tests/test_oracle.py`` checks every function below against
golden vectors produced by the reference package itself
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src/lvxattn``
and stores its outputs in ``tests/golden/*.npz``).

Everything is float64 internally, exactly like the reference
(``pkg/src/lvxattn/kernels.py:1-8``); results are cast to the numpy result
dtype of the inputs.  Layout is ``[heads, rows, d]``; the merged
log-sum-exp ``L = m + log(l)`` of the *scaled* scores is the softmax
statistic, ``(O=0, L=-inf)`` the empty state.

GQA extension (not in the reference, which is MHA-only —
``SPEC.md:176``): query head ``a`` reads key/value head ``a // (hq // hkv)``.
``expand_kv`` / ``reduce_kv_grad`` express GQA through the MHA oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# synthetic inputs — pkg/src/lvxattn/tensorio.py:62-82
# ---------------------------------------------------------------------------


def seeded_random_tensor(seed: int, shape, dtype=np.float64, scale: float = 1.0,
                         stream: int = 0) -> np.ndarray:
    """U[-scale, scale] drawn in f64 from Philox keyed (seed, stream), then cast
    (tensorio.py:62-82).  Same bits as the reference for the same key."""
    shape = tuple(int(s) for s in shape)
    if not shape or any(s <= 0 for s in shape):
        raise ValueError("empty shape")
    bitgen = np.random.Philox(key=[int(seed) & (2**64 - 1), int(stream)])
    return np.random.Generator(bitgen).uniform(-scale, scale, size=shape).astype(dtype)


def make_inputs(s_q: int, s_kv: int, h: int, d: int, seed: int, hkv: int | None = None):
    """(Q, K, V, dO) on streams 0..3 (verify.py:88-93); ``hkv`` adds GQA."""
    hkv = h if hkv is None else hkv
    return (seeded_random_tensor(seed, (h, s_q, d), stream=0),
            seeded_random_tensor(seed, (hkv, s_kv, d), stream=1),
            seeded_random_tensor(seed, (hkv, s_kv, d), stream=2),
            seeded_random_tensor(seed, (h, s_q, d), stream=3))


def max_norm_error(actual, expected) -> float:
    """max|a-e| / max|e| with matching -inf treated equal (verify.py:54-68)."""
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    if a.shape != e.shape:
        return math.inf
    both = np.isneginf(a) & np.isneginf(e)
    a = np.where(both, 0.0, a)
    e = np.where(both, 0.0, e)
    if not (np.isfinite(a).all() and np.isfinite(e).all()):
        return math.inf
    if e.size == 0:
        return 0.0
    diff = float(np.abs(a - e).max())
    denom = float(np.abs(e).max())
    return diff / denom if denom else diff


# ---------------------------------------------------------------------------
# attention math — pkg/src/lvxattn/kernels.py
# ---------------------------------------------------------------------------


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)          # kernels.py:58-59


def _f64(*ts):
    return [np.asarray(t).astype(np.float64, copy=False) for t in ts]


def expand_kv(t: np.ndarray, hq: int) -> np.ndarray:
    """[hkv, S, d] -> [hq, S, d]: q head a reads kv head a // (hq // hkv)."""
    hkv = t.shape[0]
    if hq % hkv:
        raise ValueError(f"q heads {hq} not a multiple of kv heads {hkv}")
    return np.repeat(t, hq // hkv, axis=0)


def reduce_kv_grad(g: np.ndarray, hkv: int) -> np.ndarray:
    """[hq, S, d] -> [hkv, S, d]: sum the gradient over each GQA group."""
    hq, s, d = g.shape
    return g.reshape(hkv, hq // hkv, s, d).sum(axis=1)


def dense_attention(Q, K, V, scale=None):
    """Materialised softmax oracle (kernels.py:80-102).  Returns (O, L)."""
    out_dt = np.result_type(Q, K, V)
    h, sq, d = Q.shape
    scale = default_scale(d) if scale is None else scale
    if K.shape[1] == 0:
        return np.zeros((h, sq, d), out_dt), np.full((h, sq), -np.inf, out_dt)
    q, k, v = _f64(Q, expand_kv(K, h), expand_kv(V, h))
    s = scale * (q @ k.transpose(0, 2, 1))
    m = s.max(axis=2, keepdims=True)
    w = np.exp(s - m)
    tot = w.sum(axis=2, keepdims=True)
    o = (w @ v) / tot
    lse = (m + np.log(tot))[..., 0]
    return o.astype(out_dt), lse.astype(out_dt)


def blockwise_attention(Q, K, V, scale=None, tile_rows: int = 64):
    """Online-softmax partial state of one KV block (kernels.py:105-141):
    KV tiles of ``tile_rows``; running (m, l); O/=l; L = m + log l."""
    if tile_rows < 1:
        raise ValueError(f"tile_rows must be >= 1, got {tile_rows}")
    out_dt = np.result_type(Q, K, V)
    h, sq, d = Q.shape
    skv = K.shape[1]
    scale = default_scale(d) if scale is None else scale
    if skv == 0:
        return np.zeros((h, sq, d), out_dt), np.full((h, sq), -np.inf, out_dt)
    q, k, v = _f64(Q, expand_kv(K, h), expand_kv(V, h))
    run_max = np.full((h, sq), -np.inf)
    run_sum = np.zeros((h, sq))
    acc = np.zeros((h, sq, d))
    step = min(tile_rows, skv)
    for lo in range(0, skv, step):
        kt, vt = k[:, lo:lo + step], v[:, lo:lo + step]
        st = scale * (q @ kt.transpose(0, 2, 1))
        new_max = np.maximum(run_max, st.max(axis=2))
        p = np.exp(st - new_max[..., None])
        corr = np.exp(run_max - new_max)
        run_sum = corr * run_sum + p.sum(axis=2)
        acc = corr[..., None] * acc + (p @ vt)
        run_max = new_max
    return (acc / run_sum[..., None]).astype(out_dt), \
        (run_max + np.log(run_sum)).astype(out_dt)


def merge_states(Oa, La, Ob, Lb):
    """LSE merge of two partial states (kernels.py:144-161).  Rows that are
    empty in both inputs stay (0, -inf); the empty state is an exact identity."""
    if np.shape(Oa) != np.shape(Ob):
        raise ValueError(f"state shape mismatch: {np.shape(Oa)} vs {np.shape(Ob)}")
    out_dt = np.result_type(Oa, Ob)
    la, lb = _f64(La, Lb)
    lse = np.logaddexp(la, lb)
    safe = np.where(np.isneginf(lse), 0.0, lse)
    oa, ob = _f64(Oa, Ob)
    o = np.exp(la - safe)[..., None] * oa + np.exp(lb - safe)[..., None] * ob
    return o.astype(out_dt), lse.astype(out_dt)


def attention_row_stats(O, dO):
    """D = rowsum(dO * O) in f64 (kernels.py:164-169)."""
    if np.shape(dO) != np.shape(O):
        raise ValueError(f"dO shape {np.shape(dO)} != O shape {np.shape(O)}")
    o, g = _f64(O, dO)
    return (o * g).sum(axis=2)


def blockwise_attention_backward(Q, K, V, L, D, dO, scale=None):
    """Additive (dQ+, dK+, dV+) of one (Q block, KV block) pair given the final
    forward statistics L and D of the query rows (kernels.py:192-224).
    GQA: dK/dV are summed over each query-head group."""
    out_dt = np.result_type(Q, K, V)
    h, sq, d = Q.shape
    hkv = K.shape[0]
    scale = default_scale(d) if scale is None else scale
    q, k, v, g, lse, dd = _f64(Q, expand_kv(K, h), expand_kv(V, h), dO, L, D)
    p = np.exp(scale * (q @ k.transpose(0, 2, 1)) - lse[..., None])
    dv = (p.transpose(0, 2, 1) @ g)
    ds = p * ((g @ v.transpose(0, 2, 1)) - dd[..., None])
    dq = scale * (ds @ k)
    dk = scale * (ds.transpose(0, 2, 1) @ q)
    return (dq.astype(out_dt), reduce_kv_grad(dk, hkv).astype(out_dt),
            reduce_kv_grad(dv, hkv).astype(out_dt))


def dense_attention_backward(Q, K, V, O, L, dO, scale=None):
    """Full backward from saved (O, L) (kernels.py:172-189)."""
    return blockwise_attention_backward(Q, K, V, L, attention_row_stats(O, dO), dO, scale)


def project(x, W, heads: int):
    """x [S, e] @ W [e, h*d] -> [h, S, d]; head k owns cols [kd, (k+1)d)
    (kernels.py:227-240)."""
    if x.shape[1] != W.shape[0]:
        raise ValueError(f"inner dims disagree: input {x.shape[1]} vs weight {W.shape[0]}")
    if W.shape[1] % heads:
        raise ValueError(f"weight cols {W.shape[1]} not divisible by heads {heads}")
    out_dt = np.result_type(x, W)
    xf, wf = _f64(x, W)
    flat = xf @ wf
    return np.ascontiguousarray(
        flat.reshape(x.shape[0], heads, -1).transpose(1, 0, 2)).astype(out_dt)


def project_backward(x, W, dOut):
    """(dX = dOut_flat W^T, dW = x^T dOut_flat) (kernels.py:243-254)."""
    out_dt = np.result_type(x, W)
    h, s, d = dOut.shape
    g = np.asarray(dOut, np.float64).transpose(1, 0, 2).reshape(s, h * d)
    xf, wf = _f64(x, W)
    return (g @ wf.T).astype(out_dt), (xf.T @ g).astype(out_dt)


# ---------------------------------------------------------------------------
# sharding — pkg/src/lvxattn/strategies.py:47-99
# ---------------------------------------------------------------------------


def partition_rows(total: int, n: int):
    """Balanced contiguous ranges, first ``total % n`` ranks get +1 row."""
    if n < 1:
        raise ValueError(f"worker count must be >= 1, got {n}")
    if total < 0:
        raise ValueError(f"row count must be >= 0, got {total}")
    q, r = divmod(total, n)
    edges = [0]
    for i in range(n):
        edges.append(edges[-1] + q + (i < r))
    return list(zip(edges[:-1], edges[1:]))


# ---------------------------------------------------------------------------
# the four ring protocols, simulated rank-by-rank in one process
# (strategies.py:175-361).  Byte counts follow cluster.py:8-11: payload bytes
# only, loopback free.
# ---------------------------------------------------------------------------


@dataclass
class SimResult:
    O: np.ndarray
    L: np.ndarray
    dQ: np.ndarray | None = None
    dK: np.ndarray | None = None
    dV: np.ndarray | None = None
    fwd_bytes: list = field(default_factory=list)   # per rank
    bwd_bytes: list = field(default_factory=list)
    fwd_rounds: int = 0


def _nb(*arrays) -> int:
    return int(sum(np.asarray(a).nbytes for a in arrays))


def simulate(strategy: str, Q, K, V, dO=None, n: int = 1, scale=None, tile_rows: int = 64):
    """Run the reference's ``lvx`` or ``ring`` schedule for n ranks in lock-step
    and gather O, L (and grads).  Messages are exchanged as lists indexed by
    the destination rank, so round semantics are identical to the threaded
    reference (strategies.py:193-231 lvx fwd, :243-276 lvx bwd, :287-311 ring
    fwd, :322-361 ring bwd)."""
    if strategy == "head":
        return _simulate_head(Q, K, V, dO, n, scale)
    if strategy not in ("lvx", "ring"):
        raise ValueError(f"unknown strategy {strategy!r}")
    h, sq, d = Q.shape
    skv = K.shape[1]
    dt = np.result_type(Q, K, V)
    scale = default_scale(d) if scale is None else scale
    qr, kr = partition_rows(sq, n), partition_rows(skv, n)
    qs = [Q[:, a:b] for a, b in qr]
    ks = [K[:, a:b] for a, b in kr]
    vs = [V[:, a:b] for a, b in kr]
    succ = lambda i: (i + 1) % n  # noqa: E731
    fwd_b = [0] * n
    bwd_b = [0] * n

    def ship(i, payload, counter):
        if succ(i) != i:
            counter[i] += _nb(*payload)
        return payload

    if strategy == "lvx":
        # state of block (i+1) starts empty; Q_i is the first block consumed
        send_state = []
        for i in range(n):
            rows = qr[(i + 1) % n][1] - qr[(i + 1) % n][0]
            send_state.append((np.zeros((h, rows, d), dt), np.full((h, rows), -np.inf, dt)))
        q_cur = list(qs)
        for r in range(n):
            inbox = [None] * n
            deltas = [blockwise_attention(q_cur[i], ks[i], vs[i], scale, tile_rows)
                      for i in range(n)]
            for i in range(n):
                inbox[succ(i)] = ship(i, (send_state[i][0], send_state[i][1], q_cur[i]), fwd_b)
            for i in range(n):
                o_in, l_in, q_in = inbox[i]
                send_state[i] = merge_states(o_in, l_in, *deltas[i])
                q_cur[i] = q_in
        home = [None] * n
        for i in range(n):
            home[succ(i)] = ship(i, send_state[i], fwd_b)
        O = np.concatenate([home[i][0] for i in range(n)], axis=1).astype(dt)
        Lf = np.concatenate([home[i][1] for i in range(n)], axis=1).astype(dt)
    else:
        states = [(np.zeros((h, b - a, d), dt), np.full((h, b - a), -np.inf, dt)) for a, b in qr]
        kv = [(ks[i], vs[i]) for i in range(n)]
        for r in range(n):
            inbox = [None] * n
            if r < n - 1:
                for i in range(n):
                    inbox[succ(i)] = ship(i, kv[i], fwd_b)
            for i in range(n):
                states[i] = merge_states(*states[i], *blockwise_attention(
                    qs[i], kv[i][0], kv[i][1], scale, tile_rows))
            if r < n - 1:
                kv = inbox
        O = np.concatenate([s[0] for s in states], axis=1).astype(dt)
        Lf = np.concatenate([s[1] for s in states], axis=1).astype(dt)

    res = SimResult(O=O, L=Lf, fwd_bytes=fwd_b, fwd_rounds=n)
    if dO is None:
        return res

    dos = [dO[:, a:b] for a, b in qr]
    Ls = [Lf[:, a:b] for a, b in qr]
    Os = [O[:, a:b] for a, b in qr]
    Ds = [attention_row_stats(Os[i], dos[i]).astype(dt) for i in range(n)]
    if strategy == "lvx":
        tup = [(qs[i], dos[i], Ls[i], Ds[i], np.zeros_like(qs[i])) for i in range(n)]
        dk = [np.zeros_like(k) for k in ks]
        dv = [np.zeros_like(v) for v in vs]
        for r in range(n):
            inbox = [None] * n
            for i in range(n):
                qj, doj, lj, dj, dqj = tup[i]
                gq, gk, gv = blockwise_attention_backward(qj, ks[i], vs[i], lj, dj, doj, scale)
                dk[i] = dk[i] + gk
                dv[i] = dv[i] + gv
                inbox[succ(i)] = ship(i, (qj, doj, lj, dj, dqj + gq), bwd_b)
            tup = inbox
        res.dQ = np.concatenate([tup[i][4] for i in range(n)], axis=1)
        res.dK = np.concatenate(dk, axis=1)
        res.dV = np.concatenate(dv, axis=1)
    else:
        dq = [np.zeros_like(q) for q in qs]
        cur = [(ks[i], vs[i], np.zeros_like(ks[i]), np.zeros_like(vs[i])) for i in range(n)]
        for r in range(n):
            inbox = [None] * n
            for i in range(n):
                kc, vc, dkc, dvc = cur[i]
                gq, gk, gv = blockwise_attention_backward(qs[i], kc, vc, Ls[i], Ds[i], dos[i], scale)
                dq[i] = dq[i] + gq
                cur[i] = (kc, vc, dkc + gk, dvc + gv)
                if r < n - 1:
                    inbox[succ(i)] = ship(i, cur[i], bwd_b)
            if r < n - 1:
                cur = inbox
        home = [None] * n
        for i in range(n):
            home[succ(i)] = ship(i, cur[i][2:], bwd_b)
        res.dQ = np.concatenate(dq, axis=1)
        res.dK = np.concatenate([home[i][0] for i in range(n)], axis=1)
        res.dV = np.concatenate([home[i][1] for i in range(n)], axis=1)
    res.bwd_bytes = bwd_b
    return res


def _simulate_head(Q, K, V, dO, n, scale):
    """Head parallelism (strategies.py:364-432): every rank attends over the
    full sequence for h/n heads; results equal the dense oracle.  Bytes are
    the per-message payloads of the two all-to-alls per pass, src != dst."""
    h, sq, d = Q.shape
    hk = K.shape[0]
    if h % n or hk % n:
        raise ValueError(f"head count {h} not divisible by workers {n}")
    dt = np.result_type(Q, K, V)
    b = np.dtype(dt).itemsize
    qs = [b_ - a for a, b_ in partition_rows(sq, n)]
    ks = [b_ - a for a, b_ in partition_rows(K.shape[1], n)]
    O, L = dense_attention(Q, K, V, scale)
    fwd = [(n - 1) * (qs[i] * h + 2 * ks[i] * hk) // n * d * b +
           sum(qs[w] for w in range(n) if w != i) * (h // n) * (d + 1) * b for i in range(n)]
    if n == 1:
        fwd = [0]
    res = SimResult(O=O.astype(dt), L=L.astype(dt), fwd_bytes=fwd, fwd_rounds=1)
    if dO is None:
        return res
    dq, dk, dv = dense_attention_backward(Q, K, V, O, L, dO, scale)
    res.dQ, res.dK, res.dV = dq, dk, dv
    res.bwd_bytes = [0] if n == 1 else [
        ((n - 1) * qs[i] * h // n + sum(qs[w] * h + 2 * ks[w] * hk for w in range(n) if w != i)
         // n) * d * b for i in range(n)]
    return res


# ---------------------------------------------------------------------------
# closed-form volumes — pkg/src/lvxattn/volumes.py:71-120 (GQA-aware:
# K/V/dK/dV rows carry hkv*d elements, the rest hq*d / hq)
# ---------------------------------------------------------------------------


def lvx_forward_bytes(q_sizes, hq, d, b_o, b_l=None, b_q=None):
    n = len(q_sizes)
    if n == 1:
        return [0]
    b_l = b_o if b_l is None else b_l
    b_q = b_o if b_q is None else b_q
    ol = lambda rows: rows * hq * (d * b_o + b_l)  # noqa: E731
    out = []
    for i in range(n):
        tot = sum(ol(q_sizes[(i - r + 1) % n]) + q_sizes[(i - r) % n] * hq * d * b_q
                  for r in range(n))
        out.append(tot + ol(q_sizes[(i + 1) % n]))
    return out


def lvx_backward_bytes(q_sizes, hq, d, b):
    n = len(q_sizes)
    return [0] if n == 1 else [sum(q_sizes) * hq * (3 * d + 2) * b] * n


def ring_forward_bytes(kv_sizes, hkv, d, b):
    n = len(kv_sizes)
    if n == 1:
        return [0]
    return [sum(kv_sizes[(i - r) % n] for r in range(n - 1)) * 2 * hkv * d * b
            for i in range(n)]


def ring_backward_bytes(kv_sizes, hkv, d, b):
    n = len(kv_sizes)
    if n == 1:
        return [0]
    return [(sum(kv_sizes[(i - r) % n] for r in range(n - 1)) * 4
             + kv_sizes[(i + 1) % n] * 2) * hkv * d * b for i in range(n)]


def attention_flops(s_q, s_kv, hq, d, backward: bool = True) -> float:
    """4 (fwd) + 10 (bwd) x Sq Skv h d (analytics.py:113-115)."""
    return (14.0 if backward else 4.0) * s_q * s_kv * hq * d


# ---------------------------------------------------------------------------
# cross-attention block with K/V recompute — pkg/src/lvxattn/mllm.py
# ---------------------------------------------------------------------------


def _flat_heads(t):
    h, s, d = t.shape
    return np.ascontiguousarray(t.transpose(1, 0, 2)).reshape(s, h * d)


def _unflat_heads(t, h):
    s, hd = t.shape
    return np.ascontiguousarray(t.reshape(s, h, hd // h).transpose(1, 0, 2))


def ca_block_forward(x, y, w_q, w_k, w_v, w_o, hq, hkv=None, scale=None):
    """mllm.py:290-301: q = x W_Q, k = y W_K, v = y W_V, attention,
    out = x + flatten(O) W_O.  Returns (out, O, L)."""
    hkv = hq if hkv is None else hkv
    q, k, v = project(x, w_q, hq), project(y, w_k, hkv), project(y, w_v, hkv)
    O, L = blockwise_attention(q, k, v, scale)
    return x + _flat_heads(O) @ w_o, O, L


def ca_block_backward(g, x, O, L, y, w_q, w_k, w_v, w_o, hq, hkv=None, scale=None):
    """mllm.py:343-370 (either policy — both recompute q from x; K/V come
    from y).  Returns (d_x, d_y, g_wq, g_wk, g_wv, g_wo)."""
    hkv = hq if hkv is None else hkv
    d_o = _unflat_heads(g @ w_o.T, hq)
    g_wo = _flat_heads(O).T @ g
    q, k, v = project(x, w_q, hq), project(y, w_k, hkv), project(y, w_v, hkv)
    dq, dk, dv = dense_attention_backward(q, k, v, O, L, d_o, scale)
    d_x_q, g_wq = project_backward(x, w_q, dq)
    d_y_k, g_wk = project_backward(y, w_k, dk)
    d_y_v, g_wv = project_backward(y, w_v, dv)
    return g + d_x_q, d_y_k + d_y_v, g_wq, g_wk, g_wv, g_wo


# ---------------------------------------------------------------------------
# toy MLLM stack, memory ledger, frame budget — pkg/src/lvxattn/mllm.py
# ---------------------------------------------------------------------------


def mllm_stack_forward(x0, y, ca_params: dict, lm_params: list, ca_positions, hq, hkv=None,
                       store_kv: bool = False, scale=None):
    """mllm.py:274-305: for every block, a CA layer first when the block is
    in ``ca_positions`` (x += flatten(O) W_O), then u = x, x = u + tanh(u W1) W2.
    ``ca_params[pos] = (w_q, w_k, w_v, w_o)``, ``lm_params[i] = (w1, w2)``.
    Returns (out, saved) with saved = {"lm_inputs": [...], "ca": {pos: {...}}}."""
    saved = {"lm_inputs": [], "ca": {}}
    x = x0
    for blk, (w1, w2) in enumerate(lm_params):
        if blk in ca_positions:
            w_q, w_k, w_v, w_o = ca_params[blk]
            xn, O, L = ca_block_forward(x, y, w_q, w_k, w_v, w_o, hq, hkv, scale)
            entry = {"x": x, "O": O, "L": L}
            if store_kv:   # mllm.py:297-299
                h2 = hq if hkv is None else hkv
                entry["K"], entry["V"] = project(y, w_k, h2), project(y, w_v, h2)
            saved["ca"][blk] = entry
            x = xn
        saved["lm_inputs"].append(x)
        x = x + np.tanh(x @ w1) @ w2
    return x, saved


def mllm_stack_backward(g, saved, y, ca_params: dict, lm_params: list, ca_positions, hq,
                        hkv=None, scale=None):
    """mllm.py:314-371 (both policies give the same gradients).  Returns
    (d_x0, d_y, {pos: (g_wq, g_wk, g_wv, g_wo)}, [(g_w1, g_w2)])."""
    d_y = np.zeros_like(y, dtype=np.float64)
    ca_g, lm_g = {}, [None] * len(lm_params)
    for blk in reversed(range(len(lm_params))):
        w1, w2 = lm_params[blk]
        u = saved["lm_inputs"][blk]
        t = np.tanh(u @ w1)
        d_pre = (g @ w2.T) * (1.0 - t * t)
        lm_g[blk] = (u.T @ d_pre, t.T @ g)
        g = g + d_pre @ w1.T
        if blk in ca_positions:
            e = saved["ca"][blk]
            g, dy, *gw = ca_block_backward(g, e["x"], e["O"], e["L"], y, *ca_params[blk],
                                           hq, hkv, scale)
            d_y = d_y + dy
            ca_g[blk] = tuple(gw)
    return g, d_y, ca_g, lm_g


def analytic_ledger(num_lm_blocks, num_ca_layers, d_embed, h, d, s_q, s_kv, store_kv: bool,
                    b: int, hkv=None, b_state=None, b_params=None):
    """mllm.py:190-210 peak activation ledger.  With one element size b (and
    hkv = h) it is the reference's formula; the extra arguments express the
    B200 layout: K/V with hkv heads, O/L in the fp32 state dtype (b_state),
    parameters in their own dtype (b_params)."""
    hkv = h if hkv is None else hkv
    b_state = b if b_state is None else b_state
    b_params = b if b_params is None else b_params
    c = num_ca_layers
    params = (c * (2 * d_embed * h * d + 2 * d_embed * hkv * d) +
              num_lm_blocks * 2 * d_embed * d_embed) * b_params
    yb = s_kv * d_embed * b
    x = s_q * d_embed * b if c else 0
    o_l = (s_q * h * d + s_q * h) * b_state if c else 0
    kv = 2 * s_kv * hkv * d * b if (c and store_kv) else 0
    peak = params + yb + c * (x + o_l + kv)
    return {"params_bytes": params, "visual_features_y": yb, "per_layer_saved_x": x,
            "per_layer_saved_o_l": o_l, "per_layer_saved_kv": kv, "num_ca_layers": c,
            "peak_total": peak}


def max_frames_under_budget(peak_of_frames, budget_bytes: int) -> int:
    """mllm.py:374-397: largest frame count whose peak fits; 0 when even the
    frame-independent part does not (doubling, then bisection)."""
    if budget_bytes <= 0:
        raise ValueError(f"budget must be positive, got {budget_bytes}")
    if peak_of_frames(0) > budget_bytes:
        return 0
    lo, hi = 0, 1
    while peak_of_frames(hi) <= budget_bytes:
        lo, hi = hi, hi * 2
        if hi > 2 ** 60:
            raise ValueError("budget admits an absurd frame count; check inputs")
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if peak_of_frames(mid) <= budget_bytes:
            lo = mid
        else:
            hi = mid
    return lo
