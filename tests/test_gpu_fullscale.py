"""BASELINE configs[1] (C2, Llama-3-V: Lq 2048, hq 32, hkv 8, d 128, Lkv 1,048,576,
bf16) at FULL size on one B200, checked against the CPU oracle on sampled rows
(SURVEY.md §8(c) "full-scale parity"):

* query side: for sampled query rows the oracle runs the reference's own
  blockwise algorithm in f64 over ALL 1M KV rows in chunks (blockwise_attention
  + merge_states per chunk, then blockwise_attention_backward per chunk with
  the oracle's own L and D) -> O, L, dQ of those rows, independent of the GPU;
* KV side: dK / dV rows are independent given (L, D) of every query row, so for
  sampled KV rows the oracle's blockwise_attention_backward runs over all 2048
  query rows with L from the GPU forward (checked above) and D = rowsum(dO*O)
  from the GPU O in f64.

Tolerance (stated): max-normalised error <= 1e-2 against the f64 oracle on the
same bf16-rounded inputs, as the other bf16 tests.  Runtime ~1 min (the CPU
oracle over 1M KV rows dominates)."""
import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc

pytestmark = pytest.mark.gpu
TOL = 1e-2
HQ, HKV, SQ, SKV, D = 32, 8, 2048, 1 << 20, 128
Q_ROWS = [0, 777, 2047]
KV_ROWS = [0, 123457, 524288, 1048575]
CHUNK = 1 << 14   # KV rows per oracle chunk (expanded to hq heads in f64: 512 MB)


@pytest.fixture(scope="module")
def c2_run():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_02406_b200 import build
    build.build()
    from paper_2502_02406_b200.comm import DeviceContext
    from paper_2502_02406_b200.kernels import default_scale
    from paper_2502_02406_b200.strategies import ShardSpec, lvx_backward, lvx_forward
    g = torch.Generator(device="cuda").manual_seed(2502)

    def u(*shape):
        return (torch.rand(*shape, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    q, k, v, do = u(HQ, SQ, D), u(HKV, SKV, D), u(HKV, SKV, D), u(HQ, SQ, D)
    ctx = DeviceContext(0, 1)
    shards = ShardSpec.balanced(SQ, SKV, 1)
    scale = default_scale(D)
    st = lvx_forward(ctx, shards, q, k, v, scale)
    dq, dk, dv = lvx_backward(ctx, shards, q, k, v, st, do, scale)
    torch.cuda.synchronize()
    out = {"Q": q.double().cpu().numpy(), "dO": do.double().cpu().numpy(),
           "K": k.cpu(), "V": v.cpu(),   # bf16 on the host; f64 per chunk
           "O": st.O.double().cpu().numpy(), "L": st.L.double().cpu().numpy(),
           "dQ": dq.double().cpu().numpy(), "dK": dk[:, KV_ROWS].double().cpu().numpy(),
           "dV": dv[:, KV_ROWS].double().cpu().numpy(), "scale": scale}
    del q, k, v, do, st, dq, dk, dv
    torch.cuda.empty_cache()
    return out


def _kv_chunks(r):
    for a in range(0, SKV, CHUNK):
        yield (r["K"][:, a:a + CHUNK].double().numpy(), r["V"][:, a:a + CHUNK].double().numpy())


def test_c2_fullscale_sampled_query_rows(c2_run):
    r = c2_run
    Qs, dOs = r["Q"][:, Q_ROWS], r["dO"][:, Q_ROWS]
    O, L = np.zeros((HQ, len(Q_ROWS), D)), np.full((HQ, len(Q_ROWS)), -np.inf)
    for Kc, Vc in _kv_chunks(r):
        Oc, Lc = orc.blockwise_attention(Qs, Kc, Vc, r["scale"], tile_rows=CHUNK)
        O, L = orc.merge_states(O, L, Oc, Lc)
    Dv = orc.attention_row_stats(O, dOs)
    dQ = np.zeros_like(Qs)
    for Kc, Vc in _kv_chunks(r):
        dq_c, _, _ = orc.blockwise_attention_backward(Qs, Kc, Vc, L, Dv, dOs, r["scale"])
        dQ += dq_c
    errs = {"O": orc.max_norm_error(r["O"][:, Q_ROWS], O),
            "L": orc.max_norm_error(r["L"][:, Q_ROWS], L),
            "dQ": orc.max_norm_error(r["dQ"][:, Q_ROWS], dQ)}
    print(f"\nC2 full-scale, query rows {Q_ROWS}: {errs}")
    assert max(errs.values()) <= TOL, errs


def test_c2_fullscale_sampled_kv_rows(c2_run):
    r = c2_run
    Ks = r["K"][:, KV_ROWS].double().numpy()
    Vs = r["V"][:, KV_ROWS].double().numpy()
    Dv = orc.attention_row_stats(r["O"], r["dO"])
    _, dK, dV = orc.blockwise_attention_backward(r["Q"], Ks, Vs, r["L"], Dv, r["dO"], r["scale"])
    errs = {"dK": orc.max_norm_error(r["dK"], dK), "dV": orc.max_norm_error(r["dV"], dV)}
    print(f"\nC2 full-scale, kv rows {KV_ROWS}: {errs}")
    assert max(errs.values()) <= TOL, errs
