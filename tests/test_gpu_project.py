"""Projection entry points (lvx_project / lvx_project_bwd / lvx_kv_recompute /
lvx_gemm: the library's tcgen05 GEMM behind the C ABI) vs the reference's
golden vectors and vs torch.

Tolerances: f64 1e-12 and f32 1e-5 max-normalised against the reference's own
outputs (tests/golden/golden_kernels.npz: kernels.py:227-254 run in this
container); bf16 layouts against a torch fp32 matmul of the same bf16 inputs,
1e-2."""
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


@pytest.mark.parametrize("dt,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_project_vs_reference(golden_kernels, dt, tol):
    from paper_2502_02406_b200 import kernels as K
    g = golden_kernels
    x, W, gr = (g[k].astype(dt) for k in ("proj_x", "proj_W", "proj_g"))
    out = K.project(x, W, 2)
    dx, dw = K.project_backward(x, W, gr)
    assert out.dtype == dt and dx.dtype == dt
    assert orc.max_norm_error(out, g["proj_out"]) <= tol
    assert orc.max_norm_error(dx, g["proj_dX"]) <= tol
    assert orc.max_norm_error(dw, g["proj_dW"]) <= tol


def _bf(*shape, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.rand(*shape, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)


def _err(a, b):
    return orc.max_norm_error(a.double().cpu().numpy(), b.double().cpu().numpy())


@pytest.mark.parametrize("interleaved", [True, False])
def test_project_head_layouts_bf16(interleaved):
    """One GEMM into column blocks of [S, h*d] vs strided-batched GEMM into a
    contiguous [h, S, d] output; project_bwd with flat vs per-head dOut."""
    from paper_2502_02406_b200 import kernels as K
    S, e, h, d = 300, 256, 4, 64
    x, W = _bf(S, e, seed=1), _bf(e, h * d, seed=2)
    if interleaved:
        out = torch.empty(S, h * d, dtype=torch.bfloat16, device="cuda").view(S, h, d).transpose(0, 1)
    else:
        out = torch.empty(h, S, d, dtype=torch.bfloat16, device="cuda")
    K.project_into(x, W, out)
    ref = (x.float() @ W.float()).view(S, h, d).transpose(0, 1)
    assert _err(out, ref) <= 1e-2
    g = _bf(h, S, d, seed=3)
    if interleaved:
        g = g.transpose(0, 1).contiguous().transpose(0, 1)   # [h, S, d] view, head stride d
    dx = torch.empty_like(x)
    dw = torch.empty_like(W)
    K.project_backward_into(x, W, g, dx, dw)
    gf = g.float().transpose(0, 1).reshape(S, h * d)
    assert _err(dx, gf @ W.float().T) <= 1e-2
    assert _err(dw, x.float().T @ gf) <= 1e-2


@pytest.mark.parametrize("fused", [True, False])
def test_kv_recompute_bf16(fused):
    from paper_2502_02406_b200 import kernels as K
    S, e, hkv, d = 513, 384, 2, 128
    y = _bf(S, e, seed=4)
    wkv = _bf(e, 2 * hkv * d, seed=5)
    wk, wv = (wkv[:, :hkv * d], wkv[:, hkv * d:]) if fused else \
        (wkv[:, :hkv * d].contiguous(), wkv[:, hkv * d:].contiguous())
    if fused:
        kv = torch.empty(S, 2 * hkv * d, dtype=torch.bfloat16, device="cuda")
        k = kv[:, :hkv * d].view(S, hkv, d).transpose(0, 1)
        v = kv[:, hkv * d:].view(S, hkv, d).transpose(0, 1)
    else:
        k = torch.empty(hkv, S, d, dtype=torch.bfloat16, device="cuda")
        v = torch.empty(hkv, S, d, dtype=torch.bfloat16, device="cuda")
    K.kv_recompute(y, wk, wv, k, v)
    ref = (y.float() @ wkv.float()).view(S, 2 * hkv, d).transpose(0, 1)
    assert _err(k, ref[:hkv]) <= 1e-2 and _err(v, ref[hkv:]) <= 1e-2


GEMM_SHAPES = [  # M, N, K
    (128, 256, 64), (300, 264, 200), (1000, 1024, 512), (7, 8, 9),
    (256, 256, 65536),          # few tiles, tall K: split-K with fp32 reduce
    (4096, 1024, 4096),         # many tiles, persistent loop over both TMEM buffers
]


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_tcgen05_gemm_vs_torch_fp32(shape, ta, tb):
    """lvx_gemm (tcgen05 kernel, all four operand majors) against a torch fp32
    matmul of the same bf16 operands.  Gate 4e-3 max-normalised: one bf16
    rounding of the output is up to half an ulp, 2^-8 of the largest element
    (3.9e-3), plus fp32 summation order."""
    from paper_2502_02406_b200 import kernels as K
    M, N, Kd = shape
    a = _bf(*((Kd, M) if ta else (M, Kd)), seed=M + 3 * N)
    b = _bf(*((N, Kd) if tb else (Kd, N)), seed=Kd + 7)
    ref = (a.float().T if ta else a.float()) @ (b.float().T if tb else b.float())
    c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    K.gemm_into(a, ta, b, tb, c)
    e1 = _err(c, ref)
    c0 = _bf(M, N, seed=11)
    c2 = c0.clone()
    K.gemm_into(a, ta, b, tb, c2, accumulate=True)
    e2 = _err(c2, ref + c0.float())
    print(f"\ngemm {shape} ta={ta} tb={tb}: {e1:.2e} / accumulate {e2:.2e}")
    assert e1 <= 4e-3 and e2 <= 4e-3


def test_gemm_strided_operands():
    """Leading dimensions larger than the logical widths (column blocks of a
    wider matrix), as the recompute layer's [W_K | W_V] halves are."""
    from paper_2502_02406_b200 import kernels as K
    big_a, big_b = _bf(640, 1024, seed=21), _bf(1024, 768, seed=22)
    a, b = big_a[:, 256:768], big_b[256:768, 128:640]
    out = torch.empty(640, 1024, dtype=torch.bfloat16, device="cuda")[:, 256:768]
    K.gemm_into(a, False, b, False, out)
    assert _err(out, a.float() @ b.float()) <= 4e-3


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_simt_gemm_exact_dtypes(dt):
    from paper_2502_02406_b200 import kernels as K
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.rand(77, 130, device="cuda", generator=g, dtype=dt)
    b = torch.rand(90, 130, device="cuda", generator=g, dtype=dt)
    c = torch.empty(77, 90, device="cuda", dtype=dt)
    K.gemm_into(a, False, b, True, c)
    ref = a.double() @ b.double().T
    assert _err(c, ref) <= (1e-6 if dt == torch.float32 else 1e-13)


@pytest.mark.parametrize("shape", [(300, 264, 200), (256, 256, 65536), (1000, 1024, 512)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_gemm_bf16_into_fp32(shape, accumulate):
    """bf16 operands into an fp32 C (the visual tokens' gradient accumulator
    shared by the CA layers): stored or reduce-added in the epilogue, one or
    several K splits.  Only fp32 summation order differs from torch (1e-5)."""
    from paper_2502_02406_b200 import kernels as K
    M, N, Kd = shape
    a, b = _bf(M, Kd, seed=31), _bf(N, Kd, seed=32)
    ref = a.float() @ b.float().T
    c0 = torch.randn(M, N, device="cuda") if accumulate else torch.full((M, N), float("nan"),
                                                                         device="cuda")
    c = c0.clone()
    K.gemm_into(a, False, b, True, c, accumulate=accumulate)
    want = ref + c0 if accumulate else ref
    e = _err(c, want)
    print(f"\ngemm bf16->fp32 {shape} acc={accumulate}: {e:.2e}")
    assert e <= 1e-5


@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("accumulate", [False, True])
def test_split_k_gemm_is_deterministic(out_dtype, accumulate):
    """A tall-K product with few output tiles runs split-K (every split stores
    its own fp32 slice; the finish sums them in a fixed order), so repeated
    calls give the same bits — the weight gradients y^T dKV / x^T dQ of the
    layers are such products."""
    from paper_2502_02406_b200 import kernels as K
    a, b = _bf(65536, 512, seed=41), _bf(65536, 256, seed=42)   # a^T b: M 512, N 256, K 65536
    c0 = _bf(512, 256, seed=43).to(out_dtype)
    outs = []
    for _ in range(3):
        c = c0.clone() if accumulate else torch.empty(512, 256, dtype=out_dtype, device="cuda")
        K.gemm_into(a, True, b, False, c, accumulate=accumulate)
        outs.append(c)
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    ref = a.float().T @ b.float() + (c0.float() if accumulate else 0)
    assert _err(outs[0], ref) <= (4e-3 if out_dtype == torch.bfloat16 else 1e-5)
