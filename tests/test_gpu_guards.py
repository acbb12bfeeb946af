"""Out-of-bounds-write guards for the sm_100a kernels (compute-sanitizer is
closed on this GPU pool, so bad accesses are hunted with canaries instead).

Every output is a strided view into a larger buffer whose padding rows,
padding columns and padding heads hold a NaN canary; after the kernels run,
every canary must be untouched and every output element finite.  Shapes are
ragged (row counts not multiples of the 128-row tiles, KV tails, several
heads) so tile-edge predicates are exercised.  Inputs sit in guarded views
too, with the canary in their padding: a kernel that READ past its rows would
turn outputs into NaN."""
import pytest
import torch

pytestmark = pytest.mark.gpu

NAN = float("nan")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_02406_b200 import build
    build.build()


def guarded(h, rows, d, dtype, fill=None, pad_rows=37, pad_cols=16, pad_heads=1, seed=0):
    """A [h, rows, d] view into a NaN-filled [h + pad_heads, rows + pad_rows,
    d + pad_cols] buffer (row stride d + pad_cols, a multiple of 8 elements)."""
    buf = torch.full((h + pad_heads, rows + pad_rows, d + pad_cols), NAN, dtype=dtype,
                     device="cuda")
    view = buf[:h, :rows, :d]
    if fill == "rand":
        g = torch.Generator(device="cuda").manual_seed(seed)
        view.copy_((torch.rand(h, rows, d, device="cuda", generator=g) * 2 - 1).to(dtype))
    return buf, view


def guarded2(h, rows, dtype, pad_rows=37, pad_heads=1):
    buf = torch.full((h + pad_heads, rows + pad_rows), NAN, dtype=dtype, device="cuda")
    return buf, buf[:h, :rows]


def check(buf, view, name):
    torch.cuda.synchronize()
    mask = torch.ones_like(buf, dtype=torch.bool)
    if view.dim() == 3:
        mask[:view.shape[0], :view.shape[1], :view.shape[2]] = False
    else:
        mask[:view.shape[0], :view.shape[1]] = False
    outside = buf[mask]
    assert torch.isnan(outside.float()).all(), f"{name}: a kernel wrote outside its view"
    assert torch.isfinite(view.float()).all(), f"{name}: non-finite output (read past the view?)"


@pytest.mark.parametrize("shape", [(4, 2, 200, 700, 128), (2, 2, 77, 300, 64),
                                   (8, 8, 129, 1000, 64), (32, 8, 64, 640, 128)])
def test_attention_kernels_stay_in_bounds(shape):
    from paper_2502_02406_b200 import kernels as K
    hq, hkv, sq, skv, d = shape
    bf = torch.bfloat16
    _, q = guarded(hq, sq, d, bf, "rand", seed=1)
    _, k = guarded(hkv, skv, d, bf, "rand", seed=2)
    _, v = guarded(hkv, skv, d, bf, "rand", seed=3)
    _, g = guarded(hq, sq, d, bf, "rand", seed=4)
    scale = d ** -0.5
    # forward: partial + finish into guarded O / L
    bo, o = guarded(hq, sq, d, torch.float32)
    bl, l = guarded2(hq, sq, torch.float32)
    ws = K.workspace(K.fwd_workspace_bytes(q, k), slot=0)
    K.fwd_partial(q, k, v, scale, ws)
    K.fwd_finish(q, k, ws, o, l)
    check(bo, o, "fwd O")
    check(bl, l, "fwd L")
    # row stats
    bD, D = guarded2(hq, sq, torch.float32)
    K.row_stats_into(o, g, D)
    check(bD, D, "row_stats")
    # dQ (partial + finish) and dK / dV (bf16 overwrite and fp32 accumulate)
    bq, dq = guarded(hq, sq, d, torch.float32)
    wsb = K.workspace(K.bwd_workspace_bytes(q, k), slot=1)
    K.bwd_dq_partial(q, k, v, l, D, g, scale, wsb)
    K.bwd_dq_finish(q, k, wsb, dq, accumulate=False)
    check(bq, dq, "dQ")
    for dt, acc in ((bf, False), (torch.float32, True)):
        bk, dk = guarded(hkv, skv, d, dt)
        bv, dv = guarded(hkv, skv, d, dt)
        if acc:
            dk.zero_()
            dv.zero_()
        K.bwd_dkv(q, k, v, l, D, g, scale, dk, dv, accumulate=acc)
        check(bk, dk, f"dK {dt}")
        check(bv, dv, f"dV {dt}")
    # merge
    bm, mo = guarded(hq, sq, d, torch.float32)
    bml, ml = guarded2(hq, sq, torch.float32)
    K.merge_into(o, l, o, l, mo, ml)
    check(bm, mo, "merge O")
    check(bml, ml, "merge L")


@pytest.mark.parametrize("mnk,ta,tb", [((300, 264, 200), False, False),
                                       ((129, 512, 1000), False, True),
                                       ((256, 136, 65536), True, False),
                                       ((200, 256, 96), True, True)])
def test_gemm_stays_in_bounds(mnk, ta, tb):
    from paper_2502_02406_b200 import kernels as K
    M, N, Kd = mnk
    g = torch.Generator(device="cuda").manual_seed(M)

    def mat(r, c):
        buf = torch.full((r + 19, c + 24), NAN, dtype=torch.bfloat16, device="cuda")
        view = buf[:r, :c]
        view.copy_((torch.rand(r, c, device="cuda", generator=g) * 2 - 1).bfloat16())
        return view
    a = mat(*((Kd, M) if ta else (M, Kd)))
    b = mat(*((N, Kd) if tb else (Kd, N)))
    cbuf = torch.full((M + 21, N + 32), NAN, dtype=torch.bfloat16, device="cuda")
    c = cbuf[:M, :N]
    K.gemm_into(a, ta, b, tb, c)
    check(cbuf, c, f"gemm {mnk} ta={ta} tb={tb}")
