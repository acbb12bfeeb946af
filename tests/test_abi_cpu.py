"""The C-ABI library builds for sm_100a, loads on a CPU-only host and exports
every symbol include/lvx_b200.h declares.  No compute calls (no GPU here)."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    hdr = (ROOT / "include" / "lvx_b200.h").read_text()
    return sorted(set(re.findall(r"\b(lvx_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for must in ("lvx_blockwise_fwd", "lvx_fwd_partial", "lvx_fwd_finish", "lvx_merge_states",
                 "lvx_row_stats", "lvx_blockwise_bwd"):
        assert must in names


def test_library_loads_and_exports_all_symbols():
    from paper_2502_02406_b200 import build, _lib
    build.build()
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == set(_declared())
    assert lib.lvx_abi_version() == 1
    assert lib.lvx_strerror(-1) == b"invalid shape, stride or argument"


def test_kernels_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2502_02406_b200 import blockwise_attention
    with pytest.raises(RuntimeError, match="CUDA device"):
        blockwise_attention(np.ones((1, 2, 4)), np.ones((1, 3, 4)), np.ones((1, 3, 4)))


def test_shape_errors_use_reference_messages():
    import numpy as np
    from paper_2502_02406_b200 import blockwise_attention, merge_states, empty_state
    Q, K, V = np.ones((2, 4, 3)), np.ones((2, 6, 3)), np.ones((2, 6, 3))
    with pytest.raises(ValueError, match="head counts"):
        blockwise_attention(Q, K[:1].repeat(3, 0), V)
    with pytest.raises(ValueError, match="rows"):
        blockwise_attention(Q, K, V[:, :5])
    with pytest.raises(ValueError, match="cols"):
        blockwise_attention(Q, K[:, :, :2], V)
    with pytest.raises(ValueError, match="tile_rows"):
        blockwise_attention(Q, K, V, tile_rows=0)


def test_library_links_no_cublas():
    """Every GEMM of the path is the library's own kernel (lvx_gemm_sm100.cu):
    the shared object depends on no BLAS library."""
    import subprocess
    from paper_2502_02406_b200 import build
    lib = build.build()
    deps = subprocess.run(["ldd", str(lib)], capture_output=True, text=True).stdout
    assert "cublas" not in deps.lower(), deps


def test_integration_stub_binds_declared_symbols():
    """The ctypes stub INTEGRATION.md shows a maintainer of the reference
    package compiles, and every lvx_* function it calls is declared in the
    header and exported by the library."""
    import ast
    blocks = re.findall(r"```python\n(.*?)```", (ROOT / "INTEGRATION.md").read_text(), re.S)
    assert len(blocks) >= 2
    declared = set(_declared())
    used = set()
    for b in blocks:
        ast.parse(b)                       # valid Python
        used |= set(re.findall(r"_lib\.(lvx_[a-z0-9_]+)", b))
    assert used, "the stub calls the C ABI"
    assert used <= declared, used - declared
