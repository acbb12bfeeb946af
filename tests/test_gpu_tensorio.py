"""run_files (the numeric data path of `lvxattn run`) on the GPU vs the
reference's own run on the same LVXT inputs (lvx, n = 3 -> here n = 1 and the
n-independent outputs; f64 through the exact kernels, 1e-12), plus a device
round trip of load_tensor."""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import lvx_oracle as orc

pytestmark = pytest.mark.gpu
G = Path(__file__).parent / "golden" / "lvxt"


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_02406_b200 import build
    build.build()


def test_run_files_matches_reference_run(tmp_path):
    from paper_2502_02406_b200 import tensorio as T
    stats = T.run_files("lvx", tmp_path, G / "run_in_q.lvxt", G / "run_in_k.lvxt",
                        G / "run_in_v.lvxt", G / "run_in_do.lvxt", n=1)
    assert stats["outputs"] == ["o.lvxt", "l.lvxt", "dq.lvxt", "dk.lvxt", "dv.lvxt"]
    for name in ("o", "l", "dq", "dk", "dv"):
        got = T.load_tensor(tmp_path / f"{name}.lvxt")
        ref = T.load_tensor(G / f"run_out_{name}.lvxt")
        assert got.dtype == ref.dtype == torch.float64
        assert orc.max_norm_error(got.numpy(), ref.numpy()) <= 1e-12, name
    assert json.loads((tmp_path / "stats.json").read_text())["total_bytes"] == 0   # n = 1


def test_load_tensor_to_device():
    from paper_2502_02406_b200 import tensorio as T
    t = T.load_tensor(G / "f32_3d.lvxt", device="cuda")
    torch.cuda.synchronize()
    assert t.is_cuda and np.array_equal(t.cpu().numpy(), T.load_tensor(G / "f32_3d.lvxt").numpy())
