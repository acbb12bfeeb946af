"""LVXT files (paper_2502_02406_b200.tensorio, §8(f) next 4 — the format half) vs
files the reference itself wrote (tests/golden/lvxt/, make_golden.py --only lvxt):
bit-exact reads, byte-identical writes, the reference's error classes, the
same Philox streams; the bf16 extension round-trips."""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2502_02406_b200 import tensorio as T

G = Path(__file__).parent / "golden" / "lvxt"
FILES = {"f32_3d.lvxt": (5, (3, 4, 2), np.float32, 1.0, 0),
         "f64_1d.lvxt": (6, (7,), np.float64, 2.0, 3),
         "f32_2d.lvxt": (7, (2, 5), np.float32, 1.0, 9)}


@pytest.mark.parametrize("name", sorted(FILES))
def test_reads_reference_files_and_writes_identical_bytes(name, tmp_path):
    seed, shape, dt, scale, stream = FILES[name]
    ref = T.seeded_random_tensor(seed, shape, dt, scale=scale, stream=stream)
    got = T.load_tensor(G / name)
    assert got.dtype == (torch.float32 if dt == np.float32 else torch.float64)
    assert np.array_equal(got.numpy(), ref)                     # same Philox bits
    T.store_tensor(ref, tmp_path / name)
    assert (tmp_path / name).read_bytes() == (G / name).read_bytes()
    T.store_tensor(torch.from_numpy(ref), tmp_path / "t.lvxt")   # torch input, same bytes
    assert (tmp_path / "t.lvxt").read_bytes() == (G / name).read_bytes()


def test_errors_match_reference_classes(tmp_path):
    raw = (G / "f32_3d.lvxt").read_bytes()
    with pytest.raises(T.BadMagicError):
        T.decode(b"XVXT" + raw[4:])
    bad = bytearray(raw)
    bad[8] = 7
    with pytest.raises(T.UnknownDtypeError):
        T.decode(bytes(bad))
    with pytest.raises(T.TruncatedPayloadError):
        T.decode(raw[:-1])
    with pytest.raises(T.TruncatedPayloadError):
        T.decode(raw[:12])
    with pytest.raises(T.LvxtError):
        T.decode(raw + b"\0")
    with pytest.raises(T.LvxtError):
        T.store_tensor(np.zeros((1, 1, 1, 1), np.float32), tmp_path / "x.lvxt")
    with pytest.raises(T.LvxtError):
        T.store_tensor(np.zeros(3, np.int32), tmp_path / "x.lvxt")
    assert issubclass(T.BadMagicError, ValueError)


def test_bf16_extension_round_trip(tmp_path):
    t = torch.randn(2, 3, 8).to(torch.bfloat16)
    T.store_tensor(t, tmp_path / "b.lvxt")
    raw = (tmp_path / "b.lvxt").read_bytes()
    assert raw[8] == 2 and len(raw) == 10 + 3 * 8 + t.numel() * 2
    back = T.load_tensor(tmp_path / "b.lvxt")
    assert back.dtype == torch.bfloat16 and torch.equal(back, t)


def test_run_golden_files_present():
    stats = json.loads((G / "run_stats.json").read_text())
    assert stats["rounds_forward"] == 3 and len(stats["per_worker_bytes_sent"]) == 3
