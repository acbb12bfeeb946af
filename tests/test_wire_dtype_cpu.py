"""The rotating forward state's wire dtype (DESIGN §5 "Wire dtypes"): fp32
(O, L) on the wire adds nothing beyond the final bf16 rounding; a bf16 wire,
as the paper's Q + O volume model assumes, at least doubles it."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))

import wire_dtype_error as W  # noqa: E402


def test_fp32_wire_is_free_and_bf16_wire_is_not():
    for sharp in (1.0, 8.0):
        r = W.run(8, 64, 256, 64, sharp, 7)
        assert r["O f32, L f32 (this repo)"]["x_final_rounding"] < 1.05
        assert r["O bf16, L f32"]["x_final_rounding"] > 2.0
        assert r["O bf16, L bf16 (paper's bf16 Q+O model)"]["x_final_rounding"] > 3.0


def test_bf16_rounding_is_round_to_nearest_even():
    import numpy as np
    assert W.bf16(np.float32(1.0 + 2 ** -8)) == 1.0            # tie -> even
    assert W.bf16(np.float32(1.0 + 3 * 2 ** -8)) == 1.0 + 2 ** -6
    assert W.bf16(np.float32(1.0 + 2 ** -8 + 2 ** -12)) == 1.0 + 2 ** -7
