"""Hand-off timeline of one forward CTA (profiling build only).

    bash tools/build_variant.sh ftrace "-DLVX_FWD_TRACE=0"
    LVX_B200_LIB=build/ab/ftrace.so python tools/fwd_trace.py [--shape c2gath]

clock64 stamps per KV tile j (SM clocks), averaged over the middle tiles:
softmax of query tile t: s_full returned, p_full arrived; MMA warp: V_j /
K_{j+1} landed, p_full[0] / p_full[1] returned.  Ideal tile = 4 MMAs of
128x128x128 = 2048 clk at the nominal tensor rate.
"""
import argparse
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SHAPES = {"c2gath": (32, 8, 2048, 131072, 128), "c2round": (32, 8, 256, 131072, 128),
          "c2full": (32, 8, 2048, 1 << 20, 128)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="c2gath")
    a = ap.parse_args()
    from paper_2502_02406_b200 import kernels as K
    hq, hkv, sq, skv, d = SHAPES[a.shape]
    dev = torch.device("cuda")
    q = (torch.rand(hq, sq, d, device=dev) * 2 - 1).bfloat16()
    k, v = [(torch.rand(hkv, skv, d, device=dev) * 2 - 1).bfloat16() for _ in range(2)]
    ws = K.workspace(K.fwd_workspace_bytes(q, k))
    for _ in range(3):
        K.fwd_partial(q, k, v, d ** -0.5, ws)
    torch.cuda.synchronize()
    lib = ctypes.CDLL(os.environ["LVX_B200_LIB"])
    buf = np.zeros((4, 128, 6), dtype=np.int64)
    assert lib.lvx_dbg_fwd_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    s0, s1, mma = buf[0], buf[1], buf[2]
    nt = int((s0[:, 0] != 0).sum())
    st = slice(4, nt - 4)
    nx = slice(5, nt - 3)
    per = np.diff(s0[:nt, 0])[st]
    out = {
        "kv_tiles": nt, "tile_clk": float(per.mean()), "tile_clk_min": float(per.min()),
        "ideal_clk_at_full_tensor_rate": 2048,
        "single_pass_share": float((s0[st, 3] != 0).mean()),
        "t0_softmax": float((s0[st, 1] - s0[st, 0]).mean()),
        "t1_softmax": float((s1[st, 1] - s1[st, 0]).mean()),
        "t1_s_full_after_t0": float((s1[st, 0] - s0[st, 0]).mean()),
        "t0_idle_until_next_s": float((s0[nx, 0] - s0[st, 1]).mean()),
        "mma_V_wait_after_prev_p1": float((mma[nx, 0] - mma[st, 3]).mean()),
        "mma_K_wait": float((mma[st, 1] - mma[st, 0]).mean()),
        "mma_p0_after_t0_s_full": float((mma[st, 2] - s0[st, 0]).mean()),
        "mma_p1_after_t1_s_full": float((mma[st, 3] - s1[st, 0]).mean()),
        "t0_s_full_next_after_p0": float((s0[nx, 0] - mma[st, 2]).mean()),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
