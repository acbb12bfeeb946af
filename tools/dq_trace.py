"""Hand-off timeline of one dQ CTA (profiling build only).

    bash tools/build_variant.sh dqtrace "-DLVX_DQ_TRACE=0"
    LVX_B200_LIB=build/ab/dqtrace.so python tools/dq_trace.py [--shape c2gath]

clock64 stamps per 128-row KV step (SM clocks), averaged over the middle steps:
softmax wg w: s_full returned, s_read arrived, dp_full returned, ds_full arrived;
MMA warp: K|V(j+1) landed, s_read(j) returned, ds_full(j) returned; producer:
slot free.  Ideal step = 3 MMAs of 128x128x128 = 1536 clk at the nominal rate.
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

SHAPES = {"c2gath": (32, 8, 2048, 131072, 128), "c2full": (32, 8, 2048, 1 << 20, 128)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="c2gath")
    a = ap.parse_args()
    from paper_2502_02406_b200 import kernels as K
    hq, hkv, sq, skv, d = SHAPES[a.shape]
    dev = torch.device("cuda")
    q, g = [(torch.rand(hq, sq, d, device=dev) * 2 - 1).bfloat16() for _ in range(2)]
    k, v = [(torch.rand(hkv, skv, d, device=dev) * 2 - 1).bfloat16() for _ in range(2)]
    ws = K.workspace(K.fwd_workspace_bytes(q, k))
    O = torch.empty(hq, sq, d, device=dev)
    L = torch.empty(hq, sq, device=dev)
    K.fwd_partial(q, k, v, d ** -0.5, ws)
    K.fwd_finish(q, k, ws, O, L, O, L)
    D = (O * g.float()).sum(-1)
    dq = torch.zeros(hq, sq, d, device=dev)
    wsb = K.workspace(K.bwd_ws_bytes(q, k), dev, slot=3)
    for _ in range(3):
        K.bwd_dq_partial(q, k, v, L, D, g, d ** -0.5, wsb)
    torch.cuda.synchronize()
    lib = ctypes.CDLL(os.environ["LVX_B200_LIB"])
    buf = np.zeros((4, 128, 8), dtype=np.int64)
    assert lib.lvx_dbg_dq_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    w0, w1, mma, prod = buf
    nt = int((w0[:, 0] != 0).sum())
    st, nx = slice(4, nt - 4), slice(5, nt - 3)
    per = np.diff(w0[:nt, 0])[st]
    out = {
        "kv_steps": nt, "step_clk": float(per.mean()), "step_clk_min": float(per.min()),
        "ideal_clk_at_full_tensor_rate": 1536,
        "wg0": {"phaseA": float((w0[st, 1] - w0[st, 0]).mean()),
                "dp_wait": float((w0[st, 2] - w0[st, 1]).mean()),
                "phaseB": float((w0[st, 3] - w0[st, 2]).mean()),
                "s_wait_next": float((w0[nx, 0] - w0[st, 3]).mean())},
        "wg1": {"phaseA": float((w1[st, 1] - w1[st, 0]).mean()),
                "phaseB": float((w1[st, 3] - w1[st, 2]).mean())},
        "mma": {"kv_next_landed_after_s_full": float((mma[st, 0] - w0[st, 0]).mean()),
                "s_read_after_s_full": float((mma[st, 1] - w0[st, 0]).mean()),
                "ds_full_after_dp_full": float((mma[st, 2] - w0[st, 2]).mean()),
                "s_full_next_after_s_read": float((w0[nx, 0] - mma[st, 1]).mean()),
                "dp_full_next_after_ds_full": float((w0[nx, 2] - mma[st, 2]).mean())},
        "producer_slot_free_after_s_full": float((prod[st, 0] - w0[st, 0]).mean()),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
