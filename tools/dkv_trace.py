"""Hand-off timeline of one dK/dV CTA (profiling build only).

    bash tools/build_variant.sh trace "-DLVX_DKV_TRACE=100"
    LVX_B200_LIB=build/ab/trace.so python tools/dkv_trace.py [--shape c2gath]

clock64 stamps (SM clocks) per 128-row query step, averaged over steps 4..59:
softmax wg w: s_full returned, chunk arrivals, dp_full returned, phase B done;
MMA warp: p_ready[c] / next Q / ds_ready / next dO returned; producer: Q / dO slot free.
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
    dkg = torch.zeros(hkv, skv, d, device=dev, dtype=torch.bfloat16)
    dvg = torch.zeros_like(dkg)
    wsb = K.workspace(K.bwd_ws_bytes(q, k), dev, slot=3)
    for _ in range(3):
        K.bwd_dkv(q, k, v, L, D, g, d ** -0.5, dkg, dvg, False, ws=wsb)
    torch.cuda.synchronize()
    lib = ctypes.CDLL(os.environ["LVX_B200_LIB"])
    buf = np.zeros((4, 64, 8), dtype=np.int64)
    assert lib.lvx_dbg_dkv_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    sm0, sm1, mma, prod = buf
    st = slice(4, 60)
    per = np.diff(sm0[:, 0])[st]
    out = {
        "step_clk": float(per.mean()), "step_clk_min": float(per.min()),
        "ideal_clk_at_full_tensor_rate": 2048,
        "wg0": {
            "phaseA_chunk0_done": float((sm0[st, 1] - sm0[st, 0]).mean()),
            "phaseA_done": float((sm0[st, 2] - sm0[st, 0]).mean()),
            "dp_wait": float((sm0[st, 5] - sm0[st, 2]).mean()),
            "phaseB": float((sm0[st, 6] - sm0[st, 5]).mean()),
            "s_wait_next": float((sm0[5:61, 0] - sm0[st, 6]).mean()),
        },
        "wg1": {
            "phaseA_done": float((sm1[st, 2] - sm1[st, 0]).mean()),
            "phaseB": float((sm1[st, 6] - sm1[st, 5]).mean()),
            "s_full_skew_vs_wg0": float((sm1[st, 0] - sm0[st, 0]).mean()),
        },
        "mma": {
            "p_ready0_after_s_full": float((mma[st, 0] - sm0[st, 0]).mean()),
            "p_ready1_after_s_full": float((mma[st, 1] - sm0[st, 0]).mean()),
            "ds_ready_after_dp_full": float((mma[st, 5] - sm0[st, 5]).mean()),
            "next_Q_wait_after_p1": float((mma[st, 4] - mma[st, 1]).mean()),
            "next_dO_wait_after_ds_ready": float((mma[st, 6] - mma[st, 5]).mean()),
            "s_full_next_after_p_ready1": float((sm0[5:61, 0] - mma[st, 1]).mean()),
            "dp_full_next_after_ds_ready": float((sm0[5:61, 5] - mma[st, 5]).mean()),
        },
        "producer_Q_slot_free_after_s_full": float((prod[5:61, 0] - sm0[st, 0]).mean()),
        "producer_dO_slot_free_after_s_full": float((prod[5:61, 1] - sm0[st, 0]).mean()),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
