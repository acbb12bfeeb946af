"""Small invocations of every sm_100a kernel of the library (forward, dK/dV,
dQ, combine, GEMM, HBM kernels) for compute-sanitizer runs:
    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_small.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_02406_b200 import kernels as K  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1).bfloat16()  # noqa: E731
    for hq, hkv, sq, skv, d in ((4, 2, 200, 700, 128), (2, 2, 128, 384, 64)):
        q, k, v, do = r(hq, sq, d), r(hkv, skv, d), r(hkv, skv, d), r(hq, sq, d)
        st = K.blockwise_attention(q, k, v)
        dq, dk, dv = K.blockwise_attention_backward(q, k, v, st.L, K.attention_row_stats(st, do),
                                                    do)
        m = K.merge_states(st, st)
    a, b = r(300, 256), r(256, 512)
    c = torch.empty(300, 512, device="cuda", dtype=torch.bfloat16)
    K.gemm_into(a, False, b, False, c)
    K.gemm_into(r(4096, 256), True, r(4096, 256), False, torch.empty(256, 256, device="cuda",
                                                                  dtype=torch.bfloat16))
    torch.cuda.synchronize()
    print("sanitize_small ok", float(dq.float().abs().sum()), float(m.O.abs().sum()))


if __name__ == "__main__":
    main()
