import sys; sys.path.insert(0, '.')
import torch, numpy as np
from oracle import lvx_oracle as orc
from paper_2502_02406_b200 import kernels as K
for (hq, hkv, sq, skv) in [(1,1,128,128),(1,1,256,128),(1,1,200,128),(2,2,128,128),(1,1,128,1000),(2,2,200,1000),(1,1,512,128),(1,1,320,128)]:
    Q, Kt, V, G = orc.make_inputs(sq, skv, hq, 128, seed=3, hkv=hkv)
    q, k, v, g = (torch.from_numpy(t).to("cuda", torch.bfloat16) for t in (Q, Kt, V, G))
    Qr, Kr, Vr, Gr = (t.double().cpu().numpy() for t in (q, k, v, g))
    O, L = orc.dense_attention(Qr, Kr, Vr); D = orc.attention_row_stats(O, Gr)
    Lt, Dt = torch.from_numpy(L).float().cuda(), torch.from_numpy(D).float().cuda()
    dk = torch.zeros(k.shape, device="cuda"); dv = torch.zeros(v.shape, device="cuda")
    K.bwd_dkv(q, k, v, Lt, Dt, g, 128**-0.5, dk, dv, False)
    _, rk, rv = orc.blockwise_attention_backward(Qr, Kr, Vr, L, D, Gr)
    ek = orc.max_norm_error(dk.cpu().numpy(), rk); ev = orc.max_norm_error(dv.cpu().numpy(), rv)
    # per 128-row kv tile error for dK
    tiles = [orc.max_norm_error(dk.cpu().numpy()[:, a:a+128], rk[:, a:a+128]) for a in range(0, skv, 128)]
    print((hq,hkv,sq,skv), f"dK {ek:.2e} dV {ev:.2e}", "tiles", [f"{t:.1e}" for t in tiles])
