"""Trace check that the forward's second-half fallback path runs (profiling build:
    bash tools/build_variant.sh fhalft "-DLVX_FWD_TRACE=0"; LVX_B200_LIB=build/ab/fhalft.so
    python tools/fwd_half_fallback_check.py).  ev3 = single pass accepted, ev2 = exact path."""
import ctypes, numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2502_02406_b200 as lvx
from oracle import lvx_oracle as orc
Q,K,V,_ = orc.make_inputs(200, 1536, 2, 128, 33, hkv=1)
q,k,v = (torch.from_numpy(t).to("cuda", torch.bfloat16) for t in (Q,K,V))
q = (q.float()*4).bfloat16()
rows = torch.arange(1536, device="cuda")
sc = torch.where((rows % 128) >= 64, 3.0 ** (rows//128).float(), torch.ones_like(rows, dtype=torch.float32))
k = (k.float()*sc[None,:,None]).bfloat16()
st = lvx.blockwise_attention(q, k, v); torch.cuda.synchronize()
lib = ctypes.CDLL("build/ab/fhalft.so"); buf = np.zeros((4,128,6), dtype=np.int64)
lib.lvx_dbg_fwd_trace(buf.ctypes.data_as(ctypes.c_void_p))
n = int((buf[0,:,0]!=0).sum()); print("tiles", n, "accepted flags (ev3)", (buf[0,:n,3]!=0).astype(int).tolist(), "exact (ev2)", (buf[0,:n,2]!=0).astype(int).tolist(), "second-half fallback (ev4)", (buf[0,:n,4]!=0).astype(int).tolist())
