import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2502_02406_b200 import kernels as K
S, e, hkd = 131072, 4096, 1024
y = (torch.rand(S, e, device="cuda") - 0.5).bfloat16()
w = (torch.rand(e, 2 * hkd, device="cuda") - 0.5).bfloat16()
kv = torch.empty(S, 2 * hkd, device="cuda", dtype=torch.bfloat16)
k = kv[:, :hkd].view(S, 8, 128).transpose(0, 1); v = kv[:, hkd:].view(S, 8, 128).transpose(0, 1)
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
fl = 2 * S * e * 2 * hkd
for name, fn in (("torch.mm", lambda: torch.mm(y, w, out=kv)),
                 ("lvx_kv_recompute", lambda: K.kv_recompute(y, w[:, :hkd], w[:, hkd:], k, v)),
                 ("torch.mm N=1024 x2", lambda: (torch.mm(y, w[:, :hkd].contiguous()), torch.mm(y, w[:, hkd:].contiguous())))):
    ms = t(fn); print(name, round(ms, 3), "ms", round(fl / ms / 1e9), "TFLOP/s")
