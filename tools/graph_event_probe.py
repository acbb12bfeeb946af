"""Do timing events recorded inside a CUDA graph capture give per-kernel
times after a replay (torch.cuda.Event(external=True))?"""
import torch

x = torch.randn(8192, 8192, device="cuda")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
ev = []
with torch.cuda.graph(g, stream=s):
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True, external=True)
        b = torch.cuda.Event(enable_timing=True, external=True)
        a.record()
        y = x @ x
        b.record()
        ev.append((a, b))
for rep in range(3):
    g.replay()
    torch.cuda.synchronize()
    print("replay", rep, [round(a.elapsed_time(b), 3) for a, b in ev])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); y = x @ x; e1.record(); torch.cuda.synchronize()
print("eager matmul ms", round(e0.elapsed_time(e1), 3))
