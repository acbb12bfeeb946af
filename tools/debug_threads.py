"""Debug: thread ranks on one GPU through the copy-engine transport, smallest
cases first, with a stack dump of every thread if anything hangs."""
import faulthandler
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("DBG_TIMEOUT", "90")), exit=True)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_02406_b200 as lvx  # noqa: E402
from oracle import lvx_oracle as orc  # noqa: E402
from paper_2502_02406_b200.comm import ClusterSpec  # noqa: E402
from paper_2502_02406_b200.launch import spawn_ranks  # noqa: E402


def log(*a):
    print(f"[{time.monotonic():.2f}]", *a, flush=True)


# 1. a bare shift between 2 thread ranks
def body(ctx):
    with ctx.call() as call:
        buf = call.alloc({"r": ((2, 8, 16), torch.float32)})["r"]
        t = torch.full((2, 8, 16), float(ctx.rank + 1), device="cuda")
        hop, _ = ctx.shift([t], [buf])
        hop.wait()
        out = buf.clone()
    ctx.synchronize()
    return float(out[0, 0, 0])


log("bare shift n=2")
res = spawn_ranks(ClusterSpec(2), body, timeout=20)
log("bare shift ok", res.results)

g = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                              "golden_strategies.npz")))
for t in ["s6_lvx_float32", "s6_ring_float32", "s6_head_float32", "s1_lvx_float32",
          "s2_ring_float64", "s5_lvx_float32"]:
    n = int(g[t + "_n"])
    log("case", t, "n", n)
    res = lvx.run_distributed(t.split("_")[1], g[t + "_Q"], g[t + "_K"], g[t + "_V"],
                              dO=g[t + "_dO"], spec=lvx.ClusterSpec(n), ranks="threads",
                              timeout=20)
    e = max(orc.max_norm_error(res.O, g[t + "_O"]), orc.max_norm_error(res.grads.dQ, g[t + "_dQ"]))
    log("case", t, "err", e)
log("all ok")
