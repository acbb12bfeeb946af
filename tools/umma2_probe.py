"""Run tools/umma2_probe.cu (2-CTA tcgen05 MMA probe) against torch.
    nvcc ... -o build/umma2_probe.so tools/umma2_probe.cu ; python tools/umma2_probe.py"""
import ctypes
import sys
from pathlib import Path

import torch

lib = ctypes.CDLL(str(Path(__file__).resolve().parent.parent / "build" / "umma2_probe.so"))
lib.umma2_probe.argtypes = [ctypes.c_void_p] * 4
torch.manual_seed(0)
A = torch.randn(256, 64, device="cuda").bfloat16()
B = torch.randn(128, 64, device="cuda").bfloat16()
D = torch.full((256, 128), float("nan"), device="cuda")
rc = lib.umma2_probe(A.data_ptr(), B.data_ptr(), D.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ref = A.float() @ B.float().T
err = (D - ref).abs().max().item()
print("rc", rc, "max abs err", err, "rows 0-127 ok", torch.allclose(D[:128], ref[:128], atol=1e-2),
      "rows 128-255 ok", torch.allclose(D[128:], ref[128:], atol=1e-2))
sys.exit(0 if rc == 0 and err < 1e-2 else 1)
