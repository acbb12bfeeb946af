"""ctypes binding of ``liblvx_b200.so`` (declared in ``include/lvx_b200.h``).

The library is built in-tree by ``paper_2502_02406_b200.build``.  There is no
fallback: if the library is missing, or no CUDA device is visible when a
kernel is called, the call raises.  Loading the library itself works on a
CPU-only host (static CUDA runtime), which the CPU test-suite uses to check
the exported symbols.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "liblvx_b200.so"

LVX_F32, LVX_F64, LVX_BF16 = 0, 1, 2
_DT = {torch.float32: LVX_F32, torch.float64: LVX_F64, torch.bfloat16: LVX_BF16}

EXPORTS = ("lvx_abi_version", "lvx_kernel_launches", "lvx_strerror", "lvx_tc_eligible", "lvx_blockwise_fwd_workspace",
           "lvx_blockwise_fwd", "lvx_fwd_partial", "lvx_fwd_finish", "lvx_merge_states",
           "lvx_row_stats", "lvx_blockwise_bwd_workspace", "lvx_blockwise_bwd",
           "lvx_fill_empty_state", "lvx_convert", "lvx_bwd_workspace", "lvx_bwd_dq_partial",
           "lvx_bwd_dq_finish", "lvx_bwd_dkv", "lvx_project", "lvx_project_bwd",
           "lvx_kv_recompute", "lvx_gemm", "lvx_accumulate", "lvx_peer_create", "lvx_peer_destroy",
           "lvx_peer_base", "lvx_peer_handle_bytes", "lvx_peer_export", "lvx_peer_open",
           "lvx_peer_attach", "lvx_peer_put", "lvx_peer_signal", "lvx_peer_wait",
           "lvx_stream_create", "lvx_stream_destroy")


class LvxView(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("heads", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("d", ctypes.c_int64), ("head_stride", ctypes.c_int64),
                ("row_stride", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


class LvxMatrix(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("row_stride", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


class LvxError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: {msg} (status {status})")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and prototype the library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    # LVX_B200_LIB: an alternate build of the same library (same-box A/B tooling)
    path = Path(os.environ.get("LVX_B200_LIB") or LIB_PATH)
    if not path.exists():
        raise RuntimeError(f"{path} not built: run `python -m paper_2502_02406_b200.build`"
                           " (there is no CPU fallback)")
    lib = ctypes.CDLL(str(path))
    P = ctypes.POINTER(LvxView)
    M = ctypes.POINTER(LvxMatrix)
    vp, sz, dbl, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_double, ctypes.c_int
    u64 = ctypes.c_uint64
    proto = {
        "lvx_abi_version": (i32, []),
        "lvx_kernel_launches": (ctypes.c_ulonglong, []),
        "lvx_strerror": (ctypes.c_char_p, [i32]),
        "lvx_tc_eligible": (i32, [P, P]),
        "lvx_blockwise_fwd_workspace": (sz, [P, P]),
        "lvx_blockwise_fwd": (i32, [P, P, P, dbl, P, P, P, P, vp, sz, vp]),
        "lvx_fwd_partial": (i32, [P, P, P, dbl, vp, sz, vp]),
        "lvx_fwd_finish": (i32, [P, P, P, P, P, P, vp, sz, vp]),
        "lvx_merge_states": (i32, [P, P, P, P, P, P, vp]),
        "lvx_row_stats": (i32, [P, P, P, vp]),
        "lvx_blockwise_bwd_workspace": (sz, [P, P]),
        "lvx_blockwise_bwd": (i32, [P, P, P, P, P, P, dbl, P, P, P, i32, vp, sz, vp]),
        "lvx_fill_empty_state": (i32, [P, P, vp]),
        "lvx_bwd_workspace": (sz, [P, P]),
        "lvx_bwd_dq_partial": (i32, [P, P, P, P, P, P, dbl, vp, sz, vp]),
        "lvx_bwd_dq_finish": (i32, [P, P, P, i32, vp, sz, vp]),
        "lvx_bwd_dkv": (i32, [P, P, P, P, P, P, dbl, P, P, i32, vp, sz, vp]),
        "lvx_convert": (i32, [P, P, vp]),
        "lvx_project": (i32, [M, M, P, vp]),
        "lvx_project_bwd": (i32, [M, M, P, M, M, vp]),
        "lvx_kv_recompute": (i32, [M, M, M, P, P, vp]),
        "lvx_gemm": (i32, [M, i32, M, i32, M, i32, vp]),
        "lvx_accumulate": (i32, [P, P, vp]),
        "lvx_peer_create": (i32, [u64, i32, i32, ctypes.POINTER(vp)]),
        "lvx_peer_destroy": (i32, [vp]),
        "lvx_peer_base": (vp, [vp]),
        "lvx_peer_handle_bytes": (u64, []),
        "lvx_peer_export": (i32, [vp, vp]),
        "lvx_peer_open": (i32, [vp, i32, vp]),
        "lvx_peer_attach": (i32, [vp, i32, vp]),
        "lvx_peer_put": (i32, [vp, i32, u64, u64, vp, u64, u64, u64, vp]),
        "lvx_peer_signal": (i32, [vp, i32, u64, ctypes.c_uint32, vp]),
        "lvx_peer_wait": (i32, [vp, u64, ctypes.c_uint32, vp]),
        "lvx_stream_create": (i32, [ctypes.POINTER(vp)]),
        "lvx_stream_destroy": (i32, [vp]),
    }
    for name, (res, args) in proto.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


def lvx_dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}; expected float32, float64 or bfloat16")


def view(t: torch.Tensor | None):
    """[h, rows, d] (or [h, rows] row statistics, as d=1) -> pointer to LvxView."""
    if t is None:
        return None
    if t.dim() == 2:
        h, r = t.shape
        hs, rs = t.stride()
        v = LvxView(t.data_ptr(), h, r, 1, hs, rs, lvx_dtype(t), 0)
    elif t.dim() == 3:
        if t.numel() and t.shape[2] > 1 and t.stride(2) != 1:
            raise ValueError("last dimension must be contiguous")
        h, r, d = t.shape
        v = LvxView(t.data_ptr(), h, r, d, t.stride(0), t.stride(1), lvx_dtype(t), 0)
    else:
        raise ValueError(f"expected a [heads, rows, d] tensor, got shape {tuple(t.shape)}")
    return ctypes.byref(v)


def matrix(t: torch.Tensor):
    """Row-major [rows, cols] matrix (unit column stride) -> pointer to LvxMatrix."""
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {tuple(t.shape)}")
    if t.numel() and t.shape[1] > 1 and t.stride(1) != 1:
        raise ValueError("matrix columns must be contiguous")
    rs = t.stride(0) if t.shape[0] > 1 else max(t.shape[1], 1)
    return ctypes.byref(LvxMatrix(t.data_ptr(), t.shape[0], t.shape[1], rs, lvx_dtype(t), 0))


def check(fn: str, status: int) -> None:
    if status != 0:
        msg = load().lvx_strerror(status).decode()
        if status in (-1, -2, -4):
            raise ValueError(f"{fn}: {msg}")
        raise LvxError(fn, status, msg)


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class OwnStream:
    """A CUDA stream of its own (lvx_stream_create) usable as a torch stream;
    destroyed with ``close()``."""

    def __init__(self, device):
        import torch
        self.device = torch.device(device)
        p = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check("lvx_stream_create", load().lvx_stream_create(ctypes.byref(p)))
        self.ptr = p.value
        self.stream = torch.cuda.ExternalStream(self.ptr, device=self.device)

    def close(self) -> None:
        if self.ptr:
            self.stream.synchronize()
            load().lvx_stream_destroy(ctypes.c_void_p(self.ptr))
            self.ptr = None
