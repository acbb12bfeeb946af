"""LVXT tensor files and the numeric file-to-file run (reference
``pkg/src/lvxattn/tensorio.py`` and the data path of ``cli.cmd_run``,
``cli.py:96-177``; SURVEY.md §8(f) next 4 — the format half; the CLI itself is
out of scope).

LVXT layout (tensorio.py:7-16, all integers little-endian)::

    0   4        magic b"LVXT"
    4   4        version u32 (1)
    8   1        dtype code u8: 0 = f32, 1 = f64 (reference); 2 = bf16 (this
                 implementation's extension, written only for bf16 tensors)
    9   1        ndim u8 (1..3)
    10  8 ndim   dims, u64 each
    ..           payload, row-major little-endian scalars

Files written here for f32 / f64 tensors are byte-identical to the
reference's, and the reference's files load bit-exactly (tests/
test_tensorio_cpu.py against files the reference wrote).  Tensors may be
numpy arrays or torch tensors on any device; ``load_tensor(path, device=...)``
reads into pinned host memory and copies to the device asynchronously.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np
import torch

MAGIC = b"LVXT"
FORMAT_VERSION = 1
_CODES = {0: (np.dtype("<f4"), torch.float32), 1: (np.dtype("<f8"), torch.float64),
          2: (np.dtype("<u2"), torch.bfloat16)}
_CODE_FOR = {torch.float32: 0, torch.float64: 1, torch.bfloat16: 2}
DTYPE_NAMES = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}


class LvxtError(ValueError):
    """Base class for LVXT parse / encode failures (tensorio.py:40-53)."""


class BadMagicError(LvxtError):
    pass


class UnknownDtypeError(LvxtError):
    pass


class TruncatedPayloadError(LvxtError):
    pass


def dtype_from_name(name: str) -> torch.dtype:
    try:
        return DTYPE_NAMES[name]
    except KeyError:
        raise ValueError(f"unknown dtype name {name!r}, expected one of {sorted(DTYPE_NAMES)}")


def seeded_random_tensor(seed: int, shape, dtype=np.float64, scale: float = 1.0,
                         stream: int = 0) -> np.ndarray:
    """U[-scale, scale] from Philox keyed (seed, stream), drawn in f64 and cast
    (tensorio.py:62-82) — the same bits as the reference's generator."""
    shape = tuple(int(s) for s in shape)
    if len(shape) == 0:
        raise ValueError("empty shape")
    if any(s <= 0 for s in shape):
        raise ValueError("empty shape: all axes must be positive")
    if not scale > 0:
        raise ValueError(f"scale must be positive, got {scale}")
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"unsupported dtype {dt}")
    gen = np.random.Generator(np.random.Philox(key=[int(seed) & (2 ** 64 - 1), int(stream)]))
    return gen.uniform(-scale, scale, size=shape).astype(dt)


def _as_cpu_tensor(t) -> torch.Tensor:
    if isinstance(t, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(t))
    if isinstance(t, torch.Tensor):
        return t.detach().to("cpu").contiguous()
    raise LvxtError(f"expected a numpy array or torch tensor, got {type(t).__name__}")


def encode(t) -> bytes:
    """LVXT bytes of a tensor (numpy or torch, any device)."""
    c = _as_cpu_tensor(t)
    if c.dtype not in _CODE_FOR:
        raise LvxtError(f"unsupported dtype {c.dtype}")
    if c.dim() < 1 or c.dim() > 3:
        raise LvxtError(f"rank must be 1..3, got {c.dim()}")
    code = _CODE_FOR[c.dtype]
    header = MAGIC + struct.pack("<IBB", FORMAT_VERSION, code, c.dim())
    header += b"".join(struct.pack("<Q", int(d)) for d in c.shape)
    raw = c.view(torch.int16) if c.dtype == torch.bfloat16 else c
    return header + raw.numpy().astype(_CODES[code][0].newbyteorder("<"), copy=False).tobytes()


def store_tensor(t, path) -> None:
    """Write one tensor in LVXT form; round-trips bit-exactly with load_tensor."""
    Path(path).write_bytes(encode(t))


def decode(raw: bytes) -> torch.Tensor:
    """Parse LVXT bytes into a CPU tensor; distinct errors for bad magic,
    unknown dtype, truncation and trailing data (tensorio.py:100-130)."""
    if len(raw) < 4 or raw[:4] != MAGIC:
        raise BadMagicError(f"bad magic: expected {MAGIC!r}, got {raw[:4]!r}")
    if len(raw) < 10:
        raise TruncatedPayloadError(f"truncated header: {len(raw)} bytes")
    version, code, ndim = struct.unpack_from("<IBB", raw, 4)
    if version != FORMAT_VERSION:
        raise LvxtError(f"unsupported version {version}")
    if code not in _CODES:
        raise UnknownDtypeError(f"unknown dtype code {code}")
    if ndim < 1 or ndim > 3:
        raise LvxtError(f"rank must be 1..3, got {ndim}")
    dims_end = 10 + 8 * ndim
    if len(raw) < dims_end:
        raise TruncatedPayloadError(f"truncated header: {len(raw)} bytes, need {dims_end}")
    dims = struct.unpack_from("<" + "Q" * ndim, raw, 10)
    npdt, tdt = _CODES[code]
    count = 1
    for d in dims:
        count *= d
    expected = dims_end + count * npdt.itemsize
    if len(raw) < expected:
        raise TruncatedPayloadError(
            f"truncated payload: have {len(raw) - dims_end} bytes, expected {expected - dims_end}")
    if len(raw) > expected:
        raise LvxtError(f"trailing data: {len(raw) - expected} extra bytes")
    flat = np.frombuffer(raw, dtype=npdt, count=count, offset=dims_end)
    arr = flat.astype(npdt.newbyteorder("="), copy=True).reshape(dims)
    t = torch.from_numpy(arr)
    return t.view(torch.bfloat16) if tdt == torch.bfloat16 else t


def load_tensor(path, device: torch.device | str | None = None) -> torch.Tensor:
    """Read an LVXT file; with ``device`` the payload goes through pinned host
    memory to the device (asynchronous on the current stream)."""
    t = decode(Path(path).read_bytes())
    if device is None or torch.device(device).type == "cpu":
        return t
    return t.pin_memory().to(device, non_blocking=True)


def run_files(strategy: str, out_dir, q_path, k_path, v_path, do_path=None, n: int = 1,
              dtype: str | None = None, scale: float | None = None, stats_path=None) -> dict:
    """The numeric data path of ``lvxattn run`` (cli.py:96-177) on B200: LVXT
    inputs -> ``run_distributed`` over n GPUs -> o / l (+ dq / dk / dv).lvxt and
    a stats JSON with the transport byte counters and round traces.  ``dtype``
    casts the inputs (the reference's --dtype); None keeps the files' dtype."""
    from .comm import ClusterSpec
    from .strategies import run_distributed
    Q, K, V = (load_tensor(p) for p in (q_path, k_path, v_path))
    dO = load_tensor(do_path) if do_path else None
    if dtype is not None:
        dt = dtype_from_name(dtype)
        Q, K, V = Q.to(dt), K.to(dt), V.to(dt)
        dO = dO.to(dt) if dO is not None else None
    res = run_distributed(strategy, Q, K, V, dO=dO, spec=ClusterSpec(n), scale=scale)
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = []
    outs = [("o", res.O), ("l", res.L)]
    if res.grads is not None:
        outs += [("dq", res.grads.dQ), ("dk", res.grads.dK), ("dv", res.grads.dV)]
    for name, t in outs:
        store_tensor(t, out / f"{name}.lvxt")
        written.append(f"{name}.lvxt")
    stats = {"strategy": strategy, "n": n,
             "workload": {"s_q": int(Q.shape[1]), "s_kv": int(K.shape[1]), "h": int(Q.shape[0]),
                          "hkv": int(K.shape[0]), "d": int(Q.shape[2]),
                          "dtype": str(Q.dtype).replace("torch.", "")},
             "total_bytes": res.stats.total_bytes(),
             "per_worker_bytes_sent": [res.stats.bytes_sent_by(i) for i in range(n)],
             "rounds_forward": res.traces_forward[0].num_rounds,
             "traces": {"forward": [t.as_dict() for t in res.traces_forward],
                        "backward": ([t.as_dict() for t in res.traces_backward]
                                     if res.traces_backward else None)},
             "outputs": written}
    Path(stats_path or out / "stats.json").write_text(json.dumps(stats, indent=1))
    return stats
