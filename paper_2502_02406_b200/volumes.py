"""Closed-form NVLink bytes of the ring protocols (reference
``pkg/src/lvxattn/volumes.py``), extended for GQA and mixed wire dtypes.

Which tensor classes travel per round is fixed by the reference
(volumes.py:48-59); here every class carries its own head count and element
size, because on B200 Q/K/V/dO travel in bf16 while the softmax state
(O, L, D) and gradient accumulators (dQ, dK, dV) travel in fp32, and K/V have
``hkv`` heads while the query-side classes have ``hq``.  With hq = hkv and one
element size the functions reduce exactly to the reference's closed forms
(tests/test_oracle.py and the protocol tests check them against the byte
counters the reference itself produced, tests/golden/golden_strategies.npz).
"""
from __future__ import annotations

from dataclasses import dataclass

ROUND_PAYLOAD = {
    ("lvx", "forward"): ("O", "L", "Q"),
    ("lvx", "backward"): ("Q", "dO", "L", "D", "dQ"),
    ("ring", "forward"): ("K", "V"),
    ("ring", "backward"): ("K", "V", "dK", "dV"),
}
EPILOGUE_PAYLOAD = {
    ("lvx", "forward"): ("O", "L"),
    ("lvx", "backward"): (),
    ("ring", "forward"): (),
    ("ring", "backward"): ("dK", "dV"),
}
# The B200 lvx backward moves the same bytes per rank on a different message
# schedule (strategies.lvx_backward): the immutable (Q, dO, L, D) block is sent
# at the START of each round and dQ lags one hop, so round 0 carries no dQ
# and a dQ epilogue hop takes the last one home — n + 1 messages per rank
# instead of the reference's n.  The B200 Ring backward sends K/V and the dK/dV
# partials as separate hops (the partial lags its block by one round), so
# 2 (n - 1) + 1 messages.  Per-rank byte totals are unchanged everywhere.
B200_ROUND_PAYLOAD = {**ROUND_PAYLOAD,
                      ("lvx", "backward", 0): ("Q", "dO", "L", "D")}
B200_EPILOGUE_PAYLOAD = {**EPILOGUE_PAYLOAD, ("lvx", "backward"): ("dQ",)}


def messages_per_rank(strategy: str, phase: str, n: int, schedule: str = "b200") -> int:
    """Hops one rank sends in one call (0 at n = 1): rounds with a send plus
    the epilogue, if the schedule has one."""
    if n == 1:
        return 0
    rounds = n if strategy == "lvx" else n - 1
    if schedule == "b200" and (strategy, phase) == ("ring", "backward"):
        rounds *= 2   # K/V lead, the dK/dV partial of the same block follows one round later
    epi = (B200_EPILOGUE_PAYLOAD if schedule == "b200" else EPILOGUE_PAYLOAD)[(strategy, phase)]
    return rounds + (1 if epi else 0)


_QSIDE = {"Q", "O", "dO", "dQ", "L", "D"}
_ROWSTAT = {"L", "D"}


@dataclass(frozen=True)
class Wire:
    """Shape/dtype of one rotated row per class."""

    hq: int
    hkv: int
    d: int
    in_bytes: int      # Q, K, V, dO element size
    state_bytes: int   # O, L, D, dQ, dK, dV element size

    def row_bytes(self, cls: str) -> int:
        heads = self.hq if cls in _QSIDE else self.hkv
        width = 1 if cls in _ROWSTAT else self.d
        size = self.in_bytes if cls in ("Q", "K", "V", "dO") else self.state_bytes
        return heads * width * size

    @classmethod
    def reference(cls, h: int, d: int, elem_bytes: int) -> "Wire":
        return cls(h, h, d, elem_bytes, elem_bytes)

    @classmethod
    def b200(cls, hq: int, hkv: int, d: int, in_bytes: int = 2) -> "Wire":
        return cls(hq, hkv, d, in_bytes, 8 if in_bytes == 8 else 4)


def _rows_bytes(w: Wire, classes, rows: int) -> int:
    return rows * sum(w.row_bytes(c) for c in classes)


def lvx_forward_bytes_by_worker(q_sizes, w: Wire) -> list[int]:
    """Round r ships (O, L) of block i-r+1 and Q of block i-r; the epilogue
    ships (O, L) of block i+1 (volumes.py:71-85)."""
    n = len(q_sizes)
    if n == 1:
        return [0]
    out = []
    for i in range(n):
        tot = sum(_rows_bytes(w, ("O", "L"), q_sizes[(i - r + 1) % n]) +
                  _rows_bytes(w, ("Q",), q_sizes[(i - r) % n]) for r in range(n))
        out.append(tot + _rows_bytes(w, ("O", "L"), q_sizes[(i + 1) % n]))
    return out


def lvx_backward_bytes_by_worker(q_sizes, w: Wire) -> list[int]:
    """Every (Q, dO, L, D, dQ) block is forwarded once by every rank
    (volumes.py:88-94)."""
    n = len(q_sizes)
    if n == 1:
        return [0]
    return [_rows_bytes(w, ROUND_PAYLOAD[("lvx", "backward")], sum(q_sizes))] * n


def ring_forward_bytes_by_worker(kv_sizes, w: Wire) -> list[int]:
    n = len(kv_sizes)
    if n == 1:
        return [0]
    return [_rows_bytes(w, ("K", "V"), sum(kv_sizes[(i - r) % n] for r in range(n - 1)))
            for i in range(n)]


def ring_backward_bytes_by_worker(kv_sizes, w: Wire) -> list[int]:
    n = len(kv_sizes)
    if n == 1:
        return [0]
    return [_rows_bytes(w, ("K", "V", "dK", "dV"),
                        sum(kv_sizes[(i - r) % n] for r in range(n - 1))) +
            _rows_bytes(w, ("dK", "dV"), kv_sizes[(i + 1) % n]) for i in range(n)]


def head_parallel_forward_bytes_by_worker(q_sizes, kv_sizes, w: Wire) -> list[int]:
    """Gather (Q, K, V head chunks of the own rows) to n-1 ranks, scatter
    (O, L) rows back (volumes.py:123-137); hq, hkv divisible by n."""
    n = len(q_sizes)
    if n == 1:
        return [0]
    out = []
    for i in range(n):
        gather = (n - 1) * (q_sizes[i] * w.row_bytes("Q") +
                            kv_sizes[i] * (w.row_bytes("K") + w.row_bytes("V"))) // n
        scatter = sum(q_sizes[x] for x in range(n) if x != i) * \
            (w.row_bytes("O") + w.row_bytes("L")) // n
        out.append(gather + scatter)
    return out


def head_parallel_backward_bytes_by_worker(q_sizes, kv_sizes, w: Wire) -> list[int]:
    """Gather dO head chunks, scatter (dQ, dK, dV) rows (volumes.py:140-152)."""
    n = len(q_sizes)
    if n == 1:
        return [0]
    out = []
    for i in range(n):
        gather = (n - 1) * q_sizes[i] * w.row_bytes("dO") // n
        scatter = sum(q_sizes[x] * w.row_bytes("dQ") +
                      kv_sizes[x] * (w.row_bytes("dK") + w.row_bytes("dV"))
                      for x in range(n) if x != i) // n
        out.append(gather + scatter)
    return out


def bytes_by_worker(strategy: str, phase: str, q_sizes, kv_sizes, w: Wire) -> list[int]:
    fn = {("head", "forward"): lambda: head_parallel_forward_bytes_by_worker(q_sizes, kv_sizes, w),
          ("head", "backward"): lambda: head_parallel_backward_bytes_by_worker(q_sizes, kv_sizes, w),
          ("lvx", "forward"): lambda: lvx_forward_bytes_by_worker(q_sizes, w),
          ("lvx", "backward"): lambda: lvx_backward_bytes_by_worker(q_sizes, w),
          ("ring", "forward"): lambda: ring_forward_bytes_by_worker(kv_sizes, w),
          ("ring", "backward"): lambda: ring_backward_bytes_by_worker(kv_sizes, w)}
    return fn[(strategy, phase)]()


def paper_hop_bytes(s_q: int, n: int, hq: int, d: int, b: int) -> float:
    """The paper's per-round LV-XAttn volume, Q + O (+ L) of one block:
    (2 (S_Q/n) h d + (S_Q/n) h) b (Table 1)."""
    rows = s_q / n
    return (2 * rows * hq * d + rows * hq) * b


def attention_flops(s_q: int, s_kv: int, hq: int, d: int, phase: str = "both") -> float:
    """4 Sq Skv h d forward, 10 Sq Skv h d backward (PAPER.md:67,
    analytics.py:113-115); h = query heads."""
    f = {"forward": 4.0, "backward": 10.0, "both": 14.0}[phase]
    return f * s_q * s_kv * hq * d
