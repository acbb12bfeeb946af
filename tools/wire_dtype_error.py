"""Error cost of the wire dtype of the rotating forward state.

    python tools/wire_dtype_error.py [--n 8] [--rows 256] [--kv 2048] [--d 128]

The LV-XAttn forward (src/strategies.py:175-231) carries each query block's
running (O, L) around the ring and merges one KV shard's partial into it per
round (src/kernels.py:144-161).  This tool replays that merge chain in f64 with
the carried state rounded to a candidate wire dtype after every hop and reports
the error of the final O against the exact attention, in units of the error the
final bf16 output rounding alone makes.  Inputs are uniform[-1,1] like the
bench; a second case sharpens the scores (x 8) so that L moves more per round.
Host-only (numpy); writes one JSON line."""
import argparse
import json

import numpy as np


def bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def partial(q, k, v, scale):
    s = (q @ k.T) * scale
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    l_sum = p.sum(axis=1, keepdims=True)
    return (p @ v) / l_sum, (m + np.log(l_sum))[:, 0]


def merge(o1, l1, o2, l2):
    m = np.maximum(l1, l2)
    w1, w2 = np.exp(l1 - m), np.exp(l2 - m)
    lse = m + np.log(w1 + w2)
    return (o1 * (w1 / (w1 + w2))[:, None] + o2 * (w2 / (w1 + w2))[:, None]), lse


def run(n, rows, kv, d, sharp, seed):
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (rows, d)) * sharp
    k = rng.uniform(-1, 1, (n * kv, d))
    v = rng.uniform(-1, 1, (n * kv, d))
    scale = d ** -0.5
    exact, _ = partial(q, k, v, scale)
    ref_scale = np.abs(exact).max()
    out_round = np.abs(bf16(exact) - exact).max() / ref_scale
    res = {"sharpen": sharp, "final_bf16_rounding": out_round}
    for name, o_wire, l_wire in (("O f32, L f32 (this repo)", f32, f32),
                                 ("O bf16, L f32", bf16, f32),
                                 ("O bf16, L bf16 (paper's bf16 Q+O model)", bf16, bf16)):
        o, lse = None, None
        for r in range(n):
            po, pl = partial(q, k[r * kv:(r + 1) * kv], v[r * kv:(r + 1) * kv], scale)
            if o is None:
                o, lse = po, pl
            else:
                o, lse = merge(o, lse, po, pl)
            if r < n - 1:                  # the state crosses a link after every round but the last
                o, lse = o_wire(o), l_wire(lse)
        err = np.abs(bf16(o) - exact).max() / ref_scale
        res[name] = {"max_norm_error": err, "x_final_rounding": err / out_round}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--kv", type=int, default=2048)
    ap.add_argument("--d", type=int, default=128)
    a = ap.parse_args()
    out = {"tool": "wire_dtype_error", "n": a.n, "rows": a.rows, "kv_rows_per_shard": a.kv,
           "d": a.d, "cases": [run(a.n, a.rows, a.kv, a.d, s, 7) for s in (1.0, 8.0)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
