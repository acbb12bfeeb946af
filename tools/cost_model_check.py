"""Cost model (paper_2502_02406_b200.analytics) vs measured bench runs.

    python tools/cost_model_check.py [profiles/r02_bench_c2_n2.json ...]

For each committed bench line: the model's per-round compute / comm times at
the B200 GEMM peak, the same with the compute side calibrated to the
measured kernel times, and the predicted vs measured LV-XAttn step and
Ring / LV-XAttn ratio.  Prints a markdown table."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2502_02406_b200 import analytics as A  # noqa: E402


def row(path: Path) -> dict:
    d = json.loads([ln for ln in path.read_text().splitlines() if ln.startswith("{")][-1])
    c = d["config"]
    n = d["n_gpus"]
    w = A.WorkloadSpec.b200(c["s_q"], c["s_kv"], c["hq"], c["hkv"], c["d"], n)
    ph = d["roofline"]["phase_ms_per_step"]
    fwd_round = ph["fwd_kernel"] / 1e3 / n
    bwd_round = (ph["dq_kernel"] + ph["dkv_kernel"] + ph.get("dq_finish", 0)) / 1e3 / n
    peak = A.HardwareSpec.b200(sustained=True)
    t_peak = A.round_times(w, peak)
    hf, hb = A.calibrate(w, fwd_round, bwd_round)
    t_f, t_b = A.round_times(w, hf), A.round_times(w, hb)
    lvx_pred = n * (t_f["lvx"].round_fwd + t_b["lvx"].round_bwd)
    ring_pred = n * (t_f["ring"].round_fwd + t_b["ring"].round_bwd)
    out = {"n": n, "measured_step_ms": d["ms_per_step"],
           "model_step_ms_at_peak": 1e3 * n * (t_peak["lvx"].round_fwd + t_peak["lvx"].round_bwd),
           "model_step_ms_calibrated": 1e3 * lvx_pred,
           "fwd_round_ms_measured": fwd_round * 1e3,
           "fwd_round_ms_model_peak": t_peak["lvx"].compute_fwd * 1e3,
           "lvx_comm_fwd_ms": t_peak["lvx"].comm_fwd * 1e3,
           "ring_comm_fwd_ms": t_peak["ring"].comm_fwd * 1e3,
           "regime": A.classify_regime(w, peak).as_dict()}
    rb = d.get("ring_baseline") or {}
    if rb:
        out["ring_over_lvx_measured"] = rb["ms_per_step"] / d["ms_per_step"]
        out["ring_over_lvx_model_calibrated"] = ring_pred / lvx_pred
        if P2P and n > 1:   # the same with the measured shift bandwidth per hop size (p2p_bw.py)
            def at(nbytes):
                return A.HardwareSpec(1.0, p2p_bandwidth(nbytes))
            ring_t = 0.0
            for phase, hw in (("forward", hf), ("backward", hb)):
                comp = A.attention_round_flops(w, phase) / hw.gpu_flops
                nb = A.round_comm_bytes("ring", phase, w)
                ring_t += n * max(comp, nb / at(nb).net_bandwidth)
            out["ring_over_lvx_model_measured_net"] = ring_t / lvx_pred
            out["ring_hop_GBps_measured"] = p2p_bandwidth(A.round_comm_bytes("ring", "forward", w)) / 1e9
    return out


P2P = None
# the ring's transport: the copy-engine shift of round 2 (tools/p2p_bw.py)
_p2p = ROOT / "profiles" / "r02_p2p_bw_ce_n4.json"
if _p2p.exists():
    P2P = sorted((int(k[:-3]) << 20, v["GBps_per_direction"] * 1e9)
                 for k, v in json.loads([ln for ln in _p2p.read_text().splitlines()
                                         if ln.startswith("{")][-1])["shift"].items())


def p2p_bandwidth(nbytes: float) -> float:
    """Measured shift bandwidth (tools/p2p_bw.py), log-interpolated in size."""
    import math
    if nbytes <= P2P[0][0]:
        return P2P[0][1]
    for (s0, b0), (s1, b1) in zip(P2P, P2P[1:]):
        if nbytes <= s1:
            f = (math.log(nbytes) - math.log(s0)) / (math.log(s1) - math.log(s0))
            return b0 + f * (b1 - b0)
    return P2P[-1][1]


def main():
    paths = [Path(p) for p in sys.argv[1:]] or [
        ROOT / "profiles" / f for f in ("r02_bench_c2_n2.json", "r02_bench_c2_n4.json",
                                        "r02_bench_c2_n4_skv524288.json")]
    rows = [row(p) for p in paths]
    print("| n | measured ms/step | model @sustained peak | model calibrated | fwd round meas / model (ms) "
          "| LVX / Ring fwd hop (ms @900 GB/s) | regime (lvx / ring) | Ring/LVX meas | Ring/LVX model "
          "| Ring/LVX model, measured shift GB/s |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['n']} | {r['measured_step_ms']:.1f} | {r['model_step_ms_at_peak']:.1f} | "
              f"{r['model_step_ms_calibrated']:.1f} | {r['fwd_round_ms_measured']:.2f} / "
              f"{r['fwd_round_ms_model_peak']:.2f} | {r['lvx_comm_fwd_ms']:.3f} / "
              f"{r['ring_comm_fwd_ms']:.2f} | {r['regime']['lvx_bound']} / "
              f"{r['regime']['ring_bound']} | {r.get('ring_over_lvx_measured', float('nan')):.2f} | "
              f"{r.get('ring_over_lvx_model_calibrated', float('nan')):.2f} | "
              f"{r.get('ring_over_lvx_model_measured_net', float('nan')):.2f} "
              f"({r.get('ring_hop_GBps_measured', float('nan')):.0f} GB/s) |")
    print()
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
