"""LV-XAttn fwd+bwd benchmark on B200 (BASELINE.json configs[1], Llama-3-V).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--strategy lvx|ring]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)
    python bench.py --impl reference ...                   (the reference CPU path)

Workload (strong scaling; total work fixed as N grows): one cross-attention
layer, Lq = 2048 text queries, 32 query heads / 8 KV heads (GQA), head_dim 128,
Lkv = 1,048,576 visual tokens, bf16 inputs, forward + backward.  Each rank
holds its 1/N shard of K/V (and of Q/dO) resident in HBM; a step is one
lvx_forward + lvx_backward (Algorithm 1 + its backward) over NCCL.
Inputs are synthetic uniform[-1, 1] (seeded, generated on the device); every
rank's K/V shard (>= 512 MiB) is larger than the 126 MB L2, so no L2 flush is
needed between steps.

Printed (rank 0, one JSON line): value = whole-job attention TFLOP/s
(14 Lq Lkv hq d per step), ms_per_step = ms per layer fwd+bwd,
the roofline of the dominant kernel, the no-communication arm (same schedule,
hops skipped) and the overhead against it, measured NVLink
bytes per step against the closed form and the paper's Q+O model, the
Ring-Attention baseline (N > 1), the CPU reference timed on the host, the
end-to-end number through the host-buffer API, clocks, and kernel launches.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# BASELINE.json configs[1..4]; C2 is the headline (the driver's default run)
WORKLOADS = {
    "c2": dict(workload="llama3v-cross-attn-C2", s_q=2048, s_kv=1 << 20, hq=32, hkv=8, d=128),
    # mPLUG-Owl3: Lkv sweep 256K..4M (headline point 1M)
    "c3": dict(workload="owl3-cross-attn-C3", s_q=5514, s_kv=1 << 20, hq=28, hkv=4, d=128,
               sweep=[1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22]),
    # OpenFlamingo gated cross-attn: L layers sharing one visual-token copy y,
    # K/V recomputed from y in the backward (d_embed 2048, OpenFlamingo-3B-like)
    "c4": dict(workload="openflamingo-xattn-C4", s_q=1024, s_kv=1 << 19, hq=8, hkv=8, d=64,
               layers=4, d_embed=2048),
    # scaling sweep, Llama-3-V heads: Lkv 64K..15M, LV-XAttn vs Ring
    "c5": dict(workload="lkv-sweep-C5", s_q=2048, s_kv=1 << 20, hq=32, hkv=8, d=128,
               sweep=[1 << 16, 1 << 18, 1 << 20, 1 << 22, 15_000_000]),
}
CFG = dict(WORKLOADS["c2"])
METRIC = "cross-attn fwd+bwd ms/layer & TFLOP/s at 1/2/4/8 B200; overhead vs no-comm bound"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--strategy", default="lvx", choices=["lvx", "ring"])
    ap.add_argument("--no-ring-compare", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay leg")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS),
                    help="BASELINE config (c2 = the headline; c3 / c5 sweep Lkv, c4 = layers "
                         "with K/V recompute)")
    ap.add_argument("--skv", type=int, default=None, help="Lkv (default: the workload's)")
    ap.add_argument("--sweep", default=None,
                    help="comma-separated Lkv list (default: the workload's sweep, if any)")
    a = ap.parse_args()
    wl = WORKLOADS[a.workload]
    CFG.clear()
    CFG.update({k: v for k, v in wl.items() if k != "sweep"})
    if a.skv is not None:
        CFG["s_kv"] = a.skv
    if a.sweep:
        a.points = [int(float(x)) for x in a.sweep.split(",")]
    elif a.skv is None and "sweep" in wl:
        a.points = list(wl["sweep"])
    else:
        a.points = [CFG["s_kv"]]
    a.skv = CFG["s_kv"]
    return a


# ---------------------------------------------------------------- helpers

def peaks():
    """(burst, sustained, hbm, kind, SM MHz the sustained GEMM ran at)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        mhz = (j.get("clocks_under_load") or {}).get("sm_mhz_median")
        return j["bf16_tflops"], j["bf16_tflops_sustained"], j["hbm_gbs"], "measured", mhz
    return 1590.0, 1400.0, 6650.0, "fallback", None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "window", (0.0, float("inf")))
        inside = [ln for ts, ln in self.lines if t0 - 0.05 <= ts <= t1 + 0.15]
        if not inside:   # timed region shorter than one sample: nearest samples
            inside = [ln for ts, ln in sorted(self.lines, key=lambda x: abs(x[0] - t1))[:3]]
        for ln in inside:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


def cpu_reference_rate(budget_s: float = 12.0):
    """The reference algorithm on the host cores (oracle port of
    strategies.py lvx fwd+bwd, numpy f64 + multithreaded BLAS), on a bounded
    sample of the C2 workload: Lq=64 query rows x Lkv=16384 visual tokens, same
    heads/head_dim, repeated until ``budget_s``.  Returns (TFLOP/s, sample)."""
    import numpy as np
    from oracle import lvx_oracle as orc
    sq, skv = 64, 16384
    Q, K, V, dO = orc.make_inputs(sq, skv, CFG["hq"], CFG["d"], seed=7, hkv=CFG["hkv"])
    Q, K, V, dO = (t.astype(np.float32) for t in (Q, K, V, dO))
    flops = orc.attention_flops(sq, skv, CFG["hq"], CFG["d"])
    # all host cores for BLAS, whatever OMP_NUM_THREADS torchrun exported
    from threadpoolctl import threadpool_info, threadpool_limits
    with threadpool_limits(limits=os.cpu_count(), user_api="blas"):
        threads = max((i.get("num_threads", 1) for i in threadpool_info()
                       if i.get("user_api") == "blas"), default=1)
        reps, t0 = 0, time.perf_counter()
        while True:
            orc.simulate("lvx", Q, K, V, dO, n=1)
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget_s or reps >= 50:
                break
    sample = (f"oracle port of lvx fwd+bwd (numpy f64, {threads} host threads BLAS), "
              f"Lq={sq} x Lkv={skv}, hq=32/hkv=8, d=128, fp32 in, {reps} reps in {el:.1f}s")
    return flops * reps / el / 1e12, sample, threads


def reference_arm(args):
    """The reference's algorithm on the host cores (the oracle port of
    strategies.py lvx fwd + bwd, numpy f64 + multithreaded BLAS).  A step is
    ONE bounded sample of the workload — the C2 heads / head_dim on 64 query
    rows x 16384 KV rows — because the full layer takes about an hour of CPU;
    ms_per_step is that sample step's wall time and value its TFLOP/s, so the
    rate is comparable with the GPU's and every step is really run."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from threadpoolctl import threadpool_info, threadpool_limits
    from oracle import lvx_oracle as orc
    sq, skv = 64, 16384
    Q, K, V, dO = orc.make_inputs(sq, skv, CFG["hq"], CFG["d"], seed=7, hkv=CFG["hkv"])
    Q, K, V, dO = (t.astype(np.float32) for t in (Q, K, V, dO))
    flops = orc.attention_flops(sq, skv, CFG["hq"], CFG["d"])
    times = []
    with threadpool_limits(limits=os.cpu_count(), user_api="blas"):
        threads = max((i.get("num_threads", 1) for i in threadpool_info()
                       if i.get("user_api") == "blas"), default=1)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            orc.simulate("lvx", Q, K, V, dO, n=1)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    sec = statistics.median(times)
    val = flops / sec / 1e12
    sample = (f"oracle port of lvx fwd+bwd (numpy f64, {threads} host threads BLAS) on "
              f"Lq={sq} x Lkv={skv} rows of the workload, hq={CFG['hq']}/hkv={CFG['hkv']}, "
              f"d={CFG['d']}, fp32 in; one sample per step")
    line = {"metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**CFG, "sample_s_q": sq, "sample_s_kv": skv,
                       "note": "a step = one bounded sample of the workload (same heads, "
                               "head_dim and dtype path); the rate is the compared quantity"},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- native arm

class Env:
    """Per-process run context shared by the measurement legs."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.world}; "
                             "launch N>1 with torchrun")
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.group = None
        if self.world > 1:
            # the process group carries only setup, barriers and the timing
            # reduction; the ring hops are copy-engine transfers (comm.py)
            dist.init_process_group("nccl", device_id=self.dev)
            self.group = dist.group.WORLD
        from paper_2502_02406_b200 import build
        if self.rank == 0 and not build.LIB.exists():
            build.build()
        if self.world > 1:
            dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return x
        t = torch.tensor([x], device=self.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()


def native_arm(args):
    import torch
    env = Env(args)
    if args.workload == "c4":
        out = layer_arm(args, env)
    else:
        import paper_2502_02406_b200 as lvx
        ctx = lvx.DeviceContext(env.rank, env.world, group=env.group, device=env.dev)
        # the no-comm arm: its own arena and side stream; its hops are local
        # copies of the send blocks into its receive slots
        ctx_nc = lvx.DeviceContext(env.rank, env.world, group=env.group, device=env.dev,
                                   comm_enabled=False)
        head_skv = CFG["s_kv"] if CFG["s_kv"] in args.points else args.points[-1]
        lines = []
        for skv in args.points:
            lines.append(measure_point(args, env, ctx, ctx_nc, skv, head=(skv == head_skv)))
            gc.collect()               # the point's closures hold its shard tensors
            ctx.release_arena()        # the Ring's K/V slots are sized for this point
            ctx_nc.release_arena()
            torch.cuda.empty_cache()
        out = next(ln for ln, skv in zip(lines, args.points) if skv == head_skv)
        if len(lines) > 1:
            out["sweep"] = [_summary(ln) for ln in lines]
    if env.rank == 0 and env.world == 1 and not args.no_cpu:
        v, sample, threads = cpu_reference_rate()
        out["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                               "sample": sample + " (TFLOP/s on a sample, not the full workload)",
                               "c1": cpu_c1_timing()}
    if env.rank == 0:
        print(json.dumps(out), flush=True)
    if env.world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _summary(line: dict) -> dict:
    keep = ("value", "ms_per_step", "overhead_vs_no_comm", "no_comm_ms_per_step",
            "host_submit_ms_per_step")
    out = {"s_kv": line["config"]["s_kv"], **{k: line.get(k) for k in keep}}
    gr = line.get("graph_replay") or {}
    if "ms_per_step" in gr:
        out["graph_ms_per_step"] = gr["ms_per_step"]
        out["graph_value"] = gr["value"]
    out["roofline_frac"] = line["roofline"]["frac"]
    out["fwd_tflops"] = line["roofline"]["fwd_tflops"]
    out["bwd_tflops"] = line["roofline"]["bwd_tflops"]
    rb = line.get("ring_baseline") or {}
    if "ms_per_step" in rb:
        out["ring_ms_per_step"] = rb["ms_per_step"]
        out["speedup_lvx_over_ring"] = rb["speedup_lvx_over_ring"]
    elif rb:
        out["ring"] = rb.get("skipped")
    return out


def measure_point(args, env, ctx, ctx_nc, s_kv, head=True):
    """One (workload, Lkv) point: the timed lvx (or ring) fwd+bwd steps, the
    dominant kernel's roofline, the no-comm A/B and the Ring baseline at
    N > 1, and (``head``) the end-to-end host-buffer leg."""
    import torch
    from paper_2502_02406_b200 import _lib, volumes
    from paper_2502_02406_b200.strategies import (RoundTrace, ShardSpec, lvx_backward,
                                                  lvx_forward, ring_backward,
                                                  ring_backward_reference_schedule, ring_forward)
    world, rank, local, dev = env.world, env.rank, env.local, env.dev
    s_q, hq, hkv, d = CFG["s_q"], CFG["hq"], CFG["hkv"], CFG["d"]
    scale = 1.0 / d ** 0.5
    shards = ShardSpec.balanced(s_q, s_kv, world)
    qa, qb = shards.q_ranges[rank]
    ka, kb = shards.kv_ranges[rank]
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def rnd(h, rows, dd):
        # uniform[-1, 1) bf16, generated by row chunks: no full-size fp32
        # temporaries (at Lkv 15M one would be 61 GB)
        t = torch.empty((h, rows, dd), device=dev, dtype=torch.bfloat16)
        for a in range(0, rows, 1 << 20):
            b = min(rows, a + (1 << 20))
            t[:, a:b] = torch.rand((h, b - a, dd), device=dev, generator=gen) * 2 - 1
        return t

    q_i, k_i, v_i, do_i = rnd(hq, qb - qa, d), rnd(hkv, kb - ka, d), rnd(hkv, kb - ka, d), \
        rnd(hq, qb - qa, d)
    fwd, bwd = (lvx_forward, lvx_backward) if args.strategy == "lvx" else \
        (ring_forward, ring_backward)

    def step(c, traces=None, strategy=None):
        f, b = (fwd, bwd) if strategy is None else strategy
        tf = RoundTrace("x", "forward") if traces is not None else None
        tb = RoundTrace("x", "backward") if traces is not None else None
        st = f(c, shards, q_i, k_i, v_i, scale, 64, tf)
        g = b(c, shards, q_i, k_i, v_i, st, do_i, scale, tb)
        if traces is not None:
            traces.append((tf, tb))
        return st, g

    host_stats = {}

    def timed(c, steps, warm, strategy=None, sampler=False):
        cs = ClockSampler(local) if sampler else None
        if cs:
            cs.__enter__()
        for _ in range(warm):
            step(c, strategy=strategy)
        torch.cuda.synchronize()
        env.barrier()
        traces = []
        launches0 = _lib.load().lvx_kernel_launches()
        w0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for _ in range(steps):
            step(c, traces, strategy)
        host_ms = (time.perf_counter() - h0) * 1e3 / steps   # host submission time per step
        e1.record()
        torch.cuda.synchronize()
        if cs:
            cs.mark(w0, time.time())
            time.sleep(0.15)
            cs.__exit__()
        env.barrier()
        launches = _lib.load().lvx_kernel_launches() - launches0
        ms = e0.elapsed_time(e1) / steps
        for tf, tb in traces:
            tf.resolve()
            tb.resolve()
        host_stats["host_ms"] = env.max_over_ranks(host_ms)
        return env.max_over_ranks(ms), traces, launches, (cs.summary() if cs else None)

    ms, traces, launches, clocks = timed(ctx, args.steps, args.warmup, sampler=True)
    flops = volumes.attention_flops(s_q, s_kv, hq, d)
    value = flops / (ms * 1e-3) / 1e12

    # --- kernel roofline: dominant kernel by device time inside the timed region
    def sec(tr_list, name):
        return statistics.mean(t.sections.get(name, 0.0) for t in tr_list)

    tfs, tbs = [tf for tf, _ in traces], [tb for _, tb in traces]
    n_rounds = len(traces[0][0].rounds)
    qrows, kvrows = s_q / world, kb - ka
    unit = qrows * kvrows * hq * d                      # one (q block, kv shard) pair
    phases = {"fwd_kernel": sec(tfs, "fwd_kernel"), "fwd_finish": sec(tfs, "fwd_finish"),
              "fwd_wait": sec(tfs, "wait"), "dq_kernel": sec(tbs, "dq_kernel"),
              "dq_finish": sec(tbs, "dq_finish"), "bwd_wait": sec(tbs, "wait"),
              "dkv_kernel": sec(tbs, "dkv_kernel")}
    # algorithmic FLOP per launch (PAPER.md:67 split by product): fwd 4 units per
    # round; dQ kernel 2 (dS K) + the S, dP it recomputes are counted in dkv;
    # dkv kernel 8 (S, dP, dV, dK) over all n blocks in one launch.
    kernels = {"fwd_kernel (tcgen05)": (4.0 * unit, phases["fwd_kernel"] / n_rounds),
               "dkv_kernel (tcgen05)": (8.0 * unit * n_rounds, phases["dkv_kernel"]),
               "dq_kernel (tcgen05)": (2.0 * unit, phases["dq_kernel"] / n_rounds)}
    if args.strategy == "ring":   # ring backward runs the fused per-round backward
        rb = statistics.mean(sum(r.compute_seconds for r in tb.rounds) for tb in tbs)
        kernels = {"fwd_kernel (tcgen05)": kernels["fwd_kernel (tcgen05)"],
                   "ring_bwd (dkv+dq per round)": (10.0 * unit, rb / n_rounds)}
    kernels = {k: v for k, v in kernels.items() if v[1] > 0}
    kname = max(kernels, key=lambda k: kernels[k][1] * (n_rounds if "dkv" not in k else 1))
    kflops, kdur = kernels[kname]
    burst, sust, hbm, pk_kind, sust_mhz = peaks()
    achieved = kflops / kdur / 1e12
    # The sustained peak is cuBLAS under the power cap at the SM clock in
    # MEASURED_PEAKS clocks_under_load; tensor throughput scales with the SM
    # clock, so a timed region that ran faster (less work per GPU at N > 1) is
    # measured against that peak scaled up to its clock, never above burst.
    # Never scaled DOWN: the clock is a median over the whole step, not the
    # dominant kernel's own clock, and the measured sustained figure is what a
    # capped B200 delivers.
    run_mhz = (clocks or {}).get("sm_mhz")
    if run_mhz and sust_mhz:
        peak = min(burst, max(sust, sust * run_mhz / sust_mhz))
        peak_kind = (f"{pk_kind} bf16 sustained {sust} TFLOP/s at {sust_mhz} MHz, scaled up to "
                     f"the {run_mhz} MHz SM clock of this timed region when higher (capped at "
                     f"burst {burst})")
    else:
        peak = sust
        peak_kind = f"{pk_kind} bf16 sustained (kernel timed inside a long step)"
    traffic, traffic_src = None, None
    tj = ROOT / "profiles" / "r02_traffic.json"
    if world == 1 and args.strategy == "lvx" and args.workload == "c2" and \
            s_kv == WORKLOADS["c2"]["s_kv"] and tj.exists():
        # ncu DRAM bytes per launch of this kernel at this exact launch shape
        rec = json.loads(tj.read_text())["per_launch"].get(kname)
        if rec:
            traffic = rec["dram_bytes_read"] + rec["dram_bytes_write"]
            traffic_src = {"file": "profiles/r02_traffic.json", "read": rec["dram_bytes_read"],
                           "write": rec["dram_bytes_write"], "algorithmic": rec["algorithmic_bytes"]}
    roofline = {"kernel": kname, "bound": "tensor", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_detail": traffic_src, "peak_kind": peak_kind,
                "frac_of_sustained": achieved / sust, "frac_of_burst": achieved / burst,
                "frac_of_nominal_2250": achieved / 2250.0,
                "per_launch_ms": kdur * 1e3,
                "phase_ms_per_step": {k: v * 1e3 for k, v in phases.items()},
                # every hot kernel: algorithmic FLOP (the paper's 4 / 10 units)
                # and the tensor work it actually issues (dK/dV and dQ both
                # recompute S and dP: 8 + 6 issued units for 10 algorithmic)
                "kernels": {name: {
                    "ms_per_step": phases[ph] * 1e3,
                    "algorithmic_tflops": alg * unit * n_rounds / max(phases[ph], 1e-9) / 1e12,
                    "issued_tflops": iss * unit * n_rounds / max(phases[ph], 1e-9) / 1e12,
                    "issued_frac_of_peak": iss * unit * n_rounds / max(phases[ph], 1e-9) / 1e12
                    / peak}
                    for name, ph, alg, iss in (("fwd_kernel", "fwd_kernel", 4.0, 4.0),
                                               ("dq_kernel", "dq_kernel", 2.0, 6.0),
                                               ("dkv_kernel", "dkv_kernel", 8.0, 8.0))
                    if phases.get(ph, 0) > 0 and args.strategy == "lvx"},
                "fwd_tflops": 4.0 * unit * n_rounds / max(phases["fwd_kernel"], 1e-9) / 1e12,
                "bwd_tflops": 10.0 * unit * n_rounds /
                max(phases["dkv_kernel"] + phases["dq_kernel"] + phases["dq_finish"], 1e-9) / 1e12}

    # --- measured NVLink bytes vs closed form and the paper's model
    tf0, tb0 = traces[0]
    sent = tf0.total_sent_bytes() + tb0.total_sent_bytes()
    w = volumes.Wire.b200(hq, hkv, d, 2)
    model = (volumes.bytes_by_worker(args.strategy, "forward", shards.q_sizes, shards.kv_sizes, w)[rank]
             + volumes.bytes_by_worker(args.strategy, "backward", shards.q_sizes, shards.kv_sizes, w)[rank])
    comm = {"transport": ctx.transport_kind,
            "bytes_per_step_rank0": sent, "closed_form_rank0": model,
            "paper_q_plus_o_hop_bytes_bf16": volumes.paper_hop_bytes(s_q, world, hq, d, 2),
            "measured_fwd_hop_bytes": (tf0.rounds[0].sent_bytes if world > 1 else 0),
            "exposed_comm_ms_per_step": sum(r.comm_seconds for r in tf0.rounds + tb0.rounds) * 1e3}

    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_layer": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (uniform[-1,1], seeded, generated on device)",
           "config": {**CFG, "s_kv": s_kv, "strategy": args.strategy,
                      "parallelism": f"kv-seq-parallel x{world} (query rotation)"
                      if args.strategy == "lvx" else f"kv-rotation x{world}",
                      "l2": "inputs larger than L2 (K/V shard >= 16 MiB per rank and the "
                            "step touches > 126 MB)"},
           "roofline": roofline, "comm": comm, "clocks": clocks,
           "gpu_launches": int(launches),
           # host time to submit one step (Python schedulers + C ABI calls); a
           # step whose device time is not well above it is launch-bound
           "host_submit_ms_per_step": host_stats["host_ms"]}

    # --- the same step recorded once as a CUDA graph and replayed (no host
    # work per step: the kernels, copy-engine hops and one-shot flags replay)
    if not args.no_graph:
        out["graph_replay"] = graph_replay(env, ctx, lambda: step(ctx), args.steps, flops)

    # --- no-communication arm and the Ring baseline
    if world > 1:
        # the identical schedule with every hop skipped, measured as interleaved
        # A/B step pairs so power-cap and clock drift hit both arms equally
        pairs = max(20, 2 * args.steps)
        step(ctx_nc)     # the no-comm arm's first call (outside the pairs)
        a_ms, b_ms = [], []
        for pi in range(pairs):
            # ABBA order: whichever arm runs first in a pair gets the idle gap
            arms = ((ctx, a_ms), (ctx_nc, b_ms)) if pi % 2 == 0 else ((ctx_nc, b_ms), (ctx, a_ms))
            for c, acc in arms:
                torch.cuda.synchronize()
                env.barrier()
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ea.record()
                step(c)
                eb.record()
                torch.cuda.synchronize()
                acc.append(env.max_over_ranks(ea.elapsed_time(eb)))
        ms_a, ms_b = statistics.median(a_ms), statistics.median(b_ms)
        # per-pair ratios: clock drift under the power cap moves both steps of
        # a pair together, so the median ratio is the robust overhead figure
        ratios = sorted(a / b for a, b in zip(a_ms, b_ms))
        out["no_comm_ms_per_step"] = ms_b
        out["overhead_vs_no_comm"] = statistics.median(ratios) - 1.0
        out["no_comm_ab"] = {"pairs": pairs, "comm_ms_median": ms_a, "no_comm_ms_median": ms_b,
                             "overhead_of_medians": ms_a / ms_b - 1.0,
                             "pair_ratio_iqr": [ratios[len(ratios) // 4] - 1.0,
                                                ratios[(3 * len(ratios)) // 4] - 1.0],
                             "comm_ms": a_ms, "no_comm_ms": b_ms}
        ms_nc, tr_nc, *_ = timed(ctx_nc, max(2, args.steps // 2), 1)
        out["no_comm_block_ms_per_step"] = ms_nc
        out["no_comm_phase_ms_per_step"] = {
            "fwd_kernel": sec([a for a, _ in tr_nc], "fwd_kernel") * 1e3,
            "dq_kernel": sec([b for _, b in tr_nc], "dq_kernel") * 1e3,
            "dkv_kernel": sec([b for _, b in tr_nc], "dkv_kernel") * 1e3}
        ring_fits = _ring_fits(env, shards, hq, hkv, d, dev)
        if not args.no_ring_compare and args.strategy == "lvx" and not ring_fits:
            out["ring_baseline"] = {"skipped": "the Ring baseline's rotating K/V slots and fp32 "
                                               "dK/dV partials do not fit in HBM at this Lkv"}
        elif not args.no_ring_compare and args.strategy == "lvx":
            ms_ring, rtr, *_ = timed(ctx, max(2, args.steps // 2), 1,
                                     strategy=(ring_forward, ring_backward))
            out["ring_baseline"] = {"ms_per_step": ms_ring,
                                    "value": flops / (ms_ring * 1e-3) / 1e12,
                                    "speedup_lvx_over_ring": ms_ring / ms,
                                    "schedule": "K/V sent at the start of each round, dK/dV "
                                                "partials one hop behind (overlapped)",
                                    "bytes_per_step_rank0": rtr[0][0].total_sent_bytes()
                                    + rtr[0][1].total_sent_bytes()}
            # the Ring in the reference's own order (compute, then shift and wait)
            if not _ring_fits(env, shards, hq, hkv, d, dev, reference_order=True):
                out["ring_baseline_reference_schedule"] = {
                    "skipped": "two (K, V, dK, dV) records do not fit in HBM at this Lkv"}
                return _finish(out, args, head, ctx, shards, q_i, k_i, v_i, do_i, scale, fwd,
                               bwd, flops, world, dev)
            ms_rref, _, *_ = timed(ctx, max(2, args.steps // 2), 1,
                                   strategy=(ring_forward, ring_backward_reference_schedule))
            out["ring_baseline_reference_schedule"] = {
                "ms_per_step": ms_rref, "value": flops / (ms_rref * 1e-3) / 1e12,
                "speedup_lvx_over_ring": ms_rref / ms,
                "schedule": "strategies.py:314-361 order: compute, then (K, V, dK, dV) shift, "
                            "then wait"}
    else:
        out["no_comm_ms_per_step"] = ms
        out["overhead_vs_no_comm"] = 0.0

    return _finish(out, args, head, ctx, shards, q_i, k_i, v_i, do_i, scale, fwd, bwd, flops,
                   world, dev)


def _finish(out, args, head, ctx, shards, q_i, k_i, v_i, do_i, scale, fwd, bwd, flops, world,
            dev):
    # --- end to end through the host-buffer API (pinned host -> HBM -> host)
    if head and not args.no_e2e:
        try:
            out["e2e"] = e2e_arm(args, ctx, shards, (q_i, k_i, v_i, do_i), scale, fwd, bwd,
                                 flops, world, dev)
        except (RuntimeError, MemoryError) as exc:   # e.g. pinned host memory; the line stands
            out["e2e"] = {"error": repr(exc)[:300]}
    return out


def _ring_fits(env, shards, hq, hkv, d, dev, reference_order: bool = False) -> bool:
    """Whether ring_backward's buffers fit beside what is resident: per rank
    RING_SLOTS bf16 K/V slots, as many fp32 dK/dV partial slots, the fp32
    homecoming, its own and a scratch fp32 dK/dV, and the bf16 gradients
    (strategies.ring_backward).  Decided collectively (min over ranks)."""
    import torch
    from paper_2502_02406_b200.strategies import RING_SLOTS
    n = env.world
    mk = max(shards.kv_sizes)
    slots = max(1, min(RING_SLOTS, n - 1))
    kv = hkv * mk * d
    if reference_order:   # two (K, V, dK, dV) records + homecoming + acc / tmp + grads
        need = 2 * (kv * 2 * 2 + kv * 4 * 2) + kv * 4 * 2 + 2 * kv * 4 * 2 + kv * 2 * 2
    else:
        need = slots * kv * 2 * 2 + slots * kv * 4 * 2 + kv * 4 * 2 + 2 * kv * 4 * 2 + kv * 2 * 2
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(dev)
    ok = torch.tensor([1.0 if need < 0.9 * free else 0.0], device=dev)
    if n > 1:
        import torch.distributed as dist
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return bool(ok.item() > 0)


def graph_replay(env, ctx, fn, steps, flops) -> dict:
    """Time ``steps`` replays of ``fn`` recorded as a StepGraph (CUDA events,
    max over ranks).  The graph and its memory pool are released after."""
    import torch
    from paper_2502_02406_b200.strategies import StepGraph
    try:
        g = StepGraph(ctx, fn)
    except Exception as exc:  # noqa: BLE001 - reported, the eager number stands
        return {"error": f"capture failed: {exc!r}"[:300]}
    g.replay()
    torch.cuda.synchronize()
    env.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(steps):
        g.replay()
    host_ms = (time.perf_counter() - h0) * 1e3 / steps
    e1.record()
    torch.cuda.synchronize()
    env.barrier()
    ms = env.max_over_ranks(e0.elapsed_time(e1) / steps)
    del g
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "value": flops / (ms * 1e-3) / 1e12,
            "host_submit_ms_per_step": env.max_over_ranks(host_ms), "steps": steps}


def cpu_c1_timing(reps: int = 3) -> dict:
    """BASELINE configs[0] exactly (Lq 128, Lkv 4096, 8 heads, d 64, fp32,
    simulated world_size 2): the oracle port of lvx fwd+bwd at 1 BLAS
    thread and at all host threads, best of ``reps`` each."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import lvx_oracle as orc
    Q, K, V, dO = (t.astype(np.float32) for t in orc.make_inputs(128, 4096, 8, 64, seed=1))
    out = {"config": "C1: Lq 128, Lkv 4096, h 8, d 64, fp32, n 2 (oracle port of the "
                     "reference's lvx fwd+bwd)", "cpu_count": os.cpu_count()}
    for key, threads in (("ms_1_thread", 1), ("ms_all_threads", os.cpu_count())):
        with threadpool_limits(limits=threads, user_api="blas"):
            best = float("inf")
            for _ in range(reps):
                t0 = time.perf_counter()
                orc.simulate("lvx", Q, K, V, dO, n=2)
                best = min(best, time.perf_counter() - t0)
        out[key] = best * 1e3
    return out


def layer_arm(args, env):
    """C4: ``layers`` OpenFlamingo cross-attention layers sharing ONE copy of
    the visual tokens y, RECOMPUTE_KV (K/V re-projected from y in the
    backward), lvx over the ranks.  A step = forward through all layers, then
    backward through them in reverse.  value = algorithmic TFLOP/s of the
    whole step: attention (14 Lq Lkv hq d per layer) + every projection GEMM
    (Q, K/V, O forward; the K/V recompute; dX, dY and weight gradients)."""
    import torch
    import paper_2502_02406_b200 as lvx
    from paper_2502_02406_b200 import _lib, volumes
    from paper_2502_02406_b200.recompute import (ActivationPolicy, CrossAttentionWeights,
                                                 OpCounter, VisualGradSink, ca_backward,
                                                 ca_forward)
    world, rank, dev = env.world, env.rank, env.dev
    s_q, s_kv, hq, hkv, d = CFG["s_q"], CFG["s_kv"], CFG["hq"], CFG["hkv"], CFG["d"]
    e, nl = CFG["d_embed"], CFG["layers"]
    sh = lvx.ShardSpec.balanced(s_q, s_kv, world)
    (qa, qb), (ka, kb) = sh.q_ranges[rank], sh.kv_ranges[rank]
    g = torch.Generator(device=dev).manual_seed(77)

    def r(*shape, sc=1.0):
        return ((torch.rand(*shape, device=dev, generator=g) * 2 - 1) * sc).bfloat16()
    ws = 0.5 / e ** 0.5
    layers = [CrossAttentionWeights(r(e, hq * d, sc=ws), r(e, hkv * d, sc=ws),
                                    r(e, hkv * d, sc=ws), r(hq * d, e, sc=ws), hq, hkv)
              for _ in range(nl)]
    x0, y, go = r(qb - qa, e), r(kb - ka, e), r(qb - qa, e)
    ctx = lvx.DeviceContext(rank, world, group=env.group, device=dev)

    def step(policy, counter=None):
        x, saved = x0, []
        for w in layers:
            x, sv = ca_forward(ctx, sh, x, y, w, policy)
            saved.append(sv)
        gx = go
        # every layer leaves [dK | dV] in the sink; dY = ONE GEMM over all layers
        sink = VisualGradSink(y, [w.kv_weight().shape[1] for w in layers])
        for w, sv in zip(reversed(layers), reversed(saved)):
            gr = ca_backward(ctx, sh, gx, sv, y, w, counter=counter, group=env.group,
                             dy_sink=sink)
            gx = gr.d_x
        return gx, sink.finish(ctx, dtype=y.dtype)   # dY in y's dtype, like the reference

    def timed(policy, steps, warm, sampler=False):
        for _ in range(warm):
            step(policy)
        torch.cuda.synchronize()
        env.barrier()
        cs = ClockSampler(env.local).__enter__() if sampler else None
        l0 = _lib.load().lvx_kernel_launches()
        w0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for _ in range(steps):
            step(policy)
        host_ms = (time.perf_counter() - h0) * 1e3 / steps
        e1.record()
        torch.cuda.synchronize()
        timed.host_ms = env.max_over_ranks(host_ms)
        if cs:
            cs.mark(w0, time.time())
            time.sleep(0.15)
            cs.__exit__()
        env.barrier()
        return env.max_over_ranks(e0.elapsed_time(e1) / steps), \
            _lib.load().lvx_kernel_launches() - l0, (cs.summary() if cs else None)

    cnt = OpCounter()
    step(ActivationPolicy.RECOMPUTE_KV, cnt)       # counts the recompute FLOP (per rank)
    ms, launches, clocks = timed(ActivationPolicy.RECOMPUTE_KV, args.steps, args.warmup, True)
    host_ms = timed.host_ms
    ms_store, _, _ = timed(ActivationPolicy.STORE_KV, max(2, args.steps // 2), 1)
    graph = None
    if not args.no_graph:   # the whole layer-stack step recorded once and replayed
        graph = graph_replay(env, ctx, lambda: step(ActivationPolicy.RECOMPUTE_KV),
                             args.steps, 0.0)
    att = volumes.attention_flops(s_q, s_kv, hq, d) * nl
    # projections per layer: fwd Q (2 sq e hq d), K+V (2 * 2 skv e hkv d), O
    # (2 sq hq d e); bwd: recompute K+V, Q re-projection, dX / dW for Q, K, V, O
    proj_fwd = 2 * s_q * e * hq * d * 2 + 2 * 2 * s_kv * e * hkv * d
    proj_bwd = (2 * 2 * s_kv * e * hkv * d + 2 * s_q * e * hq * d      # recompute K/V, Q
                + 2 * (2 * 2 * s_q * e * hq * d)                         # dX, dW of Q and O
                + 2 * (2 * 2 * s_kv * e * hkv * d))                      # dY, dW of K and V
    total = att + nl * (proj_fwd + proj_bwd)
    burst, sust, hbm, pk_kind, _ = peaks()
    value = total / (ms * 1e-3) / 1e12
    return {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_layer": ms / nl, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (uniform[-1,1] activations, U[+-0.5/sqrt(e)] weights)",
            "config": {**CFG, "policy": "recompute", "parallelism": f"kv-seq-parallel x{world}",
                       "l2": "y shard + K/V larger than L2"},
            "attention_tflops": att / (ms * 1e-3) / 1e12,
            "flop_split": {"attention": att, "projections": nl * (proj_fwd + proj_bwd),
                           "recompute_counted_per_rank": cnt.projection_flops},
            "store_kv_ms_per_step": ms_store, "recompute_overhead": ms / ms_store - 1.0,
            "host_submit_ms_per_step": host_ms,
            "graph_replay": ({**graph, "value": total / (graph["ms_per_step"] * 1e-3) / 1e12}
                             if graph and "ms_per_step" in graph else graph),
            "roofline": {"kernel": "whole step (attention + projection GEMMs), per GPU",
                         "bound": "tensor", "achieved": value / world, "peak": sust,
                         "unit": "TFLOP/s", "frac": value / world / sust, "traffic": None,
                         "peak_kind": f"{pk_kind} bf16 sustained"},
            "clocks": clocks, "gpu_launches": int(launches)}


def _bwd_is_tc(q, k):
    from paper_2502_02406_b200 import _lib
    return _lib.load().lvx_blockwise_bwd_workspace(_lib.view(q), _lib.view(k)) > 0


def e2e_arm(args, ctx, shards, dev_inputs, scale, fwd, bwd, flops, world, dev):
    """The same layer step through the public host-buffer API
    (``HostLayerPipeline``): every step copies its shard's Q, K, V, dO from
    pinned host memory and its O, L, dQ, dK, dV back, inside the timed region;
    K/V stream in by chunks and the next step's inputs prefetch behind the
    current step's compute (the first step's copies are not hidden)."""
    import torch
    import torch.distributed as dist
    from paper_2502_02406_b200.host_pipeline import HostLayerPipeline, HostStep
    host_in = [t.cpu().pin_memory() for t in dev_inputs]
    base = HostStep.allocate(*host_in)
    h2d, d2h = base.h2d_bytes(), base.d2h_bytes()
    pipe = HostLayerPipeline(ctx, shards, scale, chunks=8, prefetch=True)
    steps = max(2, args.steps)
    pcie = _pcie_rates(dev, world)
    pipe.run([base, base])   # warm-up (allocations, both slots)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.run([base] * steps)
    el = (time.perf_counter() - t0) / steps
    if world > 1:
        t = torch.tensor([el, h2d, d2h], device=dev, dtype=torch.float64)
        tm = t.clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        el, h2d, d2h = tm[0].item(), int(t[1].item()), int(t[2].item())
    per_rank_h2d, per_rank_d2h = base.h2d_bytes(), base.d2h_bytes()
    pcie["copy_bound_ms_per_step"] = 1e3 * max(per_rank_h2d / (pcie["h2d_gbs"] * 1e9),
                                               per_rank_d2h / (pcie["d2h_gbs"] * 1e9))
    return {"value": flops / el / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": el * 1e3, "steps": steps,
            "pcie": pcie,
            "path": "HostLayerPipeline: pinned host shard -> HBM (chunked, prefetched) -> "
                    "lvx_forward/lvx_backward -> pinned host (host wall clock around "
                    f"{steps} steps incl. the first step's unhidden copies, max over ranks)"}


def _pcie_rates(dev, world) -> dict:
    """Pinned host <-> this GPU copy rates (GB/s, 512 MiB each way, best of 3,
    min over ranks — all ranks copy at once, as in the e2e steps): what bounds
    the e2e step when its copies are longer than its kernels."""
    import torch
    import torch.distributed as dist
    n = 512 << 20
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    buf = torch.empty(n, dtype=torch.uint8, device=dev)
    rates = []
    for src, dst in ((host, buf), (buf, host)):
        best = float("inf")
        for _ in range(3):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        rates.append(n / best / 1e9)
    if world > 1:
        t = torch.tensor(rates, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        rates = t.tolist()
    del host, buf
    return {"h2d_gbs": rates[0], "d2h_gbs": rates[1], "probe_bytes": n}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        native_arm(args)


if __name__ == "__main__":
    main()
