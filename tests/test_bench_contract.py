"""bench.py keeps the driver's JSON-line contract (task spec).

The reference arm runs on the host (the CPU oracle port), so it is checked
here without a GPU; the native arm is a GPU test at a reduced Lkv."""
import json
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["config"]["workload"] == "llama3v-cross-attn-C2"
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= cb.keys()
    assert cb["kind"] in ("port", "reference") and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_native_arm_contract():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--steps", "2", "--warmup", "3", "--skv", "65536", "--no-cpu")
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    assert d["dtype"] == "bf16" and d["scaling"] in ("weak", "strong")
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.5 and r["peak"] >= 1000
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["gpu_launches"] > 0
