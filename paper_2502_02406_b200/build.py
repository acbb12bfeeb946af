"""Build liblvx_b200.so in-tree with nvcc for sm_100a (no torch JIT cache).

    python -m paper_2502_02406_b200.build [--verbose]

Each ``csrc/*.cu`` is compiled to an object in parallel with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked into
``paper_2502_02406_b200/liblvx_b200.so`` with the static CUDA runtime, so the
library loads on a CPU-only host (the driver is reached at run time through
``cudaGetDriverEntryPoint``).  ``-Xptxas -v`` output goes to
``build/ptxas.log``.  ``LVX_NVCC_EXTRA`` appends flags (variant builds for
same-box A/B runs: tools/build_variant.sh).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "liblvx_b200.so"
BUILD = ROOT / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include")] + os.environ.get("LVX_NVCC_EXTRA", "").split()


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) +
                  list((ROOT / "include").glob("*.h")))


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def _compile(src: Path):
    obj = BUILD / (src.stem + ".o")
    cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, r


def build(verbose: bool = False, force: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    BUILD.mkdir(exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, _sources()))
    log = []
    for src, _, r in results:
        log.append(f"== {src.name}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
    (BUILD / "ptxas.log").write_text("\n".join(log))
    tmp = LIB.with_suffix(".so.tmp")
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
            *[str(o) for _, o, _ in results], "-cudart", "static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
