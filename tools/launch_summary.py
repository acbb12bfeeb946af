"""Aggregate an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
by kernel: launches, total ms, share of kernel time.

    python tools/launch_summary.py gpurun_out/<tag>_launches.csv [--skip N]
``--skip`` drops the first N launches (input generation, warm-up)."""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return re.sub(r"at::native::|at::<unnamed>::|\(anonymous namespace\)::|<unnamed>::", "", name)[:80]


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    lines = [ln for ln in open(path) if ln.startswith('"')]   # drop ==PROF== / ==WARNING== lines
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    rows = rows[skip:]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit == "us" else v
        k = short(r["Kernel Name"])
        tot[k] += ms
        cnt[k] += 1
    all_ms = sum(tot.values())
    print(f"| kernel | launches | ms | share |\n|---|---|---|---|")
    for k, ms in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {ms:.3f} | {ms / all_ms:.1%} |")
    print(f"\n{len(rows)} launches, {all_ms:.2f} ms of kernel time (serialised, cold-cache under ncu)")


if __name__ == "__main__":
    main()
