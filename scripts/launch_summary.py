"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a
bench.py run: per-kernel launches, average ms and share of the step (the
library's kernels; torch kernels are input setup outside the timed region).
    python scripts/launch_summary.py launches.csv "<command line>" > summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in rows:
    v = float(r["Metric Value"].replace(",", ""))
    v = {"ns": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "nsecond": v / 1e6, "ms": v, "msecond": v}.get(
        r["Metric Unit"], v / 1e6)
    a = agg.setdefault(r["Kernel Name"][:70], [0, 0.0])
    a[0] += 1
    a[1] += v
import os
import re

# kernels of the timed step (default: the fused config-3 sweeps); everything
# else -- torch's input generation, the inputs' solve and relayout, the FP64
# peak microbenchmarks -- runs outside the timed region
STEP = re.compile(os.environ.get("STEP_RE", r"t1::|mlik"))
setup = lambda k: not STEP.search(k)  # noqa: E731
step = {k: t / c for k, (c, t) in agg.items() if not setup(k)}
per_step = sum(step.values())
print(sys.argv[2] if len(sys.argv) > 2 else "")
print("(cold-cache, serialised per-launch times; setup kernels = input generation outside the timed region)\n")
print(f"{'kernel':70s} launches    avg ms share of step")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    share = "setup" if setup(k) else f"{100 * (t / c) / per_step:.1f}%"
    print(f"{k:70s} {c:8d} {t / c:9.4f} {share:>12s}")
print(f"\nsum of per-step kernel averages: {per_step:.4f} ms")
