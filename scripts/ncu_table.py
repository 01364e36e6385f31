"""Per-kernel table from an ncu --metrics --csv log (one row per launch):
python scripts/ncu_table.py LOG [--skip-setup]"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
by = collections.OrderedDict()
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    by.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
agg = collections.OrderedDict()
for (i, name), m in by.items():
    nm = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")[:60]
    t = float(m["gpu__time_duration.sum"][0].replace(",", ""))
    u = m["gpu__time_duration.sum"][1]
    t = t / 1e6 if u in ("ns", "nsecond") else t / 1e3 if u in ("us", "usecond") else t
    a = agg.setdefault(nm, {"n": 0, "ms": 0.0, "m": m})
    a["n"] += 1
    a["ms"] += t
tot = sum(a["ms"] for a in agg.values())
print(f"{'kernel':60s} {'n':>3s} {'ms':>8s} {'share':>6s} tensor% fp64% warps% issue% regs grid x block")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
    m = a["m"]
    g = lambda k: m.get(k, ("-", ""))[0]  # noqa: E731
    print(f"{nm:60s} {a['n']:3d} {a['ms']:8.3f} {100 * a['ms'] / tot:5.1f}% "
          f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):>7s} "
          f"{g('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):>5s} "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):>6s} "
          f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):>6s} "
          f"{g('launch__registers_per_thread'):>4s} {g('launch__grid_size')}x{g('launch__block_size')}")
print(f"total {tot:.3f} ms")
