"""Compact per-op view of bench.py JSON lines: python scripts/show_ops2.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no json", e)
        continue
    r = d["roofline"]
    p = d.get("parity") or {}
    sp = d.get("scaling_proxy") or {}
    print(d["config"]["workload"], "ms", d["ms_per_step"], "suite", d["suite_roofline"].get("suite_frac_of_step", d["suite_roofline"].get("fused_floor_frac")),
          {n: v["ms"] for n, v in r.get("per_op", {}).items()}, "parity", p.get("pass"),
          "proxy8", sp.get("8", {}).get("efficiency"), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
