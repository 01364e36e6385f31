"""Pretty-prints bench_ops.py JSON lines: python scripts/show_ops.py FILE"""
import json
import sys

for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print(d["config"], d["dtype"], "suite", d["suite_ms"], "roof", d["suite_roofline_ms"], "frac", d["suite_frac"])
    for o in d["ops"]:
        print("   %-22s %8.3f ms  roof %7.3f  frac %.3f" % (o["op"], o["ms"], o["roofline_ms"], o["frac"]))
