"""Program-order view of an ncu --page source --print-source sass CSV: every
instruction holding at least MIN % of the stall samples, with its dominant
stall reasons, plus running totals per region between BAR / branch targets:
python scripts/sass_flow.py FILE [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
src, smp, ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "not_issued" not in c.lower()]
body = [r for r in rows[2:] if len(r) > src and r[src].split()]
T = sum(float(r[smp] or 0) for r in body)
acc = 0.0
for n, r in enumerate(body):
    v = float(r[smp] or 0)
    acc += v
    s = r[src]
    mark = "BAR" in s or "EXIT" in s
    if 100 * v / T >= mn or mark:
        st = sorted(((float(r[i] or 0), c[6:]) for i, c in stall_cols), reverse=True)[:2]
        why = " ".join(f"{c}:{100 * x / T:.1f}" for x, c in st if x > 0)
        print(f"{n:5d} {100 * v / T:5.1f}% cum {100 * acc / T:5.1f}%  ex {float(r[ex] or 0):9.3g}  {s[:60]:60s} {why}")
