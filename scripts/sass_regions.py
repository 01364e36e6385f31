"""Stall samples of an ncu SASS source CSV summed per region (between BAR /
EXIT instructions), by stall reason and by opcode: python scripts/sass_regions.py FILE"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
src, smp, ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
body = [r for r in rows[2:] if len(r) > src and r[src].split()]
T = sum(float(r[smp] or 0) for r in body)
reg, start = None, 0


def flush(n):
    global reg
    if reg and reg["v"] > 0.002 * T:
        st = " ".join(f"{k}:{100 * v / T:.1f}" for k, v in sorted(reg["st"].items(), key=lambda x: -x[1])[:5] if v > 0)
        op = " ".join(f"{k}:{100 * v / T:.1f}" for k, v in sorted(reg["op"].items(), key=lambda x: -x[1])[:6] if v > 0)
        print(f"[{start:5d},{n:5d}) {100 * reg['v'] / T:5.1f}%  inst/exec {reg['ex']:.3g}  n={n - start}\n      stalls {st}\n      ops    {op}")
    reg = {"v": 0.0, "ex": 0.0, "st": {}, "op": {}}


flush(0)
for n, r in enumerate(body):
    v = float(r[smp] or 0)
    t = r[src].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    reg["v"] += v
    reg["ex"] += float(r[ex] or 0)
    reg["op"][op] = reg["op"].get(op, 0) + v
    for i, c in stall_cols:
        reg["st"][c] = reg["st"].get(c, 0) + float(r[i] or 0)
    if op in ("BAR", "EXIT"):
        flush(n + 1)
        start = n + 1
flush(len(body))
