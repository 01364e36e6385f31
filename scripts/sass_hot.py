"""Opcode and hottest-instruction stall breakdown of an ncu --page source
--print-source sass CSV: python scripts/sass_hot.py FILE [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
src, smp, ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ops, inst = {}, []
T = 0.0
for r in rows[2:]:
    if len(r) <= src or not r[src].split():
        continue
    t = r[src].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    v = float(r[smp] or 0)
    T += v
    o = ops.setdefault(op, [0.0, 0.0])
    o[0] += v
    o[1] += float(r[ex] or 0)
    inst.append((v, r[0], r[src]))
for k, (v, e) in sorted(ops.items(), key=lambda x: -x[1][0])[:14]:
    print(f"{k:8s} {100 * v / T:5.1f}% of samples  executed {e:.3g}")
print("--- hottest instructions")
for v, a, s in sorted(inst, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{100 * v / T:5.1f}%  {a}  {s[:70]}")
