"""Runs one bench.py suite workload's step PROF_REPS times (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

dev = torch.device("cuda", 0)
wl = dict(bench.WORKLOADS[os.environ.get("PROF_WL", "cfg4_k64_f64")])
B = int(os.environ.get("PROF_B", str(wl["B"])))
w = bench.make_workload(wl, B, 0, dev)
torch.cuda.synchronize()
for _ in range(int(os.environ.get("PROF_REPS", "1"))):
    w.step()
torch.cuda.synchronize()
print("ok")
