"""Runs the config-3 fused step a few times at full size (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1902_10078_b200 as bgm

B = int(os.environ.get("PROF_B", "256"))
n = int(os.environ.get("PROF_N", "65536"))
reps = int(os.environ.get("PROF_REPS", "2"))
dev = torch.device("cuda", 0)
L, y = bench.MlikWorkload.make_inputs(B, n, 16, 1234, dev)
for _ in range(reps):
    loss, lbar, tb = bgm.marginal_likelihood_grad(L, y, 0.01)
torch.cuda.synchronize()
print("ok", float(loss.sum()))
