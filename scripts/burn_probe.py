"""Repairs and step time of the config-3 step vs the burn-in length (BGM_BURN)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1902_10078_b200 as bgm
from paper_1902_10078_b200 import api

dev = torch.device("cuda", 0)
L, y = bench.make_inputs(256, 65536, 16, 1234, dev)
ref = None
for burn in [int(a) for a in sys.argv[1:]] or (128, 96, 80, 64, 48):
    os.environ["BGM_BURN"] = str(burn)
    api.debug_repairs(reset=True)
    loss, lbar, tb = bgm.marginal_likelihood_grad(L, y, 0.01, check=False)
    torch.cuda.synchronize()
    reps = api.debug_repairs()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        bgm.marginal_likelihood_grad(L, y, 0.01, check=False)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = (loss.clone(), lbar.data.clone(), tb.clone())
    dl = float(((loss - ref[0]).abs() / ref[0].abs()).max())
    dg = float(((lbar.data - ref[1]).abs().max() / ref[1].abs().max()))
    print(f"burn={burn} repairs={reps} ms={e0.elapsed_time(e1) / 5:.3f} dloss={dl:.2e} dlbar={dg:.2e}", flush=True)
