"""Print the burn-in check mismatches of the config-3 step (BGM_DEBUG=1) at a short burn-in."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1902_10078_b200 as bgm
from paper_1902_10078_b200 import api
dev = torch.device("cuda", 0)
wl = dict(bench.WORKLOADS["cfg3"])
wl["n"] = int(os.environ.get("DBG_N", "2048"))
w = bench.MlikWorkload(wl, 32, 0, dev, int(os.environ.get("DBG_TILE", "32")))
bgm.set_segment_rows(int(os.environ.get("DBG_SEG", "256")))
api.debug_repairs(reset=True)
w.step()
torch.cuda.synchronize()
print("repairs", api.debug_repairs(with_dev=True), flush=True)
