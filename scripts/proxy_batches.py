"""Config-3 step at the per-GPU batches of a strong-scaling run (B/G), one at a time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
wl = bench.WORKLOADS["cfg3"]
for B in [int(a) for a in sys.argv[1:]] or (256, 128, 64, 32):
    for stage in ("inputs", "step"):
        try:
            if stage == "inputs":
                w = bench.MlikWorkload(wl, B, 0, dev)
            else:
                w.step()
            torch.cuda.synchronize()
            print(B, stage, "ok", flush=True)
        except Exception as e:
            print(B, stage, "FAILED", repr(e)[:300], flush=True)
            sys.exit(1)
    del w
    torch.cuda.empty_cache()
