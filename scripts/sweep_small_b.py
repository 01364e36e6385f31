"""Config-3 step time at small per-GPU batches vs burn-in and segment length
(the strong-scaling proxy's per-rank work).  Prints one JSON line per setting."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1902_10078_b200 as bgm
from paper_1902_10078_b200 import api

dev = torch.device("cuda", 0)
wl = dict(bench.WORKLOADS["cfg3"])
batches = [int(x) for x in os.environ.get("SWEEP_B", "256,32").split(",")]
burns = [int(x) for x in os.environ.get("SWEEP_BURN", "96,64,48,32").split(",")]
segs = [int(x) for x in os.environ.get("SWEEP_SEG", "0,64,96,128,192").split(",")]
tiles = [int(x) for x in os.environ.get("SWEEP_TILE", "32").split(",")]
for tile in tiles:
    for B in batches:
        w = bench.MlikWorkload(wl, B, 0, dev, tile)
        for burn in burns:
            os.environ["BGM_BURN"] = str(burn)
            for seg in segs:
                bgm.set_segment_rows(seg)
                api.debug_repairs(reset=True)
                w.step()
                torch.cuda.synchronize()
                reps = api.debug_repairs()
                g, _ = bench.capture(w.step)
                run = g.replay if g is not None else w.step
                for _ in range(3):
                    run()
                ms = bench.time_steps(run, 10)
                print(json.dumps({"tile": tile, "B": B, "burn": burn, "seg": seg, "ms": round(ms, 4), "fixups_repairs": reps}), flush=True)
                del g
        bgm.set_segment_rows(0)
        del w
        torch.cuda.empty_cache()
