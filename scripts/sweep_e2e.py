"""Config-3 end-to-end (host buffers) step time vs the host pipeline's chunk
size and stream count (paper_1902_10078_b200/host.py)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1902_10078_b200.host import marginal_likelihood_grad_host

dev = torch.device("cuda", 0)
wl = dict(bench.WORKLOADS["cfg3"])
w = bench.MlikWorkload(wl, wl["B"], 0, dev)
Lr, yr = w.L.to_reference(), w.y.to_reference()
hL = torch.empty(Lr.shape, dtype=Lr.dtype, pin_memory=True)
hy = torch.empty(yr.shape, dtype=yr.dtype, pin_memory=True)
hL.copy_(Lr)
hy.copy_(yr)
del Lr, yr
hout = (torch.empty(w.B, dtype=torch.float64, pin_memory=True), torch.empty(hL.shape, dtype=torch.float64, pin_memory=True),
        torch.empty(w.B, dtype=torch.float64, pin_memory=True))
for chunk in (8, 16, 32, 64):
    for streams in (2, 3, 4, 6):
        run = lambda: marginal_likelihood_grad_host(hL, hy, 0.01, out_host=hout, tile=32, chunk=chunk, streams=streams)
        run()
        torch.cuda.synchronize()
        ms = bench.time_steps(run, 4)
        print(json.dumps({"chunk": chunk, "streams": streams, "ms": round(ms, 2)}), flush=True)
