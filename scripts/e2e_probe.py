"""e2e (host buffers) step time vs chunk size / streams, and raw PCIe copy rates."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1902_10078_b200.host import marginal_likelihood_grad_host

dev = torch.device("cuda", 0)
B, n, k = 256, 65536, 16
L, y = bench.make_inputs(B, n, k, 1234, dev)
Lr, yr = L.to_reference(), y.to_reference()
hL = torch.empty(Lr.shape, dtype=Lr.dtype, pin_memory=True)
hy = torch.empty(yr.shape, dtype=yr.dtype, pin_memory=True)
hL.copy_(Lr)
hy.copy_(yr)
hout = (torch.empty(B, dtype=torch.float64, pin_memory=True), torch.empty(hL.shape, dtype=torch.float64, pin_memory=True),
        torch.empty(B, dtype=torch.float64, pin_memory=True))
# raw copy rates
d = torch.empty_like(Lr)
for name, fn in (("h2d", lambda: d.copy_(hL, non_blocking=True)), ("d2h", lambda: hout[1].copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name}: {hL.numel() * 8 / dt / 1e9:.1f} GB/s", flush=True)
s2 = torch.cuda.Stream()
t0 = time.perf_counter()
with torch.cuda.stream(s2):
    hout[1].copy_(d, non_blocking=True)
d.copy_(hL, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"both directions concurrently: {2 * hL.numel() * 8 / dt / 1e9:.1f} GB/s total", flush=True)
del d
for chunk, streams in ((32, 4), (16, 4), (8, 4), (8, 6), (4, 6), (16, 6)):
    marginal_likelihood_grad_host(hL, hy, 0.01, out_host=hout, chunk=chunk, streams=streams)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        marginal_likelihood_grad_host(hL, hy, 0.01, out_host=hout, chunk=chunk, streams=streams)
    torch.cuda.synchronize()
    print(f"chunk={chunk} streams={streams}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms", flush=True)
