"""Timing scopes of the wide forward kernels (cholesky, subset) at config-4 size (fp64)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor

for k in [int(a) for a in sys.argv[1:]] or (64, 128):
    dev = torch.device("cuda", 0)
    B, n = 64, 32768
    L0 = factor(B, n, k, torch.float64, dev, 0.02 / k ** 0.5, 105, tile=1)
    Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
    L = bgm.cholesky(Q)
    S = bgm.sparse_inverse_subset(L)
    torch.cuda.synchronize()
    lib = bgm.library()
    lib.bgm_timing_enable(1)
    bgm.cholesky(Q, check=False)
    bgm.sparse_inverse_subset(L, check=False)
    torch.cuda.synchronize()
    out = []
    for i in range(lib.bgm_timing_read(-1, None, 0, None, None)):
        nm, tot, c = C.create_string_buffer(128), C.c_double(), C.c_int64()
        lib.bgm_timing_read(i, nm, 128, C.byref(tot), C.byref(c))
        out.append(f"{nm.value.decode()}={tot.value:.2f}")
    lib.bgm_timing_enable(0)
    print(k, " ".join(out), flush=True)
