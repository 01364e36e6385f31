"""Per-kernel breakdown (library timing scopes) of a few API calls at config-4
size: python scripts/time_ops.py [k] [f64|f32]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_vec

k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dt = torch.float32 if len(sys.argv) > 2 and sys.argv[2] == "f32" else torch.float64
dev = torch.device("cuda", 0)
B, n = 64, 32768
L0 = factor(B, n, k, dt, dev, 0.02 / k ** 0.5, 41 + k, tile=1)
Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
L = bgm.cholesky(Q)
b = normal_vec(B, n, dt, dev, 42, tile=1)
lib = bgm.library()
for name, fn in (("cholesky", lambda: bgm.cholesky(Q, check=False)),
                 ("subset", lambda: bgm.sparse_inverse_subset(L, check=False)),
                 ("solve", lambda: bgm.solve_vec(L, b, False, check=False)),
                 ("solve_t", lambda: bgm.solve_vec(L, b, True, check=False))):
    fn()
    torch.cuda.synchronize()
    lib.bgm_timing_enable(1)
    fn()
    torch.cuda.synchronize()
    cnt = lib.bgm_timing_read(-1, None, 0, None, None)
    parts = []
    for i in range(cnt):
        nm = C.create_string_buffer(128)
        tot = C.c_double()
        c = C.c_int64()
        lib.bgm_timing_read(i, nm, 128, C.byref(tot), C.byref(c))
        parts.append(f"{nm.value.decode()}={tot.value:.3f}ms")
    lib.bgm_timing_enable(0)
    print(name, " ".join(parts), flush=True)
