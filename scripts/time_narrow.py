"""Per-kernel breakdown of the narrow per-op paths at config-3 / config-1 size."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1902_10078_b200 as bgm
from scripts.bench_ops import factor, normal_vec

B, n, k = [(256, 65536, 16), (4096, 2048, 4)][int(sys.argv[1]) if len(sys.argv) > 1 else 0]
dev = torch.device("cuda", 0)
L0 = factor(B, n, k, torch.float64, dev, 0.1, 31)
Q = bgm.product_band_band_restricted(L0, bgm.T(L0), k, 0)
L = bgm.cholesky(Q)
y = normal_vec(B, n, torch.float64, dev, 32)
lib = bgm.library()
for name, fn in (("cholesky", lambda: bgm.cholesky(Q, check=False)),
                 ("solve", lambda: bgm.solve_vec(L, y, False, check=False)),
                 ("solve_t", lambda: bgm.solve_vec(L, y, True, check=False)),
                 ("subset", lambda: bgm.sparse_inverse_subset(L, check=False))):
    fn()
    torch.cuda.synchronize()
    lib.bgm_timing_enable(1)
    fn()
    torch.cuda.synchronize()
    parts = []
    for i in range(lib.bgm_timing_read(-1, None, 0, None, None)):
        nm, tot, c = C.create_string_buffer(128), C.c_double(), C.c_int64()
        lib.bgm_timing_read(i, nm, 128, C.byref(tot), C.byref(c))
        parts.append(f"{nm.value.decode()}={tot.value:.3f}ms")
    lib.bgm_timing_enable(0)
    print(name, " ".join(parts), flush=True)
