"""Device time of the drop-in's check_scaling ops on one matrix (B = 1,
reference layout, bw = 5): what the GPU spends inside the drop-in calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1902_10078_b200 as bgm
from tests import common as cm

dev = torch.device("cuda", 0)
for n in (50000, 100000, 200000):
    rng = np.random.default_rng(n)
    q = cm.random_spd_band(rng, 1, n, 5)
    Q = bgm.Bands.from_reference(q, 5, 0, tile=1)
    def chol():
        return bgm.cholesky(Q, check=False)
    L = chol()
    Lb = bgm.vjp_log_det_from_cholesky(L, 1.0)
    res = {}
    for name, fn in (("cholesky", chol), ("log_det", lambda: bgm.log_det_from_cholesky(L, check=False)),
                     ("vjp_log_det", lambda: bgm.vjp_log_det_from_cholesky(L, 1.0)),
                     ("vjp_cholesky", lambda: bgm.vjp_cholesky(L, Lb))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record(); torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 5, 3)
    print(n, res, flush=True)
