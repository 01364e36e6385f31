import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as orc
from tests import common as cm
from tests import exact
from tests.gpu_adapter import GpuOracle
from paper_1902_10078_b200 import api
O = orc.Oracle("restatement")
rng = np.random.default_rng(5)
B, n, k, tau2 = 3, 1500, 16, 0.01
L = cm.config_factor(rng, B, n, k)
y = rng.normal(0, 1, (B, n))
lo, lb, tb, st, _ = O.marginal_likelihood_grad(L, y, tau2)
for burn in ("128", "16"):
    os.environ["BGM_BURN"] = burn
    api.set_segment_rows(64)
    api.debug_repairs(reset=True)
    lg, lbg, tbg, _, _ = GpuOracle(tile=32).marginal_likelihood_grad(L, y, tau2)
    print("burn", burn, "reps", api.debug_repairs(), "err(floor1e-6)", cm.max_rel_err(lbg, lb, floor_scale=1e-6),
          "err(floor1e-5)", cm.max_rel_err(lbg, lb, floor_scale=1e-5),
          "normwise", np.linalg.norm(lbg - lb) / np.linalg.norm(lb))
    idx = np.unravel_index(np.argmax(np.abs(lbg - lb) / np.maximum(np.maximum(np.abs(lbg), np.abs(lb)), 1e-6 * np.abs(lb).max())), lb.shape)
    print("   worst", idx, lbg[idx], lb[idx], "max", np.abs(lb).max())
