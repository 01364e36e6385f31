"""Debug helper: run the fast config-3 path on a small problem, report repairs
and parity against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as orc
import paper_1902_10078_b200 as bgm
from paper_1902_10078_b200 import api
from tests import common as cm

B, n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 2, int(sys.argv[2]) if len(sys.argv) > 2 else 2048, 16
seg = int(sys.argv[3]) if len(sys.argv) > 3 else 256
rng = np.random.default_rng(0)
L = cm.config_factor(rng, B, n, k)
y = rng.normal(0, 1, (B, n))
api.set_segment_rows(seg)
api.debug_repairs(reset=True)
Ld = bgm.Bands.from_reference(L, k, 0, tile=1)
Yd = bgm.Vecs.from_reference(y, tile=1)
loss, lbar, tb = bgm.marginal_likelihood_grad(Ld, Yd, 0.01)
torch.cuda.synchronize()
print("repairs", api.debug_repairs())
o = orc.Oracle("restatement")
lo, lbo, tbo, st, _ = o.marginal_likelihood_grad(L, y, 0.01)
print("loss err", cm.max_rel_err(loss.cpu().numpy(), lo), "lbar err", cm.max_rel_err(lbar.numpy(), lbo),
      "tbar err", cm.max_rel_err(tb.cpu().numpy(), tbo))
g = lbar.numpy()
bad = np.argwhere(np.abs(g - lbo) > 1e-9 * np.abs(lbo).max())
print("bad cells", len(bad), bad[:10])
