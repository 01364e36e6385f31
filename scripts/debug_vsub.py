import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as orc
from tests import common as cm
from tests.gpu_adapter import GpuOracle
O = orc.Oracle("restatement")
rng = np.random.default_rng(1)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = 4 * k + 20
q = cm.random_spd_band(rng, 1, n, k)
l = O.cholesky(q)[0]
s = O.sparse_inverse_subset(l)[0]
sb = cm.random_band(rng, 1, n, k, 0)
ref = O.vjp_sparse_inverse_subset(l, s, sb)[0][0]
g = GpuOracle(tile=1).vjp_sparse_inverse_subset(l, s, sb)[0][0]
d = np.abs(g - ref)
bad = np.argwhere(d > 1e-9 * np.abs(ref).max())
print("n", n, "bad cells", len(bad), "first", bad[:5], "cols with bad", np.unique(bad[:, 0])[:20])
print("g col0", g[0, :4], "ref", ref[0, :4])
print("g col n-1", g[n - 1, :2], "ref", ref[n - 1, :2])
colbad = [(c, int((d[c] > 1e-9 * np.abs(ref).max()).sum())) for c in range(n)]
print("per-col bad:", colbad[:6], "...", colbad[-k - 3:-k + 3], "...", colbad[-3:])
