"""The host-buffer entry (paper_1902_10078_b200/host.py): a batch in host memory in the reference
layout goes through the three-stage copy-in / sweeps / copy-out pipeline; results equal the device
API's on the same inputs (bitwise when the chunk matches a whole device batch) and the oracle's."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("chunk,streams", [(16, 2), (5, 3), (64, 4)])
def test_host_pipeline_matches_oracle(cuda, oracle, tile, chunk, streams):
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200.host import marginal_likelihood_grad_host
    rng = np.random.default_rng(100 + chunk)
    B, n, k, tau2 = 37, 1200, 16, 0.01
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    hL = torch.from_numpy(np.ascontiguousarray(L)).pin_memory()
    hy = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
    loss, lbar, tbar = marginal_likelihood_grad_host(hL, hy, tau2, chunk=chunk, streams=streams, tile=tile)
    torch.cuda.synchronize()
    lo, lbo, tbo, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert not st.any()
    assert cm.max_rel_err(loss.numpy(), lo) <= 1e-9
    assert cm.max_rel_err(lbar.numpy(), lbo, floor_scale=1e-6) <= 1e-9
    assert np.max(np.abs(tbar.numpy() - tbo)) <= 1e-9 * max(1.0, float(np.max(np.abs(tbo))))
    # a second call reuses nothing from the first and overwrites the same outputs
    out = (loss, lbar, tbar)
    l2, lb2, t2 = marginal_likelihood_grad_host(hL, hy, tau2, out_host=out, chunk=chunk, streams=streams, tile=tile)
    torch.cuda.synchronize()
    assert l2 is loss and cm.max_rel_err(lb2.numpy(), lbo, floor_scale=1e-6) <= 1e-9
