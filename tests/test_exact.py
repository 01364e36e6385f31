"""Accuracy against extended precision: the reference route (oracle) and
the CUDA fused sweeps are both within a few ulps of max|.| of the exact
config-3 gradients (tests/exact.py, x87 long double)."""
import numpy as np
import pytest

from tests import common as cm
from tests.exact import abs_rel, mlik_exact


@pytest.fixture(scope="module")
def instance():
    rng = np.random.default_rng(31)
    B, n, k, tau2 = 2, 160, 16, 0.01
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    return L, y, tau2, mlik_exact(L, y, tau2)


def test_oracle_is_accurate(oracle, instance):
    L, y, tau2, (lo_x, lb_x, tb_x) = instance
    lo, lb, tb, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert np.all(st == 0)
    assert abs_rel(lb, lb_x) < 1e-14
    assert abs_rel(lo, lo_x) < 1e-13
    assert abs_rel(tb, tb_x) < 1e-11  # tau2_bar cancels ~1e6-sized terms


@pytest.mark.gpu
@pytest.mark.parametrize("tile", [1, 32])
def test_gpu_is_as_accurate_as_reference(cuda, oracle, instance, tile):
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    L, y, tau2, (lo_x, lb_x, tb_x) = instance
    lo, lb, tb, _, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    api.set_segment_rows(32)  # several segments even at n=160 (tile 1 -> fast path)
    try:
        lg, lbg, tbg, _, _ = GpuOracle(tile=tile).marginal_likelihood_grad(L, y, tau2)
    finally:
        api.set_segment_rows(0)
    assert abs_rel(lbg, lb_x) <= max(2 * abs_rel(lb, lb_x), 1e-15)
    assert abs_rel(lg, lo_x) <= max(2 * abs_rel(lo, lo_x), 1e-15)
    assert abs_rel(tbg, tb_x) <= max(2 * abs_rel(tb, tb_x), 1e-13)
