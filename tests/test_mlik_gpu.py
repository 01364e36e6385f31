"""GPU parity of the fused config-3 learning step against the reference's
tape composition (oracle: inference.cpp:140-163 + tape.cpp:435-451 +
grad.cpp:145-151, restated bit-exactly in oracle/bandgm_oracle.c)."""
import numpy as np
import pytest

from tests import common as cm

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _check(gpu, oracle, B, n, k, tau2, seed):
    rng = np.random.default_rng(seed)
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    lo, lb, tb, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert np.all(st == 0)
    lg, lbg, tbg, _, _ = gpu.marginal_likelihood_grad(L, y, tau2)
    for name, g, o in (("loss", lg, lo), ("l_bar", lbg, lb), ("tau2_bar", tbg, tb)):
        err = cm.max_rel_err(g, o)
        assert err <= TOL, f"{name} B={B} n={n} k={k}: {err:.3e}"


@pytest.mark.parametrize("B,n,k,tau2", [(1, 1, 0, 0.5), (3, 50, 1, 0.3), (5, 400, 4, 0.01),
                                        (33, 700, 16, 0.01), (2, 2000, 16, 0.01), (4, 257, 8, 2.0)])
def test_mlik_matches_tape_composition(cuda, oracle, B, n, k, tau2):
    from tests.gpu_adapter import GpuOracle
    _check(GpuOracle(tile=32), oracle, B, n, k, tau2, seed=B * 1000 + n)
