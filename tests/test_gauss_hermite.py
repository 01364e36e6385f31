"""infer::gauss_hermite (inference.cpp:120-137): the library's Golub-Welsch
rule equals numpy's hermgauss (ascending nodes, weights for e^{-x^2}).
Host function of the C ABI: runs without a GPU."""
import numpy as np
import pytest


@pytest.mark.parametrize("k", [1, 2, 5, 20, 64])
def test_gauss_hermite_matches_numpy(k):
    import paper_1902_10078_b200 as bgm
    x, w = bgm.gauss_hermite(k)
    if k == 1:
        assert x[0] == 0.0 and abs(w[0] - np.sqrt(np.pi)) < 1e-15
        return
    rx, rw = np.polynomial.hermite.hermgauss(k)
    assert np.max(np.abs(x - rx)) <= 1e-12 * max(1.0, np.max(np.abs(rx)))
    assert np.max(np.abs(w - rw) / rw) <= 1e-9
