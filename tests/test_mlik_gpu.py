"""GPU parity of the fused config-3 learning step against the reference's
tape composition (oracle: inference.cpp:140-163 + tape.cpp:435-451 +
grad.cpp:145-151, restated bit-exactly in oracle/bandgm_oracle.c).

Metric: |a-b| / max(|a|, |b|, floor), floor = 1e-6 max|ref| for the
gradient arrays.  The fused sweep and the reference tape reach L_bar by
different (equally accurate) operation orders; entries that cancel to below
~1e-6 of the array maximum then differ by rounding (~1e-16 max), which a
1e-12 floor would report as ~1e-9 "relative" error.  test_exact.py pins both
implementations against an extended-precision evaluation instead."""
import numpy as np
import pytest

from tests import common as cm

pytestmark = pytest.mark.gpu
TOL = 1e-9
FLOOR = 1e-6


def _check(gpu, oracle, B, n, k, tau2, seed):
    rng = np.random.default_rng(seed)
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    lo, lb, tb, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert np.all(st == 0)
    lg, lbg, tbg, _, _ = gpu.marginal_likelihood_grad(L, y, tau2)
    for name, g, o in (("loss", lg, lo), ("l_bar", lbg, lb), ("tau2_bar", tbg, tb)):
        err = cm.max_rel_err(g, o, floor_scale=FLOOR)
        assert err <= TOL, f"{name} B={B} n={n} k={k}: {err:.3e}"
        # normwise agreement, as the survey also asks to report
        assert np.linalg.norm(g - o) <= 1e-10 * np.linalg.norm(o), name


@pytest.mark.parametrize("B,n,k,tau2", [(1, 1, 0, 0.5), (3, 50, 1, 0.3), (5, 400, 4, 0.01),
                                        (33, 700, 16, 0.01), (2, 2000, 16, 0.01), (4, 257, 8, 2.0)])
def test_mlik_matches_tape_composition(cuda, oracle, B, n, k, tau2):
    from tests.gpu_adapter import GpuOracle
    _check(GpuOracle(tile=32), oracle, B, n, k, tau2, seed=B * 1000 + n)


# ---------------------------------------------------------------- fast path
# k = 16 in the tile-1 layout routes to the team sweeps (bgm_mlik_fast.cu),
# k in {4, 8, 16} in the tile-32 layout to the one-thread-per-unit sweeps
# (bgm_mlik_t1.cu); small segment lengths force many segments + burn-in.
FAST = [(1, 16), (32, 16), (32, 8), (32, 4)]


@pytest.mark.parametrize("tile,k", FAST)
@pytest.mark.parametrize("B,n,seg", [(2, 300, 0), (3, 1000, 64), (5, 2048, 128), (33, 777, 96),
                                     (1, 17, 16), (4, 4096, 0), (70, 1200, 0)])
def test_mlik_fast_segments(cuda, oracle, B, n, seg, tile, k):
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    api.set_segment_rows(seg)
    try:
        api.debug_repairs(reset=True)
        _check(GpuOracle(tile=tile), oracle, B, n, k, 0.01, seed=B * 7 + n + k)
        assert api.debug_repairs() == 0  # well-conditioned: every burn-in converged
    finally:
        api.set_segment_rows(0)


@pytest.mark.parametrize("tile", [1, 32])
def test_mlik_fast_repair_path(cuda, oracle, monkeypatch, tile):
    """A 4- (16-) row burn-in cannot converge: the verification flags every segment
    boundary; flagged segments are recomputed from their neighbour's exact
    end state (tile 32) or the matrix by the exact single-unit sweep.
    Results must still match the reference."""
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(5)
    B, n, k, tau2 = 3, 1500, 16, 0.01
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    lo, lb, tb, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert np.all(st == 0)
    monkeypatch.setenv("BGM_BURN", "16" if tile == 1 else "4")  # team sweeps round to 16-row blocks
    api.set_segment_rows(64)
    try:
        api.debug_repairs(reset=True)
        lg, lbg, tbg, _, _ = GpuOracle(tile=tile).marginal_likelihood_grad(L, y, tau2)
        reps = api.debug_repairs()
    finally:
        api.set_segment_rows(0)
    assert reps > 0
    for name, g, o in (("loss", lg, lo), ("l_bar", lbg, lb), ("tau2_bar", tbg, tb)):
        assert cm.max_rel_err(g, o, floor_scale=FLOOR) <= TOL, name


@pytest.mark.parametrize("tile", [1, 32])
def test_mlik_fast_not_pd(cuda, oracle, tile):
    """A zero on L's diagonal mid-matrix: the reference throws at the
    log-det of L (inference.cpp:143); the fused step reports that row."""
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(11)
    B, n, k = 3, 900, 16
    L = cm.config_factor(rng, B, n, k)
    L[1, 500, 0] = 0.0
    y = rng.normal(0, 1, (B, n))
    api.set_segment_rows(128)
    try:
        _, _, _, st, row = GpuOracle(tile=tile).marginal_likelihood_grad(L, y, 0.01)
    finally:
        api.set_segment_rows(0)
    assert st[0] == 0 and st[2] == 0
    assert st[1] != 0 and row[1] == 500


@pytest.mark.parametrize("tile,k", [(1, 16), (32, 16), (32, 8)])
def test_mlik_fast_extreme_diagonals(cuda, oracle, tile, k):
    """Pivots and |L_ii| outside [1e-30, 1e30] send a matrix to the exact
    sweeps.  The reverse must be redone too: its fast path seeds 1/L_ii from a
    float reciprocal, which overflows for |L_ii| < ~3e-39.
    Matrix 0 has one L_ii = 1e-39 (its row otherwise zero, so chol(L L^T) in
    the reference still reproduces it), matrices 1 and 2 are scaled by 1e35 and
    1e-35, matrix 3 is an ordinary control."""
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(17 + k)
    B, n, tau2, i = 4, 900, 0.01, 300
    L = cm.config_factor(rng, B, n, k)
    L[0, i, 0] = 1e-39
    for r in range(1, k + 1):
        L[0, i - r, r] = 0.0
    L[1] *= 1e35
    L[2] *= 1e-35
    y = rng.normal(0, 1, (B, n))
    lo, lb, tb, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert np.all(st == 0)
    api.set_segment_rows(128)
    try:
        lg, lbg, tbg, stg, _ = GpuOracle(tile=tile).marginal_likelihood_grad(L, y, tau2)
    finally:
        api.set_segment_rows(0)
    assert np.all(stg == 0)
    assert np.all(np.isfinite(lbg))
    assert cm.max_rel_err(lg, lo, floor_scale=FLOOR) <= TOL
    # d tau2 cancels summands of ~yTy / (2 tau2^2) to ~1e-9 on the 1e-35
    # matrix: compare relative to the summands
    summ = n / (2 * tau2) + (y * y).sum(axis=1) / (2 * tau2 ** 2)
    assert np.all(np.abs(tbg - tb) <= 1e-12 * np.maximum(summ, np.abs(tb)))
    # L_bar(i, i) = ... + 1/L_ii = ~1e39 on matrix 0
    assert abs(lbg[0, i, 0] - lb[0, i, 0]) <= TOL * abs(lb[0, i, 0])
    # Matrix 0: the reference tape differentiates chol(L L^T) through the
    # 1e-39 pivot and returns ~1e21 for L_bar(i, i-r) where the true value is
    # O(1) (tests/exact.py, long double).  There the yardstick is the
    # extended-precision evaluation, and the reference is shown to be worse.
    ex = _exact_matrix0(L[:1], y[:1], tau2)
    g, e = lbg[0].copy(), ex.copy()
    assert abs(g[i, 0] - e[i, 0]) <= TOL * abs(e[i, 0])
    g[i, 0] = e[i, 0] = 0.0
    assert cm.max_rel_err(g, e, floor_scale=FLOOR) <= TOL
    r0 = lb[0].copy()
    r0[i, 0] = 0.0
    assert cm.max_rel_err(r0, e, floor_scale=FLOOR) > 1e3 * max(cm.max_rel_err(g, e, floor_scale=FLOOR), 1e-16)
    for b in range(1, B):  # per matrix: the scales differ by 1e70
        g, o = lbg[b].copy(), lb[b].copy()
        # floor relative to the summands' scale (1/L_ii): at 1e35 the
        # log|A| and log|L_Q| adjoints cancel exactly in the reference (A = Q
        # in fp64), leaving zeros that the fused form reaches as ~1e-16 of them
        scale = max(np.abs(o).max(), np.abs(1.0 / L[b, :, 0]).max() if b else 0.0)
        den = np.maximum(np.maximum(np.abs(g), np.abs(o)), FLOOR * scale)
        assert float(np.max(np.abs(g - o) / den)) <= TOL, b


_EXACT0 = {}


def _exact_matrix0(L, y, tau2):
    """L_bar of one matrix in long double along the banded route (cached per k)."""
    from tests import exact
    key = (L.shape, float(L.sum()))
    if key not in _EXACT0:
        _EXACT0[key] = np.asarray(exact.mlik_exact(L, y, tau2)[1], dtype=np.float64)[0]
    return _EXACT0[key]
