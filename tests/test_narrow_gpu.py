"""GPU parity of the narrow-band (k <= 16, tile 32) per-operator fast paths
(csrc/bgm_narrow.cu): cholesky, solve_vec (L, L^T), sparse_inverse_subset
against the oracle, with automatic and forced segmentation, a batch that is
not a multiple of the 32-matrix tile, the burn-in repair path and the
reference's error rows.  Tolerance 1e-9 (fp64), metric of
test_util.hpp:19-21."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = pytest.mark.gpu


@pytest.fixture
def segrows():
    from paper_1902_10078_b200 import api
    yield api.set_segment_rows
    api.set_segment_rows(0)


def _factor(oracle, rng, B, n, k, kind):
    if kind == "config":
        return oracle.cholesky(cm.precision(oracle, cm.config_factor(rng, B, n, k), k))[0]
    return oracle.cholesky(cm.random_spd_band(rng, B, n, k))[0]


@pytest.mark.parametrize("k", [1, 2, 3, 4, 8, 16])
@pytest.mark.parametrize("B,n,seg", [(37, 700, 0), (5, 1500, 300), (64, 257, 80)])
@pytest.mark.parametrize("kind", ["config", "dominant"])
def test_narrow_ops(cuda, oracle, segrows, k, B, n, seg, kind):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(k * 1000 + n + seg)
    gpu = GpuOracle(tile=32)
    q = cm.precision(oracle, cm.config_factor(rng, B, n, k), k) if kind == "config" else cm.random_spd_band(rng, B, n, k)
    segrows(seg)
    l_g, st, _ = gpu.cholesky(q)
    l_o, st_o, _ = oracle.cholesky(q)
    assert np.array_equal(st, st_o)
    assert cm.max_rel_err(l_g, l_o) <= 1e-9, "cholesky"
    v = cm.random_vec(rng, B, n)
    for tr in (False, True):
        x_g = gpu.solve_vec(l_o, v, tr)[0]
        assert cm.max_rel_err(x_g, oracle.solve_vec(l_o, v, tr)[0]) <= 1e-9, f"solve {tr}"
    s_g = gpu.sparse_inverse_subset(l_o)[0]
    assert cm.max_rel_err(s_g, oracle.sparse_inverse_subset(l_o)[0]) <= 1e-9, "subset"
    lbar = cm.random_band(rng, B, n, k, 0)
    assert cm.max_rel_err(gpu.vjp_cholesky(l_o, lbar), oracle.vjp_cholesky(l_o, lbar)) <= 1e-9, "vjp_cholesky"


def test_narrow_repair_and_errors(cuda, oracle, segrows, monkeypatch):
    """A 2-row burn-in cannot converge: every boundary is flagged and the
    single-unit sweeps recompute.  Error rows match the reference."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(3)
    B, n, k = 33, 900, 4
    gpu = GpuOracle(tile=32)
    q = cm.random_spd_band(rng, B, n, k)
    q[7, 640, 0] = -5.0
    monkeypatch.setenv("BGM_NARROW_BURN", "2")
    segrows(100)
    l_g, st, row = gpu.cholesky(q)
    l_o, st_o, row_o = oracle.cholesky(q)
    assert np.array_equal(st, st_o) and row[7] == row_o[7]
    ok = np.nonzero(st_o == 0)[0]
    assert cm.max_rel_err(l_g[ok], l_o[ok]) <= 1e-9
    l = l_o.copy()
    l[ok[0]] = oracle.cholesky(cm.random_spd_band(rng, 1, n, k))[0][0]
    l[7] = l[ok[1]]
    l[7, 100, 0] = 0.0
    l[7, 700, 0] = 0.0
    v = cm.random_vec(rng, B, n)
    for tr in (False, True):
        x_g, st, row = gpu.solve_vec(l, v, tr)
        x_o, st_o, row_o = oracle.solve_vec(l, v, tr)
        assert np.array_equal(st, st_o) and row[7] == row_o[7] == (700 if tr else 100)
        good = np.nonzero(st_o == 0)[0]
        assert cm.max_rel_err(x_g[good], x_o[good]) <= 1e-9
    s_g, st, row = gpu.sparse_inverse_subset(l)
    s_o, st_o, row_o = oracle.sparse_inverse_subset(l)
    assert np.array_equal(st, st_o) and row[7] == 100
    good = np.nonzero(st_o == 0)[0]
    assert cm.max_rel_err(s_g[good], s_o[good]) <= 1e-9
    lbar = cm.random_band(rng, B, n, k, 0)
    assert cm.max_rel_err(gpu.vjp_cholesky(l[good], lbar[good]), oracle.vjp_cholesky(l[good], lbar[good])) <= 1e-9


def test_narrow_fp32(cuda, oracle, segrows):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(8)
    B, n, k = 40, 800, 8
    g32 = GpuOracle(tile=32, dtype=torch.float32)
    q = cm.precision(oracle, cm.config_factor(rng, B, n, k, off_std=0.02 / np.sqrt(k)), k)
    q = q.astype(np.float32).astype(np.float64)
    segrows(200)
    l_o = oracle.cholesky(q)[0]
    for g, o in ((g32.cholesky(q)[0], l_o),
                 (g32.sparse_inverse_subset(l_o)[0], oracle.sparse_inverse_subset(l_o)[0])):
        assert cm.max_rel_err(g, o, floor_scale=1e-5) < 1e-4
    v = cm.random_vec(rng, B, n).astype(np.float32).astype(np.float64)
    for tr in (False, True):
        assert cm.max_rel_err(g32.solve_vec(l_o, v, tr)[0], oracle.solve_vec(l_o, v, tr)[0], floor_scale=1e-5) < 1e-4
