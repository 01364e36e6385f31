"""GPU parity of the wide-band (k = 64, 128) fast paths (csrc/bgm_wide.cu)
against the oracle: both layouts, fp64 and fp32, automatic and forced
segmentation, the burn-in repair path and the reference's error rows.

Inputs follow BASELINE.md §4 config 4 (diag U[1,2], off-diagonal std
0.02 k^-1/2) plus the reference gradcheck's diagonally dominant generator
(gradcheck.cpp:23-38) whose Schur complements forget their start state more
slowly.  Tolerance 1e-9 (fp64) / 1e-4 (fp32, vs the fp64 oracle on the
rounded inputs), metric of test_util.hpp:19-21."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = pytest.mark.gpu
FP32_FLOOR = 1e-5
FP32_FLOOR_VJP = 1e-4  # adjoints of random-sign cotangents cancel harder


def _fp32_ok(g, o, floor=FP32_FLOOR):
    err = cm.max_rel_err(g, o, floor_scale=floor)
    assert err < 1e-4, err
    assert np.linalg.norm(g - o) <= 1e-5 * np.linalg.norm(o)


def _seg(rows):
    from paper_1902_10078_b200 import api
    api.set_segment_rows(rows)


@pytest.fixture
def segrows():
    yield _seg
    _seg(0)


def _q(oracle, rng, B, n, k, kind):
    if kind == "cfg4":
        L = cm.config_factor(rng, B, n, k, off_std=0.02 / np.sqrt(k))
        return cm.precision(oracle, L, k)
    return cm.random_spd_band(rng, B, n, k)


@pytest.mark.parametrize("k,n", [(64, 700), (128, 1100)])
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("seg", [0, 270])
@pytest.mark.parametrize("kind", ["cfg4", "dominant"])
def test_wide_cholesky(cuda, oracle, segrows, k, n, tile, seg, kind):
    from paper_1902_10078_b200 import api
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(k + n + seg)
    q = _q(oracle, rng, 3, n, k, kind)
    segrows(seg)
    api.debug_repairs(reset=True)
    l_g, st, _ = GpuOracle(tile=tile).cholesky(q)
    l_o, st_o, _ = oracle.cholesky(q)
    assert np.array_equal(st, st_o)
    assert cm.max_rel_err(l_g, l_o) <= 1e-9


@pytest.mark.parametrize("k,n", [(64, 700), (128, 1100)])
def test_wide_cholesky_fp32(cuda, oracle, segrows, k, n):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(3 * k)
    q = _q(oracle, rng, 2, n, k, "cfg4").astype(np.float32).astype(np.float64)
    segrows(256)
    l_g = GpuOracle(tile=1, dtype=torch.float32).cholesky(q)[0]
    _fp32_ok(l_g, oracle.cholesky(q)[0])


def test_wide_cholesky_repair_and_errors(cuda, oracle, segrows, monkeypatch):
    """A 4-row burn-in cannot converge: every boundary is flagged and the
    single-unit sweep recomputes the matrix.  One matrix is not positive
    definite in a late segment: its status / row match the reference."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(9)
    k, n = 64, 900
    q = _q(oracle, rng, 3, n, k, "dominant")
    q[1, 700, 0] = -1.0
    monkeypatch.setenv("BGM_WIDE_BURN", "4")
    segrows(180)
    l_g, st, row = GpuOracle(tile=1).cholesky(q)
    l_o, st_o, row_o = oracle.cholesky(q)
    assert list(st) == list(st_o) and st[1] == 1 and row[1] == row_o[1] == 700
    for b in (0, 2):
        assert cm.max_rel_err(l_g[b], l_o[b]) <= 1e-9


@pytest.mark.parametrize("k,n", [(64, 700), (128, 1100)])
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("seg", [0, 270])
@pytest.mark.parametrize("kind", ["cfg4", "dominant"])
def test_wide_subset(cuda, oracle, segrows, k, n, tile, seg, kind):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(2 * k + n + seg)
    q = _q(oracle, rng, 3, n, k, kind)
    l = oracle.cholesky(q)[0]
    segrows(seg)
    s_g, st, _ = GpuOracle(tile=tile).sparse_inverse_subset(l)
    s_o, st_o, _ = oracle.sparse_inverse_subset(l)
    assert np.array_equal(st, st_o)
    assert cm.max_rel_err(s_g, s_o) <= 1e-9


@pytest.mark.parametrize("k,n", [(64, 700), (128, 1100)])
def test_wide_subset_fp32(cuda, oracle, segrows, k, n):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(5 * k)
    l = oracle.cholesky(_q(oracle, rng, 2, n, k, "cfg4"))[0].astype(np.float32).astype(np.float64)
    segrows(256)
    s_g = GpuOracle(tile=1, dtype=torch.float32).sparse_inverse_subset(l)[0]
    _fp32_ok(s_g, oracle.sparse_inverse_subset(l)[0])


def test_wide_subset_repair_and_singular(cuda, oracle, segrows, monkeypatch):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(12)
    k, n = 64, 900
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, "dominant"))[0]
    l[2, 333, 0] = 0.0
    monkeypatch.setenv("BGM_WIDE_BURN", "4")
    segrows(180)
    s_g, st, row = GpuOracle(tile=1).sparse_inverse_subset(l)
    s_o, st_o, row_o = oracle.sparse_inverse_subset(l)
    assert list(st) == list(st_o) and st[2] == 2 and row[2] == 333
    for b in (0, 1):
        assert cm.max_rel_err(s_g[b], s_o[b]) <= 1e-9


@pytest.mark.parametrize("k,n", [(64, 1400), (128, 2600)])
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("seg", [0, 600])
@pytest.mark.parametrize("tr", [False, True])
def test_wide_solve(cuda, oracle, segrows, k, n, tile, seg, tr):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(7 * k + n + seg + tr)
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, "cfg4"))[0]
    v = cm.random_vec(rng, 3, n)
    segrows(seg)
    x_g, st, _ = GpuOracle(tile=tile).solve_vec(l, v, tr)
    x_o, st_o, _ = oracle.solve_vec(l, v, tr)
    assert np.array_equal(st, st_o)
    assert cm.max_rel_err(x_g, x_o) <= 1e-9
    lb_g, vb_g = GpuOracle(tile=tile).vjp_solve_vec(l, x_o, v, tr)[:2]
    lb_o, vb_o = oracle.vjp_solve_vec(l, x_o, v, tr)[:2]
    assert cm.max_rel_err(vb_g, vb_o) <= 1e-9
    assert cm.max_rel_err(lb_g, lb_o) <= 1e-9


@pytest.mark.parametrize("tr", [False, True])
def test_wide_solve_repair_singular_fp32(cuda, oracle, segrows, monkeypatch, tr):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(21 + tr)
    k, n = 64, 1500
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, "dominant"))[0]
    v = cm.random_vec(rng, 3, n)
    l[0, 100, 0] = 0.0
    l[0, 1200, 0] = 0.0
    monkeypatch.setenv("BGM_WIDE_BURN", "2")
    segrows(600)
    x_g, st, row = GpuOracle(tile=1).solve_vec(l, v, tr)
    x_o, st_o, row_o = oracle.solve_vec(l, v, tr)
    assert list(st) == list(st_o) and row[0] == row_o[0] == (1200 if tr else 100)
    for b in (1, 2):
        assert cm.max_rel_err(x_g[b], x_o[b]) <= 1e-9
    # fp32 on config-4 inputs (fp64 inputs rounded to fp32)
    l32 = oracle.cholesky(_q(oracle, rng, 2, n, k, "cfg4"))[0].astype(np.float32).astype(np.float64)
    v32 = v[1:].astype(np.float32).astype(np.float64)
    _fp32_ok(GpuOracle(tile=1, dtype=torch.float32).solve_vec(l32, v32, tr)[0], oracle.solve_vec(l32, v32, tr)[0])


@pytest.mark.parametrize("k,n", [(64, 1504), (128, 2048)])
@pytest.mark.parametrize("tr", [False, True])
def test_wide_solve_blocked_panels(cuda, oracle, segrows, monkeypatch, k, n, tr):
    """n a multiple of 8 in the reference layout runs the blocked solves (csrc/bgm_wide_solve.cu):
    whole matrix in one unit, forced segments with the regular burn-in, a burn-in too short to
    converge (check + exact repair), singular rows in the first and last segment, and fp32 storage."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(5 * k + n + tr)
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, "dominant"))[0]
    v = cm.random_vec(rng, 3, n)
    x_o = oracle.solve_vec(l, v, tr)[0]
    for seg in (0, 8 * k + 8, 3 * k):
        segrows(seg)
        x_g, st, _ = GpuOracle(tile=1).solve_vec(l, v, tr)
        assert not st.any()
        assert cm.max_rel_err(x_g, x_o) <= 1e-9, seg
    monkeypatch.setenv("BGM_WIDE_BURN", "8")
    segrows(3 * k)
    ls = l.copy()
    ls[1, 40, 0] = 0.0
    ls[1, n - 9, 0] = 0.0
    x_g, st, row = GpuOracle(tile=1).solve_vec(ls, v, tr)
    x_s, st_o, row_o = oracle.solve_vec(ls, v, tr)
    assert list(st) == list(st_o) and st[1] != 0 and row[1] == row_o[1] == (n - 9 if tr else 40)
    for b in (0, 2):
        assert cm.max_rel_err(x_g[b], x_s[b]) <= 1e-9
    monkeypatch.delenv("BGM_WIDE_BURN")
    segrows(0)
    l32 = oracle.cholesky(_q(oracle, rng, 2, n, k, "cfg4"))[0].astype(np.float32).astype(np.float64)
    v32 = v[1:].astype(np.float32).astype(np.float64)
    _fp32_ok(GpuOracle(tile=1, dtype=torch.float32).solve_vec(l32, v32, tr)[0], oracle.solve_vec(l32, v32, tr)[0])


@pytest.mark.parametrize("k,n", [(64, 1600), (128, 2304)])
def test_wide_cholesky_lookahead_interior(cuda, oracle, segrows, k, n):
    """n a multiple of 8 with several segments: the look-ahead kernel's interior loops (no stores during
    the burn-in, fast stores / loads inside), the tail panels, both warp-role assignments at k = 64
    (odd and even CTAs) and a failing pivot in the last panel."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(11 * k + n)
    q = _q(oracle, rng, 5, n, k, "cfg4")
    q[3, n - 3, 0] = -0.5
    l_o, st_o, row_o = oracle.cholesky(q)
    for seg in (0, 8 * k, 5 * k + 8):
        segrows(seg)
        l_g, st, row = GpuOracle(tile=1).cholesky(q)
        assert list(st) == list(st_o) and row[3] == row_o[3] == n - 3
        for b in (0, 1, 2, 4):
            assert cm.max_rel_err(l_g[b], l_o[b]) <= 1e-9, (seg, b)


@pytest.mark.parametrize("k,n", [(64, 700), (128, 1100)])
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("seg", [0, 270])
@pytest.mark.parametrize("kind", ["cfg4", "dominant"])
def test_wide_vjp_cholesky(cuda, oracle, segrows, k, n, tile, seg, kind):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(11 * k + n + seg)
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, kind))[0]
    lbar = cm.random_band(rng, 3, n, k, 0)
    segrows(seg)
    g = GpuOracle(tile=tile).vjp_cholesky(l, lbar)
    assert cm.max_rel_err(g, oracle.vjp_cholesky(l, lbar)) <= 1e-9


def test_wide_vjp_cholesky_fp32_and_repair(cuda, oracle, segrows, monkeypatch):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(77)
    k, n = 64, 900
    l = oracle.cholesky(_q(oracle, rng, 2, n, k, "cfg4"))[0]
    lbar = cm.random_band(rng, 2, n, k, 0)
    segrows(256)
    l32, lb32 = (a.astype(np.float32).astype(np.float64) for a in (l, lbar))
    _fp32_ok(GpuOracle(tile=1, dtype=torch.float32).vjp_cholesky(l32, lb32), oracle.vjp_cholesky(l32, lb32),
             FP32_FLOOR_VJP)
    monkeypatch.setenv("BGM_WIDE_BURN", "3")
    segrows(200)
    assert cm.max_rel_err(GpuOracle(tile=1).vjp_cholesky(l, lbar), oracle.vjp_cholesky(l, lbar)) <= 1e-9


@pytest.mark.parametrize("k,n", [(64, 700), (128, 1100)])
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("seg", [0, 270])
@pytest.mark.parametrize("kind", ["cfg4", "dominant"])
def test_wide_vjp_subset(cuda, oracle, segrows, k, n, tile, seg, kind):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(13 * k + n + seg)
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, kind))[0]
    s = oracle.sparse_inverse_subset(l)[0]
    sbar = cm.random_band(rng, 3, n, k, 0)
    segrows(seg)
    g, st, _ = GpuOracle(tile=tile).vjp_sparse_inverse_subset(l, s, sbar)
    o, st_o, _ = oracle.vjp_sparse_inverse_subset(l, s, sbar)
    assert np.array_equal(st, st_o)
    assert cm.max_rel_err(g, o) <= 1e-9


@pytest.mark.parametrize("k,n,ctas", [(64, 1000, 7), (64, 1203, 5), (128, 2000, 3)])
def test_wide_vjp_subset_row_spans(cuda, oracle, segrows, monkeypatch, k, n, ctas):
    """Row-span geometry: the batch's rows, matrices end to end, cut into equal runs over a forced
    number of CTAs, so runs cross matrix ends (several pieces per CTA) and pieces start inside
    matrices (burn-in + check against the previous CTA's last piece); n % 8 != 0 pads each matrix."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(17 * k + n)
    B = 5
    l = oracle.cholesky(_q(oracle, rng, B, n, k, "cfg4"))[0]
    s = oracle.sparse_inverse_subset(l)[0]
    sbar = cm.random_band(rng, B, n, k, 0)
    o = oracle.vjp_sparse_inverse_subset(l, s, sbar)[0]
    monkeypatch.setenv("BGM_WIDE_SPAN_CTAS", str(ctas))
    segrows(0)
    g, st, _ = GpuOracle(tile=1).vjp_sparse_inverse_subset(l, s, sbar)
    assert not st.any()
    assert cm.max_rel_err(g, o) <= 1e-9
    sub, st, _ = GpuOracle(tile=1).sparse_inverse_subset(l)
    assert not st.any()
    assert cm.max_rel_err(sub, s) <= 1e-9
    lbar = cm.random_band(rng, B, n, k, 0)
    qb_o = oracle.vjp_cholesky(l, lbar)
    assert cm.max_rel_err(GpuOracle(tile=1).vjp_cholesky(l, lbar), qb_o) <= 1e-9
    # a burn-in too short to converge: the span check must flag it and the exact path repair it
    monkeypatch.setenv("BGM_WIDE_BURN", "8")
    g, st, _ = GpuOracle(tile=1).vjp_sparse_inverse_subset(l, s, sbar)
    assert cm.max_rel_err(g, o) <= 1e-9
    assert cm.max_rel_err(GpuOracle(tile=1).vjp_cholesky(l, lbar), qb_o) <= 1e-9


def test_wide_vjp_subset_fp32_repair_singular(cuda, oracle, segrows, monkeypatch):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(78)
    k, n = 64, 900
    l = oracle.cholesky(_q(oracle, rng, 3, n, k, "cfg4"))[0]
    s = oracle.sparse_inverse_subset(l)[0]
    sbar = cm.random_band(rng, 3, n, k, 0)
    segrows(256)
    a32 = [a[:2].astype(np.float32).astype(np.float64) for a in (l, s, sbar)]
    _fp32_ok(GpuOracle(tile=1, dtype=torch.float32).vjp_sparse_inverse_subset(*a32)[0],
             oracle.vjp_sparse_inverse_subset(*a32)[0], FP32_FLOOR_VJP)
    monkeypatch.setenv("BGM_WIDE_BURN", "3")
    segrows(200)
    l[2, 500, 0] = 0.0
    g, st, row = GpuOracle(tile=1).vjp_sparse_inverse_subset(l, s, sbar)
    o, st_o, row_o = oracle.vjp_sparse_inverse_subset(l, s, sbar)
    assert list(st) == list(st_o) and row[2] == row_o[2] == 500
    assert cm.max_rel_err(g[:2], o[:2]) <= 1e-9
