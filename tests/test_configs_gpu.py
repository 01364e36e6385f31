"""Parity on every BASELINE.json configuration at its exact (n, k, dtype),
with a bounded batch (north_star: "every operator and
gradient matches the CPU oracle within tolerance on all 5 configs").

Inputs are built as BASELINE.md §4 says (seeded here with numpy, identical
arrays to the GPU and the oracle); the oracle is the plain-C restatement,
itself bit-identical to the verbatim reference (test_oracle.py).  The
batches are small, but the matrix sizes are the configs' own, so the
segmentation / burn-in / check machinery runs exactly as at full scale
(more segments per matrix, in fact, with fewer tiles to fill the GPU).
Tolerances: 1e-9 (fp64, floor 1e-12 max|ref|); fp32 against the fp64 oracle
on the rounded inputs at 1e-4 with the floors of test_wide_gpu.py."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-9


def _ok(g, o, name, dtype=torch.float64, floor=1e-5):
    if dtype == torch.float64:
        err = cm.max_rel_err(g, o)
        assert err <= TOL, f"{name}: {err:.3e}"
    else:
        err = cm.max_rel_err(g, o, floor_scale=floor)
        assert err < 1e-4, f"{name}: {err:.3e}"
        assert np.linalg.norm(g - o) <= 1e-5 * np.linalg.norm(o), name


def _suite(gpu, oracle, L0, k, b, rng, dtype=torch.float64, subset=True):
    """chol(Q), both solves, log-det, L b / L^T b, the inverse subset and the
    VJP of each against N(0,1) cotangents (config 0's list)."""
    B, n, _ = L0.shape
    q = cm.precision(oracle, L0, k)
    if dtype == torch.float32:
        q = q.astype(np.float32).astype(np.float64)
    l_o, st, _ = oracle.cholesky(q)
    assert np.all(st == 0)
    _ok(gpu.cholesky(q)[0], l_o, "cholesky", dtype)
    if dtype == torch.float32:
        l_o = l_o.astype(np.float32).astype(np.float64)
        b = b.astype(np.float32).astype(np.float64)
    x1 = oracle.solve_vec(l_o, b, False)[0]
    x2 = oracle.solve_vec(l_o, x1, True)[0]
    _ok(gpu.solve_vec(l_o, b, False)[0], x1, "solve L", dtype)
    _ok(gpu.solve_vec(l_o, x1, True)[0], x2, "solve L^T", dtype)
    _ok(gpu.log_det(l_o)[0], oracle.log_det(l_o)[0], "log_det", dtype)
    s_o = None
    if subset:
        s_o = oracle.sparse_inverse_subset(l_o)[0]
        _ok(gpu.sparse_inverse_subset(l_o)[0], s_o, "subset", dtype)
    # reverse, N(0,1) cotangents
    fl = FP32_VJP if dtype == torch.float32 else 1e-5
    lbar = cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0)
    sbar = rng.normal(0, 1, (B, n))
    if dtype == torch.float32:
        lbar, sbar = (a.astype(np.float32).astype(np.float64) for a in (lbar, sbar))
    _ok(gpu.vjp_cholesky(l_o, lbar), oracle.vjp_cholesky(l_o, lbar), "vjp_cholesky", dtype, fl)
    for tr, x in ((False, x1), (True, x2)):
        g = gpu.vjp_solve_vec(l_o, x, sbar, tr)
        o = oracle.vjp_solve_vec(l_o, x, sbar, tr)
        _ok(g[0], o[0], f"vjp_solve l_bar tr={tr}", dtype, fl)
        _ok(g[1], o[1], f"vjp_solve v_bar tr={tr}", dtype, fl)
    cb = rng.normal(0, 1, B)
    _ok(gpu.vjp_log_det(l_o, cb), oracle.vjp_log_det(l_o, cb), "vjp_log_det", dtype, fl)
    if subset:
        s_bar = cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0)
        if dtype == torch.float32:
            s_bar = s_bar.astype(np.float32).astype(np.float64)
        _ok(gpu.vjp_sparse_inverse_subset(l_o, s_o, s_bar)[0], oracle.vjp_sparse_inverse_subset(l_o, s_o, s_bar)[0],
            "vjp_subset", dtype, fl)
    return l_o


FP32_VJP = 1e-4


@pytest.mark.parametrize("tile", [1, 32])
def test_config0(cuda, oracle, tile):
    """configs[0]: one SPD band, n=1024, k=2, fp64 -- the full operator list
    plus L b, L^T b and their VJPs."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(0)
    n, k = 1024, 2
    L0 = cm.config_factor(rng, 1, n, k)
    b = rng.normal(0, 1, (1, n))
    gpu = GpuOracle(tile=tile)
    l_o = _suite(gpu, oracle, L0, k, b, rng)
    for tr in (False, True):
        _ok(gpu.product_band_vec(l_o, k, 0, b, tr), oracle.product_band_vec(l_o, k, 0, b, tr), f"band_vec tr={tr}")
        p = rng.normal(0, 1, (1, n))
        g = gpu.vjp_product_band_vec(l_o, k, 0, b, p, tr)
        o = oracle.vjp_product_band_vec(l_o, k, 0, b, p, tr)
        _ok(g[0], o[0], f"vjp_band_vec b_bar tr={tr}")
        _ok(g[1], o[1], f"vjp_band_vec v_bar tr={tr}")


def test_config1(cuda, oracle):
    """configs[1]: n=2048, k=4, fp64, tile 32 (forward chol + solves + log-det
    are the config's list; the VJPs ride along)."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(1)
    B, n, k = 37, 2048, 4
    _suite(GpuOracle(tile=32), oracle, cm.config_factor(rng, B, n, k), k, rng.normal(0, 1, (B, n)), rng,
           subset=False)


def test_config2(cuda, oracle):
    """configs[2]: n=65536, k=8, entries N(0,1): L L^T (8,8), A(8,8) B(3,3),
    A v and their VJPs, tile 32 (the staged product kernels)."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(2)
    B, n = 3, 65536
    gpu = GpuOracle(tile=32)
    L = cm.random_band(rng, B, n, 8, 0, dist="normal")
    Lt = cm.transpose_ref(L, 8, 0)
    A = cm.random_band(rng, B, n, 8, 8, dist="normal")
    Bm = cm.random_band(rng, B, n, 3, 3, dist="normal")
    v = rng.normal(0, 1, (B, n))
    # the product kernels accumulate in the reference's order without FMA
    # contraction: fp64 results are bitwise the reference's (restatement
    # compiled with -ffp-contract=off, itself bitwise the verbatim reference)
    same = lambda g, o, name: np.testing.assert_array_equal(g, o, err_msg=name)  # noqa: E731
    same(gpu.product_band_band(L, 8, 0, Lt, 0, 8)[0], oracle.product_band_band(L, 8, 0, Lt, 0, 8)[0], "L L^T")
    same(gpu.product_band_band(A, 8, 8, Bm, 3, 3)[0], oracle.product_band_band(A, 8, 8, Bm, 3, 3)[0], "A B")
    same(gpu.product_band_vec(A, 8, 8, v), oracle.product_band_vec(A, 8, 8, v), "A v")
    for (a, al, au, b, bl, bu, pl, pu, name) in ((L, 8, 0, Lt, 0, 8, 8, 8, "vjp L L^T"),
                                                 (A, 8, 8, Bm, 3, 3, 11, 11, "vjp A B")):
        p = cm.random_band(rng, B, n, pl, pu, dist="normal")
        g = gpu.vjp_product_band_band(a, al, au, b, bl, bu, p, pl, pu)
        o = oracle.vjp_product_band_band(a, al, au, b, bl, bu, p, pl, pu)
        same(g[0], o[0], name + " a_bar")
        same(g[1], o[1], name + " b_bar")
    p = rng.normal(0, 1, (B, n))
    g = gpu.vjp_product_band_vec(A, 8, 8, v, p, False)
    o = oracle.vjp_product_band_vec(A, 8, 8, v, p, False)
    same(g[0], o[0], "vjp A v b_bar")
    same(g[1], o[1], "vjp A v v_bar")


def test_config3(cuda, oracle):
    """configs[3]: n=65536, k=16, tau2=0.01: the fused learning step against
    the reference's tape composition (tolerances of test_mlik_gpu.py), and
    the op-by-op kernels of that composition at k=16."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(3)
    B, n, k, tau2 = 2, 65536, 16, 0.01
    L = cm.config_factor(rng, B, n, k)
    z = rng.normal(0, 1, (B, n))
    x = oracle.solve_vec(L, z, True)[0]  # x = L^-T z, BASELINE.md §4
    y = x + rng.normal(0, 0.1, (B, n))
    gpu = GpuOracle(tile=32)
    lo, lb, tb, st, _ = oracle.marginal_likelihood_grad(L, y, tau2)
    assert np.all(st == 0)
    lg, lbg, tbg, _, _ = gpu.marginal_likelihood_grad(L, y, tau2)
    for name, g, o in (("loss", lg, lo), ("l_bar", lbg, lb)):
        assert cm.max_rel_err(g, o, floor_scale=1e-6) <= TOL, name
        assert np.linalg.norm(g - o) <= 1e-10 * np.linalg.norm(o), name
    # tau2_bar = -n/(2 tau2) + y'y/(2 tau2^2) + ... is a cancelling sum: at
    # n = 65536 its summands are ~3e8 and the result ~1e3, so two fp64
    # evaluation orders differ by ~n^1/2 eps x 3e8.  Compared relative to the
    # summands' magnitude (the accuracy any fp64 order guarantees).
    scale = n / (2 * tau2) + (y * y).sum(axis=1) / (2 * tau2 ** 2)
    assert np.all(np.abs(tbg - tb) <= 1e-12 * scale), (tbg, tb)
    lt = cm.transpose_ref(L, k, 0)
    _ok(gpu.product_band_band(L, k, 0, lt, 0, k, k, 0)[0], oracle.product_band_band(L, k, 0, lt, 0, k, k, 0)[0],
        "band(L L^T)")
    G = cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0)
    g = gpu.vjp_product_band_band(L, k, 0, lt, 0, k, G, k, 0)
    o = oracle.vjp_product_band_band(L, k, 0, lt, 0, k, G, k, 0)
    _ok(g[0], o[0], "dL a_bar")
    _ok(g[1], o[1], "dL b_bar")
    _suite(gpu, oracle, L, k, y, rng, subset=False)


@pytest.mark.parametrize("k", [64, 128])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config4(cuda, oracle, k, dtype):
    """configs[4]: n=32768, k in {64, 128}, off-diagonal std 0.02 k^-1/2,
    fp64 and fp32, the full forward + reverse suite in the reference layout
    (tile 1, the layout config 4 is benchmarked in)."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(4 + k)
    B, n = 1, 32768
    L0 = cm.config_factor(rng, B, n, k, off_std=0.02 / np.sqrt(k))
    _suite(GpuOracle(tile=1, dtype=dtype), oracle, L0, k, rng.normal(0, 1, (B, n)), rng, dtype=dtype)


def test_config4_batch_row_spans(cuda, oracle, monkeypatch):
    """configs[4] at its full length with several matrices (k = 64, fp64): the full suite, with the
    adjoints' row-span geometry forced to 37 CTAs so their runs cross matrix ends at config size."""
    from tests.gpu_adapter import GpuOracle
    monkeypatch.setenv("BGM_WIDE_SPAN_CTAS", "37")
    rng = np.random.default_rng(4464)
    B, n, k = 5, 32768, 64
    L0 = cm.config_factor(rng, B, n, k, off_std=0.02 / np.sqrt(k))
    _suite(GpuOracle(tile=1, dtype=torch.float64), oracle, L0, k, rng.normal(0, 1, (B, n)), rng, dtype=torch.float64)

