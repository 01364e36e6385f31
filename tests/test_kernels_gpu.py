"""GPU parity: every operator and adjoint through the C ABI vs the oracle.

Mirrors proj/tests/test_kernels.cpp and test_grad.cpp: the golden vectors
(reference compiled verbatim), random shapes against the C restatement, the
reference's error rows, both device layouts (tile 32 / tile 1) and fp32.
Tolerance: north_star's 1e-9 relative (fp64), 1e-4 (fp32), metric of
test_util.hpp:19-21 with floor 1e-12 max|ref|.
"""
import os

import numpy as np
import pytest
import torch

from tests import common as cm
from tests.golden.cases import CASES, run_case

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")
TOL64 = 1e-9


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="module", params=[32, 1], ids=["tile32", "tile1"])
def gpu(request, cuda):
    from tests.gpu_adapter import GpuOracle
    return GpuOracle(tile=request.param)


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_cases(gpu, golden, name):
    got = run_case(name, gpu)
    for key, val in got.items():
        want = golden[f"{name}/{key}"]
        if key == "status":
            assert np.array_equal(val, want)
            continue
        err = cm.max_rel_err(val, want)
        assert err <= TOL64, f"{name}/{key}: max rel err {err:.3e}"


def test_error_rows(gpu):
    q = np.zeros((2, 4, 1))
    q[:, :, 0] = 1.0
    q[1, 2, 0] = -1.0  # test_kernels.cpp:48-58: first bad pivot at row 2
    _, st, row = gpu.cholesky(q)
    assert list(st) == [0, 1] and row[1] == 2
    ind = np.array([[[1.0, 2.0], [1.0, 0.0]]])  # indefinite 2x2 -> row 1
    _, st, row = gpu.cholesky(ind)
    assert st[0] == 1 and row[0] == 1
    l = np.zeros((1, 3, 2))
    l[0, :, 0] = [1.0, 0.0, 1.0]  # test_kernels.cpp:102-115
    _, st, row = gpu.solve_vec(l, np.ones((1, 3)), False)
    assert st[0] == 2 and row[0] == 1
    _, st, row = gpu.log_det(np.array([[[1.0], [-2.0]]]))  # test_kernels.cpp:237-245
    assert st[0] == 3 and row[0] == 1


def test_log_det_pivot_ranges(gpu, oracle):
    """log_det sums one log of a mantissa product per 64-row chunk: pivots
    across the whole exponent range, near 1 (small log-det), exactly at the
    sqrt 2 mantissa split, and chunks with subnormal / inf pivots (the per-row
    loop) against the reference's per-row sum."""
    rng = np.random.default_rng(11)
    B, n = 6, 300
    l = np.zeros((B, n, 3))
    l[0, :, 0] = 10.0 ** rng.uniform(-300, 300, n)
    l[1, :, 0] = 1.0 + rng.uniform(-1e-3, 1e-3, n)
    l[2, :, 0] = np.sqrt(2.0) * (1.0 + rng.choice([-1, 0, 1], n) * 2.0 ** -52)
    l[3, :, 0] = rng.uniform(0.5, 2.0, n)
    l[3, 70, 0] = 5e-320  # subnormal: the chunk's per-row loop
    l[4, :, 0] = rng.uniform(0.1, 10.0, n)
    l[4, 200, 0] = np.inf
    l[5, :, 0] = 2.0 ** rng.integers(-1000, 1000, n)
    got, st, _ = gpu.log_det(l)
    want, st_o, _ = oracle.log_det(l)
    assert np.array_equal(st, st_o)
    for b in (0, 1, 2, 3, 5):
        assert abs(got[b] - want[b]) <= 1e-12 * max(1.0, np.abs(np.log(l[b, :, 0])).sum()), b
    assert np.isinf(got[4]) and np.isinf(want[4])


def test_known_answers(gpu):
    l, st, _ = gpu.cholesky(np.array([[[4.0, 2.0], [5.0, 0.0]]]))
    assert np.allclose(l[0], [[2.0, 1.0], [2.0, 0.0]], rtol=0, atol=1e-15)
    s, _, _ = gpu.sparse_inverse_subset(np.array([[[1.0, 1.0], [1.0, 0.0]]]))
    assert np.allclose(s[0], [[2.0, -1.0], [1.0, 0.0]], rtol=0, atol=1e-15)
    assert gpu.vjp_cholesky(np.array([[[2.0]]]), np.array([[[1.0]]]))[0, 0, 0] == 0.25
    lb, _, _ = gpu.vjp_sparse_inverse_subset(np.array([[[1.0]]]), np.array([[[1.0]]]), np.array([[[1.0]]]))
    assert lb[0, 0, 0] == -2.0


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_vs_restatement(gpu, oracle, seed):
    rng = np.random.default_rng(100 + seed)
    B = [1, 5, 37, 64, 3, 33][seed]
    n = int(rng.integers(1, 60))
    bw = int(min(rng.integers(0, 7), n - 1))
    q = cm.random_spd_band(rng, B, n, bw)
    pairs = []
    l_o, st_o, _ = oracle.cholesky(q)
    l_g, st_g, _ = gpu.cholesky(q)
    assert np.array_equal(st_o, st_g)
    pairs.append(("cholesky", l_g, l_o))
    v = cm.random_vec(rng, B, n)
    for t in (False, True):
        pairs.append((f"solve{t}", gpu.solve_vec(l_o, v, t)[0], oracle.solve_vec(l_o, v, t)[0]))
    pairs.append(("logdet", gpu.log_det(l_o)[0], oracle.log_det(l_o)[0]))
    s_o = oracle.sparse_inverse_subset(l_o)[0]
    pairs.append(("subset", gpu.sparse_inverse_subset(l_o)[0], s_o))
    lbar = cm.random_band(rng, B, n, bw, 0)
    pairs.append(("vjp_chol", gpu.vjp_cholesky(l_o, lbar), oracle.vjp_cholesky(l_o, lbar)))
    pairs.append(("vjp_subset", gpu.vjp_sparse_inverse_subset(l_o, s_o, lbar)[0],
                  oracle.vjp_sparse_inverse_subset(l_o, s_o, lbar)[0]))
    for t in (False, True):
        x = oracle.solve_vec(l_o, v, t)[0]
        g = gpu.vjp_solve_vec(l_o, x, v, t)
        o = oracle.vjp_solve_vec(l_o, x, v, t)
        pairs += [(f"vjp_solve_l{t}", g[0], o[0]), (f"vjp_solve_v{t}", g[1], o[1])]
    al, au = int(rng.integers(0, 4)), int(rng.integers(0, 4))
    al, au = min(al, n - 1), min(au, n - 1)
    a = cm.random_band(rng, B, n, al, au)
    b = cm.random_band(rng, B, n, bw, min(2, n - 1))
    bu = min(2, n - 1)
    pairs.append(("product", gpu.product_band_band(a, al, au, b, bw, bu)[0],
                  oracle.product_band_band(a, al, au, b, bw, bu)[0]))
    pairs.append(("bandvec", gpu.product_band_vec(a, al, au, v, True), oracle.product_band_vec(a, al, au, v, True)))
    for name, g, o in pairs:
        err = cm.max_rel_err(g, o)
        assert err <= TOL64, f"{name} (B={B}, n={n}, bw={bw}): {err:.3e}"


def test_fp32_factorization_path(cuda, oracle):
    from tests.gpu_adapter import GpuOracle
    g32 = GpuOracle(tile=1, dtype=torch.float32)
    rng = np.random.default_rng(7)
    B, n, k = 4, 300, 8
    L = cm.config_factor(rng, B, n, k, off_std=0.02 / np.sqrt(k))
    q = cm.precision(oracle, L, k).astype(np.float32).astype(np.float64)
    l_o = oracle.cholesky(q)[0]
    l_g = g32.cholesky(q)[0]
    assert cm.max_rel_err(l_g, l_o) < 1e-4
    v = cm.random_vec(rng, B, n).astype(np.float32).astype(np.float64)
    assert cm.max_rel_err(g32.solve_vec(l_o, v, True)[0], oracle.solve_vec(l_o, v, True)[0]) < 1e-4
    assert cm.max_rel_err(g32.sparse_inverse_subset(l_o)[0], oracle.sparse_inverse_subset(l_o)[0]) < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("shape", ["llt8", "ab", "llt16_lower"])
def test_register_blocked_products(cuda, oracle, tile, dtype, shape):
    """The register-blocked product kernels (bgm_product.cu) serve these band
    shapes only: L L^T (8,8), A(8,8) B(3,3), precision_from_factor at k=16
    (inference.cpp:23-26); n not a multiple of the 4-column block."""
    import paper_1902_10078_b200 as bgm
    from tests.gpu_adapter import GpuOracle
    g = GpuOracle(tile=tile, dtype=dtype)
    rng = np.random.default_rng({"llt8": 11, "ab": 12, "llt16_lower": 13}[shape] + tile)
    B, n = 5, 203
    if shape == "ab":
        a = cm.random_band(rng, B, n, 8, 8)
        b = cm.random_band(rng, B, n, 3, 3)
        if dtype == torch.float32:
            a, b = (x.astype(np.float32).astype(np.float64) for x in (a, b))
        got = g._np(bgm.product_band_band(g._b(a, 8, 8), g._b(b, 3, 3)))
        ref = oracle.product_band_band(a, 8, 8, b, 3, 3)[0]
    else:
        k = 8 if shape == "llt8" else 16
        l = cm.random_band(rng, B, n, k, 0)
        if dtype == torch.float32:
            l = l.astype(np.float32).astype(np.float64)
        L = g._b(l, k, 0)
        lt = cm.transpose_ref(l, k, 0)
        if shape == "llt8":
            got = g._np(bgm.product_band_band(L, bgm.T(L)))
            ref = oracle.product_band_band(l, k, 0, lt, 0, k)[0]
        else:
            got = g._np(bgm.product_band_band_restricted(L, bgm.T(L), k, 0))
            ref = oracle.product_band_band(l, k, 0, lt, 0, k, k, 0)[0]
    if dtype == torch.float64:
        assert cm.max_rel_err(got, ref) <= TOL64
    else:  # fp32 storage, fp64 accumulation (acc_t): each cell is the rounded exact dot
        assert cm.max_rel_err(got, ref) <= 1e-4
        assert np.linalg.norm(got - ref) <= 1e-6 * np.linalg.norm(ref)


STAGED_VJP = {"vjp_ab": (8, 8, 3, 3, 11, 11), "vjp_llt": (8, 0, 0, 8, 8, 8), "vjp_dl": (16, 0, 0, 16, 16, 0)}


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("shape", sorted(STAGED_VJP))
@pytest.mark.parametrize("B,n", [(5, 203), (70, 1031)])
def test_staged_vjp_products(cuda, oracle, dtype, shape, B, n):
    """The fused product VJP of bgm_stream.cu (grad.cpp:145-151: A-bar = P-bar
    B^T on band(A), B-bar = A^T P-bar on band(B), P-bar staged once) for the
    config-2 / config-3 band shapes, tile 32; B = 70 spans three tiles (a
    partial one) and n = 1031 gives each CTA runs that start mid-matrix."""
    from tests.gpu_adapter import GpuOracle
    al, au, bl, bu, pl, pu = STAGED_VJP[shape]
    g = GpuOracle(tile=32, dtype=dtype)
    rng = np.random.default_rng(100 + len(shape) + n)
    a = cm.random_band(rng, B, n, al, au)
    b = cm.random_band(rng, B, n, bl, bu)
    p = cm.random_band(rng, B, n, pl, pu)
    if dtype == torch.float32:
        a, b, p = (x.astype(np.float32).astype(np.float64) for x in (a, b, p))
    ga, gb = g.vjp_product_band_band(a, al, au, b, bl, bu, p, pl, pu)
    ra, rb = oracle.vjp_product_band_band(a, al, au, b, bl, bu, p, pl, pu)[:2]
    tol = TOL64 if dtype == torch.float64 else 1e-4
    assert cm.max_rel_err(ga, ra) <= tol
    assert cm.max_rel_err(gb, rb) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["llt8", "ab", "llt16_lower"])
def test_staged_products_multi_tile(cuda, oracle, shape):
    """Staged products over several tiles, with corner cells of the inputs
    poisoned (NaN): they must never be read (kernels_detail.hpp:16-28)."""
    import paper_1902_10078_b200 as bgm
    from tests.gpu_adapter import GpuOracle
    g = GpuOracle(tile=32, dtype=torch.float64)
    rng = np.random.default_rng({"llt8": 21, "ab": 22, "llt16_lower": 23}[shape])
    B, n = 70, 1031

    def poisoned(x, lo, up):
        y = x.copy()
        for r in range(lo + up + 1):  # storage row r of column j holds i = j - up + r
            i = np.arange(n) - up + r
            y[:, (i < 0) | (i >= n), r] = np.nan
        return y

    if shape == "ab":
        a = cm.random_band(rng, B, n, 8, 8)
        b = cm.random_band(rng, B, n, 3, 3)
        got = g._np(bgm.product_band_band(g._b(poisoned(a, 8, 8), 8, 8), g._b(poisoned(b, 3, 3), 3, 3)))
        ref = oracle.product_band_band(a, 8, 8, b, 3, 3)[0]
    else:
        k = 8 if shape == "llt8" else 16
        l = cm.random_band(rng, B, n, k, 0)
        L = g._b(poisoned(l, k, 0), k, 0)
        lt = cm.transpose_ref(l, k, 0)
        if shape == "llt8":
            got = g._np(bgm.product_band_band(L, bgm.T(L)))
            ref = oracle.product_band_band(l, k, 0, lt, 0, k)[0]
        else:
            got = g._np(bgm.product_band_band_restricted(L, bgm.T(L), k, 0))
            ref = oracle.product_band_band(l, k, 0, lt, 0, k, k, 0)[0]
    assert np.all(np.isfinite(got))
    assert cm.max_rel_err(got, ref) <= TOL64


@pytest.mark.gpu
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_band_vec_tile32_multi_tile(cuda, oracle, transpose, dtype):
    """Tile-32 band x vector and its fused VJP (kernels_detail.hpp:31-45,
    grad.cpp:153-162) over three tiles (one partial), band (8,8) as config 2
    and a ragged (2,5) band; corner cells poisoned with NaN."""
    from tests.gpu_adapter import GpuOracle
    g = GpuOracle(tile=32, dtype=dtype)
    rng = np.random.default_rng(31 + int(transpose))
    B, n = 70, 517
    tol = TOL64 if dtype == torch.float64 else 1e-4
    for lo, up in ((8, 8), (2, 5)):
        b = cm.random_band(rng, B, n, lo, up)
        v, p = cm.random_vec(rng, B, n), cm.random_vec(rng, B, n)
        if dtype == torch.float32:
            b, v, p = (x.astype(np.float32).astype(np.float64) for x in (b, v, p))
        bp = b.copy()
        for r in range(lo + up + 1):
            i = np.arange(n) - up + r
            bp[:, (i < 0) | (i >= n), r] = np.nan
        y = g.product_band_vec(bp, lo, up, v, transpose)
        assert cm.max_rel_err(y, oracle.product_band_vec(b, lo, up, v, transpose)) <= tol
        gb, gv = g.vjp_product_band_vec(bp, lo, up, v, p, transpose)
        rb, rv = oracle.vjp_product_band_vec(b, lo, up, v, p, transpose)[:2]
        assert np.all(np.isfinite(gb)) and np.all(np.isfinite(gv))
        assert cm.max_rel_err(gb, rb) <= tol
        assert cm.max_rel_err(gv, rv) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("B,n", [(1, 1), (1, 2), (33, 31), (3, 33), (2, 97)])
@pytest.mark.parametrize("lo,up", [(0, 0), (2, 1), (1, 3)])
def test_vector_kernels_edge_shapes(cuda, oracle, tile, B, n, lo, up):
    """band x vector, outer band and their VJPs on degenerate and ragged
    shapes (n = 1, bands clipped to n - 1, partial tiles, n not a multiple of
    the 32-column runs) in both layouts, bitwise against the oracle
    (kernels_detail.hpp:31-54 evaluated in the same order, uncontracted)."""
    from tests.gpu_adapter import GpuOracle
    g = GpuOracle(tile=tile)
    rng = np.random.default_rng(B * 100 + n + lo + 7 * up)
    lo, up = min(lo, n - 1), min(up, n - 1)
    b = cm.random_band(rng, B, n, lo, up)
    v, p = cm.random_vec(rng, B, n), cm.random_vec(rng, B, n)
    for tr in (False, True):
        np.testing.assert_array_equal(g.product_band_vec(b, lo, up, v, tr), oracle.product_band_vec(b, lo, up, v, tr))
        gb, gv = g.vjp_product_band_vec(b, lo, up, v, p, tr)
        rb, rv = oracle.vjp_product_band_vec(b, lo, up, v, p, tr)[:2]
        np.testing.assert_array_equal(gb, rb)
        np.testing.assert_array_equal(gv, rv)
    np.testing.assert_array_equal(g.outer_band(v, p, lo, up), oracle.outer_band(v, p, lo, up))
