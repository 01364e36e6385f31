"""Bandwidths and layouts the fast paths do not take directly are staged onto
the compiled ones (csrc/bgm_promote.cu): k in {5..7, 9..15} onto 8 / 16 in the
32-matrix interleave, narrow bands in the reference layout (the C++ drop-in's
single matrices) onto the interleave, 17..63 / 65..127 onto the DMMA kernels
at 64 / 128.  Each promoted operator is checked against the CPU oracle (the
restated reference loops, kernels_serial.cpp / grad.cpp) at the parity
tolerance, and the promoted path is shown to have run (bgm_timing's
"promote" scope), so this is not the generic kernels passing."""
import ctypes as C

import numpy as np
import pytest

from tests import common as cm

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _promoted(fn):
    """Runs fn() with per-kernel timing on; returns (result, promote launches)."""
    import torch
    import paper_1902_10078_b200 as bgm
    lib = bgm.library()
    lib.bgm_timing_enable(1)
    try:
        out = fn()
        torch.cuda.synchronize()
        cnt = 0
        for i in range(lib.bgm_timing_read(-1, None, 0, None, None)):
            name = C.create_string_buffer(64)
            tot, c = C.c_double(), C.c_int64()
            lib.bgm_timing_read(i, name, 64, C.byref(tot), C.byref(c))
            if name.value == b"promote":
                cnt += c.value
    finally:
        lib.bgm_timing_enable(0)
    return out, cnt


CASES = [  # (tile, k, B, n)
    (32, 5, 3, 700), (32, 7, 33, 300), (32, 13, 2, 900), (1, 2, 1, 1024), (1, 4, 5, 800),
    (1, 5, 1, 2000), (1, 16, 2, 700), (1, 40, 2, 1200), (1, 100, 1, 1500),
]


@pytest.mark.parametrize("tile,k,B,n", CASES)
def test_promoted_forward(cuda, oracle, tile, k, B, n):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(k * 100 + B + tile)
    off = 0.1 if k <= 16 else 0.02 / k ** 0.5
    L0 = cm.config_factor(rng, B, n, k, off_std=off)
    q = cm.precision(oracle, L0, k)
    v = rng.normal(0, 1, (B, n))
    g = GpuOracle(tile=tile)
    (lg, st, _), c1 = _promoted(lambda: g.cholesky(q))
    lo, sto, _ = oracle.cholesky(q)
    assert c1 > 0 and np.all(st == 0) and np.all(sto == 0)
    assert cm.max_rel_err(lg, lo) <= TOL
    for tr in (False, True):
        (xg, _, _), c2 = _promoted(lambda: g.solve_vec(lo, v, tr))
        xo, _, _ = oracle.solve_vec(lo, v, tr)
        assert c2 > 0
        assert cm.max_rel_err(xg, xo) <= TOL, tr
    (sg, _, _), c3 = _promoted(lambda: g.sparse_inverse_subset(lo))
    so, _, _ = oracle.sparse_inverse_subset(lo)
    assert c3 > 0
    assert cm.max_rel_err(sg, so) <= TOL


@pytest.mark.parametrize("tile,k,B,n", CASES)
def test_promoted_adjoints(cuda, oracle, tile, k, B, n):
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(k * 101 + B + tile)
    off = 0.1 if k <= 16 else 0.02 / k ** 0.5
    L0 = cm.config_factor(rng, B, n, k, off_std=off)
    lo, _, _ = oracle.cholesky(cm.precision(oracle, L0, k))
    lbar = cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0)
    g = GpuOracle(tile=tile)
    qg, c1 = _promoted(lambda: g.vjp_cholesky(lo, lbar))
    qo = oracle.vjp_cholesky(lo, lbar)
    assert c1 > 0
    assert cm.max_rel_err(qg, qo) <= TOL
    so, _, _ = oracle.sparse_inverse_subset(lo)
    sbar = cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0)
    res, c2 = _promoted(lambda: g.vjp_sparse_inverse_subset(lo, so, sbar))
    ro = oracle.vjp_sparse_inverse_subset(lo, so, sbar)
    assert c2 > 0 or (k == 16 and tile == 1)  # k = 16 in the reference layout is compiled directly
    assert cm.max_rel_err(res[0], ro[0]) <= TOL


@pytest.mark.parametrize("tile,k", [(32, 6), (1, 3), (1, 40)])
def test_promoted_error_rows(cuda, oracle, tile, k):
    """The first failing pivot row survives the staging (errors.hpp:27-50)."""
    from tests.gpu_adapter import GpuOracle
    rng = np.random.default_rng(9 + k)
    B, n = 3, 1200
    L0 = cm.config_factor(rng, B, n, k, off_std=0.1 if k <= 16 else 0.02 / k ** 0.5)
    q = cm.precision(oracle, L0, k)
    q[1, 700, 0] = -1.0  # not positive definite from row 700
    (_, st, row), c = _promoted(lambda: GpuOracle(tile=tile).cholesky(q))
    _, sto, rowo = oracle.cholesky(q)
    assert c > 0
    assert list(st) == list(sto) and list(row) == list(rowo)
