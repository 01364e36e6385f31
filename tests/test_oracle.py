"""CPU: pin the oracle.

The plain-C restatement (oracle/bandgm_oracle.c) must reproduce
  * the committed golden vectors (generated from the reference compiled
    verbatim) bit for bit,
  * the verbatim reference itself bit for bit on fresh inputs (when
    oracle/_ref is built),
  * the reference's own known answers (SPEC.md examples, test_kernels.cpp
    error rows) and dense-algebra identities (test_kernels.cpp:71-246).
The verbatim reference must pass its own finite-difference suite
(test_grad.cpp:32-40, acceptance.cpp:142-147).
"""
import os

import numpy as np
import pytest

from tests import common as cm
from tests.golden.cases import CASES, run_case

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.mark.parametrize("name", sorted(CASES))
def test_restatement_matches_golden_bitwise(oracle, golden, name):
    got = run_case(name, oracle)
    for key, val in got.items():
        want = golden[f"{name}/{key}"]
        assert np.array_equal(np.asarray(val), want), f"{name}/{key} differs from the reference"


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_restatement_matches_verbatim_reference(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    B, n, k = 4, 120, 6
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(size=(B, n))
    for fn in (lambda o: o.marginal_likelihood_grad(L, y, 0.05),
               lambda o: o.sparse_inverse_subset(L),
               lambda o: o.vjp_cholesky(L, cm.random_band(np.random.default_rng(seed), B, n, k, 0))):
        a, b = fn(oracle), fn(reference)
        a = a if isinstance(a, tuple) else (a,)
        b = b if isinstance(b, tuple) else (b,)
        for x, z in zip(a, b):
            assert np.array_equal(x, z)


def test_reference_fd_suite_passes(reference):
    # test_grad.cpp:32-40 and acceptance.cpp:142-147
    for seed, inst in ((1234, 10), (2024, 50)):
        errs = reference.run_grad_suite(seed, inst)
        assert len(errs) == 12
        assert np.all(errs < 1e-5), errs


# ------------------------------------------------ known answers (restatement)
def _sym(vals_diag, off=None):
    n = len(vals_diag)
    bw = 0 if off is None else 1
    q = np.zeros((1, n, bw + 1))
    q[0, :, 0] = vals_diag
    if off is not None:
        q[0, : n - 1, 1] = off
    return q


def test_cholesky_known_answers(oracle):
    l, st, _ = oracle.cholesky(_sym([4.0, 9.0]))  # test_kernels.cpp:37-46
    assert st[0] == 0 and l[0, 0, 0] == 2.0 and l[0, 1, 0] == 3.0
    l, st, _ = oracle.cholesky(_sym([4.0, 5.0], [2.0]))  # SPEC.md: [[4,2],[2,5]] -> [[2,0],[1,2]]
    assert np.allclose(l[0], [[2.0, 1.0], [2.0, 0.0]])


def test_cholesky_error_rows(oracle):
    _, st, row = oracle.cholesky(_sym([1.0, 1.0, -1.0, 1.0]))  # test_kernels.cpp:48-58
    assert st[0] == 1 and row[0] == 2
    _, st, row = oracle.cholesky(_sym([1.0, 1.0], [2.0]))  # indefinite 2x2 -> row 1
    assert st[0] == 1 and row[0] == 1


def test_solve_vec_singular_row(oracle):
    l = np.zeros((1, 3, 2))
    l[0, :, 0] = [1.0, 0.0, 1.0]  # test_kernels.cpp:102-115
    _, st, row = oracle.solve_vec(l, np.ones((1, 3)), False)
    assert st[0] == 2 and row[0] == 1


def test_subset_known_answers(oracle):
    s, _, _ = oracle.sparse_inverse_subset(np.array([[[1.0]]]))  # test_kernels.cpp:160-166
    assert s[0, 0, 0] == 1.0
    s, _, _ = oracle.sparse_inverse_subset(np.array([[[2.0]]]))
    assert s[0, 0, 0] == 0.25
    l = np.array([[[1.0, 1.0], [1.0, 0.0]]])  # SPEC.md: L=[[1,0],[1,1]] -> [[2,-1],[-1,1]]
    s, _, _ = oracle.sparse_inverse_subset(l)
    assert np.allclose(s[0], [[2.0, -1.0], [1.0, 0.0]])


def test_log_det_nonpositive_row(oracle):
    l = np.array([[[1.0], [-2.0]]])  # test_kernels.cpp:237-245
    _, st, row = oracle.log_det(l)
    assert st[0] == 3 and row[0] == 1


def test_scalar_adjoints(oracle):
    # SPEC.md: Q=[4], L=[2], l_bar=[1] -> q_bar=0.25; subset adjoint L=[1], s_bar=[1] -> -2
    assert oracle.vjp_cholesky(np.array([[[2.0]]]), np.array([[[1.0]]]))[0, 0, 0] == 0.25
    lb, _, _ = oracle.vjp_sparse_inverse_subset(np.array([[[1.0]]]), np.array([[[1.0]]]), np.array([[[1.0]]]))
    assert lb[0, 0, 0] == -2.0


# ------------------------------------------------ dense identities (restatement)
def _dense(a, lo, up):
    B, n, w = a.shape
    d = np.zeros((B, n, n))
    for r in range(w):
        off = r - up
        for j in range(n):
            i = j + off
            if 0 <= i < n:
                d[:, i, j] = a[:, j, r]
    return d


def test_dense_agreement(oracle):
    rng = np.random.default_rng(21)
    for _ in range(20):
        n = int(rng.integers(1, 40))
        bw = int(min(rng.integers(0, 6), n - 1))
        q = cm.random_spd_band(rng, 2, n, bw)
        qd = _dense(q, bw, 0)
        qd = qd + np.transpose(qd, (0, 2, 1)) - np.eye(n) * qd
        l, st, _ = oracle.cholesky(q)
        assert np.all(st == 0)
        assert cm.max_rel_err(_dense(l, bw, 0), np.linalg.cholesky(qd)) < 1e-12
        s, _, _ = oracle.sparse_inverse_subset(l)
        inv = np.linalg.inv(qd)
        sd = _dense(s, bw, 0)
        mask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) <= bw
        lower = np.tril(mask)
        assert cm.max_rel_err(sd[:, lower], inv[:, lower]) < 1e-9
        v = cm.random_vec(rng, 2, n)
        x, _, _ = oracle.solve_vec(l, v, False)
        assert cm.max_rel_err(x, np.linalg.solve(_dense(l, bw, 0), v[..., None])[..., 0]) < 1e-9
