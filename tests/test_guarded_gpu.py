"""Operand bounds under guard pages (compute-sanitizer is closed on this GPU
pool; tests/guarded.py places every operand flush against an unmapped guard
region, after it or before it).  Each fast path runs on guarded copies of its
operands and must neither fault nor change its result.  Checked to bite: on a
build whose paired forward runs one pair row too far (the round-2 y over-read,
bgm_mlik_t1.cu pair_end) the fused-step cases fail with an illegal address."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = pytest.mark.gpu


def _guard(x, where):
    import paper_1902_10078_b200 as bgm
    from tests.guarded import guarded_like
    if isinstance(x, bgm.Bands):
        return bgm.Bands(guarded_like(x.data, where), x.batch, x.n, x.lower, x.upper, x.tile)
    return bgm.Vecs(guarded_like(x.data, where), x.batch, x.n, x.tile)


def _np(x):
    """The B real matrices in the reference layout, corner cells zeroed
    (padding lanes and corners are not results)."""
    import paper_1902_10078_b200 as bgm
    if isinstance(x, bgm.Bands):
        return cm.zero_corners(x.to_reference().detach().cpu().numpy(), x.lower, x.upper)
    if isinstance(x, bgm.Vecs):
        return x.to_reference().detach().cpu().numpy()
    return x.detach().cpu().numpy()


def _same(a, b):
    assert np.array_equal(_np(a), _np(b))


@pytest.mark.parametrize("where", ["tail", "head"])
@pytest.mark.parametrize("tile,k,B,n", [(32, 16, 32, 1000), (32, 16, 33, 4099), (32, 8, 8, 2001), (32, 4, 40, 777),
                                        (1, 16, 3, 2100)])
def test_fused_step_guarded(cuda, where, tile, k, B, n):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(B * n + k)
    L = bgm.Bands.from_reference(cm.config_factor(rng, B, n, k), k, 0, tile=tile)
    y = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)), tile=tile)
    want = bgm.marginal_likelihood_grad(L, y, 0.01)
    Lg, yg = _guard(L, where), _guard(y, where)
    from tests.guarded import guarded_like
    out = (guarded_like(want[0], where, False), bgm.Bands(guarded_like(want[1].data, where, False), B, n, k, 0, tile),
           guarded_like(want[2], where, False), bgm.api.new_status(B))
    got = bgm.marginal_likelihood_grad(Lg, yg, 0.01, out=out)
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        _same(a, b)


@pytest.mark.parametrize("where", ["tail", "head"])
@pytest.mark.parametrize("tile,k,B,n", [(32, 4, 33, 2000), (32, 16, 5, 3000), (32, 7, 3, 900), (1, 64, 2, 1200),
                                        (1, 5, 1, 2500)])
def test_factor_solve_subset_guarded(cuda, oracle, where, tile, k, B, n):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(k * 1000 + B)
    off = 0.1 if k <= 16 else 0.02 / k ** 0.5
    q = cm.precision(oracle, cm.config_factor(rng, B, n, k, off_std=off), k)
    Q = bgm.Bands.from_reference(q, k, 0, tile=tile)
    v = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)), tile=tile)
    lb = bgm.Bands.from_reference(cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0), k, 0, tile=tile)
    L = bgm.cholesky(Q)
    S = bgm.sparse_inverse_subset(L)
    want = [L, bgm.solve_vec(L, v), bgm.solve_vec(L, v, True), S, bgm.vjp_cholesky(L, lb),
            bgm.vjp_sparse_inverse_subset(L, S, lb)]
    Qg, vg, lbg = _guard(Q, where), _guard(v, where), _guard(lb, where)
    Lg = bgm.cholesky(Qg)
    Lgg = _guard(Lg, where)
    Sg = _guard(bgm.sparse_inverse_subset(Lgg), where)
    got = [Lg, bgm.solve_vec(Lgg, vg), bgm.solve_vec(Lgg, vg, True), Sg, bgm.vjp_cholesky(Lgg, lbg),
           bgm.vjp_sparse_inverse_subset(Lgg, Sg, lbg)]
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        _same(a, b)


@pytest.mark.parametrize("where", ["tail", "head"])
def test_products_guarded(cuda, where):
    """Staged TMA products (config-2 shapes) and band x vector, partial tile."""
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(7)
    B, n, k = 33, 3001, 8
    L = bgm.Bands.from_reference(cm.zero_corners(rng.normal(0, 1, (B, n, k + 1)), k, 0), k, 0)
    A = bgm.Bands.from_reference(cm.zero_corners(rng.normal(0, 1, (B, n, 17)), 8, 8), 8, 8)
    Bm = bgm.Bands.from_reference(cm.zero_corners(rng.normal(0, 1, (B, n, 7)), 3, 3), 3, 3)
    v = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)))
    P2b = bgm.Bands.from_reference(cm.zero_corners(rng.normal(0, 1, (B, n, 23)), 11, 11), 11, 11)
    pv = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)))

    def run(L, A, Bm, v, P2b, pv):
        return [bgm.product_band_band(L, bgm.T(L)), bgm.product_band_band(A, Bm), bgm.product_band_vec(A, v),
                *bgm.vjp_product_band_band(A, Bm, P2b), *bgm.vjp_product_band_vec(A, v, pv, False)]

    want = run(L, A, Bm, v, P2b, pv)
    got = run(*(_guard(x, where) for x in (L, A, Bm, v, P2b, pv)))
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        _same(a, b)


@pytest.mark.parametrize("where", ["tail", "head"])
@pytest.mark.parametrize("tile", [1, 32])
def test_generic_and_misc_guarded(cuda, oracle, where, tile):
    """The reference-loop kernels (forced, bgm_force_generic), solve_mat and
    outer_band on guarded operands."""
    import paper_1902_10078_b200 as bgm
    lib = bgm.library()
    rng = np.random.default_rng(11 + tile)
    B, n, k = 5, 300, 3
    q = cm.precision(oracle, cm.config_factor(rng, B, n, k), k)
    Q = bgm.Bands.from_reference(q, k, 0, tile=tile)
    v = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)), tile=tile)
    R = bgm.Bands.from_reference(cm.zero_corners(rng.normal(0, 1, (B, n, 4)), 1, 2), 1, 2, tile=tile)

    def run(Q, v, R):
        L = bgm.cholesky(Q)
        return [L, bgm.solve_vec(L, v, True), bgm.sparse_inverse_subset(L), bgm.solve_mat(L, R, 4, 2),
                bgm.outer_band(v, v, 2, 1), bgm.log_det_from_cholesky(L)]

    lib.bgm_force_generic(1)
    try:
        want = run(Q, v, R)
        got = run(*(_guard(x, where) for x in (Q, v, R)))
        torch.cuda.synchronize()
    finally:
        lib.bgm_force_generic(0)
    for a, b in zip(got, want):
        _same(a, b)


@pytest.mark.parametrize("where", ["tail", "head"])
def test_vi_objectives_guarded(cuda, where):
    """KL and both ELBOs (with a partial selection) on guarded operands."""
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(5)
    B, n, kq, kp = 33, 257, 4, 2
    mq = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)) * 0.3)
    lq = bgm.Bands.from_reference(cm.config_factor(rng, B, n, kq), kq, 0)
    mp = bgm.Vecs.from_reference(rng.normal(0, 1, (B, n)))
    lp = bgm.Bands.from_reference(cm.config_factor(rng, B, n, kp), kp, 0)
    y = bgm.Vecs.from_reference(rng.poisson(1.5, (B, n)).astype(np.float64))
    wt = bgm.Vecs.from_reference(rng.uniform(0.5, 2.0, (B, n)))
    obs = bgm.selection(np.arange(0, n, 3), B, n)

    def run(mq, lq, mp, lp, y, wt, obs):
        return [*bgm.kl_divergence_grad(mq, lq, mp, lp), *bgm.elbo_gaussian_grad(mq, lq, mp, lp, y, 0.5, observed=obs),
                *bgm.elbo_poisson_grad(mq, lq, mp, lp, y, wt, 20, observed=obs)]

    want = run(mq, lq, mp, lp, y, wt, obs)
    got = run(*(_guard(x, where) for x in (mq, lq, mp, lp, y, wt, obs)))
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        _same(a, b)
