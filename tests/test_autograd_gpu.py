"""torch.autograd over the operator suite (paper_1902_10078_b200.autograd):
torch.autograd.gradcheck of every wrapped forward/VJP pair in fp64 (finite
differences over the stored cells, the reference's gradcheck convention,
gradcheck.cpp:117-126), and a composite config-3-style objective built from
the wrapped ops checked against the fused step's L-bar (inference.cpp:140-163)."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = pytest.mark.gpu


def _band(rng, B, n, lo, up, diag=None, tile=1):
    import paper_1902_10078_b200 as bgm
    a = cm.random_band(rng, B, n, lo, up)
    if diag is not None:
        a[:, :, up] = rng.uniform(*diag, (B, n))
    return bgm.Bands.from_reference(a, lo, up, tile=tile)


def _vec(rng, B, n, tile=1):
    import paper_1902_10078_b200 as bgm
    return bgm.Vecs.from_reference(cm.random_vec(rng, B, n), tile=tile)


def _req(x):
    x.data.requires_grad_(True)
    return x


def _check(fn, *inputs, atol=1e-8, rtol=1e-6):
    assert torch.autograd.gradcheck(fn, inputs, eps=1e-6, atol=atol, rtol=rtol)


def test_gradcheck_cholesky_logdet_subset(cuda, oracle):
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(1)
    B, n, k = 2, 11, 2
    L0 = cm.config_factor(rng, B, n, k)
    q = bgm.Bands.from_reference(cm.precision(oracle, L0, k), k, 0, tile=1)

    def f(qd):
        Q = bgm.Bands(qd, B, n, k, 0, 1)
        L = ag.cholesky(Q)
        return ag.log_det_from_cholesky(L), ag.sparse_inverse_subset(L).data, L.data

    _check(f, q.data.clone().requires_grad_(True))


def test_gradcheck_solves(cuda):
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(2)
    B, n, k = 2, 10, 3
    L = _band(rng, B, n, k, 0, diag=(1.0, 2.0))
    v = _vec(rng, B, n)
    R = _band(rng, B, n, 1, 2)

    def f(ld, vd, rd):
        Lb = bgm.Bands(ld, B, n, k, 0, 1)
        x = ag.solve_vec(Lb, bgm.Vecs(vd, B, n, 1), False)
        xt = ag.solve_vec(Lb, x, True)
        s = ag.solve_mat(Lb, bgm.Bands(rd, B, n, 1, 2, 1), 4, 2, False)
        return xt.data, s.data

    _check(f, L.data.clone().requires_grad_(True), v.data.clone().requires_grad_(True),
           R.data.clone().requires_grad_(True))


def test_gradcheck_products(cuda):
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(3)
    B, n = 2, 9
    a, b = _band(rng, B, n, 2, 1), _band(rng, B, n, 1, 3)
    m, v = _vec(rng, B, n), _vec(rng, B, n)

    def f(ad, bd, md, vd):
        A, Bm = bgm.Bands(ad, B, n, 2, 1, 1), bgm.Bands(bd, B, n, 1, 3, 1)
        M, V = bgm.Vecs(md, B, n, 1), bgm.Vecs(vd, B, n, 1)
        c = ag.product_band_band(A, Bm)
        cr = ag.product_band_band(A, Bm, 1, 2)
        y = ag.product_band_vec(A, V, False)
        yt = ag.product_band_vec(Bm, M, True)
        o = ag.outer_band(M, V, 2, 1)
        return c.data, cr.data, y.data, yt.data, o.data

    _check(f, *(x.data.clone().requires_grad_(True) for x in (a, b, m, v)))


def test_gradcheck_marginal_likelihood(cuda):
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(4)
    B, n, k = 2, 40, 2
    L = bgm.Bands.from_reference(cm.config_factor(rng, B, n, k), k, 0, tile=1)
    y = _vec(rng, B, n)
    tau2 = torch.tensor(0.05, dtype=torch.float64, device=L.data.device)

    def f(ld, t):
        return ag.marginal_likelihood(bgm.Bands(ld, B, n, k, 0, 1), y, t)

    # the loss is O(n / tau2) ~ 1e3: central differences carry ~1e-7 of rounding
    _check(f, L.data.clone().requires_grad_(True), tau2.clone().requires_grad_(True), atol=1e-6, rtol=1e-6)


def test_composite_objective_matches_fused_step_tile32(cuda):
    """The reference composition of config 3 written with the wrapped ops
    (Q = band(L L^T), chol(Q + tau^-2 I), chol(Q), solve, log-dets) and
    differentiated by torch autograd equals the fused step's loss and L-bar,
    over a partial 32-matrix tile (B = 5)."""
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(5)
    B, n, k, tau2 = 5, 300, 4, 0.01
    L0 = cm.config_factor(rng, B, n, k)
    yv = rng.normal(0, 1, (B, n))
    L = bgm.Bands.from_reference(L0, k, 0, tile=32)
    y = bgm.Vecs.from_reference(yv, tile=32)
    L.data.requires_grad_(True)
    # Q = band(L L^T) restricted to the lower band (inference.cpp:23-26); the
    # transpose is a materialized, differentiable copy of the stored cells
    Lt = _transpose(L)
    Q = ag.product_band_band(L, Lt, k, 0)
    shift = bgm.Bands.zeros(B, n, k, 0, tile=32)
    shift.data[:, :, 0, :] = 1.0 / tau2
    A = bgm.Bands(Q.data + shift.data, B, n, k, 0, 32)
    Lp, Lq = ag.cholesky(A), ag.cholesky(Q)
    w = ag.solve_vec(Lp, y, False)
    yy = (y.data * y.data).sum(dim=1)
    ww = (w.data * w.data).sum(dim=1)
    lane = lambda t: t.reshape(-1)[:B]  # noqa: E731  ((tiles, 32) -> the B real matrices)
    loss = (-0.5 * n * np.log(2 * np.pi) - ag.log_det_from_cholesky(Lp) + ag.log_det_from_cholesky(Lq)
            - 0.5 * n * np.log(tau2) - 0.5 * lane(yy) / tau2 + 0.5 * lane(ww) / tau2 ** 2)
    loss.sum().backward()
    f_loss, f_lbar, _ = bgm.marginal_likelihood_grad(bgm.Bands(L.data.detach(), B, n, k, 0, 32), y, tau2)
    got = bgm.Bands(L.data.grad, B, n, k, 0, 32).numpy()
    assert cm.max_rel_err(loss.detach().cpu().numpy(), f_loss.cpu().numpy()) <= 1e-9
    assert np.linalg.norm(got - f_lbar.numpy()) <= 1e-9 * np.linalg.norm(f_lbar.numpy())


def _transpose(L):
    """Differentiable materialized transpose (banded.cpp:159-167): the
    transpose's stored cells are a permutation of L's."""
    import paper_1902_10078_b200 as bgm

    class _T(torch.autograd.Function):
        @staticmethod
        def forward(ctx, d):
            return bgm.Bands(d, L.batch, L.n, L.lower, L.upper, L.tile).transpose().data

        @staticmethod
        def backward(ctx, g):
            return bgm.Bands(g.contiguous(), L.batch, L.n, L.upper, L.lower, L.tile).transpose().data

    return bgm.Bands(_T.apply(L.data), L.batch, L.n, L.upper, L.lower, L.tile)


# ------------------------------------------------------------------ vs the reference tape
# The autograd compositions against the reference's own compiled Tape
# (oracle/_ref: proj/src/tape.cpp compiled verbatim; the config-3 node graph of
# inference.cpp:140-163 and the KL of inference.cpp:247-268 built on it by
# oracle/ref_capi.cpp), not against the GPU's own finite differences.
def _config3_composite(L, y, tau2, B, n, k, tile):
    """The reference's config-3 composition written with the autograd wrappers:
    Q = band(L L^T), chol(Q + tau^-2 I), chol(Q), solve, two log-dets."""
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    Lt = _transpose(L)
    Q = ag.product_band_band(L, Lt, k, 0)
    shift = bgm.Bands.zeros(B, n, k, 0, tile=tile)
    if tile == 32:
        shift.data[:, :, 0, :] = 1.0 / tau2
    else:
        shift.data[:, :, 0] = 1.0 / tau2
    A = bgm.Bands(Q.data + shift.data, B, n, k, 0, tile)
    Lp, Lq = ag.cholesky(A), ag.cholesky(Q)
    w = ag.solve_vec(Lp, y, False)
    yy = y.data * y.data
    ww = w.data * w.data
    if tile == 32:
        lane = lambda t: t.sum(dim=1).reshape(-1)[:B]  # noqa: E731
    else:
        lane = lambda t: t.sum(dim=1)  # noqa: E731
    return (-0.5 * n * np.log(2 * np.pi) - ag.log_det_from_cholesky(Lp) + ag.log_det_from_cholesky(Lq)
            - 0.5 * n * np.log(tau2) - 0.5 * lane(yy) / tau2 + 0.5 * lane(ww) / tau2 ** 2)


@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("B,n,k", [(3, 200, 2), (5, 300, 4), (2, 257, 16)])
def test_composite_autograd_vs_reference_tape(cuda, reference, tile, B, n, k):
    """torch autograd through the wrapped operators reproduces the reference
    tape's loss and dL (tape.cpp:435-451 backward) at 1e-9."""
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(1000 + 10 * k + tile)
    tau2 = 0.01
    L0 = cm.config_factor(rng, B, n, k)
    yv = rng.normal(0, 1, (B, n))
    rl, rlb, _, st, _ = reference.marginal_likelihood_grad(L0, yv, tau2)
    assert np.all(st == 0)
    L = bgm.Bands.from_reference(L0, k, 0, tile=tile)
    y = bgm.Vecs.from_reference(yv, tile=tile)
    L.data.requires_grad_(True)
    loss = _config3_composite(L, y, tau2, B, n, k, tile)
    loss.sum().backward()
    got = bgm.Bands(L.data.grad, B, n, k, 0, tile).numpy()
    assert cm.max_rel_err(loss.detach().cpu().numpy(), rl) <= 1e-9
    assert cm.max_rel_err(got, rlb, floor_scale=1e-6) <= 1e-9
    assert np.linalg.norm(got - rlb) <= 1e-10 * np.linalg.norm(rlb)


@pytest.mark.parametrize("tile", [1, 32])
def test_fused_autograd_vs_reference_tape(cuda, reference, tile):
    """ag.marginal_likelihood (the fused step as a torch Function) under an
    upstream cotangent: dL and d tau2 equal the reference tape's, scaled."""
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(77 + tile)
    B, n, k, tau2 = 6, 700, 16, 0.01
    L0 = cm.config_factor(rng, B, n, k)
    yv = rng.normal(0, 1, (B, n))
    rl, rlb, rtb, st, _ = reference.marginal_likelihood_grad(L0, yv, tau2)
    assert np.all(st == 0)
    L = bgm.Bands.from_reference(L0, k, 0, tile=tile)
    y = bgm.Vecs.from_reference(yv, tile=tile)
    L.data.requires_grad_(True)
    t = torch.tensor(tau2, dtype=torch.float64, device=L.data.device, requires_grad=True)
    cot = torch.as_tensor(rng.normal(0, 1, B), device=L.data.device)
    loss = ag.marginal_likelihood(L, y, t)
    (loss * cot).sum().backward()
    got = bgm.Bands(L.data.grad, B, n, k, 0, tile).numpy()
    c = cot.cpu().numpy()
    assert cm.max_rel_err(loss.detach().cpu().numpy(), rl) <= 1e-9
    want = rlb * c[:, None, None]
    assert cm.max_rel_err(got, want, floor_scale=1e-6) <= 1e-9
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    # d tau2 sums cancelling ~n y'y / tau2^2 terms: judged against them
    summ = np.abs(c) @ (n / (2 * tau2) + (yv * yv).sum(axis=1) / (2 * tau2 ** 2))
    assert abs(float(t.grad) - float(c @ rtb)) <= 1e-12 * summ


@pytest.mark.parametrize("tile", [1, 32])
def test_kl_autograd_vs_reference_tape(cuda, reference, tile):
    """ag.kl_divergence under a cotangent: d m_q and d L_q equal the
    reference tape's KL gradient (inference.cpp:247-268), scaled."""
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(5 + tile)
    B, n, kq, kp = 9, 300, 4, 2
    lq0 = cm.config_factor(rng, B, n, kq)
    lp0 = cm.config_factor(rng, B, n, kp)
    mq0, mp0 = rng.normal(0, 1, (B, n)), rng.normal(0, 1, (B, n))
    rkl, rmb, rlb, st, _ = reference.kl_divergence_grad(mq0, lq0, mp0, lp0)
    assert np.all(st == 0)
    mq = bgm.Vecs.from_reference(mq0, tile=tile)
    lq = bgm.Bands.from_reference(lq0, kq, 0, tile=tile)
    mp = bgm.Vecs.from_reference(mp0, tile=tile)
    lp = bgm.Bands.from_reference(lp0, kp, 0, tile=tile)
    mq.data.requires_grad_(True)
    lq.data.requires_grad_(True)
    cot = torch.as_tensor(rng.normal(0, 1, B), device=mq.data.device)
    kl = ag.kl_divergence(mq, lq, mp, lp)
    (kl * cot).sum().backward()
    c = cot.cpu().numpy()
    gm = bgm.Vecs(mq.data.grad, B, n, tile).numpy()
    gl = bgm.Bands(lq.data.grad, B, n, kq, 0, tile).numpy()
    assert cm.max_rel_err(kl.detach().cpu().numpy(), rkl) <= 1e-9
    assert cm.max_rel_err(gm, rmb * c[:, None]) <= 1e-9
    assert cm.max_rel_err(gl, rlb * c[:, None, None]) <= 1e-9
