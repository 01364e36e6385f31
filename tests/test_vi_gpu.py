"""VI objective on the device: trace_product_sym
(tape.cpp:274-302) and infer::kl_divergence (inference.cpp:247-268) with its
gradient, against the verbatim reference tape (oracle/_ref) and a numpy
restatement of the trace; both device layouts."""
import numpy as np
import pytest
import torch

from tests import common as cm

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _trace_np(a, b):
    """tape.cpp:279-284 on (B, n, w) lower stores."""
    B, n, wa = a.shape
    bw = min(wa, b.shape[2]) - 1
    out = np.zeros(B)
    for j in range(n):
        out += a[:, j, 0] * b[:, j, 0]
        for d in range(1, min(bw, n - 1 - j) + 1):
            out += 2.0 * a[:, j, d] * b[:, j, d]
    return out


@pytest.fixture(scope="module")
def ref():
    import oracle as orc
    if not orc.available("reference"):
        pytest.skip("verbatim reference oracle not built")
    return orc.Oracle("reference")


@pytest.mark.parametrize("tile", [1, 32])
def test_trace_product_sym(cuda, tile):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(7 + tile)
    B, n = 5, 613
    a, b = cm.random_band(rng, B, n, 4, 0), cm.random_band(rng, B, n, 2, 0)
    A, Bm = bgm.Bands.from_reference(a, 4, 0, tile=tile), bgm.Bands.from_reference(b, 2, 0, tile=tile)
    got = bgm.trace_product_sym(A, Bm).cpu().numpy()
    assert cm.max_rel_err(got, _trace_np(a, b)) <= TOL
    ab, bb = bgm.vjp_trace_product_sym(A, Bm, 0.5)
    want_a = np.zeros_like(a)
    want_a[:, :, 0] = 0.5 * b[:, :, 0]
    want_a[:, :, 1:3] = b[:, :, 1:3]  # 2 * 0.5 below the diagonal, within b's band
    want_b = 0.5 * a[:, :, :3].copy()
    want_b[:, :, 1:] *= 2.0
    assert cm.max_rel_err(ab.numpy(), cm.zero_corners(want_a, 4, 0)) <= TOL
    assert cm.max_rel_err(bb.numpy(), cm.zero_corners(want_b, 2, 0)) <= TOL


def _kl_inputs(rng, B, n, kq, kp):
    lq = cm.config_factor(rng, B, n, kq)
    lp = cm.config_factor(rng, B, n, kp)
    return rng.normal(0, 1, (B, n)), lq, rng.normal(0, 1, (B, n)), lp


@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("kq,kp", [(4, 2), (3, 3), (16, 8)])
def test_kl_divergence_vs_reference_tape(cuda, ref, tile, kq, kp):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(100 * kq + kp + tile)
    B, n = 37, 401
    mq, lq, mp, lp = _kl_inputs(rng, B, n, kq, kp)
    kl, mb, lb = bgm.kl_divergence_grad(bgm.Vecs.from_reference(mq, tile=tile), bgm.Bands.from_reference(lq, kq, 0, tile=tile),
                                        bgm.Vecs.from_reference(mp, tile=tile), bgm.Bands.from_reference(lp, kp, 0, tile=tile))
    rkl, rmb, rlb, st, _ = ref.kl_divergence_grad(mq, lq, mp, lp)
    assert np.all(st == 0)
    assert cm.max_rel_err(kl.cpu().numpy(), rkl) <= TOL
    assert cm.max_rel_err(mb.numpy(), rmb) <= TOL
    assert cm.max_rel_err(lb.numpy(), rlb) <= TOL


def test_kl_errors(cuda):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(3)
    B, n = 2, 50
    mq, lq, mp, lp = _kl_inputs(rng, B, n, 2, 4)
    with pytest.raises(bgm.DimensionMismatch):  # inference.cpp:252-253
        bgm.kl_divergence_grad(bgm.Vecs.from_reference(mq), bgm.Bands.from_reference(lq, 2, 0),
                               bgm.Vecs.from_reference(mp), bgm.Bands.from_reference(lp, 4, 0))
    mq, lq, mp, lp = _kl_inputs(rng, B, n, 4, 2)
    lp[1, 7, 0] = -1.0  # log|L_p| first: NonPositiveDiagonal at row 7 of matrix 1
    with pytest.raises(bgm.NonPositiveDiagonal) as e:
        bgm.kl_divergence_grad(bgm.Vecs.from_reference(mq), bgm.Bands.from_reference(lq, 4, 0),
                               bgm.Vecs.from_reference(mp), bgm.Bands.from_reference(lp, 2, 0))
    assert e.value.row == 7 and e.value.matrix == 1


def test_kl_autograd(cuda):
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(11)
    B, n, kq, kp = 2, 12, 2, 1
    mq, lq, mp, lp = _kl_inputs(rng, B, n, kq, kp)
    Mp, Lp = bgm.Vecs.from_reference(mp, tile=1), bgm.Bands.from_reference(lp, kp, 0, tile=1)
    Mq, Lq = bgm.Vecs.from_reference(mq, tile=1), bgm.Bands.from_reference(lq, kq, 0, tile=1)

    def f(md, ld):
        return ag.kl_divergence(bgm.Vecs(md, B, n, 1), bgm.Bands(ld, B, n, kq, 0, 1), Mp, Lp)

    assert torch.autograd.gradcheck(f, (Mq.data.clone().requires_grad_(True), Lq.data.clone().requires_grad_(True)),
                                    eps=1e-6, atol=1e-7, rtol=1e-6)


@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("kq,kp", [(4, 2), (16, 8)])
def test_elbo_gaussian_vs_reference_tape(cuda, ref, tile, kq, kp):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(7 * kq + kp + tile)
    B, n, tau2 = 37, 401, 0.3
    mq, lq, mp, lp = _kl_inputs(rng, B, n, kq, kp)
    y = rng.normal(0, 1, (B, n))
    V = lambda a: bgm.Vecs.from_reference(a, tile=tile)  # noqa: E731
    el, kl, mb, lb, tb = bgm.elbo_gaussian_grad(V(mq), bgm.Bands.from_reference(lq, kq, 0, tile=tile), V(mp),
                                                bgm.Bands.from_reference(lp, kp, 0, tile=tile), V(y), tau2)
    rel, rmb, rlb, rtb, st, _ = ref.elbo_gaussian_grad(mq, lq, mp, lp, y, tau2)
    assert np.all(st == 0)
    rkl = ref.kl_divergence_grad(mq, lq, mp, lp)[0]
    assert cm.max_rel_err(el.cpu().numpy(), rel) <= TOL
    assert cm.max_rel_err(kl.cpu().numpy(), rkl) <= TOL
    assert cm.max_rel_err(mb.numpy(), rmb) <= TOL
    assert cm.max_rel_err(lb.numpy(), rlb) <= TOL
    assert cm.max_rel_err(tb.cpu().numpy(), rtb) <= TOL


@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("quad", [1, 20])
def test_elbo_poisson_vs_reference_tape(cuda, ref, tile, quad):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(31 + tile + quad)
    B, n, kq, kp = 37, 257, 4, 2
    mq, lq, mp, lp = _kl_inputs(rng, B, n, kq, kp)
    mq *= 0.3
    y = rng.poisson(1.5, (B, n)).astype(np.float64)
    wt = rng.uniform(0.5, 2.0, (B, n))
    V = lambda a: bgm.Vecs.from_reference(a, tile=tile)  # noqa: E731
    el, kl, mb, lb = bgm.elbo_poisson_grad(V(mq), bgm.Bands.from_reference(lq, kq, 0, tile=tile), V(mp),
                                           bgm.Bands.from_reference(lp, kp, 0, tile=tile), V(y), V(wt), quad)
    rel, rmb, rlb, st, _ = ref.elbo_poisson_grad(mq, lq, mp, lp, y, wt, quad)
    assert np.all(st == 0)
    assert cm.max_rel_err(el.cpu().numpy(), rel) <= TOL
    assert cm.max_rel_err(mb.numpy(), rmb) <= TOL
    assert cm.max_rel_err(lb.numpy(), rlb) <= TOL
    wt[3, 10] = 0.0
    with pytest.raises(bgm.BandgmError, match="weight"):
        bgm.elbo_poisson_grad(V(mq), bgm.Bands.from_reference(lq, kq, 0, tile=tile), V(mp),
                              bgm.Bands.from_reference(lp, kp, 0, tile=tile), V(y), V(wt), quad)


# ---------------------------------------------------------------- partial SelectionIndex
@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("frac", [0.0, 0.3, 1.0])
def test_elbo_gaussian_partial_selection(cuda, ref, tile, frac):
    """models::SelectionIndex observing a subset of the latents
    (inference.cpp:45-63, 276-287): only observed latents enter the expected
    log-likelihood; the GPU mask path against the reference tape."""
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(int(100 * frac) + tile)
    B, n, kq, kp, tau2 = 9, 300, 4, 2, 0.3
    mq, lq, mp, lp = _kl_inputs(rng, B, n, kq, kp)
    idx = np.sort(rng.choice(n, int(frac * n), replace=False))
    y = rng.normal(0, 1, (B, n))  # scattered to full length; unobserved entries ignored
    obs = np.zeros((B, n))
    obs[:, idx] = 1.0
    V = lambda a: bgm.Vecs.from_reference(a, tile=tile)  # noqa: E731
    el, kl, mb, lb, tb = bgm.elbo_gaussian_grad(V(mq), bgm.Bands.from_reference(lq, kq, 0, tile=tile), V(mp),
                                                bgm.Bands.from_reference(lp, kp, 0, tile=tile), V(y), tau2,
                                                observed=bgm.selection(idx, B, n, tile=tile))
    rel, rmb, rlb, rtb, st, _ = ref.elbo_gaussian_grad(mq, lq, mp, lp, y, tau2, observed=obs)
    assert np.all(st == 0)
    assert cm.max_rel_err(el.cpu().numpy(), rel) <= TOL
    assert cm.max_rel_err(mb.numpy(), rmb) <= TOL
    assert cm.max_rel_err(lb.numpy(), rlb) <= TOL
    assert cm.max_rel_err(tb.cpu().numpy(), rtb) <= TOL


@pytest.mark.parametrize("tile", [1, 32])
def test_elbo_poisson_partial_selection(cuda, ref, tile):
    """Poisson with a partial selection: unobserved latents' weights are not
    vetted (the reference only reads weight(i) for i in the selection)."""
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(41 + tile)
    B, n, kq, kp, quad = 9, 257, 4, 2, 20
    mq, lq, mp, lp = _kl_inputs(rng, B, n, kq, kp)
    mq *= 0.3
    idx = np.sort(rng.choice(n, 100, replace=False))
    y = rng.poisson(1.5, (B, n)).astype(np.float64)
    wt = rng.uniform(0.5, 2.0, (B, n))
    unobs = np.setdiff1d(np.arange(n), idx)
    wt[:, unobs[:5]] = 0.0  # invalid weights at unobserved latents: ignored
    obs = np.zeros((B, n))
    obs[:, idx] = 1.0
    V = lambda a: bgm.Vecs.from_reference(a, tile=tile)  # noqa: E731
    el, kl, mb, lb = bgm.elbo_poisson_grad(V(mq), bgm.Bands.from_reference(lq, kq, 0, tile=tile), V(mp),
                                           bgm.Bands.from_reference(lp, kp, 0, tile=tile), V(y), V(wt), quad,
                                           observed=bgm.selection(idx, B, n, tile=tile))
    rel, rmb, rlb, st, _ = ref.elbo_poisson_grad(mq, lq, mp, lp, y, wt, quad, observed=obs)
    assert np.all(st == 0)
    assert cm.max_rel_err(el.cpu().numpy(), rel) <= TOL
    assert cm.max_rel_err(mb.numpy(), rmb) <= TOL
    assert cm.max_rel_err(lb.numpy(), rlb) <= TOL
