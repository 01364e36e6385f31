"""The analytic reverse of the state-space prior assembly
(bgm_vjp_prior_natural_params): torch.autograd.gradcheck of the
prior_natural_params Function, and equivalence with the reference's
finite-difference hyperparameter gradient compose_precision_gradient
(inference.cpp:360-380), restated here, for Matern state-space models
parametrised by (log variance, log lengthscale)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _random_models(rng, B, T, d):
    a = rng.normal(0, 0.4, (B, T, d, d))
    b = rng.normal(0, 1, (B, T, d))
    g = rng.normal(0, 1, (B, T, d, d))
    q = np.einsum("btij,btkj->btik", g, g) + d * np.eye(d)
    mu0 = rng.normal(0, 1, (B, d))
    h = rng.normal(0, 1, (B, d, d))
    s0 = np.einsum("bij,bkj->bik", h, h) + d * np.eye(d)
    return a, b, q, mu0, s0


@pytest.mark.parametrize("tile", [1, 32])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_gradcheck_prior_natural_params(cuda, tile, d):
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(10 * d + tile)
    B, T = 3, 4
    dev = torch.device("cuda")
    xs = [torch.tensor(x, dtype=torch.float64, device=dev, requires_grad=True) for x in _random_models(rng, B, T, d)]

    def f(a, b, q, mu0, s0):
        lam, eta = ag.prior_natural_params(a, b, q, mu0, s0, tile=tile)
        return lam, eta

    assert torch.autograd.gradcheck(f, tuple(xs), eps=1e-6, atol=1e-6, rtol=1e-5)


def _matern32_torch(times, log_var, log_len):
    """models.cpp:84-122 in torch (differentiable in the hyperparameters)."""
    var, ell = torch.exp(log_var), torch.exp(log_len)
    T = len(times)
    s = np.sqrt(3.0) / ell
    p_inf = torch.diag(torch.stack([var, s * s * var]))
    a = [torch.zeros(2, 2, dtype=torch.float64, device=var.device)]
    q = [p_inf]
    for t in range(1, T):
        dt = float(times[t] - times[t - 1])
        dec = torch.exp(-s * dt)
        at = torch.stack([torch.stack([dec * (1 + s * dt), dec * dt]),
                          torch.stack([-dec * s * s * dt, dec * (1 - s * dt)])])
        a.append(at)
        q.append(p_inf - at @ p_inf @ at.T)
    z = torch.zeros(T, 2, dtype=torch.float64, device=var.device)
    return torch.stack(a)[None], z[None], torch.stack(q)[None], torch.zeros(1, 2, dtype=torch.float64,
                                                                              device=var.device), p_inf[None]


@pytest.mark.parametrize("tile", [1, 32])
def test_matches_compose_precision_gradient(cuda, tile):
    """theta_bar_j = sum over stored cells of Q_bar * (Q(theta + eps e_j) -
    Q(theta - eps e_j)) / (2 eps) (inference.cpp:360-380) against autograd
    through the analytic VJP, for theta = (log variance, log lengthscale)."""
    import paper_1902_10078_b200 as bgm
    from paper_1902_10078_b200 import autograd as ag
    rng = np.random.default_rng(3 + tile)
    dev = torch.device("cuda")
    times = np.cumsum(rng.uniform(0.05, 0.6, 40))
    theta = torch.tensor([np.log(1.7), np.log(0.8)], dtype=torch.float64, device=dev, requires_grad=True)
    lam, _ = ag.prior_natural_params(*_matern32_torch(times, theta[0], theta[1]), tile=tile)
    from tests import common as cm
    n = 2 * (len(times) + 1)  # (T + 1) d, d = 2; the band has 2d - 1 = 3 sub-diagonals
    qbar_ref = cm.zero_corners(rng.normal(0, 1, (1, n, 4)), 3, 0)  # cotangent on the stored cells
    qbar = bgm.Bands.from_reference(qbar_ref, 3, 0, tile=tile).data
    (lam * qbar).sum().backward()
    got = theta.grad.cpu().numpy()

    def assemble(th):
        with torch.no_grad():
            L, _ = bgm.prior_natural_params(*_matern32_torch(times, th[0], th[1]), tile=1)
        return L.data.cpu().numpy()

    eps = 1e-6
    want = np.zeros(2)
    th0 = theta.detach()
    for j in range(2):
        e = torch.zeros(2, dtype=torch.float64, device=dev)
        e[j] = eps
        want[j] = np.sum(qbar_ref * (assemble(th0 + e) - assemble(th0 - e))) / (2 * eps)
    assert np.allclose(got, want, rtol=1e-6, atol=1e-8), (got, want)
