"""Batched state-space prior assembly on the device (bgm_prior_natural_params,
models.cpp:165-189), pinned the way the reference's own model tests pin it
(test_models.cpp:67-130): known answers of the exponential-kernel model, and
the inverse of the joint prior precision reproducing the Matern-1/2 and
Matern-3/2 kernel grams; plus random batched models against a dense numpy
restatement of models.cpp:165-189, and the SingularBlock order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def matern12_ssm(times, variance, lengthscale):
    """models.cpp:58-82 restated (state-space form of the exponential kernel)."""
    T = len(times)
    a = np.zeros((T, 1, 1))
    q = np.full((T, 1, 1), variance)
    for t in range(1, T):
        phi = np.exp(-(times[t] - times[t - 1]) / lengthscale)
        a[t, 0, 0] = phi
        q[t, 0, 0] = variance * (1.0 - phi * phi)
    return a, np.zeros((T, 1)), q, np.zeros(1), np.full((1, 1), variance)


def matern32_ssm(times, variance, lengthscale):
    """models.cpp:84-122 restated."""
    T = len(times)
    s = np.sqrt(3.0) / lengthscale
    p_inf = np.diag([variance, s * s * variance])
    a = np.zeros((T, 2, 2))
    q = np.tile(p_inf, (T, 1, 1))
    for t in range(1, T):
        dt = times[t] - times[t - 1]
        dec = np.exp(-s * dt)
        at = np.array([[dec * (1 + s * dt), dec * dt], [-dec * s * s * dt, dec * (1 - s * dt)]])
        a[t] = at
        q[t] = p_inf - at @ p_inf @ at.T
    return a, np.zeros((T, 2)), q, np.zeros(2), p_inf


def _assemble(models, tile=32):
    import paper_1902_10078_b200 as bgm
    a, b, q, mu0, s0 = (np.stack([m[i] for m in models]) for i in range(5))
    return bgm.prior_natural_params(a, b, q, mu0, s0, tile=tile)


def _dense_sym(lam_np, n):
    """(n, w) lower store of one matrix -> dense symmetric."""
    w = lam_np.shape[1]
    D = np.zeros((n, n))
    for j in range(n):
        for r in range(w):
            if j + r < n:
                D[j + r, j] = D[j, j + r] = lam_np[j, r]
    return D


def _gram(lam_dense, T, d):
    cov = np.linalg.inv(lam_dense)
    return np.array([[cov[s * d, t * d] for t in range(1, T + 1)] for s in range(1, T + 1)])


def _times(rng, n):
    return np.cumsum(rng.uniform(0.05, 0.6, n))


@pytest.mark.parametrize("tile", [1, 32])
def test_exponential_known_answers(cuda, tile):
    lam, eta = _assemble([matern12_ssm(np.array([3.7]), 2.0, 0.8)], tile)  # test_models.cpp:68-80
    L = lam.numpy()[0]
    assert lam.n == 2 and lam.lower == 1
    assert abs(L[0, 0] - 0.5) < 1e-14 and abs(L[1, 0] - 0.5) < 1e-14 and L[0, 1] == 0.0
    assert np.all(eta.numpy() == 0.0)
    lam, _ = _assemble([matern12_ssm(np.array([0.0, 1e5, 2e5]), 1.5, 1.0)], tile)  # :82-89
    L = lam.numpy()[0]
    assert np.all(L[:3, 1] == 0.0)
    assert np.max(np.abs(L[:, 0] - 1.0 / 1.5)) < 1e-14


@pytest.mark.parametrize("tile", [1, 32])
def test_prior_inverts_to_kernel_grams(cuda, tile):
    rng = np.random.default_rng(101)
    t12, t32 = _times(rng, 40), _times(rng, 30)
    k12 = lambda r: 1.7 * np.exp(-r / 0.9)  # noqa: E731
    s = np.sqrt(3.0) / 1.1
    k32 = lambda r: 1.3 * (1 + s * r) * np.exp(-s * r)  # noqa: E731
    for ssm, times, kern, d in ((matern12_ssm(t12, 1.7, 0.9), t12, k12, 1), (matern32_ssm(t32, 1.3, 1.1), t32, k32, 2)):
        lam, _ = _assemble([ssm, ssm], tile)
        T = len(times)
        assert lam.lower == 2 * d - 1
        for L in lam.numpy():
            g = _gram(_dense_sym(L, (T + 1) * d), T, d)
            want = kern(np.abs(times[:, None] - times[None, :]))
            assert np.max(np.abs(g - want) / np.abs(want)) < 1e-8  # test_models.cpp:98-102


def _restated(a, b, q, mu0, s0):
    """models.cpp:165-189 in dense numpy."""
    T, d, _ = a.shape
    n = (T + 1) * d
    lam = np.zeros((n, n))
    qinv = [np.linalg.inv(q[t]) for t in range(T)]
    lam[:d, :d] += np.linalg.inv(s0) + a[0].T @ qinv[0] @ a[0]
    for t in range(1, T + 1):
        blk = qinv[t - 1] + (a[t].T @ qinv[t] @ a[t] if t < T else 0)
        lam[t * d:(t + 1) * d, t * d:(t + 1) * d] += blk
        sub = -qinv[t - 1] @ a[t - 1]
        lam[t * d:(t + 1) * d, (t - 1) * d:t * d] += sub
        lam[(t - 1) * d:t * d, t * d:(t + 1) * d] += sub.T
    m = np.zeros(n)
    m[:d] = mu0
    for t in range(1, T + 1):
        m[t * d:(t + 1) * d] = a[t - 1] @ m[(t - 1) * d:t * d] + b[t - 1]
    return lam, lam @ m, np.abs(lam) @ np.abs(m)


@pytest.mark.parametrize("d", [1, 3, 8])
def test_random_batch_vs_restatement(cuda, d):
    rng = np.random.default_rng(7 + d)
    B, T = 37, 25
    a = rng.normal(0, 0.5, (B, T, d, d))
    b = rng.normal(0, 1, (B, T, d))
    x = rng.normal(0, 1, (B, T, d, d))
    q = x @ np.swapaxes(x, -1, -2) + d * np.eye(d)
    mu0 = rng.normal(0, 1, (B, d))
    y = rng.normal(0, 1, (B, d, d))
    s0 = y @ np.swapaxes(y, -1, -2) + d * np.eye(d)
    import paper_1902_10078_b200 as bgm
    lam, eta = bgm.prior_natural_params(a, b, q, mu0, s0)
    L, E = lam.numpy(), eta.numpy()
    n = (T + 1) * d
    for i in range(B):
        want, weta, scale = _restated(a[i], b[i], q[i], mu0[i], s0[i])
        got = _dense_sym(L[i], n)
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
        # eta = Lambda m cancels (the propagated mean grows with T): compared
        # relative to |Lambda| |m|, the accuracy of any fp64 dot-product order
        assert np.all(np.abs(E[i] - weta) <= 1e-12 * scale)


def test_singular_block_order(cuda):
    import paper_1902_10078_b200 as bgm
    rng = np.random.default_rng(3)
    B, T, d = 3, 6, 2
    a = rng.normal(0, 0.5, (B, T, d, d))
    b = np.zeros((B, T, d))
    q = np.tile(np.eye(d), (B, T, 1, 1))
    s0 = np.tile(np.eye(d), (B, 1, 1))
    q[1, 4] = -np.eye(d)  # Q_4 of model 1 -> SingularBlock(5)
    q[1, 2] = -np.eye(d)  # ... but Q_2 comes first: SingularBlock(3)
    s0[2] = -np.eye(d)    # model 2: only Sigma0 -> SingularBlock(0)
    with pytest.raises(bgm.SingularBlock) as e:
        bgm.prior_natural_params(a, b, q, np.zeros((B, d)), s0)
    assert e.value.matrix == 1 and e.value.row == 3
    _, _ = bgm.prior_natural_params(a[2:], b[2:], q[2:], np.zeros((1, d)), s0[2:], check=False)
    with pytest.raises(bgm.SingularBlock) as e:
        bgm.prior_natural_params(a[2:], b[2:], q[2:], np.zeros((1, d)), s0[2:])
    assert e.value.row == 0
