"""Extended-precision (x87 long double, 64-bit mantissa) evaluation of the
config-3 quantities along the banded route -- an accuracy yardstick for both
the reference oracle and the CUDA kernels (tests only).

Same mathematics as bgm_mlik.cu's header: A = band(L L^T) + I/tau2 = Lp Lp^T,
w = Lp^-1 y, S = band(A^-1) (Takahashi), u = Lp^-T w,
L_bar = -band_lower[(S + u u^T/tau2^2) L] + diag(1/L_ii).
"""
import numpy as np

LD = np.longdouble


def mlik_exact(L, y, tau2):
    L = np.asarray(L, dtype=LD)
    y = np.asarray(y, dtype=LD)
    B, n, w = L.shape
    k = w - 1
    s = LD(1) / LD(tau2)
    c4 = s * s

    def lat(M, i, j):  # lower band entry (i >= j) or 0, vectorised over batch
        if j < 0 or i >= n or i - j > k or i < j:
            return np.zeros(B, dtype=LD)
        return M[:, j, i - j]

    # A = band(L L^T) + s I, lower store
    A = np.zeros((B, n, w), dtype=LD)
    for j in range(n):
        for r in range(min(w, n - j)):
            i = j + r
            acc = np.zeros(B, dtype=LD)
            for m in range(max(0, i - k), j + 1):
                acc += lat(L, i, m) * lat(L, j, m)
            A[:, j, r] = acc + (s if r == 0 else 0)
    # Cholesky (kernels_serial.cpp:12-32 order)
    P = np.zeros_like(A)
    for i in range(n):
        j0 = max(0, i - k)
        for j in range(j0, i + 1):
            acc = np.zeros(B, dtype=LD)
            for m in range(j0, j):
                acc += P[:, m, i - m] * P[:, m, j - m]
            if i == j:
                P[:, i, 0] = np.sqrt(A[:, i, 0] - acc)
            else:
                P[:, j, i - j] = (A[:, j, i - j] - acc) / P[:, j, 0]
    wv = np.zeros((B, n), dtype=LD)
    for i in range(n):
        acc = np.zeros(B, dtype=LD)
        for m in range(max(0, i - k), i):
            acc += P[:, m, i - m] * wv[:, m]
        wv[:, i] = (y[:, i] - acc) / P[:, i, 0]
    u = np.zeros((B, n), dtype=LD)
    for i in range(n - 1, -1, -1):
        acc = np.zeros(B, dtype=LD)
        for m in range(i + 1, min(n, i + k + 1)):
            acc += P[:, i, m - i] * u[:, m]
        u[:, i] = (wv[:, i] - acc) / P[:, i, 0]
    # Takahashi (kernels_serial.cpp:80-104)
    S = np.zeros_like(A)

    def sym(i, j):
        return S[:, j, i - j] if i >= j else S[:, i, j - i]

    for j in range(n - 1, -1, -1):
        for i in range(j, max(0, j - k) - 1, -1):
            acc = np.zeros(B, dtype=LD)
            for m in range(i + 1, min(n, i + k + 1)):
                acc += (P[:, i, m - i] / P[:, i, 0]) * sym(m, j)
            val = -acc + ((LD(1) / (P[:, i, 0] ** 2)) if i == j else 0)
            S[:, i, j - i] = val
    lbar = np.zeros_like(A)
    for j in range(n):
        for r in range(min(w, n - j)):
            i = j + r
            acc = np.zeros(B, dtype=LD)
            for m in range(j, min(n, j + k + 1)):
                acc += (sym(i, m) if abs(i - m) <= k else 0) * L[:, j, m - j] + c4 * u[:, i] * u[:, m] * L[:, j, m - j]
            lbar[:, j, r] = -acc + ((LD(1) / L[:, j, 0]) if r == 0 else 0)
    yy = (y * y).sum(1)
    ww = (wv * wv).sum(1)
    uu = (u * u).sum(1)
    tr = S[:, :, 0].sum(1)
    ldp = np.log(P[:, :, 0]).sum(1)
    ldl = np.log(np.abs(L[:, :, 0])).sum(1)
    nn = LD(n)
    log2pi = LD("1.837877066409345483560659472811235279722794947275566825634")
    loss = -0.5 * nn * log2pi - ldp + ldl - 0.5 * nn * np.log(LD(tau2)) - 0.5 * yy * s + 0.5 * ww * c4
    tbar = -nn * 0.5 * s + 0.5 * yy * c4 + 0.5 * c4 * tr - ww * c4 * s + 0.5 * uu * c4 * c4
    return loss, lbar, tbar


def abs_rel(got, exact):
    """max |got - exact| / max |exact|."""
    got = np.asarray(got, dtype=LD)
    return float(np.max(np.abs(got - exact)) / np.max(np.abs(exact)))
