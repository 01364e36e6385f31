"""Seeded generators, layout helpers and the reference's comparison metric.

Band arrays use the reference storage layout batch-major: a[b, j, r] is
storage row r (= i - j + upper) of column j (banded.hpp:1-11)."""
from __future__ import annotations

import numpy as np


def zero_corners(a: np.ndarray, lower: int, upper: int) -> np.ndarray:
    B, n, w = a.shape
    for r in range(w):
        i_off = r - upper  # i = j + i_off
        if i_off < 0:
            a[:, : min(-i_off, n), r] = 0.0
        elif i_off > 0:
            a[:, max(n - i_off, 0):, r] = 0.0
    return a


def random_band(rng, B, n, lower, upper, dist="uniform"):
    """gradcheck.cpp:12-21 shape (U(-1,1)); dist='normal' for config 2."""
    w = lower + upper + 1
    a = rng.uniform(-1, 1, (B, n, w)) if dist == "uniform" else rng.normal(0, 1, (B, n, w))
    return zero_corners(a, lower, upper)


def random_vec(rng, B, n, dist="uniform"):
    return rng.uniform(-1, 1, (B, n)) if dist == "uniform" else rng.normal(0, 1, (B, n))


def random_cholesky_factor(rng, B, n, bw):
    """gradcheck.cpp:40-49: diag U(0.6,1.6), off-diagonals U(-0.5,0.5)."""
    l = np.empty((B, n, bw + 1))
    l[:, :, 0] = rng.uniform(0.6, 1.6, (B, n))
    l[:, :, 1:] = rng.uniform(-0.5, 0.5, (B, n, bw))
    return zero_corners(l, bw, 0)


def random_spd_band(rng, B, n, bw):
    """gradcheck.cpp:23-38: U(-1,1) off-diagonals, diagonally dominant diagonal."""
    q = np.zeros((B, n, bw + 1))
    q[:, :, 1:] = rng.uniform(-1, 1, (B, n, bw))
    zero_corners(q, bw, 0)
    row = np.zeros((B, n))
    for r in range(1, bw + 1):
        row[:, : n - r] += np.abs(q[:, : n - r, r])  # entries (j+r, j) feed rows j and j+r
        row[:, r:] += np.abs(q[:, : n - r, r])
    q[:, :, 0] = row + rng.uniform(0.5, 1.5, (B, n))
    return q


def config_factor(rng, B, n, k, off_std=0.1):
    """BASELINE.md §4 "as in config 0": diag ~U[1,2], off-diagonals ~N(0, off_std^2)."""
    l = np.empty((B, n, k + 1))
    l[:, :, 0] = rng.uniform(1.0, 2.0, (B, n))
    l[:, :, 1:] = rng.normal(0.0, off_std, (B, n, k))
    return zero_corners(l, k, 0)


def transpose_ref(a: np.ndarray, lower: int, upper: int) -> np.ndarray:
    """banded.cpp:159-167 on reference-layout arrays; result has (upper, lower)."""
    B, n, w = a.shape
    t = np.zeros_like(a)
    for r in range(w):
        d = r - upper  # i - j
        rt = -d + lower  # storage row of (j, i) in the transposed band (upper'=lower)
        if d >= 0:
            t[:, d:, rt] = a[:, : n - d, r] if d < n else 0
        else:
            t[:, : n + d, rt] = a[:, -d:, r] if -d < n else 0
    return zero_corners(t, upper, lower)


def precision(orc, L, k):
    """Q = band(L L^T) as a symmetric lower store (inference.cpp:23-26)."""
    q, _, _ = orc.product_band_band(L, k, 0, transpose_ref(L, k, 0), 0, k, k, 0)
    return q


def max_rel_err(a, b, floor_scale=1e-12):
    """test_util.hpp:19-21 metric |a-b|/max(|a|,|b|,floor), floor = 1e-12 max|b|."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    floor = max(floor_scale * float(np.max(np.abs(b))), 1e-300)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / den))
