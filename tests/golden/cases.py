"""Golden cases: seeded small inputs for every hot-path operator.

``make_golden.py`` evaluates each case with the reference compiled verbatim
(oracle/_ref) and stores inputs + outputs in ``golden_v1.npz``.  The tests
re-evaluate the same cases with the C restatement (must match bit for bit)
and with the CUDA library (must match within the north-star tolerance).

Every case is a function ``case(impl, rng_inputs)`` that calls the oracle-style
numpy API (``oracle.Oracle`` or ``tests.gpu_adapter.GpuOracle``) and returns a
dict of named output arrays.  Inputs are drawn once, from a fixed seed, by
``inputs(name)``, so every implementation sees identical bytes.
"""
from __future__ import annotations

import zlib

import numpy as np

from tests import common as cm


def _q(orc, rng, B, n, k):
    L = cm.config_factor(rng, B, n, k)
    return cm.precision(orc, L, k)


def inputs(name: str):
    return np.random.default_rng(zlib.crc32(name.encode()))


# Each entry: name -> (shape params, builder).  Builders receive (impl, rng)
# and return {output_name: array}; the rng draws are identical for every impl
# because each builder draws all inputs before calling impl.

def case_cholesky(impl, rng, B=3, n=37, bw=3):
    q = cm.random_spd_band(rng, B, n, bw)
    l, st, row = impl.cholesky(q)
    return {"q": q, "l": l, "status": st}


def case_cholesky_cfg0(impl, rng):
    L = cm.config_factor(rng, 1, 1024, 2)
    q = cm.precision(impl, L, 2)
    l, st, row = impl.cholesky(q)
    return {"q": q, "l": l}


def case_solve_vec(impl, rng, B=3, n=45, bw=4):
    l = cm.random_cholesky_factor(rng, B, n, bw)
    v = cm.random_vec(rng, B, n)
    x, _, _ = impl.solve_vec(l, v, False)
    xt, _, _ = impl.solve_vec(l, v, True)
    return {"l": l, "v": v, "x": x, "xt": xt}


def case_log_det(impl, rng, B=3, n=25, bw=2):
    q = cm.random_spd_band(rng, B, n, bw)
    l, _, _ = impl.cholesky(q)
    ld, _, _ = impl.log_det(l)
    return {"l": l, "logdet": ld}


def case_subset(impl, rng, B=3, n=40, bw=5):
    q = cm.random_spd_band(rng, B, n, bw)
    l, _, _ = impl.cholesky(q)
    s, _, _ = impl.sparse_inverse_subset(l)
    return {"l": l, "s": s}


def case_products(impl, rng, B=2, n=33):
    out = {}
    for (al, au, bl, bu) in [(2, 1, 1, 2), (3, 0, 0, 3), (0, 0, 2, 2), (4, 4, 3, 3)]:
        a = cm.random_band(rng, B, n, al, au)
        b = cm.random_band(rng, B, n, bl, bu)
        c, ol, ou = impl.product_band_band(a, al, au, b, bl, bu)
        cr, _, _ = impl.product_band_band(a, al, au, b, bl, bu, 1, 2)
        tag = f"{al}{au}{bl}{bu}"
        out.update({f"a{tag}": a, f"b{tag}": b, f"c{tag}": c, f"cr{tag}": cr})
    return out


def case_band_vec(impl, rng, B=3, n=41, bl=2, bu=3):
    b = cm.random_band(rng, B, n, bl, bu)
    v = cm.random_vec(rng, B, n)
    return {"b": b, "v": v, "y": impl.product_band_vec(b, bl, bu, v, False),
            "yt": impl.product_band_vec(b, bl, bu, v, True)}


def case_outer(impl, rng, B=2, n=20):
    m = cm.random_vec(rng, B, n)
    v = cm.random_vec(rng, B, n)
    return {"m": m, "v": v, "o": impl.outer_band(m, v, 2, 1)}


def case_solve_mat(impl, rng, B=2, n=30, bw=3, rl=1, ru=2):
    l = cm.random_cholesky_factor(rng, B, n, bw)
    r = cm.random_band(rng, B, n, rl, ru)
    s, _, _ = impl.solve_mat(l, r, rl, ru, min(rl + bw, n - 1), ru, False)
    st, _, _ = impl.solve_mat(l, r, rl, ru, rl, min(ru + bw, n - 1), True)
    return {"l": l, "r": r, "s": s, "st": st}


def case_vjp_cholesky(impl, rng, B=3, n=30, bw=3):
    q = cm.random_spd_band(rng, B, n, bw)
    l, _, _ = impl.cholesky(q)
    lbar = cm.random_band(rng, B, n, bw, 0)
    return {"l": l, "lbar": lbar, "qbar": impl.vjp_cholesky(l, lbar)}


def case_vjp_solve_vec(impl, rng, B=3, n=35, bw=2):
    l = cm.random_cholesky_factor(rng, B, n, bw)
    v = cm.random_vec(rng, B, n)
    w = cm.random_vec(rng, B, n)
    out = {"l": l, "v": v, "w": w}
    for t in (False, True):
        s, _, _ = impl.solve_vec(l, v, t)
        lb, vb, _, _ = impl.vjp_solve_vec(l, s, w, t)
        out[f"lbar{int(t)}"], out[f"vbar{int(t)}"] = lb, vb
    return out


def case_vjp_subset(impl, rng, B=3, n=30, bw=3):
    l = cm.random_cholesky_factor(rng, B, n, bw)
    sbar = cm.random_band(rng, B, n, bw, 0)
    s, _, _ = impl.sparse_inverse_subset(l)
    lb, _, _ = impl.vjp_sparse_inverse_subset(l, s, sbar)
    return {"l": l, "sbar": sbar, "lbar": lb}


def case_vjp_products(impl, rng, B=2, n=28, al=2, au=1, bl=1, bu=3):
    a = cm.random_band(rng, B, n, al, au)
    b = cm.random_band(rng, B, n, bl, bu)
    pl, pu = min(al + bl, n - 1), min(au + bu, n - 1)
    pbar = cm.random_band(rng, B, n, pl, pu)
    ab, bb = impl.vjp_product_band_band(a, al, au, b, bl, bu, pbar, pl, pu)
    v = cm.random_vec(rng, B, n)
    p = cm.random_vec(rng, B, n)
    bb0, vb0 = impl.vjp_product_band_vec(b, bl, bu, v, p, False)
    bb1, vb1 = impl.vjp_product_band_vec(b, bl, bu, v, p, True)
    m = cm.random_vec(rng, B, n)
    obar = cm.random_band(rng, B, n, 2, 1)
    mb, vb = impl.vjp_outer_band(m, v, obar, 2, 1)
    return {"abar": ab, "bbar": bb, "bvbar0": bb0, "vbar0": vb0, "bvbar1": bb1, "vbar1": vb1,
            "mbar": mb, "ovbar": vb}


def case_vjp_log_det(impl, rng, B=3, n=21, bw=2):
    l = cm.random_cholesky_factor(rng, B, n, bw)
    c = rng.uniform(-1, 1, B)
    return {"lbar": impl.vjp_log_det(l, c)}


def case_vjp_solve_mat(impl, rng, B=2, n=25, bw=2, rl=1, ru=1):
    l = cm.random_cholesky_factor(rng, B, n, bw)
    r = cm.random_band(rng, B, n, rl, ru)
    out = {}
    for t in (False, True):
        ol = rl if t else min(rl + bw, n - 1)
        ou = min(ru + bw, n - 1) if t else ru
        s, _, _ = impl.solve_mat(l, r, rl, ru, ol, ou, t)
        sbar = cm.random_band(rng, B, n, ol, ou)
        lb, rb, _, _ = impl.vjp_solve_mat(l, s, ol, ou, sbar, rl, ru, t)
        out[f"lbar{int(t)}"], out[f"rbar{int(t)}"] = lb, rb
    return out


def case_mlik(impl, rng, B=3, n=200, k=4, tau2=0.01):
    L = cm.config_factor(rng, B, n, k)
    y = rng.normal(0, 1, (B, n))
    loss, lbar, tbar, _, _ = impl.marginal_likelihood_grad(L, y, tau2)
    return {"L": L, "y": y, "loss": loss, "lbar": lbar, "tau2_bar": tbar}


def case_mlik_k16(impl, rng, B=2, n=300, k=16, tau2=0.01):
    return case_mlik(impl, rng, B, n, k, tau2)


CASES = {
    "cholesky": case_cholesky,
    "cholesky_cfg0": case_cholesky_cfg0,
    "solve_vec": case_solve_vec,
    "log_det": case_log_det,
    "subset": case_subset,
    "products": case_products,
    "band_vec": case_band_vec,
    "outer": case_outer,
    "solve_mat": case_solve_mat,
    "vjp_cholesky": case_vjp_cholesky,
    "vjp_solve_vec": case_vjp_solve_vec,
    "vjp_subset": case_vjp_subset,
    "vjp_products": case_vjp_products,
    "vjp_log_det": case_vjp_log_det,
    "vjp_solve_mat": case_vjp_solve_mat,
    "mlik": case_mlik,
    "mlik_k16": case_mlik_k16,
}


def run_case(name, impl):
    return CASES[name](impl, inputs(name))
