"""PyTorch autograd over the operator suite.

Every differentiable operator of the reference (``kernels.hpp`` forward,
``grad.hpp`` reverse) as a ``torch.autograd.Function`` whose forward and
backward are the C-ABI calls of :mod:`api` -- the same role as the
reference's tape nodes (``tape.cpp:158-272``), but composable with any
PyTorch code.  Inputs and outputs are :class:`api.Bands` / :class:`api.Vecs`
whose ``.data`` tensors carry ``requires_grad``; the gradient of a band is
with respect to its stored cells, so symmetric inputs follow the reference's
stored-cell convention (``grad.hpp:4-8``).  Corner cells and the padding
lanes of a partial 32-matrix tile get zero gradient.

The config-3 step is exposed as :func:`marginal_likelihood`; its backward
reuses the L-bar and tau2-bar the fused sweeps produce in the forward pass.
"""
from __future__ import annotations

import torch

from . import api
from .api import Bands, Vecs


def _meta(x: Bands):
    return (x.batch, x.n, x.lower, x.upper, x.tile)


def _bands(d, meta) -> Bands:
    return Bands(d, *meta)


def _vecs(d, meta) -> Vecs:
    return Vecs(d, *meta)


def _clean(d: torch.Tensor, batch: int, tile: int) -> torch.Tensor:
    """Zero the padding lanes of a partial last tile (their values are not
    part of any matrix)."""
    if tile == 32 and batch % 32:
        d[-1, ..., batch % 32:] = 0
    return d


def _g(t: torch.Tensor) -> torch.Tensor:
    return t.contiguous()


class _Cholesky(torch.autograd.Function):
    @staticmethod
    def forward(ctx, qd, meta):
        l = api.cholesky(_bands(qd, meta))
        ctx.meta = _meta(l)
        ctx.save_for_backward(l.data)
        return l.data

    @staticmethod
    def backward(ctx, gl):
        (ld,) = ctx.saved_tensors
        m = ctx.meta
        qb = api.vjp_cholesky(_bands(ld, m), _bands(_g(gl), m))
        return _clean(qb.data, m[0], m[4]), None


def cholesky(q: Bands) -> Bands:
    """ops::cholesky (kernels.hpp:25); reverse grad::vjp_cholesky (grad.hpp:24)."""
    d = _Cholesky.apply(q.data, _meta(q))
    return Bands(d, q.batch, q.n, q.lower, 0, q.tile)


class _SolveVec(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ld, vd, lmeta, vmeta, transpose):
        l, v = _bands(ld, lmeta), _vecs(vd, vmeta)
        x = api.solve_vec(l, v, transpose)
        ctx.lmeta, ctx.vmeta, ctx.tr = lmeta, vmeta, transpose
        ctx.save_for_backward(ld, x.data)
        return x.data

    @staticmethod
    def backward(ctx, gx):
        ld, xd = ctx.saved_tensors
        l = _bands(ld, ctx.lmeta)
        lb, vb = api.vjp_solve_vec(l, _vecs(xd, ctx.vmeta), _vecs(_g(gx), ctx.vmeta), ctx.tr)
        b, tile = ctx.lmeta[0], ctx.lmeta[4]
        return _clean(lb.data, b, tile), _clean(vb.data, b, tile), None, None, None


def solve_vec(l: Bands, v: Vecs, transpose_l: bool = False) -> Vecs:
    """ops::solve_vec (kernels.hpp:30-31); reverse grad::vjp_solve_vec (grad.hpp:31-32)."""
    vmeta = (v.batch, v.n, v.tile)
    return Vecs(_SolveVec.apply(l.data, v.data, _meta(l), vmeta, bool(transpose_l)), v.batch, v.n, v.tile)


class _LogDet(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ld, meta):
        l = _bands(ld, meta)
        ctx.meta = meta
        ctx.save_for_backward(ld)
        return api.log_det_from_cholesky(l)

    @staticmethod
    def backward(ctx, gc):
        (ld,) = ctx.saved_tensors
        lb = api.vjp_log_det_from_cholesky(_bands(ld, ctx.meta), _g(gc))
        return _clean(lb.data, ctx.meta[0], ctx.meta[4]), None


def log_det_from_cholesky(l: Bands) -> torch.Tensor:
    """ops::log_det_from_cholesky (kernels.hpp:72): (B,) tensor; reverse
    grad::vjp_log_det_from_cholesky (grad.hpp:73)."""
    return _LogDet.apply(l.data, _meta(l))


class _Subset(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ld, meta):
        s = api.sparse_inverse_subset(_bands(ld, meta))
        ctx.meta = meta
        ctx.save_for_backward(ld, s.data)
        return s.data

    @staticmethod
    def backward(ctx, gs):
        ld, sd = ctx.saved_tensors
        m = ctx.meta
        lb = api.vjp_sparse_inverse_subset(_bands(ld, m), _bands(sd, m), _bands(_g(gs), m))
        return _clean(lb.data, m[0], m[4]), None


def sparse_inverse_subset(l: Bands) -> Bands:
    """ops::sparse_inverse_subset (kernels.hpp:47); reverse
    grad::vjp_sparse_inverse_subset (grad.hpp:46-47)."""
    return Bands(_Subset.apply(l.data, _meta(l)), l.batch, l.n, l.lower, 0, l.tile)


class _Product(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ad, bd, ameta, bmeta, ol, ou):
        a, b = _bands(ad, ameta), _bands(bd, bmeta)
        c = api.product_band_band_restricted(a, b, ol, ou)
        ctx.ameta, ctx.bmeta, ctx.cmeta = ameta, bmeta, _meta(c)
        ctx.save_for_backward(ad, bd)
        return c.data

    @staticmethod
    def backward(ctx, gc):
        ad, bd = ctx.saved_tensors
        ab, bb = api.vjp_product_band_band(_bands(ad, ctx.ameta), _bands(bd, ctx.bmeta), _bands(_g(gc), ctx.cmeta))
        b, tile = ctx.ameta[0], ctx.ameta[4]
        return _clean(ab.data, b, tile), _clean(bb.data, b, tile), None, None, None, None


def product_band_band(a: Bands, b: Bands, out_lower: int | None = None, out_upper: int | None = None) -> Bands:
    """ops::product_band_band(_restricted) (kernels.hpp:50-57); reverse
    grad::vjp_product_band_band (grad.hpp:55-56).  Default: the full band."""
    ol = a.lower + b.lower if out_lower is None else out_lower
    ou = a.upper + b.upper if out_upper is None else out_upper
    ol, ou = min(ol, max(a.n - 1, 0)), min(ou, max(a.n - 1, 0))
    d = _Product.apply(a.data, b.data, _meta(a), _meta(b), ol, ou)
    return Bands(d, a.batch, a.n, ol, ou, a.tile)


class _BandVec(torch.autograd.Function):
    @staticmethod
    def forward(ctx, bd, vd, bmeta, vmeta, transpose):
        y = api.product_band_vec(_bands(bd, bmeta), _vecs(vd, vmeta), transpose)
        ctx.bmeta, ctx.vmeta, ctx.tr = bmeta, vmeta, transpose
        ctx.save_for_backward(bd, vd)
        return y.data

    @staticmethod
    def backward(ctx, gy):
        bd, vd = ctx.saved_tensors
        bb, vb = api.vjp_product_band_vec(_bands(bd, ctx.bmeta), _vecs(vd, ctx.vmeta), _vecs(_g(gy), ctx.vmeta),
                                          ctx.tr)
        b, tile = ctx.bmeta[0], ctx.bmeta[4]
        return _clean(bb.data, b, tile), _clean(vb.data, b, tile), None, None, None


def product_band_vec(b: Bands, v: Vecs, transpose_b: bool = False) -> Vecs:
    """ops::product_band_vec (kernels.hpp:61-62); reverse
    grad::vjp_product_band_vec (grad.hpp:62-63)."""
    vmeta = (v.batch, v.n, v.tile)
    return Vecs(_BandVec.apply(b.data, v.data, _meta(b), vmeta, bool(transpose_b)), v.batch, v.n, v.tile)


class _Outer(torch.autograd.Function):
    @staticmethod
    def forward(ctx, md, vd, vmeta, lower, upper):
        o = api.outer_band(_vecs(md, vmeta), _vecs(vd, vmeta), lower, upper)
        ctx.vmeta, ctx.ometa = vmeta, _meta(o)
        ctx.save_for_backward(md, vd)
        return o.data

    @staticmethod
    def backward(ctx, go):
        md, vd = ctx.saved_tensors
        mb, vb = api.vjp_outer_band(_vecs(md, ctx.vmeta), _vecs(vd, ctx.vmeta), _bands(_g(go), ctx.ometa))
        b, tile = ctx.vmeta[0], ctx.vmeta[2]
        return _clean(mb.data, b, tile), _clean(vb.data, b, tile), None, None, None


def outer_band(m: Vecs, v: Vecs, lower: int, upper: int) -> Bands:
    """ops::outer_band (kernels.hpp:66-67); reverse grad::vjp_outer_band (grad.hpp:69-70)."""
    vmeta = (v.batch, v.n, v.tile)
    lower, upper = min(lower, max(v.n - 1, 0)), min(upper, max(v.n - 1, 0))
    return Bands(_Outer.apply(m.data, v.data, vmeta, lower, upper), v.batch, v.n, lower, upper, v.tile)


class _SolveMat(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ld, rd, lmeta, rmeta, ol, ou, transpose):
        s = api.solve_mat(_bands(ld, lmeta), _bands(rd, rmeta), ol, ou, transpose)
        ctx.lmeta, ctx.rmeta, ctx.smeta, ctx.tr = lmeta, rmeta, _meta(s), transpose
        ctx.save_for_backward(ld, s.data)
        return s.data

    @staticmethod
    def backward(ctx, gs):
        ld, sd = ctx.saved_tensors
        lb, rb = api.vjp_solve_mat(_bands(ld, ctx.lmeta), _bands(sd, ctx.smeta), _bands(_g(gs), ctx.smeta),
                                   ctx.rmeta[2], ctx.rmeta[3], ctx.tr)
        b, tile = ctx.lmeta[0], ctx.lmeta[4]
        return _clean(lb.data, b, tile), _clean(rb.data, b, tile), None, None, None, None, None


def solve_mat(l: Bands, r: Bands, out_lower: int, out_upper: int, transpose_l: bool = False) -> Bands:
    """ops::solve_mat (kernels.hpp:40-42), band-restricted L^-1 R or L^-T R;
    reverse grad::vjp_solve_mat (grad.hpp:40-42)."""
    ol, ou = min(out_lower, l.n - 1), min(out_upper, l.n - 1)
    d = _SolveMat.apply(l.data, r.data, _meta(l), _meta(r), ol, ou, bool(transpose_l))
    return Bands(d, l.batch, l.n, ol, ou, l.tile)


class _MarginalLikelihood(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ld, yd, tau2, lmeta, ymeta):
        loss, lbar, tbar = api.marginal_likelihood_grad(_bands(ld, lmeta), _vecs(yd, ymeta), float(tau2))
        ctx.lmeta, ctx.tdev = lmeta, tau2.device
        ctx.save_for_backward(lbar.data, tbar)
        return loss

    @staticmethod
    def backward(ctx, gloss):
        lbd, tbar = ctx.saved_tensors
        b, tile = ctx.lmeta[0], ctx.lmeta[4]
        g = gloss.to(lbd.dtype)
        if tile == 32:
            gp = torch.zeros(lbd.shape[0] * 32, dtype=lbd.dtype, device=lbd.device)
            gp[:b] = g
            scale = gp.view(lbd.shape[0], 1, 1, 32)
        else:
            scale = g.view(b, 1, 1)
        gl = _clean(lbd * scale, b, tile)
        return gl, None, (g * tbar).sum().to(ctx.tdev), None, None


def marginal_likelihood(L: Bands, y: Vecs, tau2) -> torch.Tensor:
    """Config-3 objective (inference.cpp:140-163 over precision_from_factor,
    inference.cpp:23-26): per-matrix log N(y | 0, (L L^T)^-1 + tau2 I) as a
    (B,) tensor, differentiable in L (stored lower band) and tau2 (a float or
    a 0-d tensor).  One fused forward+reverse pass; y is not differentiated."""
    t = tau2 if isinstance(tau2, torch.Tensor) else torch.tensor(float(tau2), dtype=torch.float64)
    return _MarginalLikelihood.apply(L.data, y.data, t, _meta(L), (y.batch, y.n, y.tile))


class _KL(torch.autograd.Function):
    @staticmethod
    def forward(ctx, mqd, lqd, mpd, lpd, vmeta, qmeta, pmeta):
        kl, mb, lb = api.kl_divergence_grad(_vecs(mqd, vmeta), _bands(lqd, qmeta), _vecs(mpd, vmeta),
                                            _bands(lpd, pmeta))
        ctx.vmeta, ctx.qmeta = vmeta, qmeta
        ctx.save_for_backward(mb.data, lb.data)
        return kl

    @staticmethod
    def backward(ctx, gkl):
        mbd, lbd = ctx.saved_tensors
        b, tile = ctx.qmeta[0], ctx.qmeta[4]
        g = gkl.to(lbd.dtype)
        if tile == 32:
            gp = torch.zeros(lbd.shape[0] * 32, dtype=lbd.dtype, device=lbd.device)
            gp[:b] = g
            gl, gm = lbd * gp.view(lbd.shape[0], 1, 1, 32), mbd * gp.view(mbd.shape[0], 1, 32)
        else:
            gl, gm = lbd * g.view(b, 1, 1), mbd * g.view(b, 1)
        return _clean(gm, b, tile), _clean(gl, b, tile), None, None, None, None, None


def kl_divergence(m_q: Vecs, l_q: Bands, m_p: Vecs, l_p: Bands) -> torch.Tensor:
    """infer::kl_divergence (inference.cpp:247-268) as a (B,) tensor,
    differentiable in the variational parameters m_q and L_q (stored cells);
    the prior (m_p, L_p) is constant, as in the reference's VI objective."""
    return _KL.apply(m_q.data, l_q.data, m_p.data, l_p.data, (m_q.batch, m_q.n, m_q.tile), _meta(l_q), _meta(l_p))


class _PriorNaturalParams(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b, q, mu0, sigma0, tile):
        lam, eta = api.prior_natural_params(a, b, q, mu0, sigma0, tile=tile)
        ctx.save_for_backward(a, b, q, mu0, sigma0)
        ctx.meta = (_meta(lam), (eta.batch, eta.n, eta.tile))
        return lam.data, eta.data

    @staticmethod
    def backward(ctx, glam, geta):
        a, b, q, mu0, sigma0 = ctx.saved_tensors
        lmeta, vmeta = ctx.meta
        lb = _bands(_g(glam).contiguous(), lmeta)
        eb = _vecs(_g(geta).contiguous(), vmeta)
        bars = api.vjp_prior_natural_params(a, b, q, mu0, sigma0, lb, eb)
        return (*bars, None)


def prior_natural_params(a, b, q, mu0, sigma0, tile: int = 32):
    """models::prior_natural_params (models.cpp:165-189) as a torch Function:
    (Lambda, eta) differentiable in a, b, q, mu0, sigma0 through the analytic
    device VJP (bgm_vjp_prior_natural_params) -- with it, the gradient of any
    objective of (Lambda, eta) with respect to model hyperparameters theta
    follows by autograd through the user's theta -> (a, q, ...) map, replacing
    the reference's finite-difference compose_precision_gradient
    (inference.cpp:360-380).  Returns the Bands / Vecs storage tensors."""
    return _PriorNaturalParams.apply(a, b, q, mu0, sigma0, tile)
