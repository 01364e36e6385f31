"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes front end over the two CPU oracles:

* ``restatement`` -- ``oracle/liboracle.so``, the plain-C restatement of the
  reference loops (``oracle/bandgm_oracle.c``, each function cites the
  reference file:line it follows);
* ``reference``   -- ``oracle/_ref/libbandgm_ref.so``, the reference's own
  ``proj/src`` hot-path sources compiled verbatim (``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  The product package ``paper_1902_10078_b200`` never
does, and has no CPU fallback.

Array convention: a batch of bands is a float64 numpy array of shape
``(B, n, w)`` with ``w = lower + upper + 1``; ``a[b, j, r]`` is storage row
``r`` of column ``j`` -- exactly the reference's column-major storage block
(``banded.hpp:1-11``) laid out batch-major.  Vectors are ``(B, n)``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "restatement": (os.path.join(HERE, "liboracle.so"), "orc_"),
    "reference": (os.path.join(HERE, "_ref", "libbandgm_ref.so"), "ref_"),
}

STATUS_NAMES = {0: "ok", 1: "NotPositiveDefinite", 2: "SingularDiagonal",
                3: "NonPositiveDiagonal", 4: "DimensionMismatch", 5: "Other"}

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


def build(reference: bool = True) -> None:
    """Compile the restatement (and the verbatim reference when present)."""
    env = {k: v for k, v in os.environ.items() if k not in ("CC", "CXX")}
    targets = ["restatement"] + (["ref"] if reference else [])
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True, env=env)


def available(which: str) -> bool:
    return os.path.exists(LIB_PATHS[which][0])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _opt(a):
    """Pointer to an optional float64 array (None -> NULL); the array is kept
    alive by the module-level holder until the next call."""
    global _HOLD
    if a is None:
        _HOLD = None
        return _dp()
    _HOLD = np.ascontiguousarray(a, dtype=np.float64)
    return _HOLD.ctypes.data_as(_dp)


_HOLD = None


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """One CPU oracle library (restatement or verbatim reference)."""

    def __init__(self, which: str = "restatement"):
        path, prefix = LIB_PATHS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        self.which = which
        self.lib = C.CDLL(path)
        self.p = prefix

    def _fn(self, name):
        f = getattr(self.lib, self.p + name)
        f.restype = C.c_int
        return f

    @staticmethod
    def _status(batch):
        return np.zeros(batch, np.int32), np.full(batch, -1, np.int64)

    # ---------------------------------------------------------- forward
    def cholesky(self, q):
        q = _f64(q)
        B, n, w = q.shape
        l = np.zeros_like(q)
        st, row = self._status(B)
        self._fn("cholesky")(_i64(B), _i64(n), _i64(w - 1), _ptr(q), _ptr(l),
                             st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return l, st, row

    def solve_vec(self, l, v, transpose=False):
        l, v = _f64(l), _f64(v)
        B, n, w = l.shape
        x = np.zeros((B, n))
        st, row = self._status(B)
        self._fn("solve_vec")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(v), C.c_int(int(transpose)),
                              _ptr(x), st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return x, st, row

    def log_det(self, l):
        l = _f64(l)
        B, n, w = l.shape
        out = np.zeros(B)
        st, row = self._status(B)
        self._fn("log_det")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(out),
                            st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return out, st, row

    def sparse_inverse_subset(self, l):
        l = _f64(l)
        B, n, w = l.shape
        s = np.zeros_like(l)
        st, row = self._status(B)
        self._fn("sparse_inverse_subset")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(s),
                                          st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return s, st, row

    def product_band_band(self, a, al, au, b, bl, bu, ol=None, ou=None):
        """Restricted product; (ol, ou) default to the full product band."""
        a, b = _f64(a), _f64(b)
        B, n, _ = a.shape
        ol = al + bl if ol is None else ol
        ou = au + bu if ou is None else ou
        ol, ou = min(ol, max(n - 1, 0)), min(ou, max(n - 1, 0))
        c = np.zeros((B, n, ol + ou + 1))
        self._fn("product_band_band")(_i64(B), _i64(n), _i64(al), _i64(au), _ptr(a), _i64(bl),
                                      _i64(bu), _ptr(b), _i64(ol), _i64(ou), _ptr(c))
        return c, ol, ou

    def product_band_vec(self, b, bl, bu, v, transpose=False):
        b, v = _f64(b), _f64(v)
        B, n, _ = b.shape
        y = np.zeros((B, n))
        self._fn("product_band_vec")(_i64(B), _i64(n), _i64(bl), _i64(bu), _ptr(b), _ptr(v),
                                     C.c_int(int(transpose)), _ptr(y))
        return y

    def outer_band(self, m, v, lower, upper):
        m, v = _f64(m), _f64(v)
        B, n = m.shape
        lower, upper = min(lower, n - 1), min(upper, n - 1)
        o = np.zeros((B, n, lower + upper + 1))
        self._fn("outer_band")(_i64(B), _i64(n), _ptr(m), _ptr(v), _i64(lower), _i64(upper), _ptr(o))
        return o

    def solve_mat(self, l, r, rl, ru, ol, ou, transpose=False):
        l, r = _f64(l), _f64(r)
        B, n, w = l.shape
        ol, ou = min(ol, n - 1), min(ou, n - 1)
        out = np.zeros((B, n, ol + ou + 1))
        st, row = self._status(B)
        self._fn("solve_mat")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _i64(rl), _i64(ru), _ptr(r),
                              _i64(ol), _i64(ou), C.c_int(int(transpose)), _ptr(out),
                              st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return out, st, row

    # ---------------------------------------------------------- reverse
    def vjp_cholesky(self, l, lbar):
        l, lbar = _f64(l), _f64(lbar)
        B, n, w = l.shape
        qbar = np.zeros_like(l)
        self._fn("vjp_cholesky")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(lbar), _ptr(qbar))
        return qbar

    def vjp_solve_vec(self, l, s, sbar, transpose=False):
        l, s, sbar = _f64(l), _f64(s), _f64(sbar)
        B, n, w = l.shape
        lbar = np.zeros_like(l)
        vbar = np.zeros((B, n))
        st, row = self._status(B)
        self._fn("vjp_solve_vec")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(s), _ptr(sbar),
                                  C.c_int(int(transpose)), _ptr(lbar), _ptr(vbar),
                                  st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return lbar, vbar, st, row

    def vjp_sparse_inverse_subset(self, l, s, sbar):
        l, s, sbar = _f64(l), _f64(s), _f64(sbar)
        B, n, w = l.shape
        lbar = np.zeros_like(l)
        st, row = self._status(B)
        self._fn("vjp_sparse_inverse_subset")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(s),
                                              _ptr(sbar), _ptr(lbar), st.ctypes.data_as(_i32p),
                                              row.ctypes.data_as(_i64p))
        return lbar, st, row

    def vjp_product_band_band(self, a, al, au, b, bl, bu, pbar, pl, pu):
        a, b, pbar = _f64(a), _f64(b), _f64(pbar)
        B, n, _ = a.shape
        abar = np.zeros_like(a)
        bbar = np.zeros_like(b)
        self._fn("vjp_product_band_band")(_i64(B), _i64(n), _i64(al), _i64(au), _ptr(a), _i64(bl),
                                          _i64(bu), _ptr(b), _i64(pl), _i64(pu), _ptr(pbar),
                                          _ptr(abar), _ptr(bbar))
        return abar, bbar

    def vjp_product_band_vec(self, b, bl, bu, v, pbar, transpose=False):
        b, v, pbar = _f64(b), _f64(v), _f64(pbar)
        B, n, _ = b.shape
        bbar = np.zeros_like(b)
        vbar = np.zeros((B, n))
        self._fn("vjp_product_band_vec")(_i64(B), _i64(n), _i64(bl), _i64(bu), _ptr(b), _ptr(v),
                                         _ptr(pbar), C.c_int(int(transpose)), _ptr(bbar), _ptr(vbar))
        return bbar, vbar

    def vjp_outer_band(self, m, v, obar, ol, ou):
        m, v, obar = _f64(m), _f64(v), _f64(obar)
        B, n = m.shape
        mbar = np.zeros((B, n))
        vbar = np.zeros((B, n))
        self._fn("vjp_outer_band")(_i64(B), _i64(n), _ptr(m), _ptr(v), _i64(ol), _i64(ou), _ptr(obar),
                                   _ptr(mbar), _ptr(vbar))
        return mbar, vbar

    def vjp_log_det(self, l, cbar):
        l = _f64(l)
        B, n, w = l.shape
        cbar = _f64(np.broadcast_to(np.asarray(cbar, np.float64), (B,)))
        lbar = np.zeros_like(l)
        self._fn("vjp_log_det")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _ptr(cbar), _ptr(lbar))
        return lbar

    def vjp_solve_mat(self, l, s, sl, su, sbar, rl, ru, transpose=False):
        l, s, sbar = _f64(l), _f64(s), _f64(sbar)
        B, n, w = l.shape
        rlc, ruc = min(rl, n - 1), min(ru, n - 1)
        lbar = np.zeros_like(l)
        rbar = np.zeros((B, n, rlc + ruc + 1))
        st, row = self._status(B)
        self._fn("vjp_solve_mat")(_i64(B), _i64(n), _i64(w - 1), _ptr(l), _i64(sl), _i64(su), _ptr(s),
                                  _ptr(sbar), _i64(rl), _i64(ru), C.c_int(int(transpose)), _ptr(lbar),
                                  _ptr(rbar), st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return lbar, rbar, st, row

    def marginal_likelihood_grad(self, L, y, tau2):
        L, y = _f64(L), _f64(y)
        B, n, w = L.shape
        loss = np.zeros(B)
        lbar = np.zeros_like(L)
        tbar = np.zeros(B)
        st, row = self._status(B)
        self._fn("marginal_likelihood_grad")(_i64(B), _i64(n), _i64(w - 1), _ptr(L), _ptr(y),
                                             C.c_double(tau2), _ptr(loss), _ptr(lbar), _ptr(tbar),
                                             st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p))
        return loss, lbar, tbar, st, row

    def kl_divergence_grad(self, mq, lq, mp, lp):
        """infer::kl_divergence (inference.cpp:247-268) and its gradient in
        (m_q, L_q); reference (verbatim tape) only."""
        if self.which != "reference":
            raise RuntimeError("kl_divergence lives in the compiled reference tape only")
        mq, lq, mp, lp = _f64(mq), _f64(lq), _f64(mp), _f64(lp)
        B, n, wq = lq.shape
        wp = lp.shape[2]
        kl, mb, lb = np.zeros(B), np.zeros((B, n)), np.zeros_like(lq)
        st, row = self._status(B)
        self._fn("kl_divergence_grad")(_i64(B), _i64(n), _i64(wq - 1), _i64(wp - 1), _ptr(mq), _ptr(lq), _ptr(mp),
                                       _ptr(lp), _ptr(kl), _ptr(mb), _ptr(lb), st.ctypes.data_as(_i32p),
                                       row.ctypes.data_as(_i64p))
        return kl, mb, lb, st, row

    def elbo_gaussian_grad(self, mq, lq, mp, lp, y, tau2, observed=None):
        """infer::elbo (inference.cpp:276-287), GaussianLik; reference
        (verbatim tape) only.  observed: optional (B, n) 0/1 mask of the
        SelectionIndex (y scattered to full length); None = every latent.
        -> elbo, m_bar, l_bar, tau2_bar, st, row."""
        if self.which != "reference":
            raise RuntimeError("elbo lives in the compiled reference tape only")
        mq, lq, mp, lp, y = _f64(mq), _f64(lq), _f64(mp), _f64(lp), _f64(y)
        B, n, wq = lq.shape
        wp = lp.shape[2]
        el, mb, lb, tb = np.zeros(B), np.zeros((B, n)), np.zeros_like(lq), np.zeros(B)
        st, row = self._status(B)
        self._fn("elbo_gaussian_grad")(_i64(B), _i64(n), _i64(wq - 1), _i64(wp - 1), _ptr(mq), _ptr(lq), _ptr(mp),
                                       _ptr(lp), _ptr(y), C.c_double(tau2), _ptr(el), _ptr(mb), _ptr(lb), _ptr(tb),
                                       st.ctypes.data_as(_i32p), row.ctypes.data_as(_i64p), _opt(observed))
        return el, mb, lb, tb, st, row

    def elbo_poisson_grad(self, mq, lq, mp, lp, y, weight, quad_points=20, observed=None):
        """infer::elbo (inference.cpp:276-287), PoissonLik, Gauss-Hermite
        nodes from numpy's hermgauss; observed as in elbo_gaussian_grad;
        reference tape only."""
        if self.which != "reference":
            raise RuntimeError("elbo lives in the compiled reference tape only")
        gx, gw = np.polynomial.hermite.hermgauss(quad_points)
        mq, lq, mp, lp, y, weight = (_f64(a) for a in (mq, lq, mp, lp, y, weight))
        B, n, wq = lq.shape
        wp = lp.shape[2]
        el, mb, lb = np.zeros(B), np.zeros((B, n)), np.zeros_like(lq)
        st, row = self._status(B)
        self._fn("elbo_poisson_grad")(_i64(B), _i64(n), _i64(wq - 1), _i64(wp - 1), _ptr(mq), _ptr(lq), _ptr(mp),
                                      _ptr(lp), _ptr(y), _ptr(weight), _i64(quad_points), _ptr(_f64(gx)),
                                      _ptr(_f64(gw)), _ptr(el), _ptr(mb), _ptr(lb), st.ctypes.data_as(_i32p),
                                      row.ctypes.data_as(_i64p), _opt(observed))
        return el, mb, lb, st, row

    # ---------------------------------------------------------- reference only
    def mlik_exact_ld(self, L, y, tau2):
        """Config-3 loss, L_bar, tau2_bar along the banded route in x87 long
        double (restatement library only; the yardstick of tests/test_exact.py),
        rounded to float64."""
        if self.which != "restatement":
            raise RuntimeError("the long-double yardstick lives in the restatement library")
        L, y = _f64(L), _f64(y)
        B, n, w = L.shape
        loss, lbar, tbar = np.zeros(B), np.zeros_like(L), np.zeros(B)
        self._fn("mlik_exact_ld")(_i64(B), _i64(n), _i64(w - 1), _ptr(L), _ptr(y), C.c_double(tau2), _ptr(loss),
                                   _ptr(lbar), _ptr(tbar))
        return loss, lbar, tbar

    def run_grad_suite(self, seed: int, instances: int):
        if self.which != "reference":
            raise RuntimeError("gradcheck suite lives in the compiled reference only")
        out = np.zeros(32)
        f = self._fn("run_grad_suite")
        f.argtypes = [C.c_uint64, C.c_int, _dp, C.c_int]
        k = f(C.c_uint64(seed), C.c_int(instances), _ptr(out), C.c_int(32))
        return out[:k]

    def threads(self) -> int:
        if self.which == "reference":
            return int(self._fn("threads")())
        return os.cpu_count() or 1


GRAD_SUITE_OPS = ["cholesky", "solve_vec", "solve_vec_transposed", "solve_mat", "solve_mat_transposed",
                  "sparse_inverse_subset", "product_band_band", "product_band_band_restricted",
                  "product_band_vec", "product_band_vec_transposed", "outer_band", "log_det_from_cholesky"]
