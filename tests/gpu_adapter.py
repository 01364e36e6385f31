"""The CUDA library behind the oracle's numpy interface (tests only).

Lets every golden case and parity check run unchanged against
``paper_1902_10078_b200``: inputs are uploaded to the device layout
(``tile`` 32 or 1), the C ABI runs, outputs come back in the reference layout.
"""
from __future__ import annotations

import numpy as np
import torch

import paper_1902_10078_b200 as bgm
from paper_1902_10078_b200 import api


class GpuOracle:
    def __init__(self, tile: int = 32, dtype=torch.float64):
        self.tile = tile
        self.dtype = dtype

    # -- helpers
    def _b(self, a, lo, up):
        return bgm.Bands.from_reference(np.asarray(a, np.float64), lo, up, tile=self.tile, dtype=self.dtype)

    def _v(self, v):
        return bgm.Vecs.from_reference(np.asarray(v, np.float64), tile=self.tile, dtype=self.dtype)

    @staticmethod
    def _np(x):
        if isinstance(x, torch.Tensor):
            return x.double().cpu().numpy()
        return x.to_reference().double().cpu().numpy()

    @staticmethod
    def _st(s):
        return s.st.cpu().numpy(), s.row.cpu().numpy()

    # -- forward
    def cholesky(self, q):
        q = np.asarray(q)
        Q = self._b(q, q.shape[2] - 1, 0)
        L = Q.like()
        s = api.new_status(Q.batch)
        api._call("bgm_cholesky", Q.desc(), L.desc(), *s.ptrs(), api._stream())
        return (self._np(L), *self._st(s))

    def solve_vec(self, l, v, transpose=False):
        l = np.asarray(l)
        L, V = self._b(l, l.shape[2] - 1, 0), self._v(v)
        x = V.like()
        s = api.new_status(L.batch)
        api._call("bgm_solve_vec", L.desc(), V.desc(), int(transpose), x.desc(), *s.ptrs(), api._stream())
        return (self._np(x), *self._st(s))

    def log_det(self, l):
        l = np.asarray(l)
        L = self._b(l, l.shape[2] - 1, 0)
        out = torch.empty(L.batch, dtype=self.dtype, device="cuda")
        s = api.new_status(L.batch)
        import ctypes as C
        api._call("bgm_log_det", L.desc(), C.c_void_p(out.data_ptr()), *s.ptrs(), api._stream())
        return (self._np(out), *self._st(s))

    def sparse_inverse_subset(self, l):
        l = np.asarray(l)
        L = self._b(l, l.shape[2] - 1, 0)
        S = L.like()
        s = api.new_status(L.batch)
        api._call("bgm_sparse_inverse_subset", L.desc(), S.desc(), *s.ptrs(), api._stream())
        return (self._np(S), *self._st(s))

    def product_band_band(self, a, al, au, b, bl, bu, ol=None, ou=None):
        A, Bm = self._b(a, al, au), self._b(b, bl, bu)
        ol = al + bl if ol is None else ol
        ou = au + bu if ou is None else ou
        c = bgm.product_band_band_restricted(A, Bm, ol, ou)
        return self._np(c), c.lower, c.upper

    def product_band_vec(self, b, bl, bu, v, transpose=False):
        return self._np(bgm.product_band_vec(self._b(b, bl, bu), self._v(v), transpose))

    def outer_band(self, m, v, lower, upper):
        return self._np(bgm.outer_band(self._v(m), self._v(v), lower, upper))

    def solve_mat(self, l, r, rl, ru, ol, ou, transpose=False):
        l = np.asarray(l)
        L, R = self._b(l, l.shape[2] - 1, 0), self._b(r, rl, ru)
        n = L.n
        out = bgm.Bands.empty(L.batch, n, min(ol, n - 1), min(ou, n - 1), self.tile, self.dtype)
        s = api.new_status(L.batch)
        api._call("bgm_solve_mat", L.desc(), R.desc(), int(transpose), out.desc(), *s.ptrs(), api._stream())
        return (self._np(out), *self._st(s))

    # -- reverse
    def vjp_cholesky(self, l, lbar):
        l = np.asarray(l)
        k = l.shape[2] - 1
        return self._np(bgm.vjp_cholesky(self._b(l, k, 0), self._b(lbar, k, 0)))

    def vjp_solve_vec(self, l, s, sbar, transpose=False):
        l = np.asarray(l)
        L = self._b(l, l.shape[2] - 1, 0)
        lb, vb = bgm.vjp_solve_vec(L, self._v(s), self._v(sbar), transpose, check=False)
        return self._np(lb), self._np(vb), None, None

    def vjp_sparse_inverse_subset(self, l, s, sbar):
        l = np.asarray(l)
        k = l.shape[2] - 1
        L, Sd, Sb = self._b(l, k, 0), self._b(s, k, 0), self._b(sbar, k, 0)  # kept alive across the call
        lb = L.like()
        st = api.new_status(L.batch)
        api._call("bgm_vjp_sparse_inverse_subset", L.desc(), Sd.desc(), Sb.desc(), lb.desc(), *st.ptrs(),
                  api._stream())
        return (self._np(lb), *self._st(st))

    def vjp_product_band_band(self, a, al, au, b, bl, bu, pbar, pl, pu):
        ab, bb = bgm.vjp_product_band_band(self._b(a, al, au), self._b(b, bl, bu), self._b(pbar, pl, pu))
        return self._np(ab), self._np(bb)

    def vjp_product_band_vec(self, b, bl, bu, v, pbar, transpose=False):
        bb, vb = bgm.vjp_product_band_vec(self._b(b, bl, bu), self._v(v), self._v(pbar), transpose)
        return self._np(bb), self._np(vb)

    def vjp_outer_band(self, m, v, obar, ol, ou):
        mb, vb = bgm.vjp_outer_band(self._v(m), self._v(v), self._b(obar, ol, ou))
        return self._np(mb), self._np(vb)

    def vjp_log_det(self, l, cbar):
        l = np.asarray(l)
        cb = torch.as_tensor(np.broadcast_to(np.asarray(cbar, np.float64), (l.shape[0],)).copy())
        return self._np(bgm.vjp_log_det_from_cholesky(self._b(l, l.shape[2] - 1, 0), cb))

    def vjp_solve_mat(self, l, s, sl, su, sbar, rl, ru, transpose=False):
        l = np.asarray(l)
        L = self._b(l, l.shape[2] - 1, 0)
        lb, rb = bgm.vjp_solve_mat(L, self._b(s, sl, su), self._b(sbar, sl, su), rl, ru, transpose, check=False)
        return self._np(lb), self._np(rb), None, None

    def marginal_likelihood_grad(self, L, y, tau2):
        L = np.asarray(L)
        Lb = bgm.Bands.from_reference(L, L.shape[2] - 1, 0, tile=self.tile)
        Y = bgm.Vecs.from_reference(np.asarray(y), tile=self.tile)
        B = L.shape[0]
        st = api.new_status(B, Lb.data.device)
        out = (torch.empty(B, dtype=torch.float64, device=Lb.data.device), Lb.like(),
               torch.empty(B, dtype=torch.float64, device=Lb.data.device), st)
        loss, lbar, tbar = bgm.marginal_likelihood_grad(Lb, Y, tau2, check=False, out=out)
        return (self._np(loss), self._np(lbar), self._np(tbar), st.st[:B].cpu().numpy(),
                st.row[:B].cpu().numpy())
