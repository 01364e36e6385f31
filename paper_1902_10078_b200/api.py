"""Python host mirror of the reference operator API over the bandgm_b200 C ABI.

Each function cites the reference symbol it mirrors.  Inputs and outputs are
:class:`Bands` / :class:`Vecs`: batches of ``B`` matrices (vectors) living in
device memory in the batch-interleaved layout of ``include/bandgm_b200.h``.
Errors are raised as the reference's exception types (``errors.hpp:9-50``)
with the first failing matrix and row.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
_LIB = None

BGM_F64, BGM_F32 = 0, 1
BGM_OK, BGM_ERR_NOT_PD, BGM_ERR_SINGULAR, BGM_ERR_NONPOS_DIAG, BGM_ERR_DIM, BGM_ERR_ARG, BGM_ERR_CUDA = range(7)


# --------------------------------------------------------------------- errors
class BandgmError(RuntimeError):
    """Base of the reference's exception family (errors.hpp)."""


class DimensionMismatch(BandgmError):
    """errors.hpp:9-11"""


class _RowError(BandgmError):
    what = ""

    def __init__(self, row: int, matrix: int = 0):
        self.row = int(row)
        self.matrix = int(matrix)
        super().__init__(f"{self.what} (pivot at row {self.row}, batch matrix {self.matrix})")


class NotPositiveDefinite(_RowError):
    """errors.hpp:27-34"""
    what = "matrix is not positive definite"


class SingularDiagonal(_RowError):
    """errors.hpp:36-43"""
    what = "triangular factor has a near-zero diagonal"


class NonPositiveDiagonal(_RowError):
    """errors.hpp:45-50"""
    what = "factor diagonal must be strictly positive"


_ROW_ERRORS = {BGM_ERR_NOT_PD: NotPositiveDefinite, BGM_ERR_SINGULAR: SingularDiagonal,
               BGM_ERR_NONPOS_DIAG: NonPositiveDiagonal}


# --------------------------------------------------------------------- ctypes
class _Band(C.Structure):
    _fields_ = [("data", C.c_void_p), ("batch", C.c_int64), ("n", C.c_int64), ("lower", C.c_int32),
                ("upper", C.c_int32), ("tile", C.c_int32), ("dtype", C.c_int32)]


class _Vec(C.Structure):
    _fields_ = [("data", C.c_void_p), ("batch", C.c_int64), ("n", C.c_int64), ("tile", C.c_int32),
                ("dtype", C.c_int32)]


def library_path() -> str:
    # BGM_LIBRARY: load an experiment build instead of the in-tree library
    return os.environ.get("BGM_LIBRARY") or os.path.join(HERE, "libbandgm_b200.so")


def library():
    """Load libbandgm_b200.so; raise (no fallback) when it is missing."""
    global _LIB
    if _LIB is None:
        path = library_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `make -C paper_1902_10078_b200` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        lib = C.CDLL(path)
        for name in ("bgm_status_name", "bgm_last_error"):
            getattr(lib, name).restype = C.c_char_p
        _LIB = lib
    return _LIB


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _call(name, *args):
    rc = getattr(library(), name)(*args)
    if rc == BGM_ERR_DIM:
        raise DimensionMismatch(f"{name}: shape mismatch")
    if rc != BGM_OK:
        msg = library().bgm_last_error().decode() if rc == BGM_ERR_CUDA else ""
        raise BandgmError(f"{name} failed: {library().bgm_status_name(rc).decode()} {msg}")


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float64:
        return BGM_F64
    if dt == torch.float32:
        return BGM_F32
    raise TypeError(f"unsupported dtype {dt}")


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("bandgm_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _round_up(b: int, tile: int) -> int:
    return (b + tile - 1) // tile * tile


# --------------------------------------------------------------------- containers
@dataclass
class Bands:
    """B banded n x n matrices with (lower, upper) diagonals, device layout.

    ``data`` has shape ``(ceil(B/32), n, w, 32)`` for tile 32 and
    ``(B, n, w)`` for tile 1 (the reference storage block per matrix)."""

    data: torch.Tensor
    batch: int
    n: int
    lower: int
    upper: int
    tile: int = 32

    @property
    def w(self) -> int:
        return self.lower + self.upper + 1

    @property
    def dtype(self) -> torch.dtype:
        return self.data.dtype

    @property
    def T(self) -> "Transposed":
        return Transposed(self)

    def desc(self) -> _Band:
        return _Band(self.data.data_ptr(), self.batch, self.n, self.lower, self.upper, self.tile,
                     _dtype_code(self.data.dtype))

    @staticmethod
    def empty(batch, n, lower, upper, tile=32, dtype=torch.float64, device=None) -> "Bands":
        dev = _device(device)
        w = lower + upper + 1
        if tile == 32:
            data = torch.empty((_round_up(batch, 32) // 32, n, w, 32), dtype=dtype, device=dev)
        elif tile == 1:
            data = torch.empty((batch, n, w), dtype=dtype, device=dev)
        else:
            raise ValueError("tile must be 1 or 32")
        return Bands(data, batch, n, lower, upper, tile)

    @staticmethod
    def zeros(batch, n, lower, upper, tile=32, dtype=torch.float64, device=None) -> "Bands":
        out = Bands.empty(batch, n, lower, upper, tile, dtype, device)
        out.data.zero_()
        return out

    def like(self, lower=None, upper=None) -> "Bands":
        return Bands.empty(self.batch, self.n, self.lower if lower is None else lower,
                           self.upper if upper is None else upper, self.tile, self.dtype, self.data.device)

    @staticmethod
    def from_reference(arr, lower, upper, tile=32, dtype=torch.float64, device=None) -> "Bands":
        """Upload ``arr[b, j, r]`` = reference storage row r of column j."""
        dev = _device(device)
        src = torch.as_tensor(np.ascontiguousarray(arr) if isinstance(arr, np.ndarray) else arr)
        src = src.to(device=dev, dtype=dtype).contiguous()
        if src.dim() == 2:
            src = src.unsqueeze(0)
        B, n, w = src.shape
        if w != lower + upper + 1:
            raise DimensionMismatch("storage rows do not match the band")
        flat = Bands(src, B, n, lower, upper, 1)
        if tile == 1:
            return flat
        out = Bands.empty(B, n, lower, upper, tile, dtype, dev)
        if tile == 32 and B % 32:
            out.data.zero_()
        _call("bgm_relayout_band", flat.desc(), out.desc(), _stream())
        return out

    def to_reference(self) -> torch.Tensor:
        """(B, n, w) tensor on the device in the reference storage layout."""
        if self.tile == 1:
            return self.data
        out = Bands.empty(self.batch, self.n, self.lower, self.upper, 1, self.dtype, self.data.device)
        _call("bgm_relayout_band", self.desc(), out.desc(), _stream())
        return out.data

    def numpy(self) -> np.ndarray:
        return self.to_reference().cpu().numpy()

    def to_tile(self, tile: int, out: "Bands | None" = None) -> "Bands":
        """Copy into the `tile` interleave (1 = reference layout, 32)."""
        if out is None:
            out = Bands.empty(self.batch, self.n, self.lower, self.upper, tile, self.dtype, self.data.device)
        if out.tile != tile or (out.batch, out.n, out.lower, out.upper) != (self.batch, self.n, self.lower, self.upper):
            raise DimensionMismatch("to_tile: output does not match")
        _call("bgm_relayout_band", self.desc(), out.desc(), _stream())
        return out

    def transpose(self) -> "Bands":
        """bandgm::transpose (banded.cpp:159-167), materialized."""
        out = self.like(self.upper, self.lower)
        _call("bgm_transpose_band", self.desc(), out.desc(), _stream())
        return out


@dataclass
class Transposed:
    """Lazy transpose: products read the stored band transposed in place."""

    base: Bands

    @property
    def lower(self):
        return self.base.upper

    @property
    def upper(self):
        return self.base.lower


def T(b: Bands) -> Transposed:
    return Transposed(b)


@dataclass
class Vecs:
    """B vectors of length n; shape (ceil(B/32), n, 32) for tile 32, (B, n) for tile 1."""

    data: torch.Tensor
    batch: int
    n: int
    tile: int = 32

    @property
    def dtype(self):
        return self.data.dtype

    def desc(self) -> _Vec:
        return _Vec(self.data.data_ptr(), self.batch, self.n, self.tile, _dtype_code(self.data.dtype))

    @staticmethod
    def empty(batch, n, tile=32, dtype=torch.float64, device=None) -> "Vecs":
        dev = _device(device)
        if tile == 32:
            data = torch.empty((_round_up(batch, 32) // 32, n, 32), dtype=dtype, device=dev)
        else:
            data = torch.empty((batch, n), dtype=dtype, device=dev)
        return Vecs(data, batch, n, tile)

    def like(self) -> "Vecs":
        return Vecs.empty(self.batch, self.n, self.tile, self.dtype, self.data.device)

    @staticmethod
    def from_reference(arr, tile=32, dtype=torch.float64, device=None) -> "Vecs":
        dev = _device(device)
        src = torch.as_tensor(np.ascontiguousarray(arr) if isinstance(arr, np.ndarray) else arr)
        src = src.to(device=dev, dtype=dtype).contiguous()
        if src.dim() == 1:
            src = src.unsqueeze(0)
        B, n = src.shape
        flat = Vecs(src, B, n, 1)
        if tile == 1:
            return flat
        out = Vecs.empty(B, n, tile, dtype, dev)
        if B % 32:
            out.data.zero_()
        _call("bgm_relayout_vec", flat.desc(), out.desc(), _stream())
        return out

    def to_reference(self) -> torch.Tensor:
        if self.tile == 1:
            return self.data
        out = Vecs.empty(self.batch, self.n, 1, self.dtype, self.data.device)
        _call("bgm_relayout_vec", self.desc(), out.desc(), _stream())
        return out.data

    def numpy(self) -> np.ndarray:
        return self.to_reference().cpu().numpy()

    def to_tile(self, tile: int, out: "Vecs | None" = None) -> "Vecs":
        if out is None:
            out = Vecs.empty(self.batch, self.n, tile, self.dtype, self.data.device)
        if out.tile != tile or (out.batch, out.n) != (self.batch, self.n):
            raise DimensionMismatch("to_tile: output does not match")
        _call("bgm_relayout_vec", self.desc(), out.desc(), _stream())
        return out


# --------------------------------------------------------------------- status
class _Status:
    def __init__(self, batch: int, device):
        self.st = torch.zeros(max(batch, 1), dtype=torch.int32, device=device)
        self.row = torch.full((max(batch, 1),), -1, dtype=torch.int64, device=device)

    def ptrs(self):
        return C.c_void_p(self.st.data_ptr()), C.c_void_p(self.row.data_ptr())

    def raise_first(self):
        st = self.st.cpu().numpy()
        bad = np.nonzero(st)[0]
        if bad.size:
            b = int(bad[0])
            code = int(st[b])
            row = int(self.row[b].item())
            raise _ROW_ERRORS.get(code, BandgmError)(row, b)


_SCRATCH_STATUS = {}


class _ScratchStatus(_Status):
    """Uninitialized status arrays reused by unchecked calls (nobody reads
    them), so a check=False call allocates and fills nothing on the device."""

    def __init__(self, st, row):
        self.st, self.row = st, row


def _status_for(batch: int, device, check: bool) -> _Status:
    if check:
        return _Status(batch, device)
    key = (str(device), max(batch, 1))
    s = _SCRATCH_STATUS.get(key)
    if s is None:
        s = _ScratchStatus(torch.empty(max(batch, 1), dtype=torch.int32, device=device),
                           torch.empty(max(batch, 1), dtype=torch.int64, device=device))
        _SCRATCH_STATUS[key] = s
    return s


def _check(status: _Status, check: bool):
    if check:
        status.raise_first()
    return status


def _same(*xs):
    b = xs[0]
    for x in xs[1:]:
        if x.batch != b.batch or x.n != b.n:
            raise DimensionMismatch("batch/size mismatch")


# --------------------------------------------------------------------- forward ops
def cholesky(q: Bands, check: bool = True) -> Bands:
    """ops::cholesky (kernels.hpp:25): lower factor of a symmetric lower store."""
    if q.upper != 0:
        raise DimensionMismatch("cholesky expects a symmetric lower store")
    l = q.like()
    s = _status_for(q.batch, q.data.device, check)
    _call("bgm_cholesky", q.desc(), l.desc(), *s.ptrs(), _stream())
    _check(s, check)
    return l


def solve_vec(l: Bands, v: Vecs, transpose_l: bool = False, check: bool = True) -> Vecs:
    """ops::solve_vec (kernels.hpp:30-31)."""
    if l.upper != 0:
        raise DimensionMismatch("solve_vec: factor must be lower triangular")
    _same(l, v)
    x = Vecs.empty(v.batch, v.n, v.tile, v.dtype, v.data.device)
    s = _status_for(l.batch, l.data.device, check)
    _call("bgm_solve_vec", l.desc(), v.desc(), C.c_int(int(transpose_l)), x.desc(), *s.ptrs(), _stream())
    _check(s, check)
    return x


def solve_mat(l: Bands, r: Bands, out_lower: int, out_upper: int, transpose_l: bool = False,
              check: bool = True) -> Bands:
    """ops::solve_mat (kernels.hpp:40-42)."""
    if l.upper != 0:
        raise DimensionMismatch("solve_mat: factor must be lower triangular")
    _same(l, r)
    n = l.n
    out = Bands.empty(l.batch, n, min(out_lower, n - 1), min(out_upper, n - 1), l.tile, l.dtype, l.data.device)
    s = _status_for(l.batch, l.data.device, check)
    _call("bgm_solve_mat", l.desc(), r.desc(), C.c_int(int(transpose_l)), out.desc(), *s.ptrs(), _stream())
    _check(s, check)
    return out


def sparse_inverse_subset(l: Bands, check: bool = True) -> Bands:
    """ops::sparse_inverse_subset (kernels.hpp:47): symmetric lower store."""
    if l.upper != 0:
        raise DimensionMismatch("sparse_inverse_subset: factor must be lower triangular")
    out = l.like()
    s = _status_for(l.batch, l.data.device, check)
    _call("bgm_sparse_inverse_subset", l.desc(), out.desc(), *s.ptrs(), _stream())
    _check(s, check)
    return out


def _operand(x):
    return (x.base, 1) if isinstance(x, Transposed) else (x, 0)


def product_band_band_restricted(a, b, out_lower: int, out_upper: int) -> Bands:
    """ops::product_band_band_restricted (kernels.hpp:55-57); a/b may be T(x)."""
    A, ta = _operand(a)
    Bm, tb = _operand(b)
    _same(A, Bm)
    n = A.n
    c = Bands.empty(A.batch, n, min(out_lower, max(n - 1, 0)), min(out_upper, max(n - 1, 0)), A.tile,
                    A.dtype, A.data.device)
    _call("bgm_product_band_band", A.desc(), C.c_int(ta), Bm.desc(), C.c_int(tb), c.desc(), _stream())
    return c


def product_band_band(a, b) -> Bands:
    """ops::product_band_band (kernels.hpp:50): full product band."""
    return product_band_band_restricted(a, b, a.lower + b.lower, a.upper + b.upper)


def product_band_vec(b: Bands, v: Vecs, transpose_b: bool = False) -> Vecs:
    """ops::product_band_vec (kernels.hpp:61-62)."""
    _same(b, v)
    y = v.like()
    _call("bgm_product_band_vec", b.desc(), v.desc(), C.c_int(int(transpose_b)), y.desc(), _stream())
    return y


def outer_band(m: Vecs, v: Vecs, lower: int, upper: int) -> Bands:
    """ops::outer_band (kernels.hpp:66-67)."""
    _same(m, v)
    n = m.n
    out = Bands.empty(m.batch, n, min(lower, max(n - 1, 0)), min(upper, max(n - 1, 0)), m.tile, m.dtype,
                      m.data.device)
    _call("bgm_outer_band", m.desc(), v.desc(), C.c_double(1.0), out.desc(), _stream())
    return out


def log_det_from_cholesky(l: Bands, check: bool = True) -> torch.Tensor:
    """ops::log_det_from_cholesky (kernels.hpp:72): one value per matrix."""
    out = torch.empty(l.batch, dtype=l.dtype, device=l.data.device)
    s = _status_for(l.batch, l.data.device, check)
    _call("bgm_log_det", l.desc(), C.c_void_p(out.data_ptr()), *s.ptrs(), _stream())
    _check(s, check)
    return out


# --------------------------------------------------------------------- reverse ops
def vjp_cholesky(l: Bands, l_bar: Bands) -> Bands:
    """grad::vjp_cholesky (grad.hpp:24).  Like the reference (l_bar by value),
    the caller's l_bar is left untouched; a device copy is consumed."""
    if l_bar.lower != l.lower or l_bar.upper != 0 or l_bar.n != l.n:
        raise DimensionMismatch("vjp_cholesky: factor and adjoint must share a lower band")
    scratch = Bands(l_bar.data.clone(), l_bar.batch, l_bar.n, l_bar.lower, l_bar.upper, l_bar.tile)
    q_bar = l.like()
    _call("bgm_vjp_cholesky", l.desc(), scratch.desc(), q_bar.desc(), _stream())
    return q_bar


def vjp_solve_vec(l: Bands, s: Vecs, s_bar: Vecs, transpose_l: bool, check: bool = True):
    """grad::vjp_solve_vec (grad.hpp:31-32) -> (l_bar, v_bar)."""
    l_bar = l.like()
    v_bar = s.like()
    st = _status_for(l.batch, l.data.device, check)
    _call("bgm_vjp_solve_vec", l.desc(), s.desc(), s_bar.desc(), C.c_int(int(transpose_l)), l_bar.desc(),
          v_bar.desc(), *st.ptrs(), _stream())
    _check(st, check)
    return l_bar, v_bar


def vjp_solve_mat(l: Bands, s: Bands, s_bar: Bands, r_band_lower: int, r_band_upper: int,
                  transpose_l: bool, check: bool = True):
    """grad::vjp_solve_mat (grad.hpp:40-42) -> (l_bar, r_bar)."""
    n = l.n
    l_bar = l.like()
    r_bar = Bands.empty(l.batch, n, min(r_band_lower, n - 1), min(r_band_upper, n - 1), l.tile, l.dtype,
                        l.data.device)
    st = _status_for(l.batch, l.data.device, check)
    _call("bgm_vjp_solve_mat", l.desc(), s.desc(), s_bar.desc(), C.c_int(int(transpose_l)), l_bar.desc(),
          r_bar.desc(), *st.ptrs(), _stream())
    _check(st, check)
    return l_bar, r_bar


def vjp_sparse_inverse_subset(l: Bands, s: Bands, s_bar: Bands, check: bool = True) -> Bands:
    """grad::vjp_sparse_inverse_subset (grad.hpp:46-47)."""
    if s.lower != l.lower or s_bar.lower != l.lower or s.n != l.n or s_bar.n != l.n:
        raise DimensionMismatch("vjp_sparse_inverse_subset: shape mismatch")
    l_bar = l.like()
    st = _status_for(l.batch, l.data.device, check)
    _call("bgm_vjp_sparse_inverse_subset", l.desc(), s.desc(), s_bar.desc(), l_bar.desc(), *st.ptrs(),
          _stream())
    _check(st, check)
    return l_bar


def vjp_product_band_band(a: Bands, b: Bands, p_bar: Bands):
    """grad::vjp_product_band_band (grad.hpp:55-56) -> (a_bar, b_bar)."""
    a_bar = a.like()
    b_bar = b.like()
    _call("bgm_vjp_product_band_band", a.desc(), b.desc(), p_bar.desc(), a_bar.desc(), b_bar.desc(), _stream())
    return a_bar, b_bar


def vjp_product_band_vec(b: Bands, v: Vecs, p_bar: Vecs, transpose_b: bool):
    """grad::vjp_product_band_vec (grad.hpp:62-63) -> (b_bar, v_bar)."""
    b_bar = b.like()
    v_bar = v.like()
    _call("bgm_vjp_product_band_vec", b.desc(), v.desc(), p_bar.desc(), C.c_int(int(transpose_b)),
          b_bar.desc(), v_bar.desc(), _stream())
    return b_bar, v_bar


def vjp_outer_band(m: Vecs, v: Vecs, o_bar: Bands):
    """grad::vjp_outer_band (grad.hpp:69-70) -> (m_bar, v_bar)."""
    m_bar, v_bar = m.like(), v.like()
    _call("bgm_vjp_outer_band", m.desc(), v.desc(), o_bar.desc(), m_bar.desc(), v_bar.desc(), _stream())
    return m_bar, v_bar


def vjp_log_det_from_cholesky(l: Bands, c_bar) -> Bands:
    """grad::vjp_log_det_from_cholesky (grad.hpp:73); c_bar scalar or (B,)."""
    cb = torch.as_tensor(c_bar, dtype=l.dtype, device=l.data.device).expand(l.batch).contiguous()
    l_bar = l.like()
    _call("bgm_vjp_log_det", l.desc(), C.c_void_p(cb.data_ptr()), l_bar.desc(), _stream())
    return l_bar


# --------------------------------------------------------------------- VI objective
def trace_product_sym(a: Bands, b: Bands) -> torch.Tensor:
    """Tape::trace_product_sym (tape.cpp:274-284) of two symmetric lower
    stores: (B,) tensor of tr(A B) over their common band.  fp64."""
    _same(a, b)
    out = torch.empty(a.batch, dtype=torch.float64, device=a.data.device)
    _call("bgm_trace_product_sym", a.desc(), b.desc(), C.c_void_p(out.data_ptr()), _stream())
    return out


def vjp_trace_product_sym(a: Bands, b: Bands, c_bar):
    """Reverse of trace_product_sym (tape.cpp:285-301) -> (a_bar, b_bar),
    stored-cell convention; c_bar scalar or (B,)."""
    cb = torch.as_tensor(c_bar, dtype=torch.float64, device=a.data.device).expand(a.batch).contiguous()
    a_bar, b_bar = a.like(), b.like()
    _call("bgm_vjp_trace_product_sym", a.desc(), b.desc(), C.c_void_p(cb.data_ptr()), a_bar.desc(), b_bar.desc(),
          _stream())
    return a_bar, b_bar


def kl_divergence_grad(m_q: Vecs, l_q: Bands, m_p: Vecs, l_p: Bands, check: bool = True):
    """infer::kl_divergence (inference.cpp:247-268): KL(q || p) for
    q = N(m_q, (L_q L_q^T)^-1), p = N(m_p, (L_p L_p^T)^-1), per matrix, with
    its gradient in the variational parameters.  Returns (kl[B], m_q_bar,
    l_q_bar).  L_q's band must cover L_p's (DimensionMismatch otherwise)."""
    if l_q.lower < l_p.lower:
        raise DimensionMismatch("kl: variational band must cover the prior band")
    _same(l_q, m_q)
    _same(l_q, l_p)
    kl = torch.empty(l_q.batch, dtype=torch.float64, device=l_q.data.device)
    m_bar, l_bar = m_q.like(), l_q.like()
    st = _status_for(l_q.batch, l_q.data.device, check)
    _call("bgm_kl_divergence_grad", m_q.desc(), l_q.desc(), m_p.desc(), l_p.desc(), C.c_void_p(kl.data_ptr()),
          m_bar.desc(), l_bar.desc(), *st.ptrs(), _stream())
    _check(st, check)
    return kl, m_bar, l_bar


def selection(observed, batch: int, n: int, tile: int = 32, device=None) -> Vecs:
    """models::SelectionIndex (models.hpp:122-128) as the device's 0/1 mask:
    ``observed`` = sorted latent indices observed in every matrix of the batch
    (or a (batch, n) boolean array).  Pair it with y / weight scattered to full
    length (models::scatter, models.hpp:131); unobserved entries are ignored."""
    obs = np.asarray(observed)
    if obs.ndim == 2:
        if obs.shape != (batch, n):
            raise DimensionMismatch("selection mask shape")
        mask = obs.astype(np.float64)
    else:
        idx = obs.astype(np.int64)
        if idx.size and (idx.min() < 0 or idx.max() >= n or np.any(np.diff(idx) <= 0)):
            raise BandgmError("selection indices must be sorted, unique and inside [0, n)")
        mask = np.zeros((batch, n))
        mask[:, idx] = 1.0
    return Vecs.from_reference(mask, tile=tile, device=device)


def elbo_gaussian_grad(m_q: Vecs, l_q: Bands, m_p: Vecs, l_p: Bands, y: Vecs, tau2: float, check: bool = True,
                       observed: Vecs | None = None):
    """infer::elbo (inference.cpp:276-287) for a Gaussian likelihood:
    E_q log N(y | F, tau2 I) - KL(q || p) per matrix, over every latent or,
    with ``observed`` (a ``selection`` mask), over the observed ones only.
    Returns (elbo[B], kl[B], m_q_bar, l_q_bar, tau2_bar[B]) -- the ELBO's
    gradient in the variational parameters and its tau2 partial."""
    if l_q.lower < l_p.lower:
        raise DimensionMismatch("kl: variational band must cover the prior band")
    if not tau2 > 0:
        raise BandgmError("parameter 'tau2' must be strictly positive")
    _same(l_q, m_q)
    _same(l_q, l_p)
    _same(l_q, y)
    dev = l_q.data.device
    elbo, kl, tb = (torch.empty(l_q.batch, dtype=torch.float64, device=dev) for _ in range(3))
    m_bar, l_bar = m_q.like(), l_q.like()
    st = _status_for(l_q.batch, dev, check)
    if observed is None:
        _call("bgm_elbo_gaussian_grad", m_q.desc(), l_q.desc(), m_p.desc(), l_p.desc(), y.desc(), C.c_double(tau2),
              C.c_void_p(elbo.data_ptr()), C.c_void_p(kl.data_ptr()), m_bar.desc(), l_bar.desc(),
              C.c_void_p(tb.data_ptr()), *st.ptrs(), _stream())
    else:
        _same(l_q, observed)
        _call("bgm_elbo_gaussian_grad_sel", m_q.desc(), l_q.desc(), m_p.desc(), l_p.desc(), y.desc(),
              observed.desc(), C.c_double(tau2), C.c_void_p(elbo.data_ptr()), C.c_void_p(kl.data_ptr()),
              m_bar.desc(), l_bar.desc(), C.c_void_p(tb.data_ptr()), *st.ptrs(), _stream())
    _check(st, check)
    return elbo, kl, m_bar, l_bar, tb


def elbo_poisson_grad(m_q: Vecs, l_q: Bands, m_p: Vecs, l_p: Bands, y: Vecs, weight: Vecs, quad_points: int = 20,
                      check: bool = True, observed: Vecs | None = None):
    """infer::elbo (inference.cpp:276-287) for a Poisson likelihood with
    exposure weights observing every latent; the expectation by
    ``quad_points``-node Gauss-Hermite quadrature (inference.cpp:65-100).
    Returns (elbo[B], kl[B], m_q_bar, l_q_bar).  A non-positive weight raises
    (the reference's NonPositiveParam) with its observation index."""
    if l_q.lower < l_p.lower:
        raise DimensionMismatch("kl: variational band must cover the prior band")
    if not 1 <= quad_points <= 64:
        raise BandgmError("parameter 'quad_points' must be in [1, 64]")
    for x in (m_q, l_p, y, weight):
        _same(l_q, x)
    dev = l_q.data.device
    elbo, kl = (torch.empty(l_q.batch, dtype=torch.float64, device=dev) for _ in range(2))
    m_bar, l_bar = m_q.like(), l_q.like()
    st = _status_for(l_q.batch, dev, check)
    if observed is None:
        _call("bgm_elbo_poisson_grad", m_q.desc(), l_q.desc(), m_p.desc(), l_p.desc(), y.desc(), weight.desc(),
              C.c_int(quad_points), C.c_void_p(elbo.data_ptr()), C.c_void_p(kl.data_ptr()), m_bar.desc(),
              l_bar.desc(), *st.ptrs(), _stream())
    else:  # partial SelectionIndex: only observed latents' weights are vetted
        _same(l_q, observed)
        _call("bgm_elbo_poisson_grad_sel", m_q.desc(), l_q.desc(), m_p.desc(), l_p.desc(), y.desc(), weight.desc(),
              observed.desc(), C.c_int(quad_points), C.c_void_p(elbo.data_ptr()), C.c_void_p(kl.data_ptr()),
              m_bar.desc(), l_bar.desc(), *st.ptrs(), _stream())
    if check:
        stn = st.st.cpu().numpy()
        bad = np.nonzero(stn == BGM_ERR_ARG)[0]
        if bad.size:
            b = int(bad[0])
            raise BandgmError(f"parameter 'weight' must be strictly positive (observation {int(st.row[b])}, "
                              f"batch matrix {b})")
    _check(st, check)
    return elbo, kl, m_bar, l_bar


def gauss_hermite(quad_points: int):
    """infer::gauss_hermite (inference.cpp:120-137): (nodes, weights), ascending."""
    x = (C.c_double * quad_points)()
    w = (C.c_double * quad_points)()
    if library().bgm_gauss_hermite(C.c_int(quad_points), x, w) != BGM_OK:
        raise BandgmError("parameter 'quad_points' must be in [1, 64]")
    return np.array(x[:]), np.array(w[:])


# --------------------------------------------------------------------- model assembly
class SingularBlock(_RowError):
    """errors.hpp (models.cpp:27): a state-space block is not SPD; .row = block."""
    what = "state-space block is not positive definite"


def prior_natural_params(a, b, q, mu0, sigma0, tile: int = 32, check: bool = True):
    """models::prior_natural_params (models.cpp:165-189), batched: B models
    with d-dim states and T transitions, given as tensors a, q (B, T, d, d),
    b (B, T, d), mu0 (B, d), sigma0 (B, d, d).  Returns (Lambda, eta): the
    joint prior precision as a symmetric lower store (Bands, n = (T+1) d,
    band 2d-1) and eta = Lambda m (Vecs)."""
    dev = _device()
    t = [torch.as_tensor(x, dtype=torch.float64).to(dev).contiguous() for x in (a, b, q, mu0, sigma0)]
    a, b, q, mu0, sigma0 = t
    B, T, d, _ = a.shape
    if b.shape != (B, T, d) or q.shape != (B, T, d, d) or mu0.shape != (B, d) or sigma0.shape != (B, d, d):
        raise DimensionMismatch("prior_natural_params: block shapes do not agree")
    if T < 1 or d < 1:
        raise BandgmError("state-space model is empty")
    if d > 8:
        raise BandgmError("prior_natural_params: state dimension above 8 is not supported")
    n = (T + 1) * d
    lam = Bands.empty(B, n, 2 * d - 1, 0, tile, torch.float64, dev)
    eta = Vecs.empty(B, n, tile, torch.float64, dev)
    if B % tile:
        eta.data.zero_()  # padding lanes of a partial tile (lambda's are cleared on the device)
    st = _status_for(B, dev, check)
    _call("bgm_prior_natural_params", C.c_int64(B), C.c_int(d), C.c_int64(T), *(C.c_void_p(x.data_ptr()) for x in t),
          lam.desc(), eta.desc(), *st.ptrs(), _stream())
    if check:
        stn = st.st.cpu().numpy()
        bad = np.nonzero(stn)[0]
        if bad.size:
            m = int(bad[0])
            raise SingularBlock(int(st.row[m]), m)
    return lam, eta


def vjp_prior_natural_params(a, b, q, mu0, sigma0, lam_bar: Bands, eta_bar: Vecs, check: bool = True):
    """Reverse of prior_natural_params: cotangents of (Lambda, eta) -> those
    of (a, b, q, mu0, sigma0), analytically -- the replacement of the
    reference's finite-difference compose_precision_gradient
    (inference.cpp:360-380) for this assembly.  Lambda's cotangent follows the
    stored-cell convention (grad.hpp:4-8); q and sigma0 are read through their
    lower triangles, so their cotangents are lower-folded."""
    dev = _device()
    t = [torch.as_tensor(x, dtype=torch.float64).to(dev).contiguous() for x in (a, b, q, mu0, sigma0)]
    a, b, q, mu0, sigma0 = t
    B, T, d, _ = a.shape
    n = (T + 1) * d
    if (lam_bar.batch, lam_bar.n, lam_bar.lower, lam_bar.upper) != (B, n, 2 * d - 1, 0) or eta_bar.n != n:
        raise DimensionMismatch("vjp_prior_natural_params: cotangent shapes do not agree")
    bars = [torch.empty_like(x) for x in t]
    st = _status_for(B, dev, check)
    _call("bgm_vjp_prior_natural_params", C.c_int64(B), C.c_int(d), C.c_int64(T),
          *(C.c_void_p(x.data_ptr()) for x in t), lam_bar.desc(), eta_bar.desc(),
          *(C.c_void_p(x.data_ptr()) for x in bars), *st.ptrs(), _stream())
    if check:
        stn = st.st.cpu().numpy()
        bad = np.nonzero(stn)[0]
        if bad.size:
            m = int(bad[0])
            raise SingularBlock(int(st.row[m]), m)
    return tuple(bars)


# --------------------------------------------------------------------- config 3
def marginal_likelihood_grad(L: Bands, y: Vecs, tau2: float, check: bool = True, out=None):
    """Config-3 learning step: per matrix, the log marginal
    likelihood of y under precision Q = band(L L^T) with noise tau2
    (infer::marginal_likelihood_partial, inference.cpp:140-163), dL (through
    grad::vjp_product_band_band(L, L^T, Q_bar)) and d tau2.
    Returns (loss[B], l_bar, tau2_bar[B])."""
    if L.upper != 0:
        raise DimensionMismatch("marginal_likelihood_grad: L must be lower triangular")
    if not tau2 > 0:
        raise BandgmError("parameter 'tau2' must be strictly positive")
    _same(L, y)
    dev = L.data.device
    if out is None:
        loss = torch.empty(L.batch, dtype=torch.float64, device=dev)
        tbar = torch.empty(L.batch, dtype=torch.float64, device=dev)
        l_bar = L.like()
        st = _Status(L.batch, dev)
    else:
        loss, l_bar, tbar, st = out
    _call("bgm_marginal_likelihood_grad", L.desc(), y.desc(), C.c_double(tau2), C.c_void_p(loss.data_ptr()),
          l_bar.desc(), C.c_void_p(tbar.data_ptr()), *st.ptrs(), _stream())
    _check(st, check)
    return loss, l_bar, tbar


def set_segment_rows(rows: int) -> None:
    """Segment length of the segment-parallel sweeps (0 = automatic)."""
    _call("bgm_set_segment_rows", C.c_int64(rows))


def debug_repairs(reset: bool = True, with_dev: bool = False):
    """Matrices re-run on the exact single-unit path since the last reset
    (and, with BGM_DEBUG set, the largest relative burn-in deviation)."""
    v = C.c_int64(0)
    d = C.c_double(0.0)
    _call("bgm_debug_repairs", C.byref(v), C.byref(d), C.c_int(int(reset)))
    return (int(v.value), float(d.value)) if with_dev else int(v.value)


def new_status(batch: int, device=None) -> _Status:
    return _Status(batch, _device(device))


def fp64_peak():
    """Measured (DFMA, DMMA) FP64 peaks of the current device, TFLOP/s
    (microbenchmarks in csrc/bgm_peak.cu; synchronizing)."""
    a, b = C.c_double(0.0), C.c_double(0.0)
    _call("bgm_fp64_peak", C.byref(a), C.byref(b), _stream())
    return float(a.value), float(b.value)
