"""bandgm_b200 -- B200-native banded operators with reverse-mode gradients.

Python host mirror of the reference's C++ operator API
(``/root/reference/proj/include/bandgm/{kernels,grad}.hpp``) over the C ABI in
``include/bandgm_b200.h``.  Names, argument meaning and error behaviour follow
the reference (``bandgm::ops::*``, ``bandgm::grad::*``, the exception types of
``errors.hpp``), batched: every call processes ``B`` independent matrices.

PyTorch is used only for device memory, streams and ``torch.distributed``;
all arithmetic runs in the hand-written sm_100a kernels of
``libbandgm_b200.so``.  There is no CPU fallback: importing this package
without the built library, or calling it without a CUDA device, raises.
"""
from .api import (  # noqa: F401
    Bands,
    Vecs,
    BandgmError,
    DimensionMismatch,
    NotPositiveDefinite,
    NonPositiveDiagonal,
    SingularBlock,
    SingularDiagonal,
    T,
    cholesky,
    library,
    elbo_gaussian_grad,
    elbo_poisson_grad,
    gauss_hermite,
    kl_divergence_grad,
    library_path,
    log_det_from_cholesky,
    marginal_likelihood_grad,
    outer_band,
    product_band_band,
    product_band_band_restricted,
    prior_natural_params,
    product_band_vec,
    selection,
    set_segment_rows,
    solve_mat,
    solve_vec,
    sparse_inverse_subset,
    trace_product_sym,
    vjp_cholesky,
    vjp_log_det_from_cholesky,
    vjp_outer_band,
    vjp_prior_natural_params,
    vjp_product_band_band,
    vjp_product_band_vec,
    vjp_solve_mat,
    vjp_solve_vec,
    vjp_sparse_inverse_subset,
    vjp_trace_product_sym,
)

from . import autograd  # noqa: E402,F401  (torch.autograd.Function wrappers)

__all__ = [n for n in dir() if not n.startswith("_")]
