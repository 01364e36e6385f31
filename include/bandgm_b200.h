/*
 * bandgm_b200 -- C ABI of the B200 (sm_100a) banded operator library.
 *
 * This is the drop-in boundary under the reference's C++ operator API
 * (/root/reference/proj/include/bandgm/{kernels,grad}.hpp).  The reference
 * exposes no C ABI of its own; each entry point below states the reference
 * function it replaces.  The C++ drop-in layer
 * (paper_1902_10078_b200/cpp/include/bandgm/{banded,errors,kernels,grad}.hpp)
 * and the Python host
 * package call only these symbols.  INTEGRATION.md shows the bindings.
 *
 * Conventions
 * -----------
 * - All data pointers are DEVICE pointers; every call is asynchronous on
 *   `stream` (0 = legacy default stream).  No torch types cross this ABI.
 * - A batch of B independent n x n bands (`bgm_band`) is stored
 *   batch-interleaved with interleave width `tile` (1 or 32):
 *       element (b, r, j) -> ((b / tile) * n * w + j * w + r) * tile + b % tile
 *   where w = lower + upper + 1 and r = i - j + upper is the storage row of
 *   matrix entry (i, j) -- the reference storage convention (banded.hpp:1-11).
 *   tile = 1 is exactly the reference's per-matrix column-major block, one
 *   matrix after another; tile = 32 puts 32 matrices side by side so a warp
 *   reads 32 matrices' copies of one cell in one 256-byte transaction.  The
 *   allocation must cover round_up(B, tile) matrices.  Corner cells (storage
 *   cells mapping outside the matrix) are written as exact zeros.
 * - Vectors (`bgm_vec`): element (b, i) -> ((b / tile) * n + i) * tile + b % tile.
 * - Symmetric bands are stored as their lower band (upper = 0) and read
 *   mirrored; symmetric adjoints follow the reference's stored-cell
 *   convention (grad.hpp:4-8).
 * - Per-matrix error reporting: `status` (int32, device, length B; may be
 *   NULL) receives BGM_OK or the op's error code, `row` (int64, device,
 *   length B; may be NULL) the first failing row or -1 -- the row the
 *   reference's exception would carry (errors.hpp:27-50).  The returned int
 *   covers argument validation and launch errors only (synchronous part).
 * - dtype: BGM_F64 everywhere; BGM_F32 is accepted by the factorization,
 *   solve, log-det, inverse-subset and their adjoints (config 4's fp32 runs).
 */
#ifndef BANDGM_B200_H
#define BANDGM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BGM_OK = 0,
  BGM_ERR_NOT_PD = 1,        /* NotPositiveDefinite  (errors.hpp:27-34) */
  BGM_ERR_SINGULAR = 2,      /* SingularDiagonal     (errors.hpp:36-43) */
  BGM_ERR_NONPOS_DIAG = 3,   /* NonPositiveDiagonal  (errors.hpp:45-50) */
  BGM_ERR_DIM = 4,           /* DimensionMismatch    (errors.hpp:9-11)  */
  BGM_ERR_ARG = 5,           /* malformed descriptor / unsupported combination */
  BGM_ERR_CUDA = 6           /* launch or allocation failure */
};

enum { BGM_F64 = 0, BGM_F32 = 1 };

typedef struct bgm_band {
  void* data;
  int64_t batch;
  int64_t n;
  int32_t lower;
  int32_t upper;
  int32_t tile;  /* 1 or 32 */
  int32_t dtype; /* BGM_F64 / BGM_F32 */
} bgm_band;

typedef struct bgm_vec {
  void* data;
  int64_t batch;
  int64_t n;
  int32_t tile;
  int32_t dtype;
} bgm_vec;

typedef void* bgm_stream; /* cudaStream_t */

/* ---------------------------------------------------------------- info */
int bgm_abi_version(void);
const char* bgm_status_name(int status);
/* Last CUDA error text seen by the library on this thread. */
const char* bgm_last_error(void);

/* -------------------------------------------------------- layout helpers */
/* Re-lays a band batch between interleave widths (same n, lower, upper,
 * dtype).  Used to move reference-layout blocks (tile 1) in and out. */
int bgm_relayout_band(bgm_band src, bgm_band dst, bgm_stream stream);
int bgm_relayout_vec(bgm_vec src, bgm_vec dst, bgm_stream stream);
/* bandgm::transpose (banded.hpp:166; banded.cpp:159-167): dst (upper, lower)
 * receives the transpose of src (lower, upper).  The products below read
 * transposes in place, so this is only needed to materialize one. */
int bgm_transpose_band(bgm_band src, bgm_band dst, bgm_stream stream);

/* ---------------------------------------------------------------- forward */
/* ops::cholesky (kernels.hpp:25; kernels_serial.cpp:12-32).  q: lower band
 * (bw, 0) of a symmetric matrix; l: (bw, 0).  Error: BGM_ERR_NOT_PD. */
int bgm_cholesky(bgm_band q, bgm_band l, int32_t* status, int64_t* row, bgm_stream stream);

/* ops::solve_vec (kernels.hpp:30-31; kernels_serial.cpp:34-60).
 * x = L^{-1} v, or L^{-T} v when transpose != 0.  Error: BGM_ERR_SINGULAR. */
int bgm_solve_vec(bgm_band l, bgm_vec v, int transpose, bgm_vec x, int32_t* status, int64_t* row,
                  bgm_stream stream);

/* ops::log_det_from_cholesky (kernels.hpp:72; kernels.cpp:121-129).
 * out: B values (device, l's dtype).  Error: BGM_ERR_NONPOS_DIAG. */
int bgm_log_det(bgm_band l, void* out, int32_t* status, int64_t* row, bgm_stream stream);

/* ops::sparse_inverse_subset (kernels.hpp:47; kernels_serial.cpp:80-104).
 * s: lower store (bw, 0) of the band of (L L^T)^{-1}.  Error: BGM_ERR_SINGULAR. */
int bgm_sparse_inverse_subset(bgm_band l, bgm_band s, int32_t* status, int64_t* row,
                              bgm_stream stream);

/* ops::product_band_band[_restricted] (kernels.hpp:50-57; kernels_detail.hpp:16-28).
 * c = op(a) * op(b) restricted to c's band; op(x) = x^T when trans_x != 0
 * (reads the transpose in place; the reference materializes it,
 * banded.cpp:159-167).  c's band must already be clipped to n-1. */
int bgm_product_band_band(bgm_band a, int trans_a, bgm_band b, int trans_b, bgm_band c,
                          bgm_stream stream);

/* ops::product_band_vec (kernels.hpp:61-62; kernels_detail.hpp:31-45). */
int bgm_product_band_vec(bgm_band b, bgm_vec v, int transpose, bgm_vec y, bgm_stream stream);

/* ops::outer_band (kernels.hpp:66-67; kernels_detail.hpp:48-54):
 * out = scale * band(m v^T) on out's band. */
int bgm_outer_band(bgm_vec m, bgm_vec v, double scale, bgm_band out, bgm_stream stream);

/* ops::solve_mat (kernels.hpp:40-42; kernels_serial.cpp:62-78; PAPER Alg. 4).
 * out's band (already clipped) is the requested (out_lower, out_upper). */
int bgm_solve_mat(bgm_band l, bgm_band r, int transpose, bgm_band out, int32_t* status,
                  int64_t* row, bgm_stream stream);

/* ---------------------------------------------------------------- reverse */
/* grad::vjp_cholesky (grad.hpp:24; grad.cpp:11-36).  l_bar is CONSUMED
 * (overwritten), as the reference takes it by value and consumes it. */
int bgm_vjp_cholesky(bgm_band l, bgm_band l_bar_consumed, bgm_band q_bar, bgm_stream stream);

/* grad::vjp_solve_vec (grad.hpp:31-32; grad.cpp:38-49). */
int bgm_vjp_solve_vec(bgm_band l, bgm_vec s, bgm_vec s_bar, int transpose, bgm_band l_bar,
                      bgm_vec v_bar, int32_t* status, int64_t* row, bgm_stream stream);

/* grad::vjp_sparse_inverse_subset (grad.hpp:46-47; grad.cpp:84-143). */
int bgm_vjp_sparse_inverse_subset(bgm_band l, bgm_band s, bgm_band s_bar, bgm_band l_bar,
                                  int32_t* status, int64_t* row, bgm_stream stream);

/* grad::vjp_product_band_band (grad.hpp:55-56; grad.cpp:145-151). */
int bgm_vjp_product_band_band(bgm_band a, bgm_band b, bgm_band p_bar, bgm_band a_bar,
                              bgm_band b_bar, bgm_stream stream);

/* grad::vjp_product_band_vec (grad.hpp:62-63; grad.cpp:153-162). */
int bgm_vjp_product_band_vec(bgm_band b, bgm_vec v, bgm_vec p_bar, int transpose, bgm_band b_bar,
                             bgm_vec v_bar, bgm_stream stream);

/* grad::vjp_outer_band (grad.hpp:69-70; grad.cpp:164-170). */
int bgm_vjp_outer_band(bgm_vec m, bgm_vec v, bgm_band o_bar, bgm_vec m_bar, bgm_vec v_bar,
                       bgm_stream stream);

/* grad::vjp_log_det_from_cholesky (grad.hpp:73; grad.cpp:172-176).
 * c_bar: B device values (l's dtype). */
int bgm_vjp_log_det(bgm_band l, const void* c_bar, bgm_band l_bar, bgm_stream stream);

/* grad::vjp_solve_mat (grad.hpp:40-42; grad.cpp:51-82).  r_bar's band is
 * band(r) clipped to n-1. */
int bgm_vjp_solve_mat(bgm_band l, bgm_band s, bgm_band s_bar, int transpose, bgm_band l_bar,
                      bgm_band r_bar, int32_t* status, int64_t* row, bgm_stream stream);

/* ------------------------------------------------- config-3 learning step */
/* Gaussian log marginal likelihood of y under N(0, Q^{-1} + tau2 I) with
 * Q = band(L L^T), and its reverse pass, per matrix:
 *   infer::marginal_likelihood_partial (inference.cpp:140-163) with every
 *   node observed, precision_from_factor (inference.cpp:23-26), and the dL
 *   chain grad::vjp_product_band_band(L, L^T, Q_bar) (grad.cpp:145-151).
 * Outputs per matrix: loss[b], l_bar (band of L), tau2_bar[b].
 * Fused: two sweeps (forward factor+solve, reverse inverse-subset + adjoint)
 * instead of the reference's 2 x cholesky, 2 x vjp_cholesky, solve,
 * vjp_solve and products.  Errors: BGM_ERR_NOT_PD (posterior factor). */
int bgm_marginal_likelihood_grad(bgm_band l, bgm_vec y, double tau2, double* loss,
                                 bgm_band l_bar, double* tau2_bar, int32_t* status, int64_t* row,
                                 bgm_stream stream);

/* ------------------------------------------------- VI objective */
/* Tape::trace_product_sym (tape.cpp:274-302): per matrix
 * sum_j a(j,j) b(j,j) + 2 sum_{0 < i-j <= min(bw_a, bw_b)} a(i,j) b(i,j)
 * of two symmetric lower stores.  out: B device doubles.  fp64. */
int bgm_trace_product_sym(bgm_band a, bgm_band b, double* out, bgm_stream stream);

/* Reverse of trace_product_sym (tape.cpp:285-301): a_bar = c_bar * seed(b)
 * on band(a), b_bar = c_bar * seed(a) on band(b), seed(x) = x on the
 * diagonal and 2x below it (stored-cell convention).  c_bar: B device
 * doubles; either output may have data == NULL (not wanted).  fp64. */
int bgm_vjp_trace_product_sym(bgm_band a, bgm_band b, const double* c_bar, bgm_band a_bar,
                              bgm_band b_bar, bgm_stream stream);

/* infer::kl_divergence (inference.cpp:247-268) and its gradient:
 * KL(N(m_q, (L_q L_q^T)^-1) || N(m_p, (L_p L_p^T)^-1)) per matrix,
 *   = 1/2 [ tr(Q_p S_q) + 2 (log|L_q| - log|L_p|) + |L_p^T (m_p - m_q)|^2 - n ]
 * with S_q the inverse subset of L_q and Q_p = band(L_p L_p^T).  Outputs kl
 * (B device doubles), m_q_bar and l_q_bar (stored cells).  L_q's band must
 * cover L_p's (BGM_ERR_DIM otherwise, as the reference).  Errors, first of
 * log|L_p| (NONPOS_DIAG), the subset of L_q (SINGULAR), log|L_q|
 * (NONPOS_DIAG).  fp64. */
int bgm_kl_divergence_grad(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, double* kl,
                           bgm_vec m_q_bar, bgm_band l_q_bar, int32_t* status, int64_t* row,
                           bgm_stream stream);

/* infer::elbo (inference.cpp:276-287) for a Gaussian likelihood observing
 * every latent (selection = identity): E_q[log N(y | F, tau2 I)] - KL(q || p),
 * the expected log-likelihood in closed form (inference.cpp:52-63) with the
 * marginal variances diag(S_q).  Outputs elbo and kl (B device doubles each),
 * the ELBO's gradient in m_q and L_q, and optionally (tau2_bar != NULL) its
 * tau2 partial.  Errors as bgm_kl_divergence_grad; tau2 <= 0: BGM_ERR_ARG.  fp64. */
int bgm_elbo_gaussian_grad(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, double tau2,
                           double* elbo, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar, double* tau2_bar,
                           int32_t* status, int64_t* row, bgm_stream stream);

/* infer::elbo (inference.cpp:276-287) for a Poisson likelihood with
 * per-observation exposure weights observing every latent: the expected
 * log-likelihood by quad_points-node Gauss-Hermite quadrature
 * (inference.cpp:65-100, 120-137) minus KL(q || p), with the ELBO's gradient
 * in m_q and L_q.  A non-positive weight reports BGM_ERR_ARG at that
 * observation (the reference's NonPositiveParam).  quad_points in [1, 64].  fp64. */
int bgm_elbo_poisson_grad(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, bgm_vec weight,
                          int quad_points, double* elbo, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar,
                          int32_t* status, int64_t* row, bgm_stream stream);

/* The two ELBOs with a partial models::SelectionIndex (models.hpp:122-131,
 * inference.cpp:45-100): `observed` is a 0/1 fp64 mask of the observed latents
 * (same batch, n and tile as y); y (and weight) are scattered to full length
 * (models::scatter), their unobserved entries ignored.  Only observed latents
 * contribute to the expected log-likelihood and its gradients; the KL is over
 * every latent, as in the reference. */
int bgm_elbo_gaussian_grad_sel(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, bgm_vec observed,
                               double tau2, double* elbo, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar,
                               double* tau2_bar, int32_t* status, int64_t* row, bgm_stream stream);
int bgm_elbo_poisson_grad_sel(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, bgm_vec weight,
                              bgm_vec observed, int quad_points, double* elbo, double* kl, bgm_vec m_q_bar,
                              bgm_band l_q_bar, int32_t* status, int64_t* row, bgm_stream stream);

/* infer::gauss_hermite (inference.cpp:120-137): quad_points ascending nodes x
 * and weights w (host arrays), by the Golub-Welsch eigen-decomposition. */
int bgm_gauss_hermite(int quad_points, double* x, double* w);

/* ------------------------------------------------- model assembly */
/* models::prior_natural_params (models.cpp:165-189) for B state-space models
 * with d-dimensional states (1 <= d <= 8) and `steps` transitions, device
 * arrays, row-major blocks: a, q [B][steps][d][d], b [B][steps][d],
 * mu0 [B][d], sigma0 [B][d][d].  Writes the joint prior precision Lambda as a
 * symmetric lower store (n = (steps+1) d, lower = 2d-1, upper = 0) and
 * eta = Lambda m (m the propagated prior mean).  A block that is not SPD
 * (the reference's SingularBlock(t)) reports BGM_ERR_NOT_PD with row = t
 * (Q_{t-1} -> t, Sigma0 -> 0), in the reference's order.  fp64. */
int bgm_prior_natural_params(int64_t batch, int d, int64_t steps, const double* a, const double* b,
                             const double* q, const double* mu0, const double* sigma0, bgm_band lambda,
                             bgm_vec eta, int32_t* status, int64_t* row, bgm_stream stream);

/* Reverse of bgm_prior_natural_params, the analytic replacement of the
 * reference's central-difference compose_precision_gradient
 * (inference.cpp:360-380) for this assembly: cotangents of Lambda (stored
 * lower cells, grad.hpp:4-8) and eta -> cotangents of a, b, q, mu0, sigma0
 * (device arrays shaped as the inputs).  Q_t and Sigma0 are read through their
 * lower triangles (models.cpp:25-29), so their adjoints are lower-folded
 * (upper entries 0).  Status as the forward (SingularBlock). */
int bgm_vjp_prior_natural_params(int64_t batch, int d, int64_t steps, const double* a, const double* b,
                                 const double* q, const double* mu0, const double* sigma0, bgm_band lambda_bar,
                                 bgm_vec eta_bar, double* a_bar, double* b_bar, double* q_bar, double* mu0_bar,
                                 double* sigma0_bar, int32_t* status, int64_t* row, bgm_stream stream);

/* ------------------------------------------------- instrumentation */
/* Per-kernel CUDA-event timing on the launching stream (off by default).
 * bgm_timing_enable(1) clears and starts recording; bgm_timing_read(i, ...)
 * returns the number of distinct kernels and, for 0 <= i < that number, the
 * i-th kernel's name, summed milliseconds and launch count. */
int bgm_timing_enable(int on);
int bgm_timing_read(int idx, char* name, int name_len, double* total_ms, int64_t* count);

/* Number of matrices the segment-parallel sweeps re-ran exactly because a
 * segment's burn-in had not converged, and (BGM_DEBUG=1/2 only) the largest
 * relative burn-in deviation the checks saw (synchronizing; reset != 0 clears). */
int bgm_debug_repairs(int64_t* count, double* max_dev, int reset);

/* Calling thread only: route every operator to the one-thread-per-matrix
 * kernels that restate the reference loops (the drop-in's ops::serial::*). */
int bgm_force_generic(int on);

/* Tuning knob for the segment-parallel sweeps (0 = automatic). */
int bgm_set_segment_rows(int64_t rows);

/* Measured FP64 peaks of the current device in TFLOP/s: vector DFMA and
 * DMMA (mma.sync.m8n8k4.f64) microbenchmarks, timed with CUDA events on
 * `stream` (synchronizing).  The FP64 denominators of bench.py's rooflines;
 * no reference counterpart (the reference reports no rooflines). */
int bgm_fp64_peak(double* dfma_tflops, double* dmma_tflops, bgm_stream stream);

#ifdef __cplusplus
}
#endif

#endif /* BANDGM_B200_H */
