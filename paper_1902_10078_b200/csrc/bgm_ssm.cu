// Batched state-space prior assembly on the device:
// models::prior_natural_params (models.cpp:165-189).  For B linear-Gaussian
// state-space models with d-dimensional states and T transitions
// (x_0 ~ N(mu0, Sigma0), x_t = A_{t-1} x_{t-1} + b_{t-1} + N(0, Q_{t-1})),
// the joint prior over the (T+1) d stacked states has the block-tridiagonal
// precision
//   Lambda(0, 0) = Sigma0^-1 + A_0^T Q_0^-1 A_0,
//   Lambda(t, t) = Q_{t-1}^-1 + A_t^T Q_t^-1 A_t  (the second term for t < T),
//   Lambda(t, t-1) = -Q_{t-1}^-1 A_{t-1},
// a symmetric band of half-bandwidth 2d - 1, and eta = Lambda m with the
// propagated prior mean m.  One thread per (model, block row t) inverts its
// d x d SPD blocks by Cholesky (models.cpp:25-29) and writes its band cells;
// one thread per model propagates the mean; eta is a symmetric band x vector
// product in the reference's order (to_banded + product_band_vec).
#include <cuda_runtime.h>

#include "bgm_common.cuh"
#include "bgm_timing.cuh"

namespace bgm {
namespace ssm {
namespace {

constexpr int kThreads = 128;

// inverse of an SPD d x d matrix (row-major in m) via Cholesky; false when
// the factorization fails (Eigen::LLT's info() != Success)
template <int D>
__device__ bool spd_inverse(const double* m, double (&inv)[D][D]) {
  double l[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) l[i][j] = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double s = m[j * D + j];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= l[j][k] * l[j][k];
    if (!(s > 0.0)) return false;
    l[j][j] = sqrt(s);
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double t = m[i * D + j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= l[i][k] * l[j][k];
      l[i][j] = t / l[j][j];
    }
  }
  // inv = L^-T L^-1, column by column: solve L y = e_c, then L^T x = y
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double y[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double t = i == c ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) t -= l[i][k] * y[k];
      y[i] = t / l[i][i];
    }
#pragma unroll
    for (int i = D - 1; i >= 0; --i) {
      double t = y[i];
#pragma unroll
      for (int k = i + 1; k < D; ++k) t -= l[k][i] * inv[k][c];
      inv[i][c] = t / l[i][i];
    }
  }
  return true;
}

struct Model {
  const double *a, *b, *q, *mu0, *sigma0;  // [B][T][D][D], [B][T][D], [B][T][D][D], [B][D], [B][D][D]
  ix batch, steps;
};

// Failure key per model: the reference inverts Q_0 .. Q_{T-1} first (failure
// = block t+1), then Sigma0 (block 0): keys t+1 for Q_t, T+1 for Sigma0.
template <int D>
__global__ void k_blocks(Model M, Band<double> lam, unsigned long long* fail) {
  const ix g = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix T = M.steps;
  if (g >= M.batch * (T + 1)) return;
  const ix b = g / (T + 1), t = g % (T + 1);
  const double* a = M.a + b * T * D * D;
  const double* q = M.q + b * T * D * D;
  double diag[D][D], qin[D][D];
  bool ok = true;
  if (t == 0) {
    ok = spd_inverse<D>(M.sigma0 + b * D * D, diag);
    if (!ok) atomicMin(fail + b, static_cast<unsigned long long>(T + 1));
  } else {
    ok = spd_inverse<D>(q + (t - 1) * D * D, diag);  // Q_{t-1}^-1
    if (!ok) atomicMin(fail + b, static_cast<unsigned long long>(t));
  }
  if (!ok) return;
  if (t >= 1) {  // Lambda(t, t-1) = -Q_{t-1}^-1 A_{t-1}: full d x d block below the diagonal
    const double* at = a + (t - 1) * D * D;
#pragma unroll
    for (int bi = 0; bi < D; ++bi)
#pragma unroll
      for (int bj = 0; bj < D; ++bj) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += diag[bi][k] * at[k * D + bj];
        const ix i = t * D + bi, j = (t - 1) * D + bj;
        lam.cell(b, int(i - j), j) = -s;
      }
  }
  if (t < T) {  // + A_t^T Q_t^-1 A_t
    if (!spd_inverse<D>(q + t * D * D, qin)) {
      atomicMin(fail + b, static_cast<unsigned long long>(t + 1));
      return;
    }
    const double* at = a + t * D * D;
    double qa[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += qin[i][k] * at[k * D + j];
        qa[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += at[k * D + i] * qa[k][j];
        diag[i][j] += s;
      }
  }
#pragma unroll
  for (int bj = 0; bj < D; ++bj)
#pragma unroll
    for (int bi = bj; bi < D; ++bi) {
      const ix j = t * D + bj;
      lam.cell(b, bi - bj, j) = diag[bi][bj];
    }
}

// prior mean m_0 = mu0, m_t = A_{t-1} m_{t-1} + b_{t-1} (models.cpp:183-185)
template <int D>
__global__ void k_mean(Model M, Vec<double> m) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= M.batch) return;
  double cur[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    cur[i] = M.mu0[b * D + i];
    m(b, i) = cur[i];
  }
  for (ix t = 1; t <= M.steps; ++t) {
    const double* at = M.a + (b * M.steps + t - 1) * D * D;
    const double* bt = M.b + (b * M.steps + t - 1) * D;
    double nx[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += at[i * D + k] * cur[k];
      nx[i] = s + bt[i];
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      cur[i] = nx[i];
      m(b, t * D + i) = cur[i];
    }
  }
}

// eta = Lambda m over the symmetric band, in the order product_band_vec
// walks Lambda.to_banded() (kernels_detail.hpp:31-45), uncontracted
__global__ void k_sym_band_vec(Band<double> lam, Vec<double> m, Vec<double> out, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, i;
  if (lam.n == 0 || !split_bj(t, batch, lam.n, out.s, b, i)) return;
  const ix n = lam.n, w = lam.lo;
  const ix j0 = i - w > 0 ? i - w : 0, j1 = i + w < n - 1 ? i + w : n - 1;
  double s = 0.0;
  for (ix j = j0; j <= j1; ++j) {
    const double v = j <= i ? lam.cell(b, int(i - j), j) : lam.cell(b, int(j - i), i);
    s = __dadd_rn(s, __dmul_rn(v, m(b, j)));
  }
  out(b, i) = s;
}

__global__ void k_fail_init(unsigned long long* fail, ix batch, ix v) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b < batch) fail[b] = static_cast<unsigned long long>(v);
}

// SingularBlock(which) (models.cpp:27) as BGM_ERR_NOT_PD with row = block
__global__ void k_fail_report(const unsigned long long* fail, ix batch, ix T, int32_t* st, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const unsigned long long f = fail[b];
  if (f > static_cast<unsigned long long>(T + 1)) return report(st, row, b, BGM_OK, -1);
  report(st, row, b, BGM_ERR_NOT_PD, f == static_cast<unsigned long long>(T + 1) ? 0 : ix(f));
}

template <int D>
int run(const Model& M, const bgm_band& lam, const bgm_vec& eta, int32_t* st, int64_t* row, cudaStream_t s) {
  const ix B = M.batch, T = M.steps, n = (T + 1) * D;
  const size_t lam_bytes = size_t((B + lam.tile - 1) / lam.tile * lam.tile) * size_t(n) * size_t(2 * D) *
                           sizeof(double);
  cudaMemsetAsync(lam.data, 0, lam_bytes, s);
  void* ws = nullptr;
  const size_t vbytes = size_t((B + eta.tile - 1) / eta.tile * eta.tile) * size_t(n) * sizeof(double);
  if (scratch_alloc(&ws, vbytes + sizeof(unsigned long long) * size_t(B) + 256, s) != cudaSuccess) return BGM_ERR_CUDA;
  bgm_vec mean = eta;
  mean.data = ws;
  auto* fail = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + (vbytes + 255) / 256 * 256);
  timing::Scope ts("prior_natural_params", s);
  k_fail_init<<<blocks_for(B, kThreads), kThreads, 0, s>>>(fail, B, T + 2);
  k_blocks<D><<<blocks_for(B * (T + 1), kThreads), kThreads, 0, s>>>(M, view<double>(lam), fail);
  k_mean<D><<<blocks_for(B, kThreads), kThreads, 0, s>>>(M, view<double>(mean));
  const ix work = (B + eta.tile - 1) / eta.tile * eta.tile * n;
  k_sym_band_vec<<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<double>(lam), view<double>(mean),
                                                                 view<double>(eta), B);
  k_fail_report<<<blocks_for(B, kThreads), kThreads, 0, s>>>(fail, B, T, st, row);
  scratch_free(ws, s);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

// ------------------------------------------------------------------ VJP
// Reverse of prior_natural_params (replaces the reference's central-
// difference compose_precision_gradient, inference.cpp:360-380, for this
// assembly): cotangents lambda_bar (stored lower cells, grad.hpp:4-8 --
// f = sum over stored cells, so theta_bar = sum Lambda_bar * dLambda/dtheta as
// compose_precision_gradient forms it) and eta_bar give a_bar, b_bar, q_bar,
// mu0_bar, sigma0_bar.  With P_t = Q_t^-1, Gs_t the symmetrised cotangent of
// diagonal block t and H_t that of the block (t, t-1), both including the
// eta = Lambda m path (eta_bar m^T + m eta_bar^T on the stored cells):
//   a_bar_t  = 2 P_t A_t Gs_t - P_t H_{t+1} + m_bar_{t+1} m_t^T
//   P_bar_t  = A_t Gs_t A_t^T + Gs_{t+1} - H_{t+1} A_t^T,   X_bar = -P P_bar P
//   Sigma0: X_bar = -Sigma0^-1 Gs_0 Sigma0^-1
// and the mean path m_bar = Lambda eta_bar run back through
// m_t = A_{t-1} m_{t-1} + b_{t-1}.  Q_t and Sigma0 are read through their
// lower triangles (the LLT of models.cpp:25-29), so their adjoints are the
// lower folds X_bar + X_bar^T (strict lower), X_bar (diagonal), 0 (upper).

template <int D>
__device__ void lower_fold(const double (&x)[D][D], double* out) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) out[i * D + j] = i > j ? x[i][j] + x[j][i] : (i == j ? x[i][i] : 0.0);
}

// Gs (symmetrised) of diagonal block t and H of block (t, t-1), with the
// eta path folded in
template <int D>
__device__ void block_cotangents(Band<double> lb, Vec<double> eb, Vec<double> m, ix b, ix t, ix T,
                                 double (&gs)[D][D], double (&h)[D][D], bool want_h) {
  double g[D][D];
#pragma unroll
  for (int bi = 0; bi < D; ++bi)
#pragma unroll
    for (int bj = 0; bj < D; ++bj) {
      const ix i = t * D + bi, j = t * D + bj;
      double v = 0.0;
      if (bi > bj) v = lb.cell(b, bi - bj, j) + eb(b, i) * m(b, j) + m(b, i) * eb(b, j);
      else if (bi == bj) v = lb.cell(b, 0, j) + eb(b, i) * m(b, i);
      g[bi][bj] = v;
    }
#pragma unroll
  for (int bi = 0; bi < D; ++bi)
#pragma unroll
    for (int bj = 0; bj < D; ++bj) gs[bi][bj] = bi == bj ? g[bi][bi] : 0.5 * (g[bi][bj] + g[bj][bi]);
  if (!want_h) return;
#pragma unroll
  for (int bi = 0; bi < D; ++bi)
#pragma unroll
    for (int bj = 0; bj < D; ++bj) {
      const ix i = t * D + bi, j = (t - 1) * D + bj;
      h[bi][bj] = lb.cell(b, int(i - j), j) + eb(b, i) * m(b, j) + m(b, i) * eb(b, j);
    }
}

// m_bar = Lambda eta_bar (symmetric band), then back through the mean
// recursion: b_bar_{t-1} = m_bar_t, a_bar_{t-1} = m_bar_t m_{t-1}^T (the
// a_bar initial value), m_bar_{t-1} += A_{t-1}^T m_bar_t, mu0_bar = m_bar_0.
template <int D>
__global__ void k_mean_rev(Model M, Vec<double> m, Vec<double> mb, double* a_bar, double* b_bar, double* mu0_bar) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= M.batch) return;
  const ix T = M.steps;
  double cur[D];
#pragma unroll
  for (int i = 0; i < D; ++i) cur[i] = mb(b, T * D + i);
  for (ix t = T; t >= 1; --t) {
    const double* at = M.a + (b * T + t - 1) * D * D;
    double* ab = a_bar + (b * T + t - 1) * D * D;
    double* bb = b_bar + (b * T + t - 1) * D;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      bb[i] = cur[i];
#pragma unroll
      for (int j = 0; j < D; ++j) ab[i * D + j] = cur[i] * m(b, (t - 1) * D + j);
    }
    double nx[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = mb(b, (t - 1) * D + j);
#pragma unroll
      for (int i = 0; i < D; ++i) s += at[i * D + j] * cur[i];
      nx[j] = s;
    }
#pragma unroll
    for (int j = 0; j < D; ++j) cur[j] = nx[j];
  }
#pragma unroll
  for (int i = 0; i < D; ++i) mu0_bar[b * D + i] = cur[i];
}

// thread per (model, transition t): a_bar_t (added to the mean part), q_bar_t;
// t = 0 also sigma0_bar
template <int D>
__global__ void k_vjp_blocks(Model M, Band<double> lb, Vec<double> eb, Vec<double> m, double* a_bar, double* q_bar,
                             double* sigma0_bar, unsigned long long* fail) {
  const ix g = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix T = M.steps;
  if (g >= M.batch * T) return;
  const ix b = g / T, t = g % T;
  const double* at = M.a + (b * T + t) * D * D;
  double p[D][D], gs[D][D], gs1[D][D], h1[D][D], dummy[D][D];
  if (!spd_inverse<D>(M.q + (b * T + t) * D * D, p)) {
    atomicMin(fail + b, static_cast<unsigned long long>(t + 1));
    return;
  }
  block_cotangents<D>(lb, eb, m, b, t, T, gs, dummy, false);
  block_cotangents<D>(lb, eb, m, b, t + 1, T, gs1, h1, true);
  double pa[D][D], ag[D][D];  // P A, A Gs
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0, u = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        s += p[i][k] * at[k * D + j];
        u += at[i * D + k] * gs[k][j];
      }
      pa[i][j] = s;
      ag[i][j] = u;
    }
  double* ab = a_bar + (b * T + t) * D * D;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += 2.0 * pa[i][k] * gs[k][j] - p[i][k] * h1[k][j];
      ab[i * D + j] += s;
    }
  double pb[D][D];  // A Gs A^T + Gs_{t+1} - H_{t+1} A^T
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = gs1[i][j];
#pragma unroll
      for (int k = 0; k < D; ++k) s += ag[i][k] * at[j * D + k] - h1[i][k] * at[j * D + k];
      pb[i][j] = s;
    }
  double tmp[D][D], xb[D][D];  // X_bar = -P P_bar P
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += p[i][k] * pb[k][j];
      tmp[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += tmp[i][k] * p[k][j];
      xb[i][j] = -s;
    }
  lower_fold<D>(xb, q_bar + (b * T + t) * D * D);
  if (t == 0) {  // Lambda(0, 0) = Sigma0^-1 + ...: X_bar = -Sigma0^-1 Gs_0 Sigma0^-1
    double si[D][D];
    if (!spd_inverse<D>(M.sigma0 + b * D * D, si)) {
      atomicMin(fail + b, static_cast<unsigned long long>(T + 1));
      return;
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += si[i][k] * gs[k][j];
        tmp[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += tmp[i][k] * si[k][j];
        xb[i][j] = -s;
      }
    lower_fold<D>(xb, sigma0_bar + b * D * D);
  }
}

struct Bars {
  double *a, *b, *q, *mu0, *sigma0;
};

template <int D>
int run_vjp(const Model& M, const bgm_band& lam_bar, const bgm_vec& eta_bar, const Bars& out, int32_t* st,
            int64_t* row, cudaStream_t s) {
  const ix B = M.batch, T = M.steps, n = (T + 1) * D;
  const int tile = lam_bar.tile;
  const size_t lam_bytes = size_t((B + tile - 1) / tile * tile) * size_t(n) * size_t(2 * D) * sizeof(double);
  const size_t vbytes = size_t((B + tile - 1) / tile * tile) * size_t(n) * sizeof(double);
  void* ws = nullptr;
  if (scratch_alloc(&ws, lam_bytes + 2 * vbytes + sizeof(unsigned long long) * size_t(B) + 1024, s) != cudaSuccess)
    return BGM_ERR_CUDA;
  char* p = static_cast<char*>(ws);
  bgm_band lam = lam_bar;  // Lambda itself (for m_bar = Lambda eta_bar)
  lam.data = p;
  p += (lam_bytes + 255) / 256 * 256;
  bgm_vec mean = eta_bar, mbar = eta_bar;
  mean.data = p;
  p += (vbytes + 255) / 256 * 256;
  mbar.data = p;
  p += (vbytes + 255) / 256 * 256;
  auto* fail = reinterpret_cast<unsigned long long*>(p);
  timing::Scope ts("vjp_prior_natural_params", s);
  cudaMemsetAsync(lam.data, 0, lam_bytes, s);
  k_fail_init<<<blocks_for(B, kThreads), kThreads, 0, s>>>(fail, B, T + 2);
  k_blocks<D><<<blocks_for(B * (T + 1), kThreads), kThreads, 0, s>>>(M, view<double>(lam), fail);
  k_mean<D><<<blocks_for(B, kThreads), kThreads, 0, s>>>(M, view<double>(mean));
  const ix work = (B + tile - 1) / tile * tile * n;
  k_sym_band_vec<<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<double>(lam), view<double>(eta_bar),
                                                                 view<double>(mbar), B);
  k_mean_rev<D><<<blocks_for(B, kThreads), kThreads, 0, s>>>(M, view<double>(mean), view<double>(mbar), out.a, out.b,
                                                             out.mu0);
  k_vjp_blocks<D><<<blocks_for(B * T, kThreads), kThreads, 0, s>>>(M, view<double>(lam_bar), view<double>(eta_bar),
                                                                   view<double>(mean), out.a, out.q, out.sigma0, fail);
  k_fail_report<<<blocks_for(B, kThreads), kThreads, 0, s>>>(fail, B, T, st, row);
  scratch_free(ws, s);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

}  // namespace
}  // namespace ssm
}  // namespace bgm

using namespace bgm;

extern "C" int bgm_prior_natural_params(int64_t batch, int d, int64_t steps, const double* a, const double* b,
                                        const double* q, const double* mu0, const double* sigma0, bgm_band lambda,
                                        bgm_vec eta, int32_t* status, int64_t* row, bgm_stream stream) {
  if (batch < 0 || steps < 1 || d < 1 || d > 8) return BGM_ERR_ARG;  // models.cpp:166 (empty model)
  if (batch > 0 && (!a || !b || !q || !mu0 || !sigma0)) return BGM_ERR_ARG;
  if (!valid(lambda) || !valid(eta) || lambda.dtype != BGM_F64 || eta.dtype != BGM_F64) return BGM_ERR_ARG;
  const int64_t n = (steps + 1) * d;
  if (lambda.batch != batch || eta.batch != batch || lambda.n != n || eta.n != n || lambda.lower != 2 * d - 1 ||
      lambda.upper != 0 || lambda.tile != eta.tile)
    return BGM_ERR_DIM;
  if (batch == 0) return BGM_OK;
  ssm::Model M{a, b, q, mu0, sigma0, batch, steps};
  auto s = static_cast<cudaStream_t>(stream);
  switch (d) {
    case 1: return ssm::run<1>(M, lambda, eta, status, row, s);
    case 2: return ssm::run<2>(M, lambda, eta, status, row, s);
    case 3: return ssm::run<3>(M, lambda, eta, status, row, s);
    case 4: return ssm::run<4>(M, lambda, eta, status, row, s);
    case 5: return ssm::run<5>(M, lambda, eta, status, row, s);
    case 6: return ssm::run<6>(M, lambda, eta, status, row, s);
    case 7: return ssm::run<7>(M, lambda, eta, status, row, s);
    default: return ssm::run<8>(M, lambda, eta, status, row, s);
  }
}

extern "C" int bgm_vjp_prior_natural_params(int64_t batch, int d, int64_t steps, const double* a, const double* b,
                                            const double* q, const double* mu0, const double* sigma0,
                                            bgm_band lambda_bar, bgm_vec eta_bar, double* a_bar, double* b_bar,
                                            double* q_bar, double* mu0_bar, double* sigma0_bar, int32_t* status,
                                            int64_t* row, bgm_stream stream) {
  if (batch < 0 || steps < 1 || d < 1 || d > 8) return BGM_ERR_ARG;
  if (batch > 0 && (!a || !b || !q || !mu0 || !sigma0 || !a_bar || !b_bar || !q_bar || !mu0_bar || !sigma0_bar))
    return BGM_ERR_ARG;
  if (!valid(lambda_bar) || !valid(eta_bar) || lambda_bar.dtype != BGM_F64 || eta_bar.dtype != BGM_F64)
    return BGM_ERR_ARG;
  const int64_t n = (steps + 1) * d;
  if (lambda_bar.batch != batch || eta_bar.batch != batch || lambda_bar.n != n || eta_bar.n != n ||
      lambda_bar.lower != 2 * d - 1 || lambda_bar.upper != 0 || lambda_bar.tile != eta_bar.tile)
    return BGM_ERR_DIM;
  if (batch == 0) return BGM_OK;
  ssm::Model M{a, b, q, mu0, sigma0, batch, steps};
  ssm::Bars out{a_bar, b_bar, q_bar, mu0_bar, sigma0_bar};
  auto s = static_cast<cudaStream_t>(stream);
  switch (d) {
    case 1: return ssm::run_vjp<1>(M, lambda_bar, eta_bar, out, status, row, s);
    case 2: return ssm::run_vjp<2>(M, lambda_bar, eta_bar, out, status, row, s);
    case 3: return ssm::run_vjp<3>(M, lambda_bar, eta_bar, out, status, row, s);
    case 4: return ssm::run_vjp<4>(M, lambda_bar, eta_bar, out, status, row, s);
    case 5: return ssm::run_vjp<5>(M, lambda_bar, eta_bar, out, status, row, s);
    case 6: return ssm::run_vjp<6>(M, lambda_bar, eta_bar, out, status, row, s);
    case 7: return ssm::run_vjp<7>(M, lambda_bar, eta_bar, out, status, row, s);
    default: return ssm::run_vjp<8>(M, lambda_bar, eta_bar, out, status, row, s);
  }
}
