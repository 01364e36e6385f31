// Config-3 learning step: Gaussian log marginal likelihood + reverse pass.
//
// Reference composition: infer::marginal_likelihood_partial
// (inference.cpp:140-163) with every node observed over Q = band(L L^T)
// (precision_from_factor, inference.cpp:23-26), replayed by Tape::backward
// (tape.cpp:435-451), then L_bar = a_bar + b_bar^T from
// grad::vjp_product_band_band(L, L^T, Q_bar) (grad.cpp:145-151).
//
// This file computes the same quantities with two sweeps per matrix:
//   forward : A = band(L L^T) + tau^-2 I formed on the fly, A = Lp Lp^T
//             (Alg. 1), w = Lp^-1 y, log|Lp|;
//   reverse : S = band(A^-1) by the Takahashi recursion (Alg. 3) on Lp,
//             u = Lp^-T w = A^-1 y, and, column by column as soon as the
//             (k+1)x(k+1) block of S is final,
//               L_bar = -band_lower[(S + tau^-4 u u^T) L] + diag(1 / L_ii),
//             which is (G + G^T) L for the stored-cell Q_bar
//               G(i,i) = -1/2 (S_ii + tau^-4 u_i^2) + 1/2 [Q^-1]_ii ...
//             (the log|L_Q| term contributes exactly L^-T, whose lower band
//             is diag(1/L_ii)), and
//   tau2_bar = -n/(2 tau2) + y'y/(2 tau2^2) + tr(S)/(2 tau2^2)
//              - w'w/tau2^3 + u'u/(2 tau2^4).
// The reference's second factorization chol(Q) only feeds log|L_Q| and its
// gradient; since chol(L L^T) = L (positive diagonal), log|L_Q| = sum log|L_ii|.
// Parity against the reference tape composition: tests/test_mlik_gpu.py.
#include <cuda_runtime.h>

#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_mlik.cuh"
#include "bgm_wide.cuh"
#include "bgm_timing.cuh"

namespace bgm {

constexpr double kLog2Pi = 1.8378770664093454836;  // inference.cpp:15

// Generic forward sweep, one thread per matrix (row-oriented Alg. 1 on the
// fly-formed A).  Writes Lp, w; per-matrix partials into part[b*4 + .].
__global__ void k_mlik_fwd_generic(Band<double> L, Vec<double> y, double inv_tau2, Band<double> Lp,
                                   Vec<double> w, double* part, ix batch, int32_t* status,
                                   int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix n = L.n, k = L.lo;
  double ldp = 0, ldl = 0, yy = 0, ww = 0;
  for (ix i = 0; i < n; ++i) {
    const ix j0 = i - k > 0 ? i - k : 0;
    for (ix j = j0; j <= i; ++j) {
      double a = 0;
      for (ix m = j0; m <= j; ++m) a += L.at(b, i, m) * L.at(b, j, m);
      if (i == j) a += inv_tau2;
      double s = 0;
      for (ix m = j0; m < j; ++m) s += Lp.at(b, i, m) * Lp.at(b, j, m);
      if (i == j) {
        const double piv = a - s;
        if (!(piv > kPivotFloor)) {
          report(status, row, b, BGM_ERR_NOT_PD, i);
          return;
        }
        Lp.at(b, i, i) = sqrt(piv);
      } else {
        Lp.at(b, i, j) = (a - s) / Lp.at(b, j, j);
      }
    }
    double s = 0;
    for (ix m = j0; m < i; ++m) s += Lp.at(b, i, m) * w(b, m);
    const double yi = y(b, i);
    const double wi = (yi - s) / Lp.at(b, i, i);
    w(b, i) = wi;
    const double lii = fabs(L.at(b, i, i));
    if (!(lii > kPivotFloor)) {
      report(status, row, b, BGM_ERR_NOT_PD, i);
      return;
    }
    ldp += log(Lp.at(b, i, i));
    ldl += log(lii);
    yy += yi * yi;
    ww += wi * wi;
  }
  part[b * 4 + 0] = ldp;
  part[b * 4 + 1] = ldl;
  part[b * 4 + 2] = yy;
  part[b * 4 + 3] = ww;
  report(status, row, b, BGM_OK, -1);
}

// Generic reverse sweep, one thread per matrix.  S is a (k,0) symmetric
// lower store scratch, u a vector scratch.
__global__ void k_mlik_bwd_generic(Band<double> L, Band<double> Lp, Vec<double> w, double tau2,
                                   Band<double> S, Vec<double> u, Band<double> Lb,
                                   const double* part, double* loss, double* tau2_bar, ix batch,
                                   const int32_t* status) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  if (status && status[b] != BGM_OK) return;
  const ix n = L.n, k = L.lo;
  const double inv = 1.0 / tau2, c4 = inv * inv;
  double tr = 0, uu = 0;
  for (ix j = n - 1; j >= 0; --j) {
    const ix i_stop = j - k > 0 ? j - k : 0;
    const ix jend = j + k < n - 1 ? j + k : n - 1;
    for (ix i = j; i >= i_stop; --i) {  // kernels_serial.cpp:93-101
      const double piv = Lp.at(b, i, i);
      double acc = 0;
      const ix m1 = i + k < n - 1 ? i + k : n - 1;
      for (ix m = i + 1; m <= m1; ++m) acc += (Lp.at(b, m, i) / piv) * S.sym(b, m, j);
      double val = -acc;
      if (i == j) val += 1.0 / (piv * piv);
      S.at(b, j, i) = val;
    }
    double s = 0;  // u_j = (w_j - sum_{m>j} Lp(m,j) u_m) / Lp(j,j)
    for (ix m = j + 1; m <= jend; ++m) s += Lp.at(b, m, j) * u(b, m);
    const double uj = (w(b, j) - s) / Lp.at(b, j, j);
    u(b, j) = uj;
    tr += S.at(b, j, j);
    uu += uj * uj;
    double lu = 0;  // (L^T u)_j over the column's band
    for (ix m = j; m <= jend; ++m) lu += L.at(b, m, j) * u(b, m);
    Lb.write_column(b, j, [&](ix i) {
      double acc = 0;
      for (ix m = j; m <= jend; ++m) acc += S.sym(b, i, m) * L.at(b, m, j);
      acc += c4 * u(b, i) * lu;
      return -acc + (i == j ? 1.0 / L.at(b, j, j) : 0.0);
    });
  }
  const double nn = double(n);
  const double ldp = part[b * 4 + 0], ldl = part[b * 4 + 1], yy = part[b * 4 + 2],
               ww = part[b * 4 + 3];
  loss[b] = -0.5 * nn * kLog2Pi - ldp + ldl - 0.5 * nn * log(tau2) - 0.5 * yy * inv +
            0.5 * ww * c4;
  tau2_bar[b] = -nn * 0.5 * inv + 0.5 * yy * c4 + 0.5 * c4 * tr - ww * c4 * inv +
                0.5 * uu * c4 * c4;
}

static int g_segment_rows = 0;

}  // namespace bgm

using namespace bgm;

extern "C" {

int bgm_debug_repairs(int64_t* count, double* max_dev, int reset) {
  int64_t c = 0;
  const int rc = mlik_repairs(&c, max_dev, reset);
  if (rc != BGM_OK) return rc;
  const int rc2 = t1::repairs(&c, reset);
  if (count) *count = c;
  return rc2;
}

int bgm_set_segment_rows(int64_t rows) {
  if (rows < 0 || rows > INT32_MAX) return BGM_ERR_ARG;
  g_segment_rows = int(rows);
  wide::set_segment_rows(int(rows));
  narrow::set_segment_rows(int(rows));
  return BGM_OK;
}

int bgm_marginal_likelihood_grad(bgm_band l, bgm_vec y, double tau2, double* loss, bgm_band lbar,
                                 double* tau2_bar, int32_t* status, int64_t* row,
                                 bgm_stream stream) {
  if (!valid(l) || !valid(y) || !valid(lbar)) return BGM_ERR_ARG;
  if (l.dtype != BGM_F64 || y.dtype != BGM_F64 || lbar.dtype != BGM_F64) return BGM_ERR_ARG;
  if (!(tau2 > 0.0) || (l.batch > 0 && (!loss || !tau2_bar))) return BGM_ERR_ARG;
  if (l.upper != 0 || lbar.upper != 0 || lbar.lower != l.lower || l.batch != y.batch ||
      l.n != y.n || l.batch != lbar.batch || l.n != lbar.n)
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  int rc = mlik_t1(l, y, tau2, loss, lbar, tau2_bar, status, row, g_segment_rows, s);
  if (rc >= 0) return rc;
  rc = mlik_fast(l, y, tau2, loss, lbar, tau2_bar, status, row, g_segment_rows, s);
  if (rc >= 0) return rc;
  // Generic path: one thread per matrix, scratch for Lp, w, S, u.
  const ix padded = (l.batch + 31) / 32 * 32;
  const int wd = l.lower + 1;
  const size_t band_bytes = sizeof(double) * size_t(padded * l.n * wd);
  const size_t vec_bytes = sizeof(double) * size_t(padded * l.n);
  char* ws = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&ws),
                                  2 * band_bytes + 2 * vec_bytes + sizeof(double) * 4 * padded, s);
  if (e != cudaSuccess) return set_error(e);
  Band<double> Lp{reinterpret_cast<double*>(ws), l.n, l.lower, 0, wd, 5};
  Band<double> Sm{reinterpret_cast<double*>(ws + band_bytes), l.n, l.lower, 0, wd, 5};
  Vec<double> wv{reinterpret_cast<double*>(ws + 2 * band_bytes), l.n, 5};
  Vec<double> uv{reinterpret_cast<double*>(ws + 2 * band_bytes + vec_bytes), l.n, 5};
  double* part = reinterpret_cast<double*>(ws + 2 * band_bytes + 2 * vec_bytes);
  int32_t* st = status;
  int32_t* own = nullptr;
  if (!st) {
    e = scratch_alloc(reinterpret_cast<void**>(&own), sizeof(int32_t) * padded, s);
    if (e != cudaSuccess) return set_error(e);
    st = own;
  }
  {
    timing::Scope ts("mlik_fwd_generic", s);
    k_mlik_fwd_generic<<<blocks_for(l.batch, 64), 64, 0, s>>>(view<double>(l), view<double>(y),
                                                           1.0 / tau2, Lp, wv, part, l.batch, st,
                                                           row);
  }
  {
    timing::Scope ts("mlik_bwd_generic", s);
    k_mlik_bwd_generic<<<blocks_for(l.batch, 64), 64, 0, s>>>(
      view<double>(l), Lp, wv, tau2, Sm, uv, view<double>(lbar), part, loss, tau2_bar, l.batch, st);
  }
  e = cudaGetLastError();
  scratch_free(ws, s);
  if (own) scratch_free(own, s);
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

}  // extern "C"
