// Variational-inference objective on the device:
// Tape::trace_product_sym and its reverse (tape.cpp:274-302), and
// infer::kl_divergence (inference.cpp:247-268) with its gradient in the
// variational parameters, composed from the library's own operators
// (sparse inverse subset, restricted product, log-det, band x vector and
// their VJPs) plus the per-matrix reductions below.  fp64, both layouts.
#include <cuda_runtime.h>

#include "bgm_common.cuh"
#include "bgm_timing.cuh"

namespace bgm {
namespace vi {
namespace {

constexpr int kThreads = 128;
constexpr ix kChunk = 256;  // columns per partial sum

__host__ __device__ inline ix chunks(ix n) { return (n + kChunk - 1) / kChunk; }

// thread per (matrix, column chunk); consecutive threads = consecutive
// matrices of one chunk (coalesced in the tile-32 layout)
__global__ void k_trace_part(Band<double> a, Band<double> b, ix batch, double* part) {
  const ix nch = chunks(a.n);
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * nch) return;
  const ix mb = t % batch, c = t / batch, n = a.n;
  const ix j1 = (c + 1) * kChunk < n ? (c + 1) * kChunk : n;
  const int bw = a.lo < b.lo ? a.lo : b.lo;
  double s = 0.0;
  for (ix j = c * kChunk; j < j1; ++j) {  // tape.cpp:280-284
    s += a.cell(mb, 0, j) * b.cell(mb, 0, j);
    for (int d = 1; d <= bw && j + d < n; ++d) s += 2.0 * a.cell(mb, d, j) * b.cell(mb, d, j);
  }
  part[mb * nch + c] = s;
}

__global__ void k_dot_part(Vec<double> x, ix batch, double* part) {
  const ix nch = chunks(x.n);
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * nch) return;
  const ix mb = t % batch, c = t / batch;
  const ix j1 = (c + 1) * kChunk < x.n ? (c + 1) * kChunk : x.n;
  double s = 0.0;
  for (ix j = c * kChunk; j < j1; ++j) s = fma(x(mb, j), x(mb, j), s);
  part[mb * nch + c] = s;
}

// ordered per-matrix sum of the partials (deterministic)
__global__ void k_sum_parts(const double* part, ix nch, ix batch, double* out) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  double s = 0.0;
  for (ix c = 0; c < nch; ++c) s += part[b * nch + c];
  out[b] = s;
}

// a_bar = c_bar * seed(b) on band(a): x on the diagonal, 2x below it
__global__ void k_trace_seed(Band<double> out, Band<double> b, const double* cbar, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix mb, j;
  if (out.n == 0 || !split_bj(t, batch, out.n, out.s, mb, j)) return;
  const double c = cbar[mb];
  out.write_column(mb, j, [&](ix i) {
    const int d = int(i - j);
    const double v = (d <= b.lo) ? b.cell(mb, d, j) : 0.0;  // tape.cpp:290-297 (at_or_zero)
    return d == 0 ? c * v : 2.0 * c * v;
  });
}

__global__ void k_fill(double* x, ix count, double v) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t < count) x[t] = v;
}

__global__ void k_sub(Vec<double> a, Vec<double> b, Vec<double> out, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix mb, i;
  if (a.n == 0 || !split_bj(t, batch, a.n, a.s, mb, i)) return;
  out(mb, i) = a(mb, i) - b(mb, i);
}

// inference.cpp:262-267: 0.5 * (trace + 2 (logdet_q - logdet_p) + quad - n)
__global__ void k_kl_final(const double* tr, const double* ldq, const double* ldp, const double* quad, ix n,
                           ix batch, double* kl) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  double inner = tr[b] + 2.0 * (ldq[b] - ldp[b]);
  inner = inner + quad[b];
  inner = inner + (-double(n));
  kl[b] = 0.5 * inner;
}

// first error in the reference's evaluation order
__global__ void k_status3(const int32_t* s1, const int64_t* r1, const int32_t* s2, const int64_t* r2,
                          const int32_t* s3, const int64_t* r3, ix batch, int32_t* st, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const bool e1 = s1[b] != BGM_OK, e2 = s2[b] != BGM_OK;
  report(st, row, b, e1 ? s1[b] : e2 ? s2[b] : s3[b], e1 ? r1[b] : e2 ? r2[b] : r3[b]);
}

size_t band_bytes(const bgm_band& d) {
  const ix t = d.tile;
  return size_t((d.batch + t - 1) / t * t) * size_t(d.n) * size_t(d.lower + d.upper + 1) * sizeof(double);
}
size_t vec_bytes(const bgm_vec& d) {
  const ix t = d.tile;
  return size_t((d.batch + t - 1) / t * t) * size_t(d.n) * sizeof(double);
}

// bump allocator over one pool block (256-byte aligned pieces)
struct Arena {
  char* base = nullptr;
  size_t off = 0;
  cudaStream_t s;
  void* take(size_t bytes) {
    void* p = base + off;
    off += (bytes + 255) / 256 * 256;
    return p;
  }
  ~Arena() {
    if (base) scratch_free(base, s);
  }
};

bool ok_band(const bgm_band& d) { return valid(d) && d.dtype == BGM_F64; }
bool ok_vec(const bgm_vec& d) { return valid(d) && d.dtype == BGM_F64; }

}  // namespace
}  // namespace vi
}  // namespace bgm

using namespace bgm;
using namespace bgm::vi;

extern "C" {

int bgm_trace_product_sym(bgm_band a, bgm_band b, double* out, bgm_stream stream) {
  if (!ok_band(a) || !ok_band(b) || (a.batch > 0 && !out)) return BGM_ERR_ARG;
  if (a.upper != 0 || b.upper != 0 || a.batch != b.batch || a.n != b.n || a.tile != b.tile) return BGM_ERR_DIM;
  if (a.batch == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  if (a.n == 0) {
    const cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * size_t(a.batch), s);
    return e == cudaSuccess ? BGM_OK : set_error(e);
  }
  const ix nch = chunks(a.n);
  Arena ar;
  ar.s = s;
  if (scratch_alloc(reinterpret_cast<void**>(&ar.base), sizeof(double) * size_t(a.batch * nch) + 256, s) != cudaSuccess)
    return BGM_ERR_CUDA;
  double* part = static_cast<double*>(ar.take(sizeof(double) * size_t(a.batch * nch)));
  timing::Scope t("trace_product_sym", s);
  k_trace_part<<<blocks_for(a.batch * nch, kThreads), kThreads, 0, s>>>(view<double>(a), view<double>(b), a.batch, part);
  k_sum_parts<<<blocks_for(a.batch, kThreads), kThreads, 0, s>>>(part, nch, a.batch, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

int bgm_vjp_trace_product_sym(bgm_band a, bgm_band b, const double* c_bar, bgm_band a_bar, bgm_band b_bar,
                              bgm_stream stream) {
  if (!ok_band(a) || !ok_band(b) || (a.batch > 0 && !c_bar)) return BGM_ERR_ARG;
  if (a.upper != 0 || b.upper != 0 || a.batch != b.batch || a.n != b.n || a.tile != b.tile) return BGM_ERR_DIM;
  auto s = static_cast<cudaStream_t>(stream);
  const ix work = (a.batch + a.tile - 1) / a.tile * a.tile * a.n;
  if (a.batch == 0 || a.n == 0) return BGM_OK;
  if (a_bar.data) {
    if (!ok_band(a_bar) || a_bar.lower != a.lower || a_bar.upper != 0 || a_bar.n != a.n || a_bar.tile != a.tile)
      return BGM_ERR_DIM;
    k_trace_seed<<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<double>(a_bar), view<double>(b), c_bar, a.batch);
  }
  if (b_bar.data) {
    if (!ok_band(b_bar) || b_bar.lower != b.lower || b_bar.upper != 0 || b_bar.n != b.n || b_bar.tile != b.tile)
      return BGM_ERR_DIM;
    k_trace_seed<<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<double>(b_bar), view<double>(a), c_bar, a.batch);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

}  // extern "C"

namespace bgm {
namespace vi {
namespace {

constexpr double kLog2Pi = 1.8378770664093454836;  // inference.cpp:15

// Gaussian expected log-likelihood, full observation (inference.cpp:52-63):
// per matrix sum_i -1/2 (log tau2 + log 2 pi) - ((y_i - m_i)^2 + v_i) / (2 tau2)
// with v_i = S(i, i); d_mean_i = r_i / tau2 goes to dm, the tau2 partial to part2.
__global__ void k_gauss_part(Vec<double> y, Vec<double> m, Band<double> S, double t2, ix batch, double* part,
                             double* part2, Vec<double> dm, Vec<double> obs, Vec<double> dv) {
  const ix nch = chunks(y.n);
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * nch) return;
  const ix mb = t % batch, c = t / batch;
  const ix j1 = (c + 1) * kChunk < y.n ? (c + 1) * kChunk : y.n;
  const double lt = -0.5 * (log(t2) + kLog2Pi);
  double v = 0.0, dt = 0.0;
  for (ix i = c * kChunk; i < j1; ++i) {
    // partial SelectionIndex (obs.p set): unobserved latents add nothing
    // (inference.cpp:55-62 loops over sel.observed only)
    if (obs.p && obs(mb, i) == 0.0) {
      dm(mb, i) = 0.0;
      dv(mb, i) = 0.0;
      continue;
    }
    const double r = y(mb, i) - m(mb, i), var = S.cell(mb, 0, i);
    v += lt - (r * r + var) / (2.0 * t2);
    dt += (r * r + var) / (2.0 * t2 * t2) - 0.5 / t2;
    dm(mb, i) = r / t2;
    if (obs.p) dv(mb, i) = -0.5 / t2;
  }
  part[mb * nch + c] = v;
  part2[mb * nch + c] = dt;
}

// out = a - out (the ELBO's m-bar: expected-loglik minus KL parts)
__global__ void k_rsub(Vec<double> a, Vec<double> out, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix mb, i;
  if (a.n == 0 || !split_bj(t, batch, a.n, a.s, mb, i)) return;
  out(mb, i) = a(mb, i) - out(mb, i);
}

// S-bar(i, i) += d_var_i (Tape::diag_sym reverse, tape.cpp:304-312)
__global__ void k_add_diag(Band<double> sb, double v, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix mb, j;
  if (sb.n == 0 || !split_bj(t, batch, sb.n, sb.s, mb, j)) return;
  sb.cell(mb, 0, j) += v;
}

__global__ void k_scale_logdet_bar(Band<double> lb, Band<double> l, double c, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix mb, j;
  if (l.n == 0 || !split_bj(t, batch, l.n, l.s, mb, j)) return;
  lb.cell(mb, 0, j) += c / l.cell(mb, 0, j);
}

__global__ void k_elbo_final(const double* ve, const double* kl, ix batch, double* elbo) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b < batch) elbo[b] = ve[b] - kl[b];
}

constexpr int kMaxQuad = 64;
struct GH {  // Gauss-Hermite rule, ascending nodes (inference.cpp:120-137)
  int k;
  double x[kMaxQuad], w[kMaxQuad];
};

struct LikTerm {
  int kind;  // 0 Gaussian (tau2), 1 Poisson (weight, Gauss-Hermite)
  bgm_vec y, weight;
  bgm_vec obs;  // 0/1 mask of the observed latents; data == null: all
  double tau2;
  GH gh;
  double* elbo;
  double* tau2_bar;  // Gaussian only; may be null
};

// Poisson expected log-likelihood, full observation (inference.cpp:65-100):
// per observation the Gauss-Hermite expectation of y f - w e^f plus
// y log w - lgamma(y + 1), its mean / variance partials to dm / dv; the first
// non-positive weight per matrix is recorded in bad (NonPositiveParam).
__global__ void k_poisson_part(Vec<double> y, Vec<double> wt, Vec<double> m, Band<double> S, const GH gh, ix batch,
                               double* part, Vec<double> dm, Vec<double> dv, unsigned long long* bad,
                               Vec<double> obs) {
  const ix nch = chunks(y.n);
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * nch) return;
  const ix mb = t % batch, c = t / batch;
  const ix j1 = (c + 1) * kChunk < y.n ? (c + 1) * kChunk : y.n;
  const double norm = 1.0 / sqrt(3.14159265358979323846);
  double val = 0.0;
  for (ix i = c * kChunk; i < j1; ++i) {
    if (obs.p && obs(mb, i) == 0.0) {  // unobserved latent (partial SelectionIndex)
      dm(mb, i) = 0.0;
      dv(mb, i) = 0.0;
      continue;
    }
    const double w = wt(mb, i), yi = y(mb, i), mi = m(mb, i), v = S.cell(mb, 0, i);
    if (!(w > 0.0)) {
      atomicMin(bad + mb, static_cast<unsigned long long>(i));
      dm(mb, i) = 0.0;
      dv(mb, i) = 0.0;
      continue;
    }
    const double base = yi * log(w) - lgamma(yi + 1.0);
    if (v <= 0.0) {
      val += yi * mi + base - w * exp(mi);
      dm(mb, i) = yi - w * exp(mi);
      dv(mb, i) = 0.0;
      continue;
    }
    const double spread = sqrt(2.0 * v);
    double ev = 0.0, sm = 0.0, sv = 0.0;
    for (int q = 0; q < gh.k; ++q) {
      const double f = mi + spread * gh.x[q];
      const double rate = w * exp(f);
      ev += gh.w[q] * (yi * f - rate);
      const double gp = yi - rate;
      sm += gh.w[q] * gp;
      sv += gh.w[q] * gp * gh.x[q] / spread;
    }
    val += norm * ev + base;
    dm(mb, i) = norm * sm;
    dv(mb, i) = norm * sv;
  }
  part[mb * nch + c] = val;
}

// S-bar(i, i) += dv_i (Tape::diag_sym reverse with a per-entry adjoint)
__global__ void k_add_diag_vec(Band<double> sb, Vec<double> dv, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix mb, j;
  if (sb.n == 0 || !split_bj(t, batch, sb.n, sb.s, mb, j)) return;
  sb.cell(mb, 0, j) += dv(mb, j);
}

__global__ void k_bad_init(unsigned long long* bad, ix batch, ix n) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b < batch) bad[b] = static_cast<unsigned long long>(n);
}

// ELBO error order (inference.cpp:278-286): subset of L_q, likelihood
// parameters (Poisson weights), then the KL's log|L_p| and log|L_q|
__global__ void k_status_elbo(const int32_t* s_sub, const int64_t* r_sub, const unsigned long long* bad, ix n,
                              const int32_t* s_p, const int64_t* r_p, const int32_t* s_q, const int64_t* r_q,
                              ix batch, int32_t* st, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  if (s_sub[b] != BGM_OK) return report(st, row, b, s_sub[b], r_sub[b]);
  if (bad && bad[b] < static_cast<unsigned long long>(n)) return report(st, row, b, BGM_ERR_ARG, ix(bad[b]));
  if (s_p[b] != BGM_OK) return report(st, row, b, s_p[b], r_p[b]);
  report(st, row, b, s_q[b], r_q[b]);
}

// Golub-Welsch: nodes = eigenvalues of the Jacobi matrix (off-diagonal
// sqrt(k/2)), weights = sqrt(pi) v_0^2, by implicit-shift QL iterations on
// the symmetric tridiagonal matrix carrying the first eigenvector components.
bool gauss_hermite(int k, GH& gh) {
  if (k < 1 || k > kMaxQuad) return false;
  gh.k = k;
  if (k == 1) {
    gh.x[0] = 0.0;
    gh.w[0] = sqrt(3.14159265358979323846);
    return true;
  }
  double d[kMaxQuad], e[kMaxQuad], z[kMaxQuad];  // diagonal, sub-diagonal, first row of the eigenvectors
  for (int i = 0; i < k; ++i) {
    d[i] = 0.0;
    e[i] = i + 1 < k ? sqrt(0.5 * (i + 1)) : 0.0;
    z[i] = i == 0 ? 1.0 : 0.0;
  }
  for (int l = 0; l < k; ++l) {
    for (int iter = 0; iter < 200; ++iter) {
      int m = l;
      for (; m + 1 < k; ++m) {
        const double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= 1e-300 + 2.2e-16 * dd) break;
      }
      if (m == l) break;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      double sn = 1.0, cs = 1.0, p = 0.0;
      int i = m - 1;
      for (; i >= l; --i) {
        double f = sn * e[i], b = cs * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[m] = 0.0;
          break;
        }
        sn = f / r;
        cs = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * sn + 2.0 * cs * b;
        p = sn * r;
        d[i + 1] = g + p;
        g = cs * r - b;
        f = z[i + 1];
        z[i + 1] = sn * z[i] + cs * f;
        z[i] = cs * z[i] - sn * f;
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  // ascending nodes, as Eigen's SelfAdjointEigenSolver returns them
  int idx[kMaxQuad];
  for (int i = 0; i < k; ++i) idx[i] = i;
  for (int i = 1; i < k; ++i)
    for (int j = i; j > 0 && d[idx[j]] < d[idx[j - 1]]; --j) {
      const int t = idx[j];
      idx[j] = idx[j - 1];
      idx[j - 1] = t;
    }
  for (int i = 0; i < k; ++i) {
    gh.x[i] = d[idx[i]];
    gh.w[i] = sqrt(3.14159265358979323846) * z[idx[i]] * z[idx[i]];
  }
  return true;
}

// KL(q || p) (inference.cpp:247-268) and, with `g`, the Gaussian ELBO
// (inference.cpp:276-287): expected log-likelihood minus KL.  Gradients in
// (m_q, L_q) of the objective computed (KL, or the ELBO).
int vi_core(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar,
            int32_t* status, int64_t* row, bgm_stream stream, const LikTerm* g) {
  if (!ok_band(l_q) || !ok_band(l_p) || !ok_band(l_q_bar) || !ok_vec(m_q) || !ok_vec(m_p) || !ok_vec(m_q_bar))
    return BGM_ERR_ARG;
  if (g && !ok_vec(g->y)) return BGM_ERR_ARG;
  if (g && g->kind == 0 && !(g->tau2 > 0.0)) return BGM_ERR_ARG;  // NonPositiveParam("tau2")
  if (g && g->kind == 1 && !ok_vec(g->weight)) return BGM_ERR_ARG;
  const bool sel = g && g->obs.data;
  if (sel && (!ok_vec(g->obs) || g->obs.dtype != BGM_F64)) return BGM_ERR_ARG;
  const ix B = l_q.batch, n = l_q.n;
  if (B > 0 && (!kl || (g && !g->elbo))) return BGM_ERR_ARG;
  const bool same = l_p.batch == B && m_q.batch == B && m_p.batch == B && m_q_bar.batch == B && l_q_bar.batch == B &&
                    l_p.n == n && m_q.n == n && m_p.n == n && m_q_bar.n == n && l_q_bar.n == n &&
                    (!g || (g->y.batch == B && g->y.n == n)) &&
                    (!g || g->kind != 1 || (g->weight.batch == B && g->weight.n == n)) &&
                    (!sel || (g->obs.batch == B && g->obs.n == n));
  const int tile = l_q.tile;
  const bool tiles = l_p.tile == tile && m_q.tile == tile && m_p.tile == tile && m_q_bar.tile == tile &&
                     l_q_bar.tile == tile && (!g || g->y.tile == tile) &&
                     (!g || g->kind != 1 || g->weight.tile == tile) && (!sel || g->obs.tile == tile);
  if (!same || !tiles || l_q.upper != 0 || l_p.upper != 0 || l_q_bar.lower != l_q.lower || l_q_bar.upper != 0 ||
      l_q.lower < l_p.lower)  // inference.cpp:252-253
    return BGM_ERR_DIM;
  if (B == 0 || n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  timing::Scope t(g ? "elbo_grad" : "kl_divergence_grad", s);
  const ix nch = chunks(n);
  bgm_band S = l_q, Sb = l_q, Qp = l_p;
  bgm_vec d = m_q, wv = m_q, dm = m_q, dvv = m_q;
  const size_t scal = sizeof(double) * size_t(B);
  const size_t total = 2 * band_bytes(l_q) + band_bytes(l_p) + 4 * vec_bytes(m_q) + 8 * scal +
                       2 * sizeof(double) * size_t(B * nch) + 4 * (sizeof(int32_t) + sizeof(int64_t)) * size_t(B) +
                       24 * 256;
  Arena ar;
  ar.s = s;
  if (scratch_alloc(reinterpret_cast<void**>(&ar.base), total, s) != cudaSuccess) return BGM_ERR_CUDA;
  S.data = ar.take(band_bytes(l_q));
  Sb.data = ar.take(band_bytes(l_q));
  Qp.data = ar.take(band_bytes(l_p));
  d.data = ar.take(vec_bytes(m_q));
  wv.data = ar.take(vec_bytes(m_q));
  dm.data = ar.take(vec_bytes(m_q));
  dvv.data = ar.take(vec_bytes(m_q));
  unsigned long long* bad = static_cast<unsigned long long*>(ar.take(scal));
  double* tr = static_cast<double*>(ar.take(scal));
  double* ldq = static_cast<double*>(ar.take(scal));
  double* ldp = static_cast<double*>(ar.take(scal));
  double* quad = static_cast<double*>(ar.take(scal));
  double* cb = static_cast<double*>(ar.take(scal));
  double* ve = static_cast<double*>(ar.take(scal));
  double* part = static_cast<double*>(ar.take(sizeof(double) * size_t(B * nch)));
  double* part2 = static_cast<double*>(ar.take(sizeof(double) * size_t(B * nch)));
  int32_t* st[4];
  int64_t* rw[4];
  for (int q = 0; q < 4; ++q) {
    st[q] = static_cast<int32_t*>(ar.take(sizeof(int32_t) * size_t(B)));
    rw[q] = static_cast<int64_t*>(ar.take(sizeof(int64_t) * size_t(B)));
  }
  int rc;
  // forward (inference.cpp:255-267)
  if ((rc = bgm_product_band_band(l_p, 0, l_p, 1, Qp, stream))) return rc;  // precision_from_factor (:23-26)
  if ((rc = bgm_log_det(l_p, ldp, st[0], rw[0], stream))) return rc;
  if ((rc = bgm_sparse_inverse_subset(l_q, S, st[1], rw[1], stream))) return rc;
  if ((rc = bgm_trace_product_sym(S, Qp, tr, stream))) return rc;
  if ((rc = bgm_log_det(l_q, ldq, st[2], rw[2], stream))) return rc;
  const ix vwork = (B + tile - 1) / tile * tile * n;
  // d = m_q - m_p, white' = L_p^T d = -white: the quadratic form is unchanged
  k_sub<<<blocks_for(vwork, kThreads), kThreads, 0, s>>>(view<double>(m_q), view<double>(m_p), view<double>(d), B);
  if ((rc = bgm_product_band_vec(l_p, d, 1, wv, stream))) return rc;
  k_dot_part<<<blocks_for(B * nch, kThreads), kThreads, 0, s>>>(view<double>(wv), B, part);
  k_sum_parts<<<blocks_for(B, kThreads), kThreads, 0, s>>>(part, nch, B, quad);
  k_kl_final<<<blocks_for(B, kThreads), kThreads, 0, s>>>(tr, ldq, ldp, quad, n, B, kl);
  // reverse of KL: m_q-bar = -L_p white = L_p white'; S-bar = 1/2 seed(Q_p)
  // (trace node, tape.cpp:285-301); L-bar += diag(1 / L_q(j,j)) (log|L_q|).
  // The ELBO negates the KL parts and adds the expected log-likelihood's
  // d_mean (to m-bar) and d_var (to S-bar's diagonal, diag_sym).
  const double sgn = g ? -1.0 : 1.0;
  if ((rc = bgm_product_band_vec(l_p, wv, 0, m_q_bar, stream))) return rc;
  k_fill<<<blocks_for(B, kThreads), kThreads, 0, s>>>(cb, B, 0.5 * sgn);
  bgm_band none = Sb;
  none.data = nullptr;
  if ((rc = bgm_vjp_trace_product_sym(S, Qp, cb, Sb, none, stream))) return rc;
  const ix bwork = (B + tile - 1) / tile * tile * n;
  if (g) {
    Vec<double> ov{};
    if (sel) ov = view<double>(g->obs);
    if (g->kind == 0) {
      k_gauss_part<<<blocks_for(B * nch, kThreads), kThreads, 0, s>>>(view<double>(g->y), view<double>(m_q),
                                                                       view<double>(S), g->tau2, B, part, part2,
                                                                       view<double>(dm), ov, view<double>(dvv));
      if (g->tau2_bar) k_sum_parts<<<blocks_for(B, kThreads), kThreads, 0, s>>>(part2, nch, B, g->tau2_bar);
      if (sel)  // d_var = -1/(2 tau2) on the observed latents only
        k_add_diag_vec<<<blocks_for(bwork, kThreads), kThreads, 0, s>>>(view<double>(Sb), view<double>(dvv), B);
      else
        k_add_diag<<<blocks_for(bwork, kThreads), kThreads, 0, s>>>(view<double>(Sb), -0.5 / g->tau2, B);
    } else {
      k_bad_init<<<blocks_for(B, kThreads), kThreads, 0, s>>>(bad, B, n);
      k_poisson_part<<<blocks_for(B * nch, kThreads), kThreads, 0, s>>>(
          view<double>(g->y), view<double>(g->weight), view<double>(m_q), view<double>(S), g->gh, B, part,
          view<double>(dm), view<double>(dvv), bad, ov);
      k_add_diag_vec<<<blocks_for(bwork, kThreads), kThreads, 0, s>>>(view<double>(Sb), view<double>(dvv), B);
    }
    k_sum_parts<<<blocks_for(B, kThreads), kThreads, 0, s>>>(part, nch, B, ve);
    k_elbo_final<<<blocks_for(B, kThreads), kThreads, 0, s>>>(ve, kl, B, g->elbo);
    k_rsub<<<blocks_for(vwork, kThreads), kThreads, 0, s>>>(view<double>(dm), view<double>(m_q_bar), B);
  }
  if ((rc = bgm_vjp_sparse_inverse_subset(l_q, S, Sb, l_q_bar, st[3], rw[3], stream))) return rc;
  k_scale_logdet_bar<<<blocks_for(bwork, kThreads), kThreads, 0, s>>>(view<double>(l_q_bar), view<double>(l_q), sgn,
                                                                       B);
  if (g)
    k_status_elbo<<<blocks_for(B, kThreads), kThreads, 0, s>>>(st[1], rw[1], g->kind == 1 ? bad : nullptr, n, st[0],
                                                                rw[0], st[2], rw[2], B, status, row);
  else
    k_status3<<<blocks_for(B, kThreads), kThreads, 0, s>>>(st[0], rw[0], st[1], rw[1], st[2], rw[2], B, status, row);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

}  // namespace
}  // namespace vi
}  // namespace bgm

extern "C" {

int bgm_kl_divergence_grad(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, double* kl, bgm_vec m_q_bar,
                           bgm_band l_q_bar, int32_t* status, int64_t* row, bgm_stream stream) {
  return vi::vi_core(m_q, l_q, m_p, l_p, kl, m_q_bar, l_q_bar, status, row, stream, nullptr);
}

int bgm_elbo_gaussian_grad(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, double tau2,
                           double* elbo, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar, double* tau2_bar,
                           int32_t* status, int64_t* row, bgm_stream stream) {
  vi::LikTerm g{};
  g.kind = 0;
  g.y = y;
  g.tau2 = tau2;
  g.elbo = elbo;
  g.tau2_bar = tau2_bar;
  return vi::vi_core(m_q, l_q, m_p, l_p, kl, m_q_bar, l_q_bar, status, row, stream, &g);
}

int bgm_elbo_poisson_grad(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, bgm_vec weight,
                          int quad_points, double* elbo, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar,
                          int32_t* status, int64_t* row, bgm_stream stream) {
  vi::LikTerm g{};
  g.kind = 1;
  g.y = y;
  g.weight = weight;
  if (!vi::gauss_hermite(quad_points, g.gh)) return BGM_ERR_ARG;  // NonPositiveParam("quad_points")
  g.elbo = elbo;
  return vi::vi_core(m_q, l_q, m_p, l_p, kl, m_q_bar, l_q_bar, status, row, stream, &g);
}

int bgm_elbo_gaussian_grad_sel(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, bgm_vec observed,
                               double tau2, double* elbo, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar,
                               double* tau2_bar, int32_t* status, int64_t* row, bgm_stream stream) {
  if (!observed.data) return BGM_ERR_ARG;
  vi::LikTerm g{};
  g.kind = 0;
  g.y = y;
  g.obs = observed;
  g.tau2 = tau2;
  g.elbo = elbo;
  g.tau2_bar = tau2_bar;
  return vi::vi_core(m_q, l_q, m_p, l_p, kl, m_q_bar, l_q_bar, status, row, stream, &g);
}

int bgm_elbo_poisson_grad_sel(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, bgm_vec y, bgm_vec weight,
                              bgm_vec observed, int quad_points, double* elbo, double* kl, bgm_vec m_q_bar,
                              bgm_band l_q_bar, int32_t* status, int64_t* row, bgm_stream stream) {
  if (!observed.data) return BGM_ERR_ARG;
  vi::LikTerm g{};
  g.kind = 1;
  g.y = y;
  g.weight = weight;
  g.obs = observed;
  if (!vi::gauss_hermite(quad_points, g.gh)) return BGM_ERR_ARG;
  g.elbo = elbo;
  return vi::vi_core(m_q, l_q, m_p, l_p, kl, m_q_bar, l_q_bar, status, row, stream, &g);
}

int bgm_gauss_hermite(int quad_points, double* x, double* w) {
  vi::GH gh;
  if (!x || !w || !vi::gauss_hermite(quad_points, gh)) return BGM_ERR_ARG;
  for (int i = 0; i < gh.k; ++i) {
    x[i] = gh.x[i];
    w[i] = gh.w[i];
  }
  return BGM_OK;
}

}  // extern "C"
