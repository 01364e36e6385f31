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
                             double* part2, Vec<double> dm) {
  const ix nch = chunks(y.n);
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * nch) return;
  const ix mb = t % batch, c = t / batch;
  const ix j1 = (c + 1) * kChunk < y.n ? (c + 1) * kChunk : y.n;
  const double lt = -0.5 * (log(t2) + kLog2Pi);
  double v = 0.0, dt = 0.0;
  for (ix i = c * kChunk; i < j1; ++i) {
    const double r = y(mb, i) - m(mb, i), var = S.cell(mb, 0, i);
    v += lt - (r * r + var) / (2.0 * t2);
    dt += (r * r + var) / (2.0 * t2 * t2) - 0.5 / t2;
    dm(mb, i) = r / t2;
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

struct GaussTerm {
  bgm_vec y;
  double tau2;
  double* elbo;
  double* tau2_bar;  // may be null
};

// KL(q || p) (inference.cpp:247-268) and, with `g`, the Gaussian ELBO
// (inference.cpp:276-287): expected log-likelihood minus KL.  Gradients in
// (m_q, L_q) of the objective computed (KL, or the ELBO).
int vi_core(bgm_vec m_q, bgm_band l_q, bgm_vec m_p, bgm_band l_p, double* kl, bgm_vec m_q_bar, bgm_band l_q_bar,
            int32_t* status, int64_t* row, bgm_stream stream, const GaussTerm* g) {
  if (!ok_band(l_q) || !ok_band(l_p) || !ok_band(l_q_bar) || !ok_vec(m_q) || !ok_vec(m_p) || !ok_vec(m_q_bar))
    return BGM_ERR_ARG;
  if (g && (!ok_vec(g->y) || !(g->tau2 > 0.0))) return BGM_ERR_ARG;  // NonPositiveParam("tau2")
  const ix B = l_q.batch, n = l_q.n;
  if (B > 0 && (!kl || (g && !g->elbo))) return BGM_ERR_ARG;
  const bool same = l_p.batch == B && m_q.batch == B && m_p.batch == B && m_q_bar.batch == B && l_q_bar.batch == B &&
                    l_p.n == n && m_q.n == n && m_p.n == n && m_q_bar.n == n && l_q_bar.n == n &&
                    (!g || (g->y.batch == B && g->y.n == n));
  const int tile = l_q.tile;
  const bool tiles = l_p.tile == tile && m_q.tile == tile && m_p.tile == tile && m_q_bar.tile == tile &&
                     l_q_bar.tile == tile && (!g || g->y.tile == tile);
  if (!same || !tiles || l_q.upper != 0 || l_p.upper != 0 || l_q_bar.lower != l_q.lower || l_q_bar.upper != 0 ||
      l_q.lower < l_p.lower)  // inference.cpp:252-253
    return BGM_ERR_DIM;
  if (B == 0 || n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  timing::Scope t(g ? "elbo_grad" : "kl_divergence_grad", s);
  const ix nch = chunks(n);
  bgm_band S = l_q, Sb = l_q, Qp = l_p;
  bgm_vec d = m_q, wv = m_q, dm = m_q;
  const size_t scal = sizeof(double) * size_t(B);
  const size_t total = 2 * band_bytes(l_q) + band_bytes(l_p) + 3 * vec_bytes(m_q) + 7 * scal +
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
    k_gauss_part<<<blocks_for(B * nch, kThreads), kThreads, 0, s>>>(view<double>(g->y), view<double>(m_q),
                                                                     view<double>(S), g->tau2, B, part, part2,
                                                                     view<double>(dm));
    k_sum_parts<<<blocks_for(B, kThreads), kThreads, 0, s>>>(part, nch, B, ve);
    if (g->tau2_bar) k_sum_parts<<<blocks_for(B, kThreads), kThreads, 0, s>>>(part2, nch, B, g->tau2_bar);
    k_elbo_final<<<blocks_for(B, kThreads), kThreads, 0, s>>>(ve, kl, B, g->elbo);
    k_rsub<<<blocks_for(vwork, kThreads), kThreads, 0, s>>>(view<double>(dm), view<double>(m_q_bar), B);
    k_add_diag<<<blocks_for(bwork, kThreads), kThreads, 0, s>>>(view<double>(Sb), -0.5 / g->tau2, B);
  }
  if ((rc = bgm_vjp_sparse_inverse_subset(l_q, S, Sb, l_q_bar, st[3], rw[3], stream))) return rc;
  k_scale_logdet_bar<<<blocks_for(bwork, kThreads), kThreads, 0, s>>>(view<double>(l_q_bar), view<double>(l_q), sgn,
                                                                       B);
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
  const vi::GaussTerm g{y, tau2, elbo, tau2_bar};
  return vi::vi_core(m_q, l_q, m_p, l_p, kl, m_q_bar, l_q_bar, status, row, stream, &g);
}

}  // extern "C"
