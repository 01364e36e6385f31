// CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the reference bandgm library, which oracle/Makefile
// compiles verbatim from /root/reference/proj/src (banded, kernels_serial,
// kernels, grad, gradcheck, tape) against the original Eigen-subset header in
// paper_1902_10078_b200/cpp/eigen_shim.  Output goes to oracle/_ref/ only.
//
// The functions mirror oracle/bandgm_oracle.c one for one (prefix ref_
// instead of orc_) so tests can run the same checks against either.  Each
// matrix is the reference's own storage block (BandedMatrix::storage(),
// banded.hpp:77-79): column-major (lower+upper+1) x n, batch-major.
// Exceptions (errors.hpp:27-50) become per-matrix status codes + rows.
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <cstring>
#include <sstream>
#include <functional>
#include <random>
#include <string>

#include "bandgm/grad.hpp"
#include "bandgm/gradcheck.hpp"
#include "bandgm/kernels.hpp"
#include "bandgm/tape.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace bandgm;
using Index = Eigen::Index;
using ix = std::int64_t;

namespace {

enum { kOk = 0, kNotPd = 1, kSingular = 2, kNonPos = 3, kDim = 4, kOther = 5 };

BandedMatrix load(ix n, ix lo, ix up, const double* p) {
  BandedMatrix m(n, lo, up);
  std::memcpy(m.storage().data(), p, sizeof(double) * static_cast<size_t>(n * (lo + up + 1)));
  return m;
}
SymmetricBandedMatrix load_sym(ix n, ix bw, const double* p) {
  return SymmetricBandedMatrix::from_lower(load(n, bw, 0, p));
}
void store(const BandedMatrix& m, double* p) {
  std::memcpy(p, m.storage().data(), sizeof(double) * static_cast<size_t>(m.storage().size()));
}
Eigen::VectorXd load_vec(ix n, const double* p) {
  Eigen::VectorXd v(n);
  std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
  return v;
}
void store_vec(const Eigen::VectorXd& v, double* p) {
  std::memcpy(p, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
}

// Runs body, mapping the reference's exceptions to (status, row).
int guarded(const std::function<void()>& body, ix* row) {
  *row = -1;
  try {
    body();
  } catch (const NotPositiveDefinite& e) {
    *row = e.row;
    return kNotPd;
  } catch (const SingularDiagonal& e) {
    *row = e.row;
    return kSingular;
  } catch (const NonPositiveDiagonal& e) {
    *row = e.row;
    return kNonPos;
  } catch (const DimensionMismatch&) {
    return kDim;
  } catch (...) {
    return kOther;
  }
  return kOk;
}

// Batch loop: matrices in parallel, the reference's own inner OpenMP off.
template <class F>
void over_batch(ix batch, F&& f) {
#ifdef _OPENMP
  omp_set_max_active_levels(1);
#pragma omp parallel for schedule(dynamic)
#endif
  for (ix b = 0; b < batch; ++b) f(b);
}

constexpr double kLog2Pi = 1.8378770664093454836;  // inference.cpp:15

}  // namespace

extern "C" {

int ref_cholesky(ix batch, ix n, ix bw, const double* q, double* l, std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded([&] { store(ops::cholesky(load_sym(n, bw, q + b * n * w)), l + b * n * w); },
                        &row[b]);
  });
  return 0;
}

int ref_solve_vec(ix batch, ix n, ix bw, const double* l, const double* v, int tr, double* x,
                  std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          store_vec(ops::solve_vec(load(n, bw, 0, l + b * n * w), load_vec(n, v + b * n), tr != 0),
                    x + b * n);
        },
        &row[b]);
  });
  return 0;
}

int ref_log_det(ix batch, ix n, ix bw, const double* l, double* out, std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] { out[b] = ops::log_det_from_cholesky(load(n, bw, 0, l + b * n * w)); }, &row[b]);
  });
  return 0;
}

int ref_sparse_inverse_subset(ix batch, ix n, ix bw, const double* l, double* s,
                              std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          store(ops::sparse_inverse_subset(load(n, bw, 0, l + b * n * w)).lower_store(),
                s + b * n * w);
        },
        &row[b]);
  });
  return 0;
}

int ref_product_band_band(ix batch, ix n, ix al, ix au, const double* a, ix bl, ix bu,
                          const double* bm, ix ol, ix ou, double* c) {
  over_batch(batch, [&](ix b) {
    store(ops::product_band_band_restricted(load(n, al, au, a + b * n * (al + au + 1)),
                                            load(n, bl, bu, bm + b * n * (bl + bu + 1)), ol, ou),
          c + b * n * (ol + ou + 1));
  });
  return 0;
}

int ref_product_band_vec(ix batch, ix n, ix bl, ix bu, const double* bm, const double* v, int tr,
                         double* y) {
  over_batch(batch, [&](ix b) {
    store_vec(ops::product_band_vec(load(n, bl, bu, bm + b * n * (bl + bu + 1)),
                                    load_vec(n, v + b * n), tr != 0),
              y + b * n);
  });
  return 0;
}

int ref_outer_band(ix batch, ix n, const double* m, const double* v, ix lo, ix up, double* out) {
  over_batch(batch, [&](ix b) {
    store(ops::outer_band(load_vec(n, m + b * n), load_vec(n, v + b * n), lo, up),
          out + b * n * (lo + up + 1));
  });
  return 0;
}

int ref_solve_mat(ix batch, ix n, ix bw, const double* l, ix rl, ix ru, const double* r, ix ol,
                  ix ou, int tr, double* out, std::int32_t* status, ix* row) {
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          store(ops::solve_mat(load(n, bw, 0, l + b * n * (bw + 1)),
                               load(n, rl, ru, r + b * n * (rl + ru + 1)), ol, ou, tr != 0),
                out + b * n * (ol + ou + 1));
        },
        &row[b]);
  });
  return 0;
}

int ref_vjp_cholesky(ix batch, ix n, ix bw, const double* l, const double* lbar, double* qbar) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    store(grad::vjp_cholesky(load(n, bw, 0, l + b * n * w), load(n, bw, 0, lbar + b * n * w))
              .lower_store(),
          qbar + b * n * w);
  });
  return 0;
}

int ref_vjp_solve_vec(ix batch, ix n, ix bw, const double* l, const double* s, const double* sbar,
                      int tr, double* lbar, double* vbar, std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          const auto r = grad::vjp_solve_vec(load(n, bw, 0, l + b * n * w), load_vec(n, s + b * n),
                                             load_vec(n, sbar + b * n), tr != 0);
          store(r.l_bar, lbar + b * n * w);
          store_vec(r.v_bar, vbar + b * n);
        },
        &row[b]);
  });
  return 0;
}

int ref_vjp_sparse_inverse_subset(ix batch, ix n, ix bw, const double* l, const double* s,
                                  const double* sbar, double* lbar, std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          store(grad::vjp_sparse_inverse_subset(load(n, bw, 0, l + b * n * w),
                                                load_sym(n, bw, s + b * n * w),
                                                load_sym(n, bw, sbar + b * n * w)),
                lbar + b * n * w);
        },
        &row[b]);
  });
  return 0;
}

int ref_vjp_product_band_band(ix batch, ix n, ix al, ix au, const double* a, ix bl, ix bu,
                              const double* bm, ix pl, ix pu, const double* pbar, double* abar,
                              double* bbar) {
  over_batch(batch, [&](ix b) {
    const auto r = grad::vjp_product_band_band(load(n, al, au, a + b * n * (al + au + 1)),
                                               load(n, bl, bu, bm + b * n * (bl + bu + 1)),
                                               load(n, pl, pu, pbar + b * n * (pl + pu + 1)));
    store(r.a_bar, abar + b * n * (al + au + 1));
    store(r.b_bar, bbar + b * n * (bl + bu + 1));
  });
  return 0;
}

int ref_vjp_product_band_vec(ix batch, ix n, ix bl, ix bu, const double* bm, const double* v,
                             const double* pbar, int tr, double* bbar, double* vbar) {
  over_batch(batch, [&](ix b) {
    const auto r = grad::vjp_product_band_vec(load(n, bl, bu, bm + b * n * (bl + bu + 1)),
                                              load_vec(n, v + b * n), load_vec(n, pbar + b * n),
                                              tr != 0);
    store(r.b_bar, bbar + b * n * (bl + bu + 1));
    store_vec(r.v_bar, vbar + b * n);
  });
  return 0;
}

int ref_vjp_outer_band(ix batch, ix n, const double* m, const double* v, ix ol, ix ou,
                       const double* obar, double* mbar, double* vbar) {
  over_batch(batch, [&](ix b) {
    const auto r = grad::vjp_outer_band(load_vec(n, m + b * n), load_vec(n, v + b * n),
                                        load(n, ol, ou, obar + b * n * (ol + ou + 1)));
    store_vec(r.m_bar, mbar + b * n);
    store_vec(r.v_bar, vbar + b * n);
  });
  return 0;
}

int ref_vjp_log_det(ix batch, ix n, ix bw, const double* l, const double* cbar, double* lbar) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    store(grad::vjp_log_det_from_cholesky(load(n, bw, 0, l + b * n * w), cbar[b]), lbar + b * n * w);
  });
  return 0;
}

int ref_vjp_solve_mat(ix batch, ix n, ix bw, const double* l, ix sl, ix su, const double* s,
                      const double* sbar, ix rl, ix ru, int tr, double* lbar, double* rbar,
                      std::int32_t* status, ix* row) {
  const ix rlc = std::min<ix>(rl, n - 1), ruc = std::min<ix>(ru, n - 1);
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          const auto r = grad::vjp_solve_mat(load(n, bw, 0, l + b * n * (bw + 1)),
                                             load(n, sl, su, s + b * n * (sl + su + 1)),
                                             load(n, sl, su, sbar + b * n * (sl + su + 1)), rl, ru,
                                             tr != 0);
          store(r.l_bar, lbar + b * n * (bw + 1));
          store(r.r_bar, rbar + b * n * (rlc + ruc + 1));
        },
        &row[b]);
  });
  return 0;
}

// Config-3 composite: infer::marginal_likelihood_partial (inference.cpp:140-163)
// restated over the compiled reference Tape with every node observed, with
// Q = precision_from_factor(L) (inference.cpp:23-26), then the dL chain
// through grad::vjp_product_band_band(L, transpose(L), G).
int ref_marginal_likelihood_grad(ix batch, ix n, ix bw, const double* L, const double* y,
                                 double tau2, double* loss, double* lbar, double* tau2_bar,
                                 std::int32_t* status, ix* row) {
  const ix w = bw + 1;
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          const BandedMatrix l = load(n, bw, 0, L + b * n * w);
          const Eigen::VectorXd yv = load_vec(n, y + b * n);
          const SymmetricBandedMatrix q = SymmetricBandedMatrix::from_lower(
              ops::product_band_band_restricted(l, transpose(l), bw, 0));
          tape::Tape t;
          const tape::NodeRef qn = t.leaf("q", q);
          const tape::NodeRef tau = t.leaf("tau2", tau2);
          const double nn = static_cast<double>(n);
          const Eigen::VectorXd mask = Eigen::VectorXd::Ones(n);
          const tape::NodeRef inv_tau = t.div(t.constant(1.0), tau);
          const tape::NodeRef lp =
              t.cholesky(t.add_diagonal_sym(qn, t.scale_vec(t.constant(mask), inv_tau)));
          const tape::NodeRef wn = t.solve_vec(lp, t.constant(yv));
          tape::NodeRef obj = t.constant(-0.5 * nn * kLog2Pi);
          obj = t.add(obj, t.neg(t.log_det_from_cholesky(lp)));
          obj = t.add(obj, t.log_det_from_cholesky(t.cholesky(qn)));
          obj = t.add(obj, t.mul(t.constant(-0.5 * nn), t.log(tau)));
          obj = t.add(obj, t.mul(t.constant(-0.5 * yv.squaredNorm()), inv_tau));
          obj = t.add(obj, t.mul(t.constant(0.5), t.mul(t.dot(wn, wn), t.mul(inv_tau, inv_tau))));
          loss[b] = t.scalar(obj);
          auto grads = t.backward(obj);
          const auto& qbar = std::get<SymmetricBandedMatrix>(grads.at("q"));
          tau2_bar[b] = std::get<double>(grads.at("tau2"));
          const auto pv = grad::vjp_product_band_band(l, transpose(l), qbar.lower_store());
          store(add(pv.a_bar, transpose(pv.b_bar)), lbar + b * n * w);
        },
        &row[b]);
  });
  return 0;
}

// VI objective term: infer::kl_divergence (inference.cpp:247-268) restated
// over the compiled reference Tape node for node -- trace_product_sym of the
// inverse subset with the prior precision (tape.cpp:274-302), the log-det
// difference, the whitened mean difference -- with precision_from_factor
// (inference.cpp:23-26) as the restricted product.  Gradients in m_q and L_q
// (stored cells) come from Tape::backward.
int ref_kl_divergence_grad(ix batch, ix n, ix bq, ix bp, const double* mq, const double* lq,
                           const double* mp, const double* lp, double* kl, double* mq_bar,
                           double* lq_bar, std::int32_t* status, ix* row, const double* obs) {
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          const BandedMatrix l_q = load(n, bq, 0, lq + b * n * (bq + 1));
          const BandedMatrix l_p = load(n, bp, 0, lp + b * n * (bp + 1));
          const Eigen::VectorXd m_q = load_vec(n, mq + b * n);
          const Eigen::VectorXd m_p = load_vec(n, mp + b * n);
          const SymmetricBandedMatrix qp = SymmetricBandedMatrix::from_lower(
              ops::product_band_band_restricted(l_p, transpose(l_p), bp, 0));
          const double logdet_p = ops::log_det_from_cholesky(l_p);
          tape::Tape t;
          const tape::NodeRef mn = t.leaf("m", m_q);
          const tape::NodeRef ln = t.leaf("l", l_q);
          const tape::NodeRef trace = t.trace_product_sym(t.sparse_inverse_subset(ln), t.constant(qp));
          const tape::NodeRef logdets =
              t.mul(t.constant(2.0), t.sub(t.log_det_from_cholesky(ln), t.constant(logdet_p)));
          const tape::NodeRef diff = t.sub_vec(t.constant(m_p), mn);
          const tape::NodeRef white = t.product_band_vec(t.constant(l_p), diff, true);
          tape::NodeRef inner = t.add(trace, logdets);
          inner = t.add(inner, t.dot(white, white));
          inner = t.add(inner, t.constant(-static_cast<double>(n)));
          const tape::NodeRef obj = t.mul(t.constant(0.5), inner);
          kl[b] = t.scalar(obj);
          auto grads = t.backward(obj);
          store_vec(std::get<Eigen::VectorXd>(grads.at("m")), mq_bar + b * n);
          store(std::get<BandedMatrix>(grads.at("l")), lq_bar + b * n * (bq + 1));
        },
        &row[b]);
  });
  return 0;
}

// infer::elbo (inference.cpp:276-287) for a GaussianLik observing the
// latents marked in obs (every latent when obs is null): the Gaussian branch of expected_loglik (inference.cpp:52-63,
// anonymous in the reference, restated) joins the compiled reference Tape as
// a linearized scalar over (m_q, diag_sym(subset(L_q))), minus the KL built
// node for node as in ref_kl_divergence_grad.
int ref_elbo_gaussian_grad(ix batch, ix n, ix bq, ix bp, const double* mq, const double* lq,
                           const double* mp, const double* lp, const double* y, double tau2,
                           double* elbo, double* mq_bar, double* lq_bar, double* tau2_bar,
                           std::int32_t* status, ix* row, const double* obs) {
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          const BandedMatrix l_q = load(n, bq, 0, lq + b * n * (bq + 1));
          const BandedMatrix l_p = load(n, bp, 0, lp + b * n * (bp + 1));
          const Eigen::VectorXd m_q = load_vec(n, mq + b * n);
          const Eigen::VectorXd m_p = load_vec(n, mp + b * n);
          const Eigen::VectorXd yv = load_vec(n, y + b * n);
          const SymmetricBandedMatrix qp = SymmetricBandedMatrix::from_lower(
              ops::product_band_band_restricted(l_p, transpose(l_p), bp, 0));
          const double logdet_p = ops::log_det_from_cholesky(l_p);
          tape::Tape t;
          const tape::NodeRef mn = t.leaf("m", m_q);
          const tape::NodeRef ln = t.leaf("l", l_q);
          // expected log-likelihood (inference.cpp:278-285)
          const tape::NodeRef marg_var = t.diag_sym(t.sparse_inverse_subset(ln));
          const Eigen::VectorXd& mean = t.vector(mn);
          const Eigen::VectorXd& var = t.vector(marg_var);
          const double kLog2Pi = 1.8378770664093454836;
          double value = 0.0, d_tau2 = 0.0;
          Eigen::VectorXd d_mean = Eigen::VectorXd::Zero(n), d_var = Eigen::VectorXd::Zero(n);
          for (ix i = 0; i < n; ++i) {
            // SelectionIndex (models.hpp:122-128): the reference loops over
            // sel.observed with y in selection order; here y is scattered to
            // full length and obs marks the observed latents (null = all)
            if (obs && obs[b * n + i] == 0.0) continue;
            const double r = yv(i) - mean(i);
            value += -0.5 * (std::log(tau2) + kLog2Pi) - (r * r + var(i)) / (2.0 * tau2);
            d_mean(i) = r / tau2;
            d_var(i) = -0.5 / tau2;
            d_tau2 += (r * r + var(i)) / (2.0 * tau2 * tau2) - 0.5 / tau2;
          }
          const tape::NodeRef ve = t.linearized_scalar(value, {{mn, d_mean}, {marg_var, d_var}});
          // kl_divergence (inference.cpp:255-267)
          const tape::NodeRef trace = t.trace_product_sym(t.sparse_inverse_subset(ln), t.constant(qp));
          const tape::NodeRef logdets =
              t.mul(t.constant(2.0), t.sub(t.log_det_from_cholesky(ln), t.constant(logdet_p)));
          const tape::NodeRef diff = t.sub_vec(t.constant(m_p), mn);
          const tape::NodeRef white = t.product_band_vec(t.constant(l_p), diff, true);
          tape::NodeRef inner = t.add(trace, logdets);
          inner = t.add(inner, t.dot(white, white));
          inner = t.add(inner, t.constant(-static_cast<double>(n)));
          const tape::NodeRef obj = t.sub(ve, t.mul(t.constant(0.5), inner));
          elbo[b] = t.scalar(obj);
          tau2_bar[b] = d_tau2;
          auto grads = t.backward(obj);
          store_vec(std::get<Eigen::VectorXd>(grads.at("m")), mq_bar + b * n);
          store(std::get<BandedMatrix>(grads.at("l")), lq_bar + b * n * (bq + 1));
        },
        &row[b]);
  });
  return 0;
}

// infer::elbo (inference.cpp:276-287) for a PoissonLik observing the
// latents marked in obs (every latent when obs is null): the Poisson branch of expected_loglik (inference.cpp:65-100,
// restated) with the Gauss-Hermite rule passed in by the caller (the tests
// use numpy's hermgauss, independent of the library's own Golub-Welsch),
// joined to the compiled reference Tape as in ref_elbo_gaussian_grad.
int ref_elbo_poisson_grad(ix batch, ix n, ix bq, ix bp, const double* mq, const double* lq,
                          const double* mp, const double* lp, const double* y, const double* wt,
                          ix nq, const double* ghx, const double* ghw, double* elbo, double* mq_bar,
                          double* lq_bar, std::int32_t* status, ix* row, const double* obs) {
  over_batch(batch, [&](ix b) {
    status[b] = guarded(
        [&] {
          const BandedMatrix l_q = load(n, bq, 0, lq + b * n * (bq + 1));
          const BandedMatrix l_p = load(n, bp, 0, lp + b * n * (bp + 1));
          const Eigen::VectorXd m_q = load_vec(n, mq + b * n);
          const Eigen::VectorXd m_p = load_vec(n, mp + b * n);
          const Eigen::VectorXd yv = load_vec(n, y + b * n);
          const Eigen::VectorXd wv = load_vec(n, wt + b * n);
          const SymmetricBandedMatrix qp = SymmetricBandedMatrix::from_lower(
              ops::product_band_band_restricted(l_p, transpose(l_p), bp, 0));
          tape::Tape t;
          const tape::NodeRef mn = t.leaf("m", m_q);
          const tape::NodeRef ln = t.leaf("l", l_q);
          const tape::NodeRef marg_var = t.diag_sym(t.sparse_inverse_subset(ln));
          const Eigen::VectorXd& mean = t.vector(mn);
          const Eigen::VectorXd& var = t.vector(marg_var);
          const double norm = 1.0 / std::sqrt(M_PI);
          double value = 0.0;
          Eigen::VectorXd d_mean = Eigen::VectorXd::Zero(n), d_var = Eigen::VectorXd::Zero(n);
          for (ix i = 0; i < n; ++i) {
            if (obs && obs[b * n + i] == 0.0) continue;  // SelectionIndex, as in the Gaussian case
            const double w = wv(i);
            if (w <= 0.0) throw std::invalid_argument("weight");
            const double m = mean(i), v = var(i);
            const double base = yv(i) * std::log(w) - std::lgamma(yv(i) + 1.0);
            if (v <= 0.0) {
              value += yv(i) * m + base - w * std::exp(m);
              d_mean(i) = yv(i) - w * std::exp(m);
              continue;
            }
            const double spread = std::sqrt(2.0 * v);
            double ev = 0.0, dm = 0.0, dv = 0.0;
            for (ix k = 0; k < nq; ++k) {
              const double f = m + spread * ghx[k];
              const double rate = w * std::exp(f);
              ev += ghw[k] * (yv(i) * f - rate);
              const double gprime = yv(i) - rate;
              dm += ghw[k] * gprime;
              dv += ghw[k] * gprime * ghx[k] / spread;
            }
            value += norm * ev + base;
            d_mean(i) = norm * dm;
            d_var(i) = norm * dv;
          }
          const tape::NodeRef ve = t.linearized_scalar(value, {{mn, d_mean}, {marg_var, d_var}});
          const double logdet_p = ops::log_det_from_cholesky(l_p);
          const tape::NodeRef trace = t.trace_product_sym(t.sparse_inverse_subset(ln), t.constant(qp));
          const tape::NodeRef logdets =
              t.mul(t.constant(2.0), t.sub(t.log_det_from_cholesky(ln), t.constant(logdet_p)));
          const tape::NodeRef diff = t.sub_vec(t.constant(m_p), mn);
          const tape::NodeRef white = t.product_band_vec(t.constant(l_p), diff, true);
          tape::NodeRef inner = t.add(trace, logdets);
          inner = t.add(inner, t.dot(white, white));
          inner = t.add(inner, t.constant(-static_cast<double>(n)));
          const tape::NodeRef obj = t.sub(ve, t.mul(t.constant(0.5), inner));
          elbo[b] = t.scalar(obj);
          auto grads = t.backward(obj);
          store_vec(std::get<Eigen::VectorXd>(grads.at("m")), mq_bar + b * n);
          store(std::get<BandedMatrix>(grads.at("l")), lq_bar + b * n * (bq + 1));
        },
        &row[b]);
  });
  return 0;
}

// write_band_text (banded.cpp:192-202), verbatim, into a caller buffer: the
// byte-level pin of the Python band text writer.  Returns the length, or -1
// when the buffer is too small.
long long ref_write_band_text(ix n, ix lo, ix up, const double* a, char* buf, long long cap) {
  std::ostringstream os;
  write_band_text(os, load(n, lo, up, a));
  const std::string s = os.str();
  if (static_cast<long long>(s.size()) + 1 > cap) return -1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<long long>(s.size());
}

// Reference gradient suite (gradcheck.cpp:288-304), used to pin the oracle
// build against the reference's own FD tests (test_grad.cpp:32-40,
// acceptance.cpp:142-147).  Writes one max-rel-err per op in op_names() order.
int ref_run_grad_suite(std::uint64_t seed, int instances, double* max_rel_err, int max_ops) {
  const auto reps = gradcheck::run_suite(seed, instances);
  int k = 0;
  for (const auto& r : reps) {
    if (k >= max_ops) break;
    max_rel_err[k++] = r.max_rel_err;
  }
  return k;
}

int ref_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int ref_abi_version(void) { return 1; }

}  // extern "C"
