// Drop-in bandgm::ops / bandgm::grad over the bandgm_b200 C ABI.
//
// Each entry point validates shapes exactly as the reference does (same
// exception types and messages' meaning), ships the operands' storage blocks
// to the device -- the reference's column-major band storage is the tile-1
// device layout, so this is a plain copy -- runs the sm_100a kernels and
// copies the result back.  Device status codes become the reference's
// exceptions carrying the failing row (errors.hpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "bandgm/grad.hpp"
#include "bandgm/kernels.hpp"
#include "bandgm_b200.h"

namespace bandgm {
namespace {

using Index = BandedMatrix::Index;

// ---------------------------------------------------------------- device glue
cudaMemPool_t drop_pool() {
  static std::once_flag once;
  static cudaMemPool_t pool = nullptr;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    } else {
      pool = nullptr;
    }
  });
  return pool;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

class DevBuf {
 public:
  explicit DevBuf(size_t bytes) : n_(bytes ? bytes : 8) {
    cudaMemPool_t p = drop_pool();
    cuda_check(p ? cudaMallocFromPoolAsync(&p_, n_, p, 0) : cudaMalloc(&p_, n_), "device alloc");
  }
  ~DevBuf() {
    if (p_) cudaFreeAsync(p_, 0);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void* get() const { return p_; }
  double* d() const { return static_cast<double*>(p_); }
  void upload(const void* src, size_t bytes) {
    if (bytes) cuda_check(cudaMemcpy(p_, src, bytes, cudaMemcpyHostToDevice), "upload");
  }
  void download(void* dst, size_t bytes) const {
    if (bytes) cuda_check(cudaMemcpy(dst, p_, bytes, cudaMemcpyDeviceToHost), "download");
  }

 private:
  void* p_ = nullptr;
  size_t n_;
};

size_t band_bytes(const BandedMatrix& a) { return sizeof(double) * size_t(a.storage().size()); }

struct DevBand {
  DevBuf buf;
  bgm_band desc;
  DevBand(Index n, Index lo, Index up) : buf(sizeof(double) * size_t(n * (lo + up + 1))) {
    desc = bgm_band{buf.get(), 1, n, int32_t(lo), int32_t(up), 1, BGM_F64};
  }
  explicit DevBand(const BandedMatrix& a) : DevBand(a.n(), a.lower(), a.upper()) {
    buf.upload(a.storage().data(), band_bytes(a));
  }
  BandedMatrix fetch() const {
    BandedMatrix out(desc.n, desc.lower, desc.upper);
    buf.download(out.storage().data(), band_bytes(out));
    return out;
  }
};

struct DevVec {
  DevBuf buf;
  bgm_vec desc;
  explicit DevVec(Index n) : buf(sizeof(double) * size_t(n)) {
    desc = bgm_vec{buf.get(), 1, n, 1, BGM_F64};
  }
  explicit DevVec(const Eigen::VectorXd& v) : DevVec(v.size()) {
    buf.upload(v.data(), sizeof(double) * size_t(v.size()));
  }
  Eigen::VectorXd fetch() const {
    Eigen::VectorXd v(desc.n);
    buf.download(v.data(), sizeof(double) * size_t(desc.n));
    return v;
  }
};

// Per-call device status (one matrix) mapped to the reference exceptions.
struct Status {
  DevBuf st{sizeof(int32_t)}, row{sizeof(int64_t)};
  Status() {
    const int32_t z = 0;
    const int64_t m1 = -1;
    st.upload(&z, sizeof z);
    row.upload(&m1, sizeof m1);
  }
  int32_t* s() { return static_cast<int32_t*>(st.get()); }
  int64_t* r() { return static_cast<int64_t*>(row.get()); }
  void raise() const {
    int32_t code = 0;
    int64_t at = -1;
    st.download(&code, sizeof code);
    row.download(&at, sizeof at);
    switch (code) {
      case BGM_OK: return;
      case BGM_ERR_NOT_PD: throw NotPositiveDefinite(long(at));
      case BGM_ERR_SINGULAR: throw SingularDiagonal(long(at));
      case BGM_ERR_NONPOS_DIAG: throw NonPositiveDiagonal(long(at));
      default: throw std::runtime_error(std::string("bandgm_b200: ") + bgm_status_name(code));
    }
  }
};

void abi(int rc, const char* op) {
  if (rc == BGM_OK) return;
  if (rc == BGM_ERR_DIM) throw DimensionMismatch(std::string(op) + ": shape mismatch");
  throw std::runtime_error(std::string(op) + ": " + bgm_status_name(rc) + " " + bgm_last_error());
}

// Runs `body` with the calling thread pinned to the reference-loop kernels.
template <class F>
auto generic_only(F&& body) {
  struct Guard {
    Guard() { bgm_force_generic(1); }
    ~Guard() { bgm_force_generic(0); }
  } g;
  return body();
}

Index clip(Index b, Index n) { return std::min(b, n > 0 ? n - 1 : 0); }

void need_lower(const BandedMatrix& l, const char* op) {
  if (l.upper() != 0) throw DimensionMismatch(std::string(op) + ": factor must be lower triangular");
}

}  // namespace

// ==================================================================== ops
namespace ops {

BandedMatrix cholesky(const SymmetricBandedMatrix& q) {
  const BandedMatrix& qs = q.lower_store();
  if (qs.n() == 0) return BandedMatrix(0, 0, 0);
  DevBand dq(qs), dl(qs.n(), qs.lower(), 0);
  Status st;
  abi(bgm_cholesky(dq.desc, dl.desc, st.s(), st.r(), nullptr), "cholesky");
  st.raise();
  return dl.fetch();
}

Eigen::VectorXd solve_vec(const BandedMatrix& l, const Eigen::VectorXd& v, bool transpose_l) {
  need_lower(l, "solve_vec");
  if (v.size() != l.n()) throw DimensionMismatch("solve_vec: vector length mismatch");
  if (l.n() == 0) return Eigen::VectorXd(0);
  DevBand dl(l);
  DevVec dv(v), dx(l.n());
  Status st;
  abi(bgm_solve_vec(dl.desc, dv.desc, transpose_l, dx.desc, st.s(), st.r(), nullptr), "solve_vec");
  st.raise();
  return dx.fetch();
}

BandedMatrix solve_mat(const BandedMatrix& l, const BandedMatrix& r, Index out_lower,
                       Index out_upper, bool transpose_l) {
  need_lower(l, "solve_mat");
  if (r.n() != l.n()) throw DimensionMismatch("solve_mat: size mismatch");
  const Index n = l.n();
  if (n == 0) return BandedMatrix(0, 0, 0);
  DevBand dl(l), dr(r), dout(n, clip(out_lower, n), clip(out_upper, n));
  Status st;
  abi(bgm_solve_mat(dl.desc, dr.desc, transpose_l, dout.desc, st.s(), st.r(), nullptr), "solve_mat");
  st.raise();
  return dout.fetch();
}

SymmetricBandedMatrix sparse_inverse_subset(const BandedMatrix& l) {
  need_lower(l, "sparse_inverse_subset");
  if (l.n() == 0) return SymmetricBandedMatrix(0, 0);
  DevBand dl(l), ds(l.n(), l.lower(), 0);
  Status st;
  abi(bgm_sparse_inverse_subset(dl.desc, ds.desc, st.s(), st.r(), nullptr), "sparse_inverse_subset");
  st.raise();
  return SymmetricBandedMatrix::from_lower(ds.fetch());
}

BandedMatrix product_band_band_restricted(const BandedMatrix& a, const BandedMatrix& b,
                                          Index out_lower, Index out_upper) {
  if (b.n() != a.n()) throw DimensionMismatch("product_band_band: size mismatch");
  const Index n = a.n();
  if (n == 0) return BandedMatrix(0, 0, 0);
  DevBand da(a), db(b), dc(n, clip(out_lower, n), clip(out_upper, n));
  abi(bgm_product_band_band(da.desc, 0, db.desc, 0, dc.desc, nullptr), "product_band_band");
  return dc.fetch();
}

BandedMatrix product_band_band(const BandedMatrix& a, const BandedMatrix& b) {
  return product_band_band_restricted(a, b, a.lower() + b.lower(), a.upper() + b.upper());
}

Eigen::VectorXd product_band_vec(const BandedMatrix& b, const Eigen::VectorXd& v,
                                 bool transpose_b) {
  if (v.size() != b.n()) throw DimensionMismatch("product_band_vec: vector length mismatch");
  if (b.n() == 0) return Eigen::VectorXd(0);
  DevBand db(b);
  DevVec dv(v), dy(b.n());
  abi(bgm_product_band_vec(db.desc, dv.desc, transpose_b, dy.desc, nullptr), "product_band_vec");
  return dy.fetch();
}

BandedMatrix outer_band(const Eigen::VectorXd& m, const Eigen::VectorXd& v, Index lower,
                        Index upper) {
  const Index n = m.size();
  if (v.size() != n) throw DimensionMismatch("outer_band: vector length mismatch");
  if (n == 0) return BandedMatrix(0, 0, 0);
  DevVec dm(m), dv(v);
  DevBand dout(n, clip(lower, n), clip(upper, n));
  abi(bgm_outer_band(dm.desc, dv.desc, 1.0, dout.desc, nullptr), "outer_band");
  return dout.fetch();
}

double log_det_from_cholesky(const BandedMatrix& l) {
  if (l.n() == 0) return 0.0;
  DevBand dl(l);
  DevBuf out(sizeof(double));
  Status st;
  abi(bgm_log_det(dl.desc, out.get(), st.s(), st.r(), nullptr), "log_det_from_cholesky");
  st.raise();
  double v = 0.0;
  out.download(&v, sizeof v);
  return v;
}

namespace serial {
BandedMatrix cholesky_ref(const SymmetricBandedMatrix& q) {
  return generic_only([&] { return ops::cholesky(q); });
}
Eigen::VectorXd solve_vec_ref(const BandedMatrix& l, const Eigen::VectorXd& v, bool transpose_l) {
  return generic_only([&] { return ops::solve_vec(l, v, transpose_l); });
}
BandedMatrix solve_mat_ref(const BandedMatrix& l, const BandedMatrix& r, Index out_lower,
                           Index out_upper, bool transpose_l) {
  return generic_only([&] { return ops::solve_mat(l, r, out_lower, out_upper, transpose_l); });
}
SymmetricBandedMatrix sparse_inverse_subset_ref(const BandedMatrix& l) {
  return generic_only([&] { return ops::sparse_inverse_subset(l); });
}
BandedMatrix product_band_band_restricted_ref(const BandedMatrix& a, const BandedMatrix& b,
                                              Index out_lower, Index out_upper) {
  return generic_only([&] { return ops::product_band_band_restricted(a, b, out_lower, out_upper); });
}
Eigen::VectorXd product_band_vec_ref(const BandedMatrix& b, const Eigen::VectorXd& v,
                                     bool transpose_b) {
  return generic_only([&] { return ops::product_band_vec(b, v, transpose_b); });
}
BandedMatrix outer_band_ref(const Eigen::VectorXd& m, const Eigen::VectorXd& v, Index lower,
                            Index upper) {
  return generic_only([&] { return ops::outer_band(m, v, lower, upper); });
}
}  // namespace serial

}  // namespace ops

// ==================================================================== grad
namespace grad {

SymmetricBandedMatrix vjp_cholesky(const BandedMatrix& l, BandedMatrix l_bar) {
  const Index n = l.n(), bw = l.lower();
  if (l.upper() != 0 || l_bar.upper() != 0 || l_bar.lower() != bw || l_bar.n() != n)
    throw DimensionMismatch("vjp_cholesky: factor and adjoint must share a lower band");
  if (n == 0) return SymmetricBandedMatrix(0, 0);
  DevBand dl(l), dlb(l_bar), dq(n, bw, 0);  // dlb is the consumed copy
  abi(bgm_vjp_cholesky(dl.desc, dlb.desc, dq.desc, nullptr), "vjp_cholesky");
  return SymmetricBandedMatrix::from_lower(dq.fetch());
}

SolveVecVjp vjp_solve_vec(const BandedMatrix& l, const Eigen::VectorXd& s,
                          const Eigen::VectorXd& s_bar, bool transpose_l) {
  need_lower(l, "solve_vec");
  if (s.size() != l.n() || s_bar.size() != l.n())
    throw DimensionMismatch("solve_vec: vector length mismatch");
  SolveVecVjp out;
  if (l.n() == 0) {
    out.l_bar = BandedMatrix(0, 0, 0);
    out.v_bar = Eigen::VectorXd(0);
    return out;
  }
  DevBand dl(l), dlb(l.n(), l.lower(), 0);
  DevVec ds(s), dsb(s_bar), dvb(l.n());
  Status st;
  abi(bgm_vjp_solve_vec(dl.desc, ds.desc, dsb.desc, transpose_l, dlb.desc, dvb.desc, st.s(), st.r(),
                        nullptr),
      "vjp_solve_vec");
  st.raise();
  out.l_bar = dlb.fetch();
  out.v_bar = dvb.fetch();
  return out;
}

SolveMatVjp vjp_solve_mat(const BandedMatrix& l, const BandedMatrix& s, const BandedMatrix& s_bar,
                          Index r_band_lower, Index r_band_upper, bool transpose_l) {
  need_lower(l, "solve_mat");
  const Index n = l.n();
  if (s.n() != n || s_bar.n() != n || !s.same_shape(s_bar))
    throw DimensionMismatch("vjp_solve_mat: shape mismatch");
  SolveMatVjp out;
  if (n == 0) {
    out.l_bar = BandedMatrix(0, 0, 0);
    out.r_bar = BandedMatrix(0, 0, 0);
    return out;
  }
  DevBand dl(l), ds(s), dsb(s_bar), dlb(n, l.lower(), 0),
      drb(n, clip(r_band_lower, n), clip(r_band_upper, n));
  Status st;
  abi(bgm_vjp_solve_mat(dl.desc, ds.desc, dsb.desc, transpose_l, dlb.desc, drb.desc, st.s(), st.r(),
                        nullptr),
      "vjp_solve_mat");
  st.raise();
  out.l_bar = dlb.fetch();
  out.r_bar = drb.fetch();
  return out;
}

BandedMatrix vjp_sparse_inverse_subset(const BandedMatrix& l, const SymmetricBandedMatrix& s,
                                       const SymmetricBandedMatrix& s_bar) {
  const Index n = l.n(), bw = l.lower();
  if (l.upper() != 0) throw DimensionMismatch("vjp_sparse_inverse_subset: lower factor expected");
  if (s.n() != n || s.bandwidth() != bw || s_bar.n() != n || s_bar.bandwidth() != bw)
    throw DimensionMismatch("vjp_sparse_inverse_subset: shape mismatch");
  if (n == 0) return BandedMatrix(0, 0, 0);
  DevBand dl(l), ds(s.lower_store()), dsb(s_bar.lower_store()), dlb(n, bw, 0);
  Status st;
  abi(bgm_vjp_sparse_inverse_subset(dl.desc, ds.desc, dsb.desc, dlb.desc, st.s(), st.r(), nullptr),
      "vjp_sparse_inverse_subset");
  st.raise();
  return dlb.fetch();
}

ProductVjp vjp_product_band_band(const BandedMatrix& a, const BandedMatrix& b,
                                 const BandedMatrix& p_bar) {
  if (b.n() != a.n() || p_bar.n() != a.n()) throw DimensionMismatch("product_band_band: size mismatch");
  ProductVjp out;
  const Index n = a.n();
  if (n == 0) {
    out.a_bar = BandedMatrix(0, 0, 0);
    out.b_bar = BandedMatrix(0, 0, 0);
    return out;
  }
  DevBand da(a), db(b), dp(p_bar), dab(n, a.lower(), a.upper()), dbb(n, b.lower(), b.upper());
  abi(bgm_vjp_product_band_band(da.desc, db.desc, dp.desc, dab.desc, dbb.desc, nullptr),
      "vjp_product_band_band");
  out.a_bar = dab.fetch();
  out.b_bar = dbb.fetch();
  return out;
}

ProductVecVjp vjp_product_band_vec(const BandedMatrix& b, const Eigen::VectorXd& v,
                                   const Eigen::VectorXd& p_bar, bool transpose_b) {
  if (v.size() != b.n() || p_bar.size() != b.n())
    throw DimensionMismatch("product_band_vec: vector length mismatch");
  ProductVecVjp out;
  const Index n = b.n();
  if (n == 0) {
    out.b_bar = BandedMatrix(0, 0, 0);
    out.v_bar = Eigen::VectorXd(0);
    return out;
  }
  DevBand db(b), dbb(n, b.lower(), b.upper());
  DevVec dv(v), dp(p_bar), dvb(n);
  abi(bgm_vjp_product_band_vec(db.desc, dv.desc, dp.desc, transpose_b, dbb.desc, dvb.desc, nullptr),
      "vjp_product_band_vec");
  out.b_bar = dbb.fetch();
  out.v_bar = dvb.fetch();
  return out;
}

OuterVjp vjp_outer_band(const Eigen::VectorXd& m, const Eigen::VectorXd& v,
                        const BandedMatrix& o_bar) {
  const Index n = m.size();
  if (v.size() != n || o_bar.n() != n) throw DimensionMismatch("outer_band: vector length mismatch");
  OuterVjp out;
  if (n == 0) {
    out.m_bar = Eigen::VectorXd(0);
    out.v_bar = Eigen::VectorXd(0);
    return out;
  }
  DevVec dm(m), dv(v), dmb(n), dvb(n);
  DevBand dob(o_bar);
  abi(bgm_vjp_outer_band(dm.desc, dv.desc, dob.desc, dmb.desc, dvb.desc, nullptr), "vjp_outer_band");
  out.m_bar = dmb.fetch();
  out.v_bar = dvb.fetch();
  return out;
}

BandedMatrix vjp_log_det_from_cholesky(const BandedMatrix& l, double c_bar) {
  if (l.n() == 0) return BandedMatrix(0, l.lower(), 0);
  DevBand dl(l), dlb(l.n(), l.lower(), 0);
  DevBuf cb(sizeof(double));
  cb.upload(&c_bar, sizeof c_bar);
  abi(bgm_vjp_log_det(dl.desc, cb.get(), dlb.desc, nullptr), "vjp_log_det_from_cholesky");
  return dlb.fetch();
}

// Central differences with per-coordinate step eps (|x| + 1) and an absolute
// floor on the relative error (the reference's checker, grad.hpp:78-92).
FiniteDiffReport finite_diff_check(const std::function<double(const Eigen::VectorXd&)>& f,
                                   const Eigen::VectorXd& x0, const Eigen::VectorXd& analytic_grad,
                                   double eps, double abs_floor) {
  const Eigen::Index dim = x0.size();
  if (analytic_grad.size() != dim) throw DimensionMismatch("finite_diff_check: gradient length mismatch");
  FiniteDiffReport rep;
  rep.fd = Eigen::VectorXd::Zero(dim);
  rep.rel = Eigen::VectorXd::Zero(dim);
  rep.analytic = analytic_grad;
  Eigen::VectorXd x = x0;
  for (Eigen::Index k = 0; k < dim; ++k) {
    const double step = eps * (std::abs(x0(k)) + 1.0);
    x(k) = x0(k) + step;
    const double up = f(x);
    x(k) = x0(k) - step;
    const double dn = f(x);
    x(k) = x0(k);
    const double g = (up - dn) / (2.0 * step);
    const double err = std::abs(g - analytic_grad(k));
    const double den = std::max(std::max(std::abs(g), std::abs(analytic_grad(k))), abs_floor);
    rep.fd(k) = g;
    rep.rel(k) = err / den;
    rep.max_abs_err = std::max(rep.max_abs_err, err);
    if (rep.rel(k) > rep.max_rel_err) {
      rep.max_rel_err = rep.rel(k);
      rep.worst_index = k;
    }
  }
  return rep;
}

}  // namespace grad
}  // namespace bandgm
