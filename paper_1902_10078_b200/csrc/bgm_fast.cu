// Specialised kernels for the benchmarked shapes.  (Filled in incrementally;
// anything not recognised here runs the generic kernels in bgm_ops.cu.)
#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace fast {

namespace {
thread_local bool t_force_generic = false;
}

bool disabled() {
  static const bool off = [] {
    const char* e = std::getenv("BGM_GENERIC_ONLY");
    return e && e[0] == '1';
  }();
  return off || t_force_generic;
}

}  // namespace fast
}  // namespace bgm

extern "C" int bgm_force_generic(int on) {
  bgm::fast::t_force_generic = on != 0;
  return BGM_OK;
}

namespace bgm {
namespace fast {

bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  if (disabled()) return false;
  return narrow::cholesky(q, l, st, row, s) || wide::cholesky(q, l, st, row, s) ||
         promote::cholesky(q, l, st, row, s);
}
bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s) {
  if (disabled()) return false;
  return narrow::solve_vec(l, v, tr, x, st, row, s) || wide::solve_vec(l, v, tr, x, st, row, s) ||
         promote::solve_vec(l, v, tr, x, st, row, s);
}
bool log_det(const bgm_band& l, void* out, int32_t* st, int64_t* row, cudaStream_t s) {
  if (disabled()) return false;
  return wide::log_det(l, out, st, row, s);
}
bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  if (disabled()) return false;
  return narrow::subset(l, sb, st, row, s) || wide::subset(l, sb, st, row, s) || promote::subset(l, sb, st, row, s);
}
bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  if (disabled()) return false;
  return stream::product(a, ta, b, tb, c, s) || prod::product(a, ta, b, tb, c, s);
}
bool band_vec(const bgm_band& b, const bgm_vec& v, int tr, const bgm_vec& y, cudaStream_t s) {
  if (disabled()) return false;
  return prod::band_vec(b, v, tr, y, s);
}
bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  if (disabled()) return false;
  return narrow::vjp_cholesky(l, lb, qb, s) || wide::vjp_cholesky(l, lb, qb, s) ||
         promote::vjp_cholesky(l, lb, qb, s);
}
bool vjp_subset(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb, int32_t* st,
                int64_t* row, cudaStream_t s) {
  if (disabled()) return false;
  return wide::vjp_subset(l, sm, sb, lb, st, row, s) || promote::vjp_subset(l, sm, sb, lb, st, row, s);
}
bool vjp_product(const bgm_band& a, const bgm_band& b, const bgm_band& pb, const bgm_band& ab,
                 const bgm_band& bb, cudaStream_t s) {
  if (disabled()) return false;
  return stream::vjp_product(a, b, pb, ab, bb, s);
}
bool vjp_band_vec(const bgm_band& b, const bgm_vec& v, const bgm_vec& pb, int tr, const bgm_band& bb,
                  const bgm_vec& vb, cudaStream_t s) {
  if (disabled()) return false;
  return prod::vjp_band_vec(b, v, pb, tr, bb, vb, s);
}

}  // namespace fast
}  // namespace bgm
