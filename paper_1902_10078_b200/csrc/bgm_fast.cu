// Specialised kernels for the benchmarked shapes.  (Filled in incrementally;
// anything not recognised here runs the generic kernels in bgm_ops.cu.)
#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"

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

bool cholesky(const bgm_band&, const bgm_band&, int32_t*, int64_t*, cudaStream_t) { return false; }
bool solve_vec(const bgm_band&, const bgm_vec&, int, const bgm_vec&, int32_t*, int64_t*,
               cudaStream_t) {
  return false;
}
bool log_det(const bgm_band&, void*, int32_t*, int64_t*, cudaStream_t) { return false; }
bool subset(const bgm_band&, const bgm_band&, int32_t*, int64_t*, cudaStream_t) { return false; }
bool product(const bgm_band&, int, const bgm_band&, int, const bgm_band&, cudaStream_t) {
  return false;
}
bool band_vec(const bgm_band&, const bgm_vec&, int, const bgm_vec&, cudaStream_t) { return false; }
bool vjp_cholesky(const bgm_band&, const bgm_band&, const bgm_band&, cudaStream_t) { return false; }
bool vjp_subset(const bgm_band&, const bgm_band&, const bgm_band&, const bgm_band&, int32_t*,
                int64_t*, cudaStream_t) {
  return false;
}
bool vjp_product(const bgm_band&, const bgm_band&, const bgm_band&, const bgm_band&,
                 const bgm_band&, cudaStream_t) {
  return false;
}
bool vjp_band_vec(const bgm_band&, const bgm_vec&, const bgm_vec&, int, const bgm_band&,
                  const bgm_vec&, cudaStream_t) {
  return false;
}

}  // namespace fast
}  // namespace bgm
