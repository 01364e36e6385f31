// Segment-parallel config-3 sweeps (placeholder: routes to the generic path).
#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_mlik.cuh"

namespace bgm {

int mlik_fast(const bgm_band&, const bgm_vec&, double, double*, const bgm_band&, double*,
              int32_t*, int64_t*, int, cudaStream_t) {
  return -1;
}

}  // namespace bgm
