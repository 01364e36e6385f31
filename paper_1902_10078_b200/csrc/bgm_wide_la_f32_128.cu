// Look-ahead wide Cholesky, float storage, k = 128 (bgm_wide_la.cuh).
#include "bgm_wide_la.cuh"

namespace bgm {
namespace wide {

bool chol_la_f32_128(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s, int segment_rows) {
  return run_chol_la<float, 128, 4>(q, l, st, row, s, segment_rows);
}

}  // namespace wide
}  // namespace bgm
