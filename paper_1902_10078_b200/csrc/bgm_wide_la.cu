// Dispatcher of the look-ahead wide Cholesky (bgm_wide_la.cuh; one translation unit per storage type
// and bandwidth so they compile in parallel).
#include <cuda_runtime.h>

#include "bgm_common.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace wide {

bool chol_la_f64_64(const bgm_band&, const bgm_band&, int32_t*, int64_t*, cudaStream_t, int);
bool chol_la_f64_128(const bgm_band&, const bgm_band&, int32_t*, int64_t*, cudaStream_t, int);
bool chol_la_f32_64(const bgm_band&, const bgm_band&, int32_t*, int64_t*, cudaStream_t, int);
bool chol_la_f32_128(const bgm_band&, const bgm_band&, int32_t*, int64_t*, cudaStream_t, int);

bool cholesky_la(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s, int segment_rows) {
  if (q.dtype != l.dtype) return false;
  if (q.n * ix(q.lower + 1) >= (ix(1) << 31) - 4096) return false;  // 32-bit row / cell indices inside
  const bool f64 = q.dtype == BGM_F64;
  if (q.lower == 64)
    return f64 ? chol_la_f64_64(q, l, st, row, s, segment_rows) : chol_la_f32_64(q, l, st, row, s, segment_rows);
  if (q.lower == 128)
    return f64 ? chol_la_f64_128(q, l, st, row, s, segment_rows) : chol_la_f32_128(q, l, st, row, s, segment_rows);
  return false;
}

}  // namespace wide
}  // namespace bgm
