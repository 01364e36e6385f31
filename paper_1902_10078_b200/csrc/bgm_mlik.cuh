#pragma once

#include <cuda_runtime.h>

#include "bandgm_b200.h"

namespace bgm {

// Segment-parallel config-3 kernels (bgm_mlik_fast.cu).  Returns a BGM_*
// status when it handled the call, or -1 to fall back to the generic sweep.
int mlik_fast(const bgm_band& l, const bgm_vec& y, double tau2, double* loss,
              const bgm_band& lbar, double* tau2_bar, int32_t* status, int64_t* row,
              int segment_rows, cudaStream_t s);

// One-thread-per-(matrix, segment) kernels for tile-32 inputs (bgm_mlik_t1.cu).
int mlik_t1(const bgm_band& l, const bgm_vec& y, double tau2, double* loss, const bgm_band& lbar,
            double* tau2_bar, int32_t* status, int64_t* row, int segment_rows, cudaStream_t s);
namespace t1 {
int repairs(int64_t* count, int reset);
}

int mlik_repairs(int64_t* count, double* max_dev, int reset);

}  // namespace bgm
