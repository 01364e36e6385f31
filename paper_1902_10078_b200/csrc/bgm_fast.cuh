// Specialised (fast-path) launchers.  Each returns true when it recognised
// the shape/layout and launched its kernels, false to let the caller run the
// generic reference-loop kernel.  Implementations: bgm_fast.cu.
#pragma once

#include <cuda_runtime.h>

#include "bandgm_b200.h"

namespace bgm {
namespace fast {

bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s);
bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st,
               int64_t* row, cudaStream_t s);
bool log_det(const bgm_band& l, void* out, int32_t* st, int64_t* row, cudaStream_t s);
bool subset(const bgm_band& l, const bgm_band& sm, int32_t* st, int64_t* row, cudaStream_t s);
bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c,
             cudaStream_t s);
bool band_vec(const bgm_band& b, const bgm_vec& v, int tr, const bgm_vec& y, cudaStream_t s);
bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s);
bool vjp_subset(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb,
                int32_t* st, int64_t* row, cudaStream_t s);
bool vjp_product(const bgm_band& a, const bgm_band& b, const bgm_band& pb, const bgm_band& ab,
                 const bgm_band& bb, cudaStream_t s);
bool vjp_band_vec(const bgm_band& b, const bgm_vec& v, const bgm_vec& pb, int tr,
                  const bgm_band& bb, const bgm_vec& vb, cudaStream_t s);

// Process-wide switch (BGM_GENERIC_ONLY=1 in the environment) that routes
// every call to the generic kernels; used by the parity tests to cover both.
bool disabled();

}  // namespace fast
}  // namespace bgm
