// Wide-band (k = 64, 128) fast paths (bgm_wide.cu).  Each returns true when
// it recognised the shape and launched, false to fall back to the generic
// kernels.
#pragma once

#include <cuda_runtime.h>

#include "bandgm_b200.h"

namespace bgm {
namespace wide {

bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s);
bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s);
bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s);
bool log_det(const bgm_band& l, void* out, int32_t* st, int64_t* row, cudaStream_t s);
bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s);
bool vjp_subset(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb, int32_t* st,
                int64_t* row, cudaStream_t s);
void set_segment_rows(int rows);
// look-ahead DMMA Cholesky, k = 64 / 128, fp64 (bgm_wide_la.cu)
bool cholesky_la(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s,
                 int segment_rows);
// blocked solves, k = 64 / 128, reference layout, n % 8 == 0 (bgm_wide_solve.cu)
bool solve_vec_blk(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
                   cudaStream_t s, int segment_rows);

}  // namespace wide

// Narrow-band (k <= 16, tile 32) fast paths (bgm_narrow.cu).
namespace narrow {
bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s);
bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s);
bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s);
bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s);
void set_segment_rows(int rows);
}  // namespace narrow

// Other bandwidths / layouts staged onto the compiled ones (bgm_promote.cu).
namespace promote {
bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s);
bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s);
bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s);
bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s);
bool vjp_subset(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb, int32_t* st,
                int64_t* row, cudaStream_t s);
}  // namespace promote

// Band x band products with strided operand walks (bgm_product.cu).
namespace prod {
bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s);
bool band_vec(const bgm_band& b, const bgm_vec& v, int tr, const bgm_vec& y, cudaStream_t s);
bool vjp_band_vec(const bgm_band& b, const bgm_vec& v, const bgm_vec& pb, int tr, const bgm_band& bb,
                  const bgm_vec& vb, cudaStream_t s);
}

// Staged (TMA ring) products and fused product VJP, tile 32 (bgm_stream.cu).
namespace stream {
bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s);
bool vjp_product(const bgm_band& a, const bgm_band& b, const bgm_band& pb, const bgm_band& ab,
                 const bgm_band& bb, cudaStream_t s);
}  // namespace stream
}  // namespace bgm
