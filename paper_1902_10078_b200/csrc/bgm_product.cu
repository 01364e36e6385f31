// Band x band products (kernels_detail.hpp:16-28), streamlined: one thread
// per (matrix, output column j) as the generic kernel, but every operand
// walk is a pointer increment.  In the band storage both op(A)(i, k) and
// op(B)(k, j) move by a constant stride as k advances (A: (w_A - 1) cells
// per k untransposed, 1 cell transposed; B the other way round), so the
// inner product over k is two strided loads and an FMA per term with no
// index arithmetic; the column is written whole, corner cells as zeros.
// Serves product_band_band(_restricted) and both halves of
// vjp_product_band_band (grad.cpp:145-151).
#include <cuda_runtime.h>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_timing.cuh"

namespace bgm {
namespace prod {
namespace {

template <class T>
__device__ __forceinline__ const T* mbase(const Band<T>& B, ix b) {
  return B.p + ((((b >> B.s) * B.n) * B.w) << B.s) + (b & ((ix(1) << B.s) - 1));
}

template <class T>
__global__ void k_product_stride(Band<T> A, int ta, Band<T> Bm, int tb, Band<T> C, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (!split_bj(t, batch, C.n, C.s, b, j)) return;
  const ix n = C.n;
  const T* a = mbase(A, b);
  const T* bb = mbase(Bm, b);
  T* c = const_cast<T*>(mbase(C, b)) + ((j * C.w) << C.s);
  const int al = ta ? A.up : A.lo, au = ta ? A.lo : A.up;
  const int bl = tb ? Bm.up : Bm.lo, bu = tb ? Bm.lo : Bm.up;
  // strides (elements) of op(A)(i, k) and op(B)(k, j) per unit step of k
  const ix da = ix(ta ? 1 : A.w - 1) << A.s;
  const ix db = ix(tb ? Bm.w - 1 : 1) << Bm.s;
#pragma unroll 1
  for (int r = 0; r < C.w; ++r) {
    const ix i = j - C.up + r;
    T s = T(0);
    if (i >= 0 && i < n) {
      ix k0 = i - al;
      if (j - bu > k0) k0 = j - bu;
      if (k0 < 0) k0 = 0;
      ix k1 = i + au;
      if (j + bl < k1) k1 = j + bl;
      if (n - 1 < k1) k1 = n - 1;
      if (k0 <= k1) {
        // op(A)(i, k0) and op(B)(k0, j)
        const T* pa = a + ((ta ? (i * A.w + (k0 - i + A.up)) : (k0 * A.w + (i - k0 + A.up))) << A.s);
        const T* pb = bb + ((tb ? (k0 * Bm.w + (j - k0 + Bm.up)) : (j * Bm.w + (k0 - j + Bm.up))) << Bm.s);
        const int cnt = int(k1 - k0) + 1;
#pragma unroll 4
        for (int q = 0; q < cnt; ++q) {
          s = fma(*pa, *pb, s);
          pa += da;
          pb += db;
        }
      }
    }
    c[ix(r) << C.s] = s;
  }
}

}  // namespace

bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  if (a.n == 0 || c.batch == 0) return false;
  timing::Scope t("product", s);
  const ix lanes = c.tile;
  const ix work = (c.batch + lanes - 1) / lanes * lanes * c.n;
  if (a.dtype == BGM_F64)
    k_product_stride<double><<<blocks_for(work, 128), 128, 0, s>>>(view<double>(a), ta, view<double>(b), tb,
                                                                   view<double>(c), c.batch);
  else
    k_product_stride<float><<<blocks_for(work, 128), 128, 0, s>>>(view<float>(a), ta, view<float>(b), tb,
                                                                  view<float>(c), c.batch);
  return true;
}

}  // namespace prod
}  // namespace bgm
