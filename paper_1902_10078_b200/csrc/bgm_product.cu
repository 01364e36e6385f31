// Every dot product here is accumulated in the reference's order with a
// separate multiply and add (no FMA contraction), as kernels_detail.hpp:16-45
// computes it: fp64 products and band x vector results are bitwise the
// reference's.
//
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
    acc_t s = 0;
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
          s = __dadd_rn(s, __dmul_rn(acc_t(*pa), acc_t(*pb)));
          pa += da;
          pb += db;
        }
      }
    }
    c[ix(r) << C.s] = T(s);
  }
}


// Register-blocked products for the benchmarked band shapes: one thread per
// (matrix, block of J output columns).  op(A) has bands (AL, AU), op(B)
// (BL, BU), the output (CL, CU) (full or restricted); all compile-time, so
// the J x (CL+CU+1) accumulators stay in registers and every op(A) column is
// loaded once per block instead of once per output cell: for output columns
// j0 .. j0+J-1 the sweep runs k = j0-BU .. j0+J-1+BL, loads op(A)(:, k) and
// op(B)(k, j) and scatters the products into the cells they belong to.
template <class T, int TA, int TB, int AL, int AU, int BL, int BU, int CL, int CU, int J>
__global__ void __launch_bounds__(128) k_product_blk(Band<T> A, Band<T> Bm, Band<T> C, ix batch) {
  constexpr int AW = AL + AU + 1, CW = CL + CU + 1, NK = J + BL + BU;
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix n = C.n, nblk = (n + J - 1) / J;
  const ix lanes = ix(1) << C.s;
  const ix rest = t >> C.s;
  const ix b = (rest / nblk) * lanes + (t & (lanes - 1));
  const ix j0 = (rest % nblk) * J;
  if (b >= batch) return;
  const T* a = mbase(A, b);
  const T* bb = mbase(Bm, b);
  acc_t acc[J][CW];
#pragma unroll
  for (int jj = 0; jj < J; ++jj)
#pragma unroll
    for (int r = 0; r < CW; ++r) acc[jj][r] = 0;
#pragma unroll
  for (int kk = 0; kk < NK; ++kk) {
    const ix k = j0 - BU + kk;
    if (k < 0 || k >= n) continue;
    acc_t av[AW];
#pragma unroll
    for (int x = 0; x < AW; ++x) {  // op(A)(i, k), i = k - AU + x
      const ix i = k - AU + x;
      av[x] = (i >= 0 && i < n) ? (TA ? a[(i * A.w + (k - i + A.up)) << A.s] : a[(k * A.w + (i - k + A.up)) << A.s])
                                : T(0);
    }
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int d = kk - BU - jj;  // k - j, compile-time
      if (d < -BU || d > BL) continue;
      const ix j = j0 + jj;
      if (j >= n) continue;
      const acc_t bv = TB ? bb[(k * Bm.w + (j - k + Bm.up)) << Bm.s] : bb[(j * Bm.w + (k - j + Bm.up)) << Bm.s];
#pragma unroll
      for (int x = 0; x < AW; ++x) {
        const int r = d - AU + x + CU;  // output cell of row i = k - AU + x in column j
        if (r >= 0 && r < CW) acc[jj][r] = __dadd_rn(acc[jj][r], __dmul_rn(av[x], bv));
      }
    }
  }
  T* c = const_cast<T*>(mbase(C, b));
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    const ix j = j0 + jj;
    if (j >= n) break;
#pragma unroll
    for (int r = 0; r < CW; ++r) {
      const ix i = j - CU + r;
      c[(j * C.w + r) << C.s] = (i >= 0 && i < n) ? T(acc[jj][r]) : T(0);
    }
  }
}

template <class T, int TA, int TB, int AL, int AU, int BL, int BU, int CL, int CU>
bool try_blk(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  const int al = ta ? a.upper : a.lower, au = ta ? a.lower : a.upper;
  const int bl = tb ? b.upper : b.lower, bu = tb ? b.lower : b.upper;
  if (ta != TA || tb != TB || al != AL || au != AU || bl != BL || bu != BU || c.lower != CL || c.upper != CU)
    return false;
  constexpr int J = 4;
  const ix lanes = c.tile;
  const ix work = (c.batch + lanes - 1) / lanes * lanes * ((c.n + J - 1) / J);
  timing::Scope t("product_blk", s);
  k_product_blk<T, TA, TB, AL, AU, BL, BU, CL, CU, J><<<blocks_for(work, 128), 128, 0, s>>>(
      view<T>(a), view<T>(b), view<T>(c), c.batch);
  return true;
}

template <class T>
bool product_blk(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  if (c.n < 64) return false;
  // the full / lower products of configs 2 and 3 (the restricted VJP halves
  // keep the strided kernel: there most loaded op(A) cells miss the output band)
  return try_blk<T, 0, 1, 8, 0, 0, 8, 8, 8>(a, ta, b, tb, c, s) ||
         try_blk<T, 0, 0, 8, 8, 3, 3, 11, 11>(a, ta, b, tb, c, s) ||
         try_blk<T, 0, 1, 16, 0, 0, 16, 16, 0>(a, ta, b, tb, c, s);
}


// Band x vector for tile 32 (kernels_detail.hpp:31-45): thread = (matrix
// lane, output index i), y_i = sum_j op(B)(i, j) v_j with pointer walks:
// untransposed, B(i, j) for consecutive j lies (w - 1) cells apart (the
// storage diagonal); transposed, B(j, i) is column i of the storage.
// Every load is one 256-byte warp transaction; fp64 accumulation.
template <class T>
__global__ void k_band_vec32(Band<T> B, Vec<T> v, int tr, Vec<T> y, ix tiles) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const int lane = int(t & 31);
  const ix rest = t >> 5, n = B.n;
  if (rest >= tiles * n) return;
  const ix tile = rest / n, i = rest - tile * n;
  const int lo = tr ? B.up : B.lo, up = tr ? B.lo : B.up;  // bands of op(B)
  const ix j0 = i - lo > 0 ? i - lo : 0, j1 = i + up < n - 1 ? i + up : n - 1;
  const T* pb = B.p + tile * n * B.w * 32 + lane +
                (tr ? (i * B.w + (j0 - i + B.up)) : (j0 * B.w + (i - j0 + B.up))) * 32;
  const ix db = tr ? 32 : ix(B.w - 1) * 32;
  const T* pv = v.p + (tile * n + j0) * 32 + lane;
  acc_t s = 0;
#pragma unroll 4
  for (ix j = j0; j <= j1; ++j) {
    s = __dadd_rn(s, __dmul_rn(acc_t(*pb), acc_t(*pv)));
    pb += db;
    pv += 32;
  }
  y.p[(tile * n + i) * 32 + lane] = T(s);
}

// Fused vjp_product_band_vec column pass (grad.cpp:153-162), tile 32:
// thread = (matrix lane, column j of B).  B-bar's column j is p-bar_i v_j
// (untransposed) or v_i p-bar_j (transposed), i over the column's band
// rows; untransposed, v-bar_j = sum_i B(i, j) p-bar_i comes from the same
// column read.  B is read once, B-bar written once, corners zero.
template <class T, bool TR>
__global__ void k_vjp_band_vec32(Band<T> B, Vec<T> v, Vec<T> pb, Band<T> bb, Vec<T> vb, ix tiles) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const int lane = int(t & 31);
  const ix rest = t >> 5, n = B.n;
  if (rest >= tiles * n) return;
  const ix tile = rest / n, j = rest - tile * n;
  const ix col = ((tile * n + j) * B.w) * 32 + lane;
  const T* pc = B.p + col;
  T* oc = bb.p + col;
  const T* vt = v.p + tile * n * 32 + lane;
  const T* pt = pb.p + tile * n * 32 + lane;
  const acc_t cj = acc_t(TR ? pt[j * 32] : vt[j * 32]);
  acc_t s = 0;
  for (int r = 0; r < B.w; ++r) {
    const ix i = j - B.up + r;
    T o = T(0);
    if (i >= 0 && i < n) {
      const acc_t ri = acc_t(TR ? vt[i * 32] : pt[i * 32]);
      o = T(ri * cj);
      if (!TR) s = __dadd_rn(s, __dmul_rn(acc_t(pc[r * 32]), ri));
    }
    oc[r * 32] = o;
  }
  if (!TR) vb.p[(tile * n + j) * 32 + lane] = T(s);
}

template <class T>
void launch_band_vec32(const bgm_band& b, const bgm_vec& v, int tr, const bgm_vec& y, cudaStream_t s) {
  const ix tiles = (b.batch + 31) / 32;
  k_band_vec32<T><<<blocks_for(tiles * b.n * 32, 256), 256, 0, s>>>(view<T>(b), view<T>(v), tr, view<T>(y), tiles);
}

}  // namespace

bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  if (a.n == 0 || c.batch == 0) return false;
  if (a.dtype == BGM_F64 ? product_blk<double>(a, ta, b, tb, c, s) : product_blk<float>(a, ta, b, tb, c, s))
    return true;
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

bool band_vec(const bgm_band& b, const bgm_vec& v, int tr, const bgm_vec& y, cudaStream_t s) {
  if (b.tile != 32 || v.tile != 32 || y.tile != 32 || b.n == 0 || b.batch == 0) return false;
  timing::Scope t("band_vec32", s);
  if (b.dtype == BGM_F64)
    launch_band_vec32<double>(b, v, tr, y, s);
  else
    launch_band_vec32<float>(b, v, tr, y, s);
  return true;
}

bool vjp_band_vec(const bgm_band& b, const bgm_vec& v, const bgm_vec& pb, int tr, const bgm_band& bb,
                  const bgm_vec& vb, cudaStream_t s) {
  if (b.tile != 32 || v.tile != 32 || pb.tile != 32 || bb.tile != 32 || vb.tile != 32 || b.n == 0 || b.batch == 0)
    return false;
  timing::Scope t("vjp_band_vec32", s);
  const ix tiles = (b.batch + 31) / 32;
  const unsigned blocks = blocks_for(tiles * b.n * 32, 256);
  auto go = [&](auto z) {
    using T = decltype(z);
    if (tr) {  // v-bar = B p-bar (row sums), B-bar = outer(v, p-bar)
      launch_band_vec32<T>(b, pb, 0, vb, s);
      k_vjp_band_vec32<T, true><<<blocks, 256, 0, s>>>(view<T>(b), view<T>(v), view<T>(pb), view<T>(bb), view<T>(vb),
                                                       tiles);
    } else {
      k_vjp_band_vec32<T, false><<<blocks, 256, 0, s>>>(view<T>(b), view<T>(v), view<T>(pb), view<T>(bb),
                                                        view<T>(vb), tiles);
    }
  };
  if (b.dtype == BGM_F64)
    go(double(0));
  else
    go(float(0));
  return true;
}

}  // namespace prod
}  // namespace bgm
