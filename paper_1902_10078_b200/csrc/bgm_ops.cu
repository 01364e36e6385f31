// bandgm_b200: C ABI entry points and the reference-loop ("generic") kernels.
//
// Every operator of the reference's hot path
// has a generic kernel here that restates the reference loop nest on the
// batch-interleaved device layout, one thread per matrix for the length-n
// recurrences and one thread per output column/row for the data-parallel
// products.  These kernels handle every shape, both dtypes and both tiles.
// Shapes on the benchmarked paths are routed to the specialised kernels in
// bgm_fast.cu / bgm_mlik.cu (see dispatch below); the generic kernels remain
// the path for everything else.  There is no CPU fallback anywhere.
#include <cuda_runtime.h>

#include <type_traits>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"

namespace bgm {

namespace {
thread_local char g_last_error[256] = "";
}

int set_error(cudaError_t e) {
  std::snprintf(g_last_error, sizeof g_last_error, "%s", cudaGetErrorString(e));
  return BGM_ERR_CUDA;
}

static int launched() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BGM_OK : set_error(e);
}

constexpr int kThreads = 128;

// ---------------------------------------------------------------- helpers

template <class T>
__global__ void k_zero_band(Band<T> o, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (o.n == 0 || !split_bj(t, batch, o.n, o.s, b, j)) return;
  for (int r = 0; r < o.w; ++r) o.cell(b, r, j) = T(0);
}

template <class T>
__global__ void k_relayout_band(Band<T> src, Band<T> dst, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (src.n == 0 || !split_bj(t, batch, src.n, dst.s, b, j)) return;
  for (int r = 0; r < src.w; ++r) dst.cell(b, r, j) = src.cell(b, r, j);
}

template <class T>
__global__ void k_relayout_vec(Vec<T> src, Vec<T> dst, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, i;
  if (src.n == 0 || !split_bj(t, batch, src.n, dst.s, b, i)) return;
  dst(b, i) = src(b, i);
}

// banded.cpp:159-167
template <class T>
__global__ void k_transpose(Band<T> src, Band<T> dst, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (dst.n == 0 || !split_bj(t, batch, dst.n, dst.s, b, j)) return;
  dst.write_column(b, j, [&](ix i) { return src.at(b, j, i); });
}

// Copies band(src) onto dst's band, at_or_zero outside src (grad.cpp:62-66).
template <class T>
__global__ void k_restrict_copy(Band<T> src, Band<T> dst, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (dst.n == 0 || !split_bj(t, batch, dst.n, dst.s, b, j)) return;
  dst.write_column(b, j, [&](ix i) { return src.at_or_zero(b, i, j); });
}

template <class T>
static void zero_band(const Band<T>& o, ix batch, cudaStream_t st) {
  const ix work = ((batch + (ix(1) << o.s) - 1) >> o.s << o.s) * o.n;
  if (work) k_zero_band<T><<<blocks_for(work, 256), 256, 0, st>>>(o, batch);
}

static ix bj_work(ix batch, ix n, int s) { return ((batch + (ix(1) << s) - 1) >> s << s) * n; }

// ---------------------------------------------------------------- forward

// kernels_serial.cpp:12-32 (PAPER Alg. 1), one thread per matrix.
template <class T>
__global__ void k_cholesky(Band<T> q, Band<T> l, ix batch, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix n = l.n, bw = l.lo;
  for (ix i = 0; i < n; ++i) {
    const ix j0 = i - bw > 0 ? i - bw : 0;
    for (ix j = j0; j <= i; ++j) {
      T s = 0;
      for (ix m = j0; m < j; ++m) s += l.at(b, i, m) * l.at(b, j, m);
      if (i == j) {
        const T piv = q.at(b, i, i) - s;
        if (!(double(piv) > kPivotFloor)) {
          report(status, row, b, BGM_ERR_NOT_PD, i);
          return;
        }
        l.at(b, i, i) = sqrt(piv);
      } else {
        l.at(b, i, j) = (q.at(b, i, j) - s) / l.at(b, j, j);
      }
    }
  }
  for (ix j = n - bw > 0 ? n - bw : 0; j < n; ++j)
    for (int r = int(n - j); r <= bw; ++r) l.cell(b, r, j) = T(0);
  report(status, row, b, BGM_OK, -1);
}

// kernels_serial.cpp:34-60
template <class T>
__global__ void k_solve_vec(Band<T> l, Vec<T> v, int tr, Vec<T> x, ix batch, int32_t* status,
                            int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix n = l.n, bw = l.lo;
  if (!tr) {
    for (ix i = 0; i < n; ++i) {
      T s = 0;
      for (ix k = i - bw > 0 ? i - bw : 0; k < i; ++k) s += l.at(b, i, k) * x(b, k);
      const T piv = l.at(b, i, i);
      if (fabs(double(piv)) < kPivotFloor) {
        report(status, row, b, BGM_ERR_SINGULAR, i);
        return;
      }
      x(b, i) = (v(b, i) - s) / piv;
    }
  } else {
    for (ix i = n - 1; i >= 0; --i) {
      T s = 0;
      const ix k1 = i + bw < n - 1 ? i + bw : n - 1;
      for (ix k = i + 1; k <= k1; ++k) s += l.at(b, k, i) * x(b, k);
      const T piv = l.at(b, i, i);
      if (fabs(double(piv)) < kPivotFloor) {
        report(status, row, b, BGM_ERR_SINGULAR, i);
        return;
      }
      x(b, i) = (v(b, i) - s) / piv;
    }
  }
  report(status, row, b, BGM_OK, -1);
}

// kernels.cpp:121-129; accumulated in double for both dtypes.
template <class T>
__global__ void k_log_det(Band<T> l, T* out, ix batch, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  double s = 0.0;
  for (ix i = 0; i < l.n; ++i) {
    const double d = double(l.at(b, i, i));
    if (!(d > 0.0)) {
      report(status, row, b, BGM_ERR_NONPOS_DIAG, i);
      return;
    }
    s += log(d);
  }
  out[b] = T(s);
  report(status, row, b, BGM_OK, -1);
}

// kernels_serial.cpp:80-104 (PAPER Alg. 3, Takahashi)
template <class T>
__global__ void k_subset(Band<T> l, Band<T> s, ix batch, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix n = l.n, bw = l.lo;
  for (ix i = 0; i < n; ++i)
    if (fabs(double(l.at(b, i, i))) < kPivotFloor) {
      report(status, row, b, BGM_ERR_SINGULAR, i);
      return;
    }
  for (ix j = n - 1; j >= 0; --j) {
    const ix i_stop = j - bw > 0 ? j - bw : 0;
    for (ix i = j; i >= i_stop; --i) {
      const T piv = l.at(b, i, i);
      T acc = 0;
      const ix m1 = i + bw < n - 1 ? i + bw : n - 1;
      for (ix m = i + 1; m <= m1; ++m) acc += (l.at(b, m, i) / piv) * s.sym(b, m, j);
      T val = -acc;
      if (i == j) val += T(1) / (piv * piv);
      s.at(b, j, i) = val;
    }
  }
  for (ix j = n - bw > 0 ? n - bw : 0; j < n; ++j)
    for (int r = int(n - j); r <= bw; ++r) s.cell(b, r, j) = T(0);
  report(status, row, b, BGM_OK, -1);
}

// kernels_detail.hpp:16-28, one thread per output column; op(x) = x^T reads
// the stored transpose in place.
template <class T>
__global__ void k_product(Band<T> a, int ta, Band<T> bm, int tb, Band<T> c, T alpha, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (c.n == 0 || !split_bj(t, batch, c.n, c.s, b, j)) return;
  const ix n = c.n;
  const int alo = ta ? a.up : a.lo, aup = ta ? a.lo : a.up;
  const int blo = tb ? bm.up : bm.lo, bup = tb ? bm.lo : bm.up;
  c.write_column(b, j, [&](ix i) -> T {
    ix k0 = i - alo;
    if (j - bup > k0) k0 = j - bup;
    if (k0 < 0) k0 = 0;
    ix k1 = i + aup;
    if (j + blo < k1) k1 = j + blo;
    if (n - 1 < k1) k1 = n - 1;
    acc_t s = 0;
    for (ix k = k0; k <= k1; ++k) {
      const acc_t av = ta ? a.at(b, k, i) : a.at(b, i, k);
      const acc_t bv = tb ? bm.at(b, j, k) : bm.at(b, k, j);
      s = __dadd_rn(s, __dmul_rn(av, bv));  // kernels_detail.hpp:24, uncontracted
    }
    return T(acc_t(alpha) * s);
  });
}

// kernels_detail.hpp:31-45, one thread per output entry.
template <class T>
__global__ void k_band_vec(Band<T> bm, Vec<T> v, int tr, Vec<T> y, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, i;
  if (bm.n == 0 || !split_bj(t, batch, bm.n, y.s, b, i)) return;
  const ix n = bm.n;
  acc_t s = 0;
  if (!tr) {
    const ix j0 = i - bm.lo > 0 ? i - bm.lo : 0, j1 = i + bm.up < n - 1 ? i + bm.up : n - 1;
    for (ix j = j0; j <= j1; ++j) s = __dadd_rn(s, __dmul_rn(acc_t(bm.at(b, i, j)), acc_t(v(b, j))));
  } else {
    const ix j0 = i - bm.up > 0 ? i - bm.up : 0, j1 = i + bm.lo < n - 1 ? i + bm.lo : n - 1;
    for (ix j = j0; j <= j1; ++j) s = __dadd_rn(s, __dmul_rn(acc_t(bm.at(b, j, i)), acc_t(v(b, j))));
  }
  y(b, i) = T(s);
}

// kernels_detail.hpp:48-54
template <class T>
__global__ void k_outer(Vec<T> m, Vec<T> v, T alpha, Band<T> o, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (o.n == 0 || !split_bj(t, batch, o.n, o.s, b, j)) return;
  const T vj = v(b, j);
  o.write_column(b, j, [&](ix i) { return alpha * (m(b, i) * vj); });
}

// Outer-product band writers (kernels_detail.hpp:48-54: out(i, j) = m_i v_j),
// alpha in {1, -1} exact.  Tile 32: thread = (matrix lane, column j) walks
// the column's w cells (every load / store a 256-byte warp transaction).
template <class T>
__global__ void k_outer_t32(Vec<T> m, Vec<T> v, T alpha, Band<T> o, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const int lane = int(t & 31);
  const ix rest = t >> 5, n = o.n;
  const ix tiles = (batch + 31) / 32;
  if (rest >= tiles * n) return;
  const ix tile = rest / n, j = rest - tile * n;
  const T vj = v.p[(tile * n + j) * 32 + lane];
  const T* mp = m.p + (tile * n + j - o.up) * 32 + lane;
  T* op = o.p + (tile * n + j) * ix(o.w) * 32 + lane;
  const bool live = tile * 32 + lane < batch;
  for (int r = 0; r < o.w; ++r) {
    const ix i = j - o.up + r;
    op[r * 32] = (live && i >= 0 && i < n) ? alpha * (mp[r * 32] * vj) : T(0);
  }
}

// Tile 1: warp = (matrix, 32 consecutive columns), whose storage is one
// contiguous run of 32 w cells; lane l writes cells l, l+32, ... of the run
// (coalesced), stepping (column, row) incrementally; v of the 32 columns is
// loaded once and shuffled.
template <class T>
__global__ void k_outer_t1(Vec<T> m, Vec<T> v, T alpha, Band<T> o, ix batch) {
  const ix gw = (blockIdx.x * ix(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const ix n = o.n, nblk = (n + 31) / 32;
  if (gw >= batch * nblk) return;  // whole warps
  const ix b = gw / nblk, j0 = (gw - b * nblk) * 32;
  const int w = o.w;
  const int cols = int(n - j0 < 32 ? n - j0 : 32);
  const T vl = lane < cols ? v.p[b * n + j0 + lane] : T(0);
  T* run = o.p + (b * n + j0) * ix(w);
  const T* mb = m.p + b * n;
  const int total = cols * w;
  const int dj = 32 / w, dr = 32 % w;  // (column, row) step of 32 cells
  int jj = lane / w, r = lane % w;
  const int iters = (total + 31) / 32;  // warp-uniform (the shuffle needs every lane)
  for (int it = 0, e = lane; it < iters; ++it, e += 32) {
    const T vj = __shfl_sync(0xffffffffu, vl, jj & 31);
    if (e < total) {
      const ix i = j0 + jj - o.up + r;
      run[e] = (i >= 0 && i < n) ? alpha * (mb[i] * vj) : T(0);
    }
    jj += dj;
    r += dr;
    if (r >= w) {
      r -= w;
      ++jj;
    }
  }
}

// Whole-band writers in storage order: thread x of tile group g writes the
// x-th element of the group's (n, w, tile) block, so every store is
// coalesced in both layouts (tile 1 columns are contiguous w-cell runs);
// f(b, i, j, r) gives the in-band value, corners and batch padding get 0.
template <class T, class F>
__global__ void k_band_flat(Band<T> o, ix batch, F f) {
  const ix g = blockIdx.y;
  const unsigned tile = 1u << o.s;
  const unsigned per = unsigned(o.n * o.w) << o.s;
  T* base = o.p + g * ix(per);
  // two consecutive elements per thread, one 2-wide store (per is even for
  // tile 32 and for tile 1 when n * w is even)
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  if (per & 1) {  // odd block (tile 1, n * w odd): blocks of odd groups are not 2-element aligned
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < per; x += gridDim.x * blockDim.x) {
      const unsigned cr = x >> o.s;
      const unsigned j = cr / unsigned(o.w), r = cr - j * unsigned(o.w);
      const ix b = g * tile + (x & (tile - 1));
      const ix i = ix(j) - o.up + r;
      base[x] = (b < batch && i >= 0 && i < o.n) ? f(b, i, ix(j), int(r)) : T(0);
    }
    return;
  }
  // U pairs per thread and iteration: every value (the functor's loads) is
  // computed before any of the U stores, so U x 2 loads are in flight at once
  constexpr int U = 4;
  const unsigned pairs = per >> 1;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned x0 = blockIdx.x * blockDim.x + threadIdx.x; x0 < pairs; x0 += U * stride) {
    T val[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned x2 = x0 + u * stride;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const unsigned xe = (x2 << 1) + h;
        const unsigned cr = xe >> o.s;
        const unsigned j = cr / unsigned(o.w), r = cr - j * unsigned(o.w);
        const ix b = g * tile + (xe & (tile - 1));
        const ix i = ix(j) - o.up + r;
        val[u][h] = (x2 < pairs && b < batch && i >= 0 && i < o.n) ? f(b, i, ix(j), int(r)) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned x2 = x0 + u * stride;
      if (x2 >= pairs) break;
      V2 v;
      v.x = val[u][0];
      v.y = val[u][1];
      *reinterpret_cast<V2*>(base + (x2 << 1)) = v;
    }
  }
}

template <class T>
struct OuterF {  // alpha m_i v_j
  Vec<T> m, v;
  T a;
  __device__ __forceinline__ T operator()(ix b, ix i, ix j, int) const { return a * (m(b, i) * v(b, j)); }
};

template <class T>
__global__ void k_logdet_diag(Band<T> l, const T* c, Band<T> lb, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (l.n == 0 || !split_bj(t, batch, l.n, lb.s, b, j)) return;
  lb.cell(b, 0, j) = c[b] / l.cell(b, 0, j);
}


template <class T>
static bool flat_ok(const Band<T>& o, ix batch) {
  const ix groups = (batch + (ix(1) << o.s) - 1) >> o.s;
  return groups > 0 && groups <= 65535 && (o.n * o.w << o.s) < (ix(1) << 32);
}

template <class T, class F>
static void launch_flat(const Band<T>& o, ix batch, F f, cudaStream_t s) {
  const ix groups = (batch + (ix(1) << o.s) - 1) >> o.s;
  const ix per = o.n * o.w << o.s;
  ix gx = (per + 255) / 256;
  const ix cap = (ix(148) * 16 + groups - 1) / groups;  // ~16 blocks per SM in total
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  k_band_flat<T><<<dim3(unsigned(gx), unsigned(groups)), 256, 0, s>>>(o, batch, f);
}

// Pivot pre-check shared by solve_mat (kernels.cpp:43-45).
template <class T>
__global__ void k_pivot_check(Band<T> l, ix batch, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  for (ix i = 0; i < l.n; ++i)
    if (fabs(double(l.at(b, i, i))) < kPivotFloor) {
      report(status, row, b, BGM_ERR_SINGULAR, i);
      return;
    }
  report(status, row, b, BGM_OK, -1);
}

// kernels_detail.hpp:58-72 on diagonal d = i - j; entries of one diagonal
// are independent (kernels.cpp:48-63), diagonals run in launch order.
template <class T>
__global__ void k_solve_mat_diag(Band<T> l, Band<T> r, Band<T> o, int tr, ix d, ix lo_i, ix cnt,
                                 ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, e;
  if (cnt <= 0 || !split_bj(t, batch, cnt, o.s, b, e)) return;
  const ix n = l.n;
  const ix i = lo_i + e, j = i - d;
  const T piv = l.at(b, i, i);
  if (fabs(double(piv)) < kPivotFloor) return;  // reported by k_pivot_check
  T s = 0;
  if (!tr) {
    for (ix m = i - l.lo > 0 ? i - l.lo : 0; m < i; ++m) s += l.at(b, i, m) * o.at_or_zero(b, m, j);
  } else {
    const ix m1 = i + l.lo < n - 1 ? i + l.lo : n - 1;
    for (ix m = i + 1; m <= m1; ++m) s += l.at(b, m, i) * o.at_or_zero(b, m, j);
  }
  o.at(b, i, j) = (r.at_or_zero(b, i, j) - s) / piv;
}

// ---------------------------------------------------------------- reverse

// grad.cpp:11-36 (PAPER Alg. 2); lb consumed in place.
template <class T>
__global__ void k_vjp_cholesky(Band<T> l, Band<T> lb, Band<T> qb, ix batch) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix n = l.n, bw = l.lo;
  for (ix i = n - 1; i >= 0; --i) {
    const ix j_stop = i - bw > 0 ? i - bw : 0;
    for (ix j = i; j >= j_stop; --j) {
      T q;
      if (j == i) {
        q = T(0.5) * lb.at(b, i, i) / l.at(b, i, i);
      } else {
        q = lb.at(b, i, j) / l.at(b, j, j);
        lb.at(b, j, j) -= lb.at(b, i, j) * l.at(b, i, j) / l.at(b, j, j);
      }
      qb.at(b, i, j) = q;
      for (ix k = j - 1; k >= j_stop; --k) {
        lb.at(b, i, k) -= q * l.at(b, j, k);
        lb.at(b, j, k) -= q * l.at(b, i, k);
      }
    }
  }
  for (ix j = n - bw > 0 ? n - bw : 0; j < n; ++j)
    for (int r = int(n - j); r <= bw; ++r) qb.cell(b, r, j) = T(0);
}

// grad.cpp:84-143 (PAPER Alg. 5).  ws: (3bw+4) x n scratch per matrix,
// interleaved by 32 matrices.
template <class T>
__global__ void k_vjp_subset(Band<T> l, Band<T> s, Band<T> sb, Band<T> lb, Band<T> ws, ix batch,
                             int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix n = l.n;
  const int bw = l.lo;
  const int r_bu = 2 * bw + 1, r_inv = 3 * bw + 2, r_bvec = r_inv + 1;
  for (ix c = 0; c < n; ++c) {
    for (int r = 0; r < bw; ++r) ws.cell(b, r, c) = T(0);
    for (int r = 0; r <= bw; ++r) ws.cell(b, bw + r, c) = sb.cell(b, r, c);
    for (int r = 0; r <= bw; ++r) ws.cell(b, r_bu + r, c) = T(0);
    const T piv = l.at(b, c, c);
    if (fabs(double(piv)) < kPivotFloor) {
      report(status, row, b, BGM_ERR_SINGULAR, c);
      return;
    }
    ws.cell(b, r_inv, c) = T(1) / piv;
  }
  auto bs = [&](ix i, ix j) -> T& { return ws.cell(b, int(i - j + bw), j); };
  auto bu = [&](ix i, ix m) -> T& { return ws.cell(b, int(r_bu + i - m + bw), m); };
  for (ix j = 0; j < n; ++j) {
    for (ix i = j - bw > 0 ? j - bw : 0; i <= j; ++i) {
      if (i == j) ws.cell(b, r_bvec, i) = bs(i, i);
      const T tmp = bs(j, i);
      bs(j, i) = T(0);
      bs(i, j) += tmp;
      const T cur = bs(i, j);
      const T scale = cur * ws.cell(b, r_inv, i);
      const ix m1 = i + bw < n - 1 ? i + bw : n - 1;
      for (ix m = i + 1; m <= m1; ++m) {
        bu(i, m) -= s.sym(b, m, j) * cur;
        bs(m, j) -= l.at(b, m, i) * scale;
      }
      bs(i, j) = T(0);
    }
  }
  for (ix c = 0; c < n; ++c) {
    const T iv = ws.cell(b, r_inv, c);
    const ix r1 = c + bw < n - 1 ? c + bw : n - 1;
    T diag_sum = 0;
    for (ix r = c + 1; r <= r1; ++r) {
      lb.at(b, r, c) = bu(c, r) * iv;
      diag_sum += bu(c, r) * l.at(b, r, c);
    }
    for (ix r = r1 + 1; r <= c + bw; ++r) lb.cell(b, int(r - c), c) = T(0);
    lb.at(b, c, c) = (T(-2) * ws.cell(b, r_bvec, c) * iv - diag_sum) * (iv * iv);
  }
  report(status, row, b, BGM_OK, -1);
}

// grad.cpp:172-176

// ------------------------------------------------------ typed launchers

template <class T>
static int run_cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row,
                        cudaStream_t s) {
  if (fast::cholesky(q, l, st, row, s)) return launched();
  k_cholesky<T><<<blocks_for(q.batch, 64), 64, 0, s>>>(view<T>(q), view<T>(l), q.batch, st, row);
  return launched();
}

template <class T>
static int run_solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st,
                         int64_t* row, cudaStream_t s) {
  if (fast::solve_vec(l, v, tr, x, st, row, s)) return launched();
  k_solve_vec<T><<<blocks_for(l.batch, 64), 64, 0, s>>>(view<T>(l), view<T>(v), tr, view<T>(x),
                                                         l.batch, st, row);
  return launched();
}

template <class T>
static int run_product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c,
                       double alpha, cudaStream_t s) {
  if (alpha == 1.0 && fast::product(a, ta, b, tb, c, s)) return launched();
  const ix work = bj_work(c.batch, c.n, tile_shift(c.tile));
  if (work)
    k_product<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<T>(a), ta, view<T>(b), tb,
                                                                 view<T>(c), T(alpha), c.batch);
  return launched();
}

template <class T>
static int run_band_vec(const bgm_band& b, const bgm_vec& v, int tr, const bgm_vec& y,
                        cudaStream_t s) {
  if (fast::band_vec(b, v, tr, y, s)) return launched();
  const ix work = bj_work(y.batch, y.n, tile_shift(y.tile));
  if (work)
    k_band_vec<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<T>(b), view<T>(v), tr,
                                                                  view<T>(y), y.batch);
  return launched();
}

template <class T>
static int run_outer(const bgm_vec& m, const bgm_vec& v, double alpha, const bgm_band& o,
                     cudaStream_t s) {
  const ix work = bj_work(o.batch, o.n, tile_shift(o.tile));
  if (!work) return launched();
  const Band<T> ob = view<T>(o);
  if (o.tile == 32) {  // thread per (matrix lane, column): a pointer walk down the column
    k_outer_t32<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<T>(m), view<T>(v), T(alpha), ob, o.batch);
    return launched();
  }
  if (o.n >= 32 && ob.w <= 4096) {  // warp per (matrix, 32 columns): contiguous stores, no per-cell division
    const ix blocks = ix(o.batch) * ((o.n + 31) / 32);
    k_outer_t1<T><<<blocks_for(blocks * 32, 256), 256, 0, s>>>(view<T>(m), view<T>(v), T(alpha), ob, o.batch);
    return launched();
  }
  if (flat_ok(ob, o.batch)) {
    const Vec<T> mv = view<T>(m), vv = view<T>(v);
    const T a = T(alpha);
    launch_flat(ob, o.batch, OuterF<T>{mv, vv, a}, s);
  } else {
    k_outer<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<T>(m), view<T>(v), T(alpha), ob, o.batch);
  }
  return launched();
}

template <class T>
static int run_solve_mat(const bgm_band& l, const bgm_band& r, int tr, const bgm_band& o,
                         int32_t* st, int64_t* row, cudaStream_t s) {
  const ix n = l.n;
  zero_band(view<T>(o), o.batch, s);
  k_pivot_check<T><<<blocks_for(l.batch, 64), 64, 0, s>>>(view<T>(l), l.batch, st, row);
  const int sh = tile_shift(o.tile);
  auto diag = [&](ix d) {
    const ix lo_i = d > 0 ? d : 0, hi_i = n - 1 + d < n - 1 ? n - 1 + d : n - 1;
    const ix cnt = hi_i - lo_i + 1;
    const ix work = bj_work(o.batch, cnt, sh);
    if (cnt > 0 && work)
      k_solve_mat_diag<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(
          view<T>(l), view<T>(r), view<T>(o), tr, d, lo_i, cnt, o.batch);
  };
  if (!tr)
    for (ix d = -ix(o.upper); d <= o.lower; ++d) diag(d);
  else
    for (ix d = o.lower; d >= -ix(o.upper); --d) diag(d);
  return launched();
}

// ------------------------------------------------------ validation helpers

static bool same_batch(const bgm_band& a, const bgm_band& b) {
  return a.batch == b.batch && a.n == b.n && a.dtype == b.dtype;
}
static bool same_batch(const bgm_band& a, const bgm_vec& v) {
  return a.batch == v.batch && a.n == v.n && a.dtype == v.dtype;
}
static bool clipped(const bgm_band& c) {
  return c.n == 0 || (c.lower <= c.n - 1 && c.upper <= c.n - 1);
}

template <class F>
static int dispatch(int dtype, F&& f) {
  if (dtype == BGM_F64) return f(double{});
  if (dtype == BGM_F32) return f(float{});
  return BGM_ERR_ARG;
}

}  // namespace bgm

using namespace bgm;

extern "C" {

int bgm_abi_version(void) { return 1; }

const char* bgm_status_name(int st) {
  switch (st) {
    case BGM_OK: return "ok";
    case BGM_ERR_NOT_PD: return "NotPositiveDefinite";
    case BGM_ERR_SINGULAR: return "SingularDiagonal";
    case BGM_ERR_NONPOS_DIAG: return "NonPositiveDiagonal";
    case BGM_ERR_DIM: return "DimensionMismatch";
    case BGM_ERR_ARG: return "InvalidArgument";
    case BGM_ERR_CUDA: return "CudaError";
  }
  return "unknown";
}

const char* bgm_last_error(void) { return g_last_error; }

int bgm_relayout_band(bgm_band src, bgm_band dst, bgm_stream stream) {
  if (!valid(src) || !valid(dst)) return BGM_ERR_ARG;
  if (!same_batch(src, dst) || src.lower != dst.lower || src.upper != dst.upper) return BGM_ERR_DIM;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(src.dtype, [&](auto z) {
    using T = decltype(z);
    const ix work = bj_work(src.batch, src.n, tile_shift(dst.tile));
    if (work)
      k_relayout_band<T><<<blocks_for(work, 256), 256, 0, s>>>(view<T>(src), view<T>(dst), src.batch);
    return launched();
  });
}

int bgm_relayout_vec(bgm_vec src, bgm_vec dst, bgm_stream stream) {
  if (!valid(src) || !valid(dst)) return BGM_ERR_ARG;
  if (src.batch != dst.batch || src.n != dst.n || src.dtype != dst.dtype) return BGM_ERR_DIM;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(src.dtype, [&](auto z) {
    using T = decltype(z);
    const ix work = bj_work(src.batch, src.n, tile_shift(dst.tile));
    if (work)
      k_relayout_vec<T><<<blocks_for(work, 256), 256, 0, s>>>(view<T>(src), view<T>(dst), src.batch);
    return launched();
  });
}

int bgm_transpose_band(bgm_band src, bgm_band dst, bgm_stream stream) {
  if (!valid(src) || !valid(dst)) return BGM_ERR_ARG;
  if (!same_batch(src, dst) || src.lower != dst.upper || src.upper != dst.lower) return BGM_ERR_DIM;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(src.dtype, [&](auto z) {
    using T = decltype(z);
    const ix work = bj_work(src.batch, src.n, tile_shift(dst.tile));
    if (work)
      k_transpose<T><<<blocks_for(work, 256), 256, 0, s>>>(view<T>(src), view<T>(dst), src.batch);
    return launched();
  });
}

int bgm_cholesky(bgm_band q, bgm_band l, int32_t* status, int64_t* row, bgm_stream stream) {
  if (!valid(q) || !valid(l)) return BGM_ERR_ARG;
  if (!same_batch(q, l) || q.upper != 0 || l.upper != 0 || l.lower != q.lower) return BGM_ERR_DIM;
  if (q.batch == 0 || q.n == 0) return BGM_OK;
  return dispatch(q.dtype, [&](auto z) {
    return run_cholesky<decltype(z)>(q, l, status, row, static_cast<cudaStream_t>(stream));
  });
}

int bgm_solve_vec(bgm_band l, bgm_vec v, int transpose, bgm_vec x, int32_t* status, int64_t* row,
                  bgm_stream stream) {
  if (!valid(l) || !valid(v) || !valid(x)) return BGM_ERR_ARG;
  if (l.upper != 0 || !same_batch(l, v) || !same_batch(l, x)) return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  return dispatch(l.dtype, [&](auto z) {
    return run_solve_vec<decltype(z)>(l, v, transpose, x, status, row,
                                      static_cast<cudaStream_t>(stream));
  });
}

int bgm_log_det(bgm_band l, void* out, int32_t* status, int64_t* row, bgm_stream stream) {
  if (!valid(l) || (l.batch > 0 && !out)) return BGM_ERR_ARG;
  if (l.batch == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    if (fast::log_det(l, out, status, row, s)) return launched();
    k_log_det<T><<<blocks_for(l.batch, 64), 64, 0, s>>>(view<T>(l), static_cast<T*>(out), l.batch,
                                                        status, row);
    return launched();
  });
}

int bgm_sparse_inverse_subset(bgm_band l, bgm_band sb, int32_t* status, int64_t* row,
                              bgm_stream stream) {
  if (!valid(l) || !valid(sb)) return BGM_ERR_ARG;
  if (!same_batch(l, sb) || l.upper != 0 || sb.upper != 0 || sb.lower != l.lower)
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    if (fast::subset(l, sb, status, row, s)) return launched();
    k_subset<T><<<blocks_for(l.batch, 64), 64, 0, s>>>(view<T>(l), view<T>(sb), l.batch, status, row);
    return launched();
  });
}

int bgm_product_band_band(bgm_band a, int trans_a, bgm_band b, int trans_b, bgm_band c,
                          bgm_stream stream) {
  if (!valid(a) || !valid(b) || !valid(c)) return BGM_ERR_ARG;
  if (!same_batch(a, b) || !same_batch(a, c) || !clipped(c)) return BGM_ERR_DIM;
  if (a.batch == 0 || a.n == 0) return BGM_OK;
  return dispatch(a.dtype, [&](auto z) {
    return run_product<decltype(z)>(a, trans_a, b, trans_b, c, 1.0,
                                    static_cast<cudaStream_t>(stream));
  });
}

int bgm_product_band_vec(bgm_band b, bgm_vec v, int transpose, bgm_vec y, bgm_stream stream) {
  if (!valid(b) || !valid(v) || !valid(y)) return BGM_ERR_ARG;
  if (!same_batch(b, v) || !same_batch(b, y)) return BGM_ERR_DIM;
  if (b.batch == 0 || b.n == 0) return BGM_OK;
  return dispatch(b.dtype, [&](auto z) {
    return run_band_vec<decltype(z)>(b, v, transpose, y, static_cast<cudaStream_t>(stream));
  });
}

int bgm_outer_band(bgm_vec m, bgm_vec v, double scale, bgm_band out, bgm_stream stream) {
  if (!valid(m) || !valid(v) || !valid(out)) return BGM_ERR_ARG;
  if (!same_batch(out, m) || !same_batch(out, v) || !clipped(out)) return BGM_ERR_DIM;
  if (out.batch == 0 || out.n == 0) return BGM_OK;
  return dispatch(out.dtype, [&](auto z) {
    return run_outer<decltype(z)>(m, v, scale, out, static_cast<cudaStream_t>(stream));
  });
}

int bgm_solve_mat(bgm_band l, bgm_band r, int transpose, bgm_band out, int32_t* status,
                  int64_t* row, bgm_stream stream) {
  if (!valid(l) || !valid(r) || !valid(out)) return BGM_ERR_ARG;
  if (l.upper != 0 || !same_batch(l, r) || !same_batch(l, out) || !clipped(out)) return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  return dispatch(l.dtype, [&](auto z) {
    return run_solve_mat<decltype(z)>(l, r, transpose, out, status, row,
                                      static_cast<cudaStream_t>(stream));
  });
}

int bgm_vjp_cholesky(bgm_band l, bgm_band lb, bgm_band qb, bgm_stream stream) {
  if (!valid(l) || !valid(lb) || !valid(qb)) return BGM_ERR_ARG;
  if (l.upper != 0 || lb.upper != 0 || qb.upper != 0 || lb.lower != l.lower ||
      qb.lower != l.lower || !same_batch(l, lb) || !same_batch(l, qb))
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    if (fast::vjp_cholesky(l, lb, qb, s)) return launched();
    k_vjp_cholesky<T><<<blocks_for(l.batch, 64), 64, 0, s>>>(view<T>(l), view<T>(lb), view<T>(qb),
                                                              l.batch);
    return launched();
  });
}

int bgm_vjp_solve_vec(bgm_band l, bgm_vec sv, bgm_vec sbar, int transpose, bgm_band lbar,
                      bgm_vec vbar, int32_t* status, int64_t* row, bgm_stream stream) {
  if (!valid(l) || !valid(sv) || !valid(sbar) || !valid(lbar) || !valid(vbar)) return BGM_ERR_ARG;
  if (l.upper != 0 || lbar.upper != 0 || lbar.lower != l.lower || !same_batch(l, sv) ||
      !same_batch(l, sbar) || !same_batch(l, lbar) || !same_batch(l, vbar))
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    // grad.cpp:41: v_bar = solve_vec(l, s_bar, !transpose)
    int rc = run_solve_vec<T>(l, sbar, !transpose, vbar, status, row, s);
    if (rc) return rc;
    // grad.cpp:44-47: l_bar = -band(row col^T)
    return transpose ? run_outer<T>(sv, vbar, -1.0, lbar, s) : run_outer<T>(vbar, sv, -1.0, lbar, s);
  });
}

int bgm_vjp_sparse_inverse_subset(bgm_band l, bgm_band sm, bgm_band sbar, bgm_band lbar,
                                  int32_t* status, int64_t* row, bgm_stream stream) {
  if (!valid(l) || !valid(sm) || !valid(sbar) || !valid(lbar)) return BGM_ERR_ARG;
  if (l.upper != 0 || sm.upper != 0 || sbar.upper != 0 || lbar.upper != 0 ||
      sm.lower != l.lower || sbar.lower != l.lower || lbar.lower != l.lower ||
      !same_batch(l, sm) || !same_batch(l, sbar) || !same_batch(l, lbar))
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    if (fast::vjp_subset(l, sm, sbar, lbar, status, row, s)) return launched();
    const int wr = 3 * l.lower + 4;
    const ix padded = (l.batch + 31) / 32 * 32;
    void* wsp = nullptr;
    cudaError_t e = scratch_alloc(&wsp, sizeof(T) * size_t(padded * l.n * wr), s);
    if (e != cudaSuccess) return set_error(e);
    Band<T> ws{static_cast<T*>(wsp), l.n, wr - 1, 0, wr, 5};
    k_vjp_subset<T><<<blocks_for(l.batch, 64), 64, 0, s>>>(view<T>(l), view<T>(sm), view<T>(sbar),
                                                            view<T>(lbar), ws, l.batch, status, row);
    const int rc = launched();
    scratch_free(wsp, s);
    return rc;
  });
}

int bgm_vjp_product_band_band(bgm_band a, bgm_band b, bgm_band pbar, bgm_band abar, bgm_band bbar,
                              bgm_stream stream) {
  if (!valid(a) || !valid(b) || !valid(pbar) || !valid(abar) || !valid(bbar)) return BGM_ERR_ARG;
  if (!same_batch(a, b) || !same_batch(a, pbar) || !same_batch(a, abar) || !same_batch(a, bbar) ||
      abar.lower != a.lower || abar.upper != a.upper || bbar.lower != b.lower ||
      bbar.upper != b.upper)
    return BGM_ERR_DIM;
  if (a.batch == 0 || a.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(a.dtype, [&](auto z) {
    using T = decltype(z);
    if (fast::vjp_product(a, b, pbar, abar, bbar, s)) return launched();
    // grad.cpp:148-149: a_bar = P_bar B^T on band(A); b_bar = A^T P_bar on band(B)
    int rc = run_product<T>(pbar, 0, b, 1, abar, 1.0, s);
    if (rc) return rc;
    return run_product<T>(a, 1, pbar, 0, bbar, 1.0, s);
  });
}

int bgm_vjp_product_band_vec(bgm_band b, bgm_vec v, bgm_vec pbar, int transpose, bgm_band bbar,
                             bgm_vec vbar, bgm_stream stream) {
  if (!valid(b) || !valid(v) || !valid(pbar) || !valid(bbar) || !valid(vbar)) return BGM_ERR_ARG;
  if (!same_batch(b, v) || !same_batch(b, pbar) || !same_batch(b, bbar) || !same_batch(b, vbar) ||
      bbar.lower != b.lower || bbar.upper != b.upper)
    return BGM_ERR_DIM;
  if (b.batch == 0 || b.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(b.dtype, [&](auto z) {
    using T = decltype(z);
    if (fast::vjp_band_vec(b, v, pbar, transpose, bbar, vbar, s)) return launched();
    int rc = run_band_vec<T>(b, pbar, !transpose, vbar, s);  // grad.cpp:156
    if (rc) return rc;
    return transpose ? run_outer<T>(v, pbar, 1.0, bbar, s) : run_outer<T>(pbar, v, 1.0, bbar, s);
  });
}

int bgm_vjp_outer_band(bgm_vec m, bgm_vec v, bgm_band obar, bgm_vec mbar, bgm_vec vbar,
                       bgm_stream stream) {
  if (!valid(m) || !valid(v) || !valid(obar) || !valid(mbar) || !valid(vbar)) return BGM_ERR_ARG;
  if (!same_batch(obar, m) || !same_batch(obar, v) || !same_batch(obar, mbar) ||
      !same_batch(obar, vbar))
    return BGM_ERR_DIM;
  if (obar.batch == 0 || obar.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(obar.dtype, [&](auto z) {
    using T = decltype(z);
    int rc = run_band_vec<T>(obar, v, 0, mbar, s);  // grad.cpp:167
    if (rc) return rc;
    return run_band_vec<T>(obar, m, 1, vbar, s);  // grad.cpp:168
  });
}

int bgm_vjp_log_det(bgm_band l, const void* cbar, bgm_band lbar, bgm_stream stream) {
  if (!valid(l) || !valid(lbar) || (l.batch > 0 && !cbar)) return BGM_ERR_ARG;
  if (!same_batch(l, lbar) || l.upper != 0 || lbar.upper != 0 || lbar.lower != l.lower)
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    const ix work = bj_work(l.batch, l.n, tile_shift(lbar.tile));
    const Band<T> lb = view<T>(lbar), lv = view<T>(l);
    const T* c = static_cast<const T*>(cbar);
    // the band is zero but for its diagonal: a memset at copy-engine speed,
    // then c / L_jj on the diagonal (grad.cpp:172-176)
    const size_t bytes = size_t((l.batch + lbar.tile - 1) / lbar.tile * lbar.tile) * size_t(l.n) *
                         size_t(lbar.lower + 1) * sizeof(T);
    const cudaError_t e = cudaMemsetAsync(lbar.data, 0, bytes, s);
    if (e != cudaSuccess) return set_error(e);
    k_logdet_diag<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(lv, c, lb, l.batch);
    return launched();
  });
}

int bgm_vjp_solve_mat(bgm_band l, bgm_band sm, bgm_band sbar, int transpose, bgm_band lbar,
                      bgm_band rbar, int32_t* status, int64_t* row, bgm_stream stream) {
  if (!valid(l) || !valid(sm) || !valid(sbar) || !valid(lbar) || !valid(rbar)) return BGM_ERR_ARG;
  if (l.upper != 0 || lbar.upper != 0 || lbar.lower != l.lower || !same_batch(l, sm) ||
      !same_batch(l, sbar) || !same_batch(l, lbar) || !same_batch(l, rbar) ||
      sbar.lower != sm.lower || sbar.upper != sm.upper || !clipped(rbar))
    return BGM_ERR_DIM;
  if (l.batch == 0 || l.n == 0) return BGM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  const ix n = l.n;
  return dispatch(l.dtype, [&](auto z) {
    using T = decltype(z);
    // grad.cpp:59-60 / 70-71: t = solve_mat(l, s_bar, widened band, !transpose)
    bgm_band t = sbar;
    t.tile = 32;
    if (!transpose) {
      t.lower = int(std::min<ix>(sbar.lower, n - 1));
      t.upper = int(std::min<ix>(std::max(sbar.upper, rbar.upper), n - 1));
    } else {
      t.lower = int(std::min<ix>(std::max(sbar.lower, rbar.lower), n - 1));
      t.upper = int(std::min<ix>(sbar.upper, n - 1));
    }
    const ix padded = (l.batch + 31) / 32 * 32;
    void* tp = nullptr;
    cudaError_t e =
        scratch_alloc(&tp, sizeof(T) * size_t(padded * n * (t.lower + t.upper + 1)), s);
    if (e != cudaSuccess) return set_error(e);
    t.data = tp;
    int rc = run_solve_mat<T>(l, sbar, !transpose, t, status, row, s);
    if (!rc) {
      const ix work = bj_work(rbar.batch, n, tile_shift(rbar.tile));
      k_restrict_copy<T><<<blocks_for(work, kThreads), kThreads, 0, s>>>(view<T>(t), view<T>(rbar),
                                                                         rbar.batch);
      rc = launched();
    }
    // grad.cpp:67-68 / 78-79: l_bar = -band(t s^T) or -band(s t^T)
    if (!rc)
      rc = transpose ? run_product<T>(sm, 0, t, 1, lbar, -1.0, s)
                     : run_product<T>(t, 0, sm, 1, lbar, -1.0, s);
    scratch_free(tp, s);
    return rc;
  });
}

}  // extern "C"
