// Look-ahead blocked Cholesky on the FP64 tensor cores (k = 64, 128), a header
// instantiated by four small translation units (storage type x bandwidth: one unit took 7 minutes
// to compile, the four build in parallel).  Replaces k_chol_dmma / k_chol_mw as the
// default: those spend ~70% of every 8-column panel in lane-parallel 8-step
// shuffle chains (the 8x8 diagonal factorisation and the triangular solves of
// the panel tiles: ~85 dependent instructions per step, ncu
// profiles/r02b_chol_mw128_regions.txt), with the tensor pipe 13% busy.
//
// Here, per panel of 8 columns (tiles are 8x8, T = K/8 + 1 tile rows in the
// window, tile (I, J) on tile diagonal d = I - J):
//   * warp 0 owns tile diagonal d = 0 only.  In the update phase it first
//     updates tile (1, 1) -- the NEXT panel's diagonal tile -- and factors it
//     at once while the other warps are still in their DMMAs (look-ahead):
//     the tile goes through shared memory to every lane, and each lane runs
//     the same straight-line sequential 8x8 Cholesky and triangular inverse
//     (8 rsqrt, ~250 DFMA, no shuffles, no predicates) and publishes L00 and
//     L00^-1;
//   * the panel tiles (d, 0), d >= 1, are solved on the tensor cores:
//     X = W L00^-T is two DMMAs per tile with L00^-1 as the B fragments
//     (instead of an 8-step substitution chain per tile);
//   * the trailing update writes every tile straight into its shifted
//     register slot (4-operand DMMA: D = A B + C with D the slot of
//     (I-1, J-1)), so the window slides without register moves;
//   * fresh rows of Q and the L stores use one running pointer per lane with
//     compile-time offsets inside the matrix interior (the bounds logic of
//     the first / last K rows stays on a slow path).
// Two barriers per panel, as before.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_timing.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace wide {
namespace {

constexpr double kCheckTol = 1e-12;  // as bgm_wide.cu
constexpr int kBurnGen = 6;          // burn-in in units of the bandwidth (bgm_wide.cu)

struct Geo {
  ix batch, n, seg;
  int nseg, burn;
};

template <class ST>  // storage type; the arithmetic is fp64 for both (an fp32 factorisation rounds only
struct CholP {        // its inputs and outputs)
  Band<ST> q;  // symmetric lower store
  Band<ST> l;  // output factor
  ST* side;    // [unit][K][K+1] burn-in copies of the K columns before the segment
  int64_t* fail;
  int32_t* flag;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_la_init(int64_t* fail, int32_t* flag, ix batch, ix n) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  fail[b] = n;
  flag[b] = 0;
}

// burn-in copies of the K columns before each segment against the neighbour's genuine columns
template <class ST, int K>
__global__ void k_la_check(CholP<ST> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix unit = t / K;
  const int c = int(t % K);
  if (unit >= G.batch * G.nseg) return;
  const int p = int(unit % G.nseg);
  if (p == 0) return;
  const ix b = unit / G.nseg, s = ix(p) * G.seg, col = s - K + c;
  const ST* sd = C.side + (unit * K + c) * (K + 1);
  double sc = 0.0;
  for (int r = 0; r <= K; ++r) sc = fmax(sc, fabs(double(C.l.cell(b, r, col))));
  bool bad = false;
  const double tol = sizeof(ST) == 8 ? kCheckTol : 1e-5;
  for (int r = 0; r <= K; ++r)
    bad |= !(fabs(double(sd[r]) - double(C.l.cell(b, r, col))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

__global__ void k_la_status(const int64_t* fail, ix batch, ix n, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const bool ok = fail[b] >= n;
  report(status, row, b, ok ? BGM_OK : BGM_ERR_NOT_PD, ok ? -1 : fail[b]);
}


template <int K, int NW>
struct LA {
  static constexpr int T = K / 8 + 1;
  static constexpr int owner(int d) {
    if (d == 0) return 0;
    const int m = NW - 1;
    const int r = (d - 1) % (2 * m);
    return 1 + (r < m ? r : 2 * m - 1 - r);
  }
  static constexpr int ntiles(int w) {
    int c = 0;
    for (int d = 0; d < T; ++d)
      if (owner(d) == w) c += T - d;
    return c;
  }
  static constexpr int slot(int w, int d, int J) {
    int c = 0;
    for (int dd = 0; dd < d; ++dd)
      if (owner(dd) == w) c += T - dd;
    return c + J;
  }
};

// Panel tiles travel through shared memory in a permuted row layout: column c
// of row r sits at r * 8 + (c % 4) * 2 + c / 4, so the two MMA fragment
// elements of lane (r, q) -- columns q and 4 + q -- are one 16-byte load.
__device__ __forceinline__ int ppos(int c) { return (c & 3) * 2 + (c >> 2); }

template <class ST, int K, int NW>
struct LASmem {
  double dt[64];    // the next diagonal tile, on its way to the sequential factorisation
  double l00[64];   // L00, row-major, lower part
  double linv[64];  // L00^-1, row-major, upper part zero
  double pft[K / 8 + 1][64];   // panel tiles, permuted rows
  double npft[K / 8 + 1][64];  // minus the panel tiles (the A operands of the update)
  ST fresh[2][32];             // warp 0's fresh diagonal tile, per lane, by cp.async
};

template <class ST>
__device__ __forceinline__ void cpa8(ST* dst, const ST* src) {
  if (sizeof(ST) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(unsigned(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void dmma4(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// 1/sqrt(d) to full double precision for normal positive d: the hardware seed
// (MUFU.RSQ64H, ~22 bits) and two coupled Newton steps on (sqrt, 1/(2 sqrt));
// no special-case branches -- non-positive pivots are reported by the caller
// and such a matrix is recomputed by the exact path.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double g = d * y, h = 0.5 * y;
  double r = fma(-g, h, 0.5);
  g = fma(g, r, g);
  h = fma(h, r, h);
  r = fma(-g, h, 0.5);
  h = fma(h, r, h);
  return h + h;
}

// Every lane factors the 8x8 tile in `dt` (lower part) and publishes L00 and
// its inverse.  `piv(j, d)` sees pivot j before its square root;
// `hook(j)` runs after elimination step j (independent work to interleave).
template <class F, class H>
__device__ __forceinline__ void chol8_seq(const double* dt, double* l00, double* linv, F&& piv, H&& hook) {
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; j += 2) {
      const double2 v = *reinterpret_cast<const double2*>(dt + i * 8 + j);
      a[i][j] = v.x;
      if (j + 1 <= i) a[i][j + 1] = v.y;
    }
  double ri[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = a[j][j];
    piv(j, d);
    ri[j] = rsqrt_nr(d);
    a[j][j] = d * ri[j];
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i][j] *= ri[j];
#pragma unroll
    for (int c = j + 1; c < 8; ++c)
#pragma unroll
      for (int r = c; r < 8; ++r) a[r][c] = fma(-a[r][j], a[c][j], a[r][c]);
    hook(j);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; j += 2)
      *reinterpret_cast<double2*>(l00 + i * 8 + j) = make_double2(a[i][j], j + 1 <= i ? a[i][j + 1] : 0.0);
  // the inverse, two columns at a time
#pragma unroll
  for (int jp = 0; jp < 8; jp += 2) {
    double w0[8], w1[8];
    w0[jp] = ri[jp];
    w1[jp] = 0.0;
    w1[jp + 1] = ri[jp + 1];
#pragma unroll
    for (int i = jp + 1; i < 8; ++i) {
      double s0 = a[i][jp] * w0[jp];
#pragma unroll
      for (int k = jp + 1; k < i; ++k) s0 = fma(a[i][k], w0[k], s0);
      w0[i] = -s0 * ri[i];
      if (i > jp + 1) {
        double s1 = a[i][jp + 1] * w1[jp + 1];
#pragma unroll
        for (int k = jp + 2; k < i; ++k) s1 = fma(a[i][k], w1[k], s1);
        w1[i] = -s1 * ri[i];
      }
    }
#pragma unroll
    for (int i = jp; i < 8; ++i) *reinterpret_cast<double2*>(linv + i * 8 + jp) = make_double2(w0[i], w1[i]);
  }
}

template <int N>
struct Mode {
  static constexpr int value = N;
};

template <class ST, int K, int NW, int W>
__device__ void chol_la_unit(const CholP<ST>& C, ix b, int n, int s, int e, int i0, ST* side,
                             LASmem<ST, K, NW>& sm) {
  using M = LA<K, NW>;
  constexpr int T = M::T;
  const int lane = threadIdx.x & 31, rr = lane >> 2, q = lane & 3, c2 = 2 * q;
  const Band<ST>& Q = C.q;
  const Band<ST>& L = C.l;
  auto qval = [&](ix r, ix c) -> double {  // symmetric Q(r, c), identity past n
    if (r < c) {
      const ix t = r;
      r = c;
      c = t;
    }
    if (r - c > K || c < 0) return 0.0;
    if (r >= n) return r == c ? 1.0 : 0.0;
    return double(Q.cell(b, int(r - c), c));
  };
  auto store_l = [&](int g, int I, double x0, double x1) {  // general: rows 8I + rr of columns g + c2 + v
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int c = c2 + v, cell = 8 * I + rr - c;
      const int col = g + c;
      if (cell >= 0 && cell <= K && col < n) {
        const double val = (col + cell < n) ? (v ? x1 : x0) : 0.0;
        if (col >= s) L.cell(b, cell, col) = ST(val);
        else if (side && col >= s - K) side[ix(col - (s - K)) * (K + 1) + cell] = ST(val);
      }
    }
  };
  // interior fast paths: element (cell r, column j) of matrix b sits at base + ((j w + r) << sh)
  const int qsh = Q.s, lsh = L.s;
  const ix qw1 = ix(Q.w - 1) << qsh, lw1 = ix(L.w - 1) << lsh;
  const ST* const qb = &Q.cell(b, 0, 0);
  ST* const lb = &L.cell(b, 0, 0);
  const int pw0 = rr * 8 + ppos(c2), pw1 = rr * 8 + ppos(c2 + 1), pr = rr * 8 + c2;
  constexpr int NTW = M::ntiles(W) > 0 ? M::ntiles(W) : 1;
  double wt[NTW][2];  // the Schur window
#pragma unroll
  for (int d = 0; d < T; ++d)
    if (M::owner(d) == W)
#pragma unroll
      for (int J = 0; J < T - d; ++J)
#pragma unroll
        for (int v = 0; v < 2; ++v) wt[M::slot(W, d, J)][v] = qval(i0 + 8 * (J + d) + rr, i0 + 8 * J + c2 + v);
  int fail = n;
  unsigned bad = 0;  // pivots of the tile being factored that are not above the floor
  auto piv = [&bad](int j, double d) { bad |= unsigned(!(d > kPivotFloor)) << j; };
  auto settle = [&](int gp) {  // first bad pivot of panel gp inside [s, n)
    if (bad) {
      for (int j = 7; j >= 0; --j)
        if ((bad >> j & 1) && gp + j >= s && gp + j < n) fail = fail < gp + j ? fail : gp + j;
      bad = 0;
    }
  };
  if (threadIdx.x < 64) sm.linv[threadIdx.x] = 0.0;
  __syncthreads();
  if (W == 0) {
    const double* D = wt[M::slot(W, 0, 0)];
    *reinterpret_cast<double2*>(sm.dt + pr) = make_double2(D[0], D[1]);
    __syncwarp();
    chol8_seq(sm.dt, sm.l00, sm.linv, piv, [](int) {});
    settle(i0);
  }
  __syncthreads();

  // MODE 1: interior (`store` false: burn-in columns that nobody reads, no stores); 2: general.  One
  // interior body with a uniform run-time store flag: a third, store-free copy only cost compile time.
  auto panel = [&](const int g, auto mode, const bool store) -> bool {
    constexpr int MODE = decltype(mode)::value;
    // (B) warp 0 writes L00; the others solve their panel tiles on the tensor cores (X = W L00^-T with
    // L00^-1 as the B fragments), write them and publish them
    if (W == 0) {
      if (store) {
        const double2 x2 = *reinterpret_cast<const double2*>(sm.l00 + pr);
        if (MODE == 1) {
          ST* p = lb + ((ix(g + c2) * L.w + (rr - c2)) << lsh);
          if (rr >= c2) p[0] = ST(x2.x);
          if (rr >= c2 + 1) p[lw1] = ST(x2.y);
        } else {
          store_l(g, 0, x2.x, c2 + 1 <= rr ? x2.y : 0.0);
        }
      }
    } else {
      const double nb0 = sm.linv[rr * 8 + q], nb1 = sm.linv[rr * 8 + 4 + q];
#pragma unroll
      for (int d = 1; d < T; ++d)
        if (M::owner(d) == W) {
          const double* X = wt[M::slot(W, d, 0)];
          sm.pft[d][pw0] = X[0];
          sm.pft[d][pw1] = X[1];
        }
      __syncwarp();
#pragma unroll
      for (int d = 1; d < T; ++d)
        if (M::owner(d) == W) {
          double* Y = wt[M::slot(W, d, 0)];  // the slot is dead once X is staged
          const double2 af = *reinterpret_cast<const double2*>(sm.pft[d] + pr);
          dmma4(Y[0], Y[1], af.x, nb0, 0.0, 0.0);
          dmma(Y[0], Y[1], af.y, nb1);
        }
      __syncwarp();
#pragma unroll
      for (int d = 1; d < T; ++d)
        if (M::owner(d) == W) {
          const double* Y = wt[M::slot(W, d, 0)];
          sm.pft[d][pw0] = Y[0];
          sm.pft[d][pw1] = Y[1];
          sm.npft[d][pw0] = -Y[0];
          sm.npft[d][pw1] = -Y[1];
          if (MODE == 1 && store) {
            ST* p = lb + ((ix(g + c2) * L.w + (8 * d + rr - c2)) << lsh);
            if (8 * d + rr - c2 <= K) p[0] = ST(Y[0]);
            if (8 * d + rr - c2 - 1 <= K) p[lw1] = ST(Y[1]);
          } else if (MODE == 2) {
            store_l(g, d, Y[0], Y[1]);
          }
        }
    }
    __syncthreads();
    const int g2 = g + 8;
    if (g2 >= e) return false;  // the unit's last panel: nothing left to update
    // (C) trailing update into the shifted slots (window += (-X_I) X_J^T), the look-ahead
    // factorisation of the next diagonal tile (warp 0), the fresh tile row of Q
    if (W == 0) {
      auto upd = [&](int Ja, int Jb) {  // tiles (Ja, Ja), (Jb, Jb) of diagonal 0, interleaved
        const double2 fa = *reinterpret_cast<const double2*>(sm.pft[Ja] + pr);
        const double2 na = *reinterpret_cast<const double2*>(sm.npft[Ja] + pr);
        double* ta = wt[M::slot(W, 0, Ja - 1)];
        const double* oa = wt[M::slot(W, 0, Ja)];
        dmma4(ta[0], ta[1], na.x, fa.x, oa[0], oa[1]);
        if (Jb < T) {
          const double2 fb = *reinterpret_cast<const double2*>(sm.pft[Jb] + pr);
          const double2 nb = *reinterpret_cast<const double2*>(sm.npft[Jb] + pr);
          double* tb = wt[M::slot(W, 0, Jb - 1)];
          const double* ob = wt[M::slot(W, 0, Jb)];
          dmma4(tb[0], tb[1], nb.x, fb.x, ob[0], ob[1]);
          dmma(ta[0], ta[1], na.y, fa.y);
          dmma(tb[0], tb[1], nb.y, fb.y);
        } else {
          dmma(ta[0], ta[1], na.y, fa.y);
        }
      };
      if (MODE != 2) {  // the fresh diagonal tile (rows / columns g2 + K ..) by cp.async: no register
                        // scoreboard is held across the factorisation (a hoisted LDG stalled it for ~1200 clk)
        const int r = g2 + K + rr;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int c = g2 + K + c2 + v;
          const ST* src = r >= c ? qb + ((ix(c) * Q.w + (r - c)) << qsh) : qb + ((ix(r) * Q.w + (c - r)) << qsh);
          cpa8(&sm.fresh[v][lane], src);
        }
        cpa_commit();
      }
      upd(1, T);  // tile (1, 1) alone: the next diagonal tile
      const double* D = wt[M::slot(W, 0, 0)];
      *reinterpret_cast<double2*>(sm.dt + pr) = make_double2(D[0], D[1]);
      __syncwarp();
      chol8_seq(sm.dt, sm.l00, sm.linv, piv, [&](int j) {
        if (2 * j + 2 < T) upd(2 * j + 2, 2 * j + 3);
      });
      settle(g2);
    } else {
#pragma unroll
      for (int J = 1; J < T; ++J) {
        const double2 fb = *reinterpret_cast<const double2*>(sm.pft[J] + pr);
        double fay[T];
#pragma unroll
        for (int d = 1; d < T; ++d)
          if (M::owner(d) == W && J < T - d) {
            const double2 fa = *reinterpret_cast<const double2*>(sm.npft[J + d] + pr);
            fay[d] = fa.y;
            double* tn = wt[M::slot(W, d, J - 1)];
            const double* to = wt[M::slot(W, d, J)];
            dmma4(tn[0], tn[1], fa.x, fb.x, to[0], to[1]);
          }
#pragma unroll
        for (int d = 1; d < T; ++d)
          if (M::owner(d) == W && J < T - d) {
            double* tn = wt[M::slot(W, d, J - 1)];
            dmma(tn[0], tn[1], fay[d], fb.y);
          }
      }
    }
    // fresh tile (T-1, T-1-d): rows g2 + K + rr, columns g2 + 8 (T-1-d) + c2 + v
    if (MODE != 2) {
      const ST* const qp = qb + ((ix(g2 + c2) * Q.w + (K + rr - c2)) << qsh);  // (row g2+K+rr, column g2+c2)
#pragma unroll
      for (int d = 0; d < T; ++d)
        if (M::owner(d) == W) {
          double* tf = wt[M::slot(W, d, T - 1 - d)];
          if (d > 0) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int cell = 8 * d + rr - c2 - v;
              tf[v] = cell <= K ? double(__ldg(qp + (8 * (T - 1 - d) + v) * qw1)) : 0.0;
            }
          } else {
            cpa_wait0();
            tf[0] = double(sm.fresh[0][lane]);
            tf[1] = double(sm.fresh[1][lane]);
          }
        }
    } else {
#pragma unroll
      for (int d = 0; d < T; ++d)
        if (M::owner(d) == W) {
          double* tf = wt[M::slot(W, d, T - 1 - d)];
#pragma unroll
          for (int v = 0; v < 2; ++v) tf[v] = qval(g2 + 8 * (T - 1) + rr, g2 + 8 * (T - 1 - d) + c2 + v);
        }
    }
    __syncthreads();
    return true;
  };

  int g = i0;
  while (g < e) {
    auto interior = [&](int gg) { return gg + K + 16 <= n && (gg + 8 + K <= s || gg >= s); };
    if (interior(g)) {
      bool more = true;
#pragma unroll 1
      while (more && interior(g)) {
        more = panel(g, Mode<1>{}, g >= s);
        g += 8;
      }
      if (!more) break;
    } else {
      if (!panel(g, Mode<2>{}, true)) break;
      g += 8;
    }
  }
  if (W == 0 && lane == 0 && fail < n)
    atomicMin(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(fail));
}

template <class ST, int K, int NW, int W>
__device__ __forceinline__ void chol_la_dispatch(int w, const CholP<ST>& C, ix b, int n, int s, int e, int i0,
                                                 ST* side, LASmem<ST, K, NW>& sm) {
  if (w == W) chol_la_unit<ST, K, NW, W>(C, b, n, s, e, i0, side, sm);
  if constexpr (W + 1 < NW) chol_la_dispatch<ST, K, NW, W + 1>(w, C, b, n, s, e, i0, side, sm);
}

// repair != 0: one CTA per flagged matrix, a single exact unit over the whole matrix
template <class ST, int K, int NW>
__global__ void __launch_bounds__(32 * NW, K == 64 ? 4 : 2) k_chol_la(CholP<ST> C, Geo G, int repair) {
  __shared__ __align__(16) LASmem<ST, K, NW> sm;
  ix b, s, e, i0;
  ST* side = nullptr;
  if (repair) {
    b = blockIdx.x;
    if (b >= G.batch || !C.flag[b]) return;
    if (threadIdx.x == 0) C.fail[b] = G.n;
    __syncthreads();
    s = 0, e = G.n, i0 = 0;
  } else {
    const ix unit = blockIdx.x;
    b = unit / G.nseg;
    const int p = int(unit % G.nseg);
    if (b >= G.batch) return;
    s = ix(p) * G.seg;
    e = s + G.seg < G.n ? s + G.seg : G.n;
    i0 = s - G.burn;
    if (i0 < 0) i0 = 0;
    i0 -= i0 % 8;
    if (p > 0) side = C.side + unit * ix(K) * (K + 1);
  }
  // co-resident CTAs swap roles so the heavy (tile) warps do not all share one SM sub-partition's tensor pipe
  const int role = NW == 2 ? int((threadIdx.x >> 5) ^ (blockIdx.x & 1)) : int(threadIdx.x >> 5);
  chol_la_dispatch<ST, K, NW, 0>(role, C, b, int(G.n), int(s), int(e), int(i0), side, sm);
}

template <class ST, int K, int NW>
bool run_chol_la(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s, int segment_rows) {
  Geo G;
  G.batch = q.batch;
  G.n = q.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_la<ST, K, NW>, 32 * NW, 0);
  if (per < 1) per = 1;
  ix seg = requested_seg(segment_rows, K);
  if (seg <= 0) {
    ix nseg = ix(sms) * per / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  seg = (seg + 7) / 8 * 8;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t sb = (sizeof(ST) * size_t(units) * K * (K + 1) + 15) / 16 * 16;
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), sb + 12 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  CholP<ST> C;
  C.q = view<ST>(q);
  C.l = view<ST>(l);
  C.side = reinterpret_cast<ST*>(ws);
  C.fail = reinterpret_cast<int64_t*>(ws + sb);
  C.flag = reinterpret_cast<int32_t*>(C.fail + G.batch);
  k_la_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, C.flag, G.batch, G.n);
  {
    timing::Scope ts("wide_chol_dmma", s);
    k_chol_la<ST, K, NW><<<unsigned(units), 32 * NW, 0, s>>>(C, G, 0);
  }
  {
    timing::Scope ts("wide_chol_check", s);
    k_la_check<ST, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_repair", s);
    k_chol_la<ST, K, NW><<<unsigned(G.batch), 32 * NW, 0, s>>>(C, G, 1);
  }
  k_la_status<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, G.batch, G.n, st, row);
  scratch_free(ws, s);
  return true;
}

}  // namespace
}  // namespace wide
}  // namespace bgm
