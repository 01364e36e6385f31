// Wide-band (k = 64, 128) fast paths: one CTA per (matrix, segment).
//
// For wide bands the per-row work is a dense (k+1) x (k+1) rank-1 update,
// too large for one thread and too small for a GEMM.  A CTA of P x P threads
// holds the whole symmetric Schur window in REGISTERS: thread (tr, tc) owns
// the TS x TS tile of window positions [tr*TS, tr*TS+TS) x [tc*TS, tc*TS+TS)
// of an M x M circular grid (M = P*TS >= k+1).  Matrix row r lives at
// position r mod M for as long as it is in the window, so the window slides
// down the band with no data movement: the eliminated row's positions are
// reused by the row entering k steps later.  Per row:
//   (a) the entering row r = i+k is written into its positions from a
//       shared-memory stage that cp.async fills one group of TS rows ahead;
//   (b) the owner of position (i, i) takes the pivot           -- barrier
//   (c) the owners of column i scale it into l = L(i.., i) and
//       publish it (and write it to HBM)                        -- barrier
//   (d) every thread applies W -= l l^T to its tile (TS*TS FMAs, l read
//       from shared memory once per tile row / column).
// Steps are unrolled by TS so every register index is static.
//
// Long matrices are cut into segments with a burn-in (the Schur complement
// forgets its start state geometrically); a check kernel compares each
// unit's burn-in copy of the K columns before its segment with the
// neighbour's genuine columns, and flagged matrices are recomputed by a
// single-unit sweep -- the same scheme as the config-3 sweeps.
#include <cuda_runtime.h>

#include <cmath>
#include <initializer_list>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_timing.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace wide {
namespace {

constexpr double kCheckTol = 1e-12;
// Burn-in length in units of the bandwidth.  A wrong start state reaches the
// columns up to K rows further on and is damped by roughly |L(i,m)/L(m,m)|
// per such generation, so convergence is counted in generations of K rows
// (not rows): 6 generations take config-4 inputs (off-diagonals ~1e-3 of the
// diagonal) from ~1e-3 to below 1e-16.  Inputs that converge slower are
// caught by the check kernels and recomputed exactly.
constexpr int kBurnGen = 6;

struct Geo {
  ix batch, n, seg;
  int nseg, burn;
  // Row-span mode (span_rows > 0): instead of nseg equal segments per matrix, the batch's rows --
  // matrices laid end to end, each padded to n8 = round_up(n, 8) -- are cut into equal runs of
  // span_rows, one CTA each, so every resident CTA slot gets the same number of rows whatever the
  // batch size (64 matrices x 2 segments leave 20 of 148 one-CTA SMs idle).  A run that crosses a
  // matrix end gives its CTA several pieces (at most span_kmax); only a piece that starts inside a
  // matrix needs a burn-in and a check against its predecessor, the last piece of the CTA before.
  ix span_rows = 0, n8 = 0;
  int span_kmax = 0;
};

// piece k of the run of CTA c: matrix b, rows [s, e) (false: no such piece)
__device__ __forceinline__ bool span_piece(const Geo& G, ix c, int k, ix& b, ix& s, ix& e) {
  const ix g0 = c * G.span_rows, g1 = g0 + G.span_rows;
  b = g0 / G.n8 + k;
  if (b >= G.batch || b * G.n8 >= g1) return false;
  s = g0 - b * G.n8;
  if (s < 0) s = 0;
  e = g1 - b * G.n8;
  if (e > G.n) e = G.n;
  return s < e;
}

template <class T>
struct CholP {
  Band<T> q;  // symmetric lower store
  Band<T> l;  // output factor
  T* side;    // [unit][K][K+1] burn-in copies of the K columns before the segment
  int64_t* fail;
  int32_t* flag;
};

template <class T>
__device__ __forceinline__ void cpa(T* dst, const T* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int K, int P, int TS>
struct Shape {
  static constexpr int M = P * TS;
  static constexpr int NT = P * P;
  static_assert(M >= K + 1, "window grid too small");
};

// One unit: rows [s, e) owned, sweep from i0 (a multiple of TS).  `side`
// receives the columns [s-K, s) computed during burn-in (nullptr: none).
template <class T, int K, int P, int TS>
__device__ void chol_unit(const CholP<T>& C, ix b, ix n, ix s, ix e, ix i0, T* side) {
  using Sh = Shape<K, P, TS>;
  constexpr int M = Sh::M;
  __shared__ T stage[2][TS][K + 1];  // entering rows of the current / next group
  __shared__ T sh_l[M];
  __shared__ T sh_piv[2];
  const int tid = threadIdx.x, tr = tid / P, tc = tid % P;
  const Band<T>& Q = C.q;
  const Band<T>& L = C.l;

  // window-relative index of position p when the window starts at the row
  // whose position is im
  auto relp = [](int p, int im) -> int {
    const int r = p - im;
    return r < 0 ? r + M : r;
  };
  auto rel = [&](int p, ix i) -> int { return relp(p, int(i % M)); };
  // initial window: rows/cols [i0, i0+K) from Q (row i0+K enters at step i0)
  T w[TS][TS];
#pragma unroll
  for (int a = 0; a < TS; ++a) {
#pragma unroll
    for (int c = 0; c < TS; ++c) {
      const int ra = rel(tr * TS + a, i0), rc = rel(tc * TS + c, i0);
      const ix r = i0 + ra, cc = i0 + rc;
      T v = T(0);
      if (ra < K && rc < K && r < n && cc < n) v = ra >= rc ? Q.cell(b, ra - rc, cc) : Q.cell(b, rc - ra, r);
      w[a][c] = v;
    }
  }
  // stage fill for the group starting at row g: rows g+K .. g+K+TS-1
  auto fill = [&](int buf, ix g) {
    for (int idx = tid; idx < TS * (K + 1); idx += Sh::NT) {
      const int t = idx / (K + 1), d = idx % (K + 1);
      const ix r = g + K + t, c = r - d;
      if (r < n && c >= 0) cpa(&stage[buf][t][d], &Q.cell(b, d, c));
      else stage[buf][t][d] = T(0);
    }
    cpa_commit();
  };
  fill(0, i0);
  ix fail = n;
  int buf = 0;
#pragma unroll 1
  for (ix g = i0; g < e; g += TS) {
    const int gm = int(g % M);
    cpa_wait0();
    __syncthreads();  // stage[buf] complete; stage[buf^1] free
    if (g + TS < e) fill(buf ^ 1, g + TS);
#pragma unroll
    for (int st = 0; st < TS; ++st) {
      const ix i = g + st;
      if (i >= e) break;  // uniform
      const int im = gm + st < M ? gm + st : gm + st - M;  // position of row i
      const int oi = im / TS;                               // its owner index (slot st)
      // (a) row i+K enters at positions (i+K) mod M, slot (st+K) % TS
      {
        constexpr int sn_base = K % TS;
        const int sn = (st + sn_base) % TS;  // static after unrolling
        const int pn = im + K < M ? im + K : im + K - M;
        const int on = pn / TS;
        if (tr == on) {
#pragma unroll
          for (int c = 0; c < TS; ++c) {
            const int rc = relp(tc * TS + c, im);
            w[sn][c] = rc <= K ? stage[buf][st][K - rc] : T(0);
          }
        }
        if (tc == on) {
#pragma unroll
          for (int a = 0; a < TS; ++a) {
            const int ra = relp(tr * TS + a, im);
            w[a][sn] = ra <= K ? stage[buf][st][K - ra] : T(0);
          }
        }
      }
      // (b) pivot
      if (tr == oi && tc == oi) {
        const T d = w[st][st];
        if (!(double(d) > kPivotFloor) && i >= s) fail = fail < i ? fail : i;
        const T piv = sqrt(d);
        sh_piv[0] = piv;
        sh_piv[1] = T(1) / piv;
      }
      __syncthreads();
      // (c) column i -> l, published and stored
      if (tc == oi) {
        const T piv = sh_piv[0], rinv = sh_piv[1];
#pragma unroll
        for (int a = 0; a < TS; ++a) {
          const int ra = relp(tr * TS + a, im);
          const bool live = ra <= K && i + ra < n;
          const T lv = ra == 0 ? piv : (live ? w[a][st] * rinv : T(0));
          sh_l[tr * TS + a] = lv;
          if (ra <= K) {
            if (i >= s) L.cell(b, ra, i) = lv;  // corner cells (i+ra >= n) get 0
            else if (side && i >= s - K) side[(i - (s - K)) * (K + 1) + ra] = lv;
          }
        }
      }
      __syncthreads();
      // (d) rank-1 update of this thread's tile
      T lc[TS];
#pragma unroll
      for (int c = 0; c < TS; ++c) lc[c] = sh_l[tc * TS + c];
#pragma unroll
      for (int a = 0; a < TS; ++a) {
        const T lr = sh_l[tr * TS + a];
#pragma unroll
        for (int c = 0; c < TS; ++c) w[a][c] = fma(-lr, lc[c], w[a][c]);
      }
    }
    buf ^= 1;
  }
  cpa_wait0();
  if (fail < n) atomicMin(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(fail));
}

template <class T, int K, int P, int TS>
__global__ void __launch_bounds__(P* P) k_chol(CholP<T> C, Geo G) {
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix i0 = s - G.burn;
  if (i0 < 0) i0 = 0;
  i0 -= i0 % TS;
  chol_unit<T, K, P, TS>(C, b, G.n, s, e, i0, p > 0 ? C.side + unit * ix(K) * (K + 1) : nullptr);
}

// thread per (unit, column of the K before the segment)
template <class T, int K>
__global__ void k_chol_check(CholP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix unit = t / K;
  const int c = int(t % K);
  if (unit >= G.batch * G.nseg) return;
  const int p = int(unit % G.nseg);
  if (p == 0) return;
  const ix b = unit / G.nseg, s = ix(p) * G.seg, col = s - K + c;
  const T* sd = C.side + (unit * K + c) * (K + 1);
  double sc = 0.0;
  for (int r = 0; r <= K; ++r) sc = fmax(sc, fabs(double(C.l.cell(b, r, col))));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int r = 0; r <= K; ++r)
    bad |= !(fabs(double(sd[r]) - double(C.l.cell(b, r, col))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K, int P, int TS>
__global__ void __launch_bounds__(P* P) k_chol_repair(CholP<T> C, Geo G) {
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  if (threadIdx.x == 0) C.fail[b] = G.n;
  __syncthreads();
  chol_unit<T, K, P, TS>(C, b, G.n, 0, G.n, 0, nullptr);
}

__global__ void fill_fail(int64_t* fail, ix batch, ix n) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b < batch) fail[b] = n;
}

__global__ void k_init(int64_t* fail, int32_t* flag, ix batch, ix n) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  fail[b] = n;
  flag[b] = 0;
}

__global__ void k_status(const int64_t* fail, ix batch, ix n, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const bool ok = fail[b] >= n;
  report(status, row, b, ok ? BGM_OK : BGM_ERR_NOT_PD, ok ? -1 : fail[b]);
}

// ------------------------------------------------------------------ subset
// Takahashi recursion, column form (kernels_serial.cpp:80-104 computes the
// same band row-wise): with u_m = L(j+m, j) / L(j,j),
//   S(j+a, j) = -sum_m S(j+a, j+m) u_m          (a = 1..K)
//   S(j, j)   = 1/L(j,j)^2 - sum_m u_m S(j+m, j)
// The window holds S over rows / columns j+1 .. j+K in the same circular
// register tiles as the Cholesky; per row: u published -- barrier -- tile
// partial mat-vecs -- barrier -- per-position sums (the new column) and the
// diagonal dot -- barrier -- the new row / column j is written into its
// positions (row j+K leaves the window).
template <class T>
struct SubP {
  Band<T> l;
  Band<T> s;  // output, symmetric lower store
  T* side;    // [unit][K][K+1] burn-in copies of the K columns above the segment
  int32_t* flag;
};

template <class T, int K, int P, int TS>
__device__ void subset_unit(const SubP<T>& C, ix b, ix n, ix s, ix e, ix jtop, T* side) {
  using Sh = Shape<K, P, TS>;
  constexpr int M = Sh::M, NT = Sh::NT, NW = (NT + 31) / 32;
  __shared__ T stage[2][TS][K + 1];  // L columns of the current / next group
  __shared__ T sh_u[M];
  __shared__ T sh_new[M];
  __shared__ T sh_part[P][M];
  __shared__ T sh_dot[NW];
  const int tid = threadIdx.x, tr = tid / P, tc = tid % P;
  const Band<T>& L = C.l;
  const Band<T>& S = C.s;
  auto relp = [](int p, int pj) -> int {
    const int r = p - pj;
    return r < 0 ? r + M : r;
  };
  T w[TS][TS];
#pragma unroll
  for (int a = 0; a < TS; ++a)
#pragma unroll
    for (int c = 0; c < TS; ++c) w[a][c] = T(0);
  auto fill = [&](int buf, ix gb) {  // L columns gb .. gb+TS-1
    for (int idx = tid; idx < TS * (K + 1); idx += NT) {
      const int t = idx / (K + 1), m = idx % (K + 1);
      const ix j = gb + t;
      if (j >= 0 && j < n && j + m < n) cpa(&stage[buf][t][m], &L.cell(b, m, j));
      else stage[buf][t][m] = T(0);
    }
    cpa_commit();
  };
  const ix gb0 = jtop - jtop % TS;
  fill(0, gb0);
  int buf = 0;
#pragma unroll 1
  for (ix gb = gb0; gb + TS > s; gb -= TS) {
    const int gbm = int(gb % M);
    cpa_wait0();
    __syncthreads();
    if (gb - TS + TS > s && gb - TS >= 0) fill(buf ^ 1, gb - TS);
#pragma unroll
    for (int st = TS - 1; st >= 0; --st) {
      const ix j = gb + st;
      if (j > jtop || j < s) continue;  // uniform
      const int pj = gbm + st < M ? gbm + st : gbm + st - M;
      const int oj = pj / TS;
      const T inv = T(1) / stage[buf][st][0];
      // (1) u by position
      for (int p = tid; p < M; p += NT) {
        const int r = relp(p, pj);
        sh_u[p] = (r >= 1 && r <= K && j + r < n) ? stage[buf][st][r] * inv : T(0);
      }
      __syncthreads();
      // (2) tile partial mat-vecs
      {
        T uc[TS];
#pragma unroll
        for (int c = 0; c < TS; ++c) uc[c] = sh_u[tc * TS + c];
#pragma unroll
        for (int a = 0; a < TS; ++a) {
          T acc = T(0);
#pragma unroll
          for (int c = 0; c < TS; ++c) acc = fma(w[a][c], uc[c], acc);
          sh_part[tc][tr * TS + a] = acc;
        }
      }
      __syncthreads();
      // (3) the new column, its store, and the diagonal dot
      T dot = T(0);
      for (int p = tid; p < M; p += NT) {
        const int r = relp(p, pj);
        T v = T(0);
        if (r >= 1 && r <= K && j + r < n) {
          T acc = T(0);
#pragma unroll
          for (int q = 0; q < P; ++q) acc += sh_part[q][p];
          v = -acc;
          dot = fma(sh_u[p], v, dot);
        }
        sh_new[p] = v;
        if (r >= 1 && r <= K) {
          if (j < e) S.cell(b, r, j) = v;  // corner cells get 0
          else if (side && j < e + K) side[(j - e) * (K + 1) + r] = v;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if ((tid & 31) == 0) sh_dot[tid >> 5] = dot;
      __syncthreads();
      // (4) S(j, j) and the new row / column j into its positions
      T dsum = T(0);
#pragma unroll
      for (int q = 0; q < NW; ++q) dsum += sh_dot[q];
      const T sjj = inv * inv - dsum;
      if (tid == 0) {
        if (j < e) S.cell(b, 0, j) = sjj;
        else if (side && j < e + K) side[(j - e) * (K + 1)] = sjj;
      }
      if (tr == oj) {
#pragma unroll
        for (int c = 0; c < TS; ++c) {
          const int p = tc * TS + c;
          w[st][c] = p == pj ? sjj : sh_new[p];
        }
      }
      if (tc == oj) {
#pragma unroll
        for (int a = 0; a < TS; ++a) {
          const int p = tr * TS + a;
          w[a][st] = p == pj ? sjj : sh_new[p];
        }
      }
    }
    buf ^= 1;
  }
  cpa_wait0();
}

template <class T, int K, int P, int TS>
__global__ void __launch_bounds__(P* P) k_subset(SubP<T> C, Geo G) {
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix jtop = e + G.burn - 1;
  if (jtop > G.n - 1) jtop = G.n - 1;
  subset_unit<T, K, P, TS>(C, b, G.n, s, e, jtop,
                           p + 1 < G.nseg ? C.side + unit * ix(K) * (K + 1) : nullptr);
}

// thread per (unit, column of the K above the segment)
template <class T, int K>
__global__ void k_subset_check(SubP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix unit = t / K;
  const int c = int(t % K);
  ix b, e;
  if (G.span_rows > 0) {  // unit = side slot (CTA, piece): pieces that end inside a matrix burned in from below
    ix s0;
    if (!span_piece(G, unit / G.span_kmax, int(unit % G.span_kmax), b, s0, e) || e >= G.n) return;
  } else {
    if (unit >= G.batch * G.nseg) return;
    const int p = int(unit % G.nseg);
    if (p + 1 >= G.nseg) return;
    b = unit / G.nseg;
    e = ix(p + 1) * G.seg;
  }
  const ix col = e + c;
  if (col >= G.n) return;
  const T* sd = C.side + (unit * K + c) * (K + 1);
  double sc = 0.0;
  for (int r = 0; r <= K; ++r) sc = fmax(sc, fabs(double(C.s.cell(b, r, col))));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int r = 0; r <= K; ++r)
    bad |= !(fabs(double(sd[r]) - double(C.s.cell(b, r, col))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K, int P, int TS>
__global__ void __launch_bounds__(P* P) k_subset_repair(SubP<T> C, Geo G) {
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  subset_unit<T, K, P, TS>(C, b, G.n, 0, G.n, G.n - 1, nullptr);
}

// SingularDiagonal pre-check (kernels_serial.cpp:82-86): first row with
// |L(i,i)| < 1e-300, one thread per (matrix, row).
template <class T>
__global__ void k_diag_check(Band<T> l, ix batch, int64_t* fail) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * l.n) return;
  const ix b = t / l.n, i = t % l.n;
  if (fabs(double(l.cell(b, 0, i))) < kPivotFloor)
    atomicMin(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(i));
}

__global__ void k_status_code(const int64_t* fail, ix batch, ix n, int code, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const bool ok = fail[b] >= n;
  report(status, row, b, ok ? BGM_OK : code, ok ? -1 : fail[b]);
}

template <class KernelT>
ix pick_seg(KernelT kern, int threads, const Geo& G, ix min_seg) {
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, 0);
  if (per < 1) per = 1;
  ix nseg = ix(sms) * per / (G.batch > 0 ? G.batch : 1);
  if (nseg < 1) nseg = 1;
  ix seg = (G.n + nseg - 1) / nseg;
  return seg < min_seg ? min_seg : seg;
}

// ------------------------------------------------------------------ solves
// One warp per (matrix, segment).  The unit's window of K+1 residuals
// (L x = v, forward) or K solution values (L^T x = v, backward) lives in
// shared memory at positions row mod M; the columns of L stream through a
// cp.async ring D columns deep.  Forward row i: x_i = res_i / L(i,i), then
// the lanes apply res_{i+a} -= L(i+a, i) x_i (right-looking, column i read
// contiguously).  Backward row i: the lanes dot column i with the window,
// a butterfly sum, x_i = (v_i - s) / L(i,i) (kernels_serial.cpp:34-60).
// The window and the arithmetic are fp64 for both storage types (acc_t):
// an fp32 solve then rounds only its inputs and outputs, not n recurrences.
template <class T>
struct SolveP {
  Band<T> l;
  Vec<T> v, x;
  T* side;  // [unit][K] burn-in copies of the K solution values next to the segment
  int32_t* flag;
};

constexpr int kSolveWarps = 4;  // units per CTA
#ifndef WSOLVE_PF
#define WSOLVE_PF 96  // L2 bulk-prefetch distance of the wide solves, rows
#endif
#ifndef WSOLVE_RING64
#define WSOLVE_RING64 12
#endif
// columns in flight per unit (static shared memory: 4 units x ring x (K+2) cells)
template <int K>
constexpr int solve_ring() {
  return K <= 64 ? WSOLVE_RING64 : 8;
}

template <class T, int K, bool TR>
__device__ void solve_unit(const SolveP<T>& C, ix b, ix n, ix s, ix e, ix start, T* side, acc_t* win,
                           T (*ring)[K + 2]) {
  constexpr int R = (K + 1 + 31) / 32, D = solve_ring<K>();
  constexpr int M = (K + 2) <= 64 ? 64 : ((K + 2) <= 128 ? 128 : 256);  // window ring, power of two
  const int lane = threadIdx.x & 31;
  const Band<T>& L = C.l;
  const T* lb = &L.cell(b, 0, 0);
  const T* vb = &C.v(b, 0);
  const int ls = L.s, vs = C.v.s;
  const ix cstride = ix(L.w) << ls;
  // ring slot for column j: cells 0..K, then v_j (TR) or v_{j+K+1} (!TR)
  auto issue = [&](ix j, int slot) {
    if (j >= 0 && j < n) {
      const T* col = lb + j * cstride;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int a = lane + 32 * q;
        if (a <= K) {
          if (j + a < n) cpa(&ring[slot][a], col + (ix(a) << ls));
          else ring[slot][a] = T(0);
        }
      }
      if (lane == 0) {
        const ix vr = TR ? j : j + K + 1;
        if (vr < n) cpa(&ring[slot][K + 1], vb + (vr << vs));
        else ring[slot][K + 1] = T(0);
      }
    }
    cpa_commit();
  };
  const int dir = TR ? -1 : 1;
  const ix stop = TR ? s - 1 : e;
  // L2 prefetch of PB columns (and their v entries) PF columns ahead of the sweep
  constexpr int PF = WSOLVE_PF, PB = 16;
  auto l2pf = [&](ix j0) {
    ix a = j0 < 0 ? 0 : j0, z = j0 + PB < n ? j0 + PB : n;
    if (a >= z) return;
    auto pf = [](const T* lo, const T* hi) {
      const size_t p0 = reinterpret_cast<size_t>(lo) & ~size_t(15);
      const size_t p1 = (reinterpret_cast<size_t>(hi) + 15) & ~size_t(15);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0), "r"(unsigned(p1 - p0)) : "memory");
    };
    pf(&L.cell(b, 0, a), &L.cell(b, K, z - 1) + 1);
    const ix va = TR ? a : a + K + 1, vz = TR ? z : (z + K + 1 < n ? z + K + 1 : n);
    if (va < vz) pf(&C.v(b, va), &C.v(b, vz - 1) + 1);
  };
  if (lane == 0)
    for (int q = 0; q < PF; q += PB) l2pf(TR ? start - q - PB + 1 : start + q);
  for (int p = lane; p < M; p += 32) win[p] = 0.0;
  __syncwarp();
  if (!TR) {
    for (int a = lane; a <= K; a += 32)
      if (start + a < n) win[(start + a) & (M - 1)] = C.v(b, start + a);
  }
  for (int d = 0; d < D - 1; ++d) issue(start + dir * d, d);
  asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");
  __syncwarp();
  // 1 / L(i,i) one row ahead, off the row-to-row dependency chain
  acc_t rnext = 1.0 / acc_t(ring[0][0]);
  int slot = 0;
#pragma unroll 1
  for (ix i = start; i != stop; i += dir) {
    if (lane == 0 && (TR ? start - i : i - start) % PB == 0) l2pf(TR ? i - PF - PB + 1 : i + PF);
    issue(i + dir * (D - 1), slot == 0 ? D - 1 : slot - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");  // columns i and i + dir landed
    __syncwarp();
    const T* col = ring[slot];
    const int nslot = slot + 1 == D ? 0 : slot + 1;
    const acc_t rd = rnext;
    acc_t xi;
    if (!TR) {
      xi = win[i & (M - 1)] * rd;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int a = lane + 32 * q + 1;
        if (a <= K && i + a < n) {
          const int p = int((i + a) & (M - 1));
          win[p] = fma(-acc_t(col[a]), xi, win[p]);
        }
      }
      rnext = 1.0 / acc_t(ring[nslot][0]);
      __syncwarp();
      if (lane == 0) win[(i + K + 1) & (M - 1)] = col[K + 1];
    } else {
      acc_t acc = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int a = lane + 32 * q + 1;
        if (a <= K && i + a < n) acc = fma(acc_t(col[a]), win[(i + a) & (M - 1)], acc);
      }
      rnext = 1.0 / acc_t(ring[nslot][0]);
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      xi = (acc_t(col[K + 1]) - acc) * rd;
      __syncwarp();
      if (lane == 0) win[i & (M - 1)] = xi;
    }
    if (lane == 0) {
      if (i >= s && i < e) C.x(b, i) = T(xi);
      else if (side) {
        const ix o = TR ? i - e : i - (s - K);
        if (o >= 0 && o < K) side[o] = T(xi);
      }
    }
    __syncwarp();
    slot = nslot;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <class T, int K, bool TR>
__global__ void __launch_bounds__(32 * kSolveWarps) k_solve(SolveP<T> C, Geo G) {
  __shared__ acc_t win[kSolveWarps][(K + 2) <= 64 ? 64 : ((K + 2) <= 128 ? 128 : 256)];
  __shared__ T ring[kSolveWarps][solve_ring<K>()][K + 2];
  const int w = threadIdx.x >> 5;
  const ix unit = blockIdx.x * ix(kSolveWarps) + w;
  if (unit >= G.batch * G.nseg) return;  // whole warps
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix start;
  T* side = nullptr;
  if (!TR) {
    start = s - G.burn > 0 ? s - G.burn : 0;
    if (p > 0) side = C.side + unit * K;
  } else {
    start = e + G.burn - 1 < G.n - 1 ? e + G.burn - 1 : G.n - 1;
    if (p + 1 < G.nseg) side = C.side + unit * K;
  }
  solve_unit<T, K, TR>(C, b, G.n, s, e, start, side, win[w], ring[w]);
}

// thread per (unit, value): burn-in copy vs the neighbour's genuine values
template <class T, int K, bool TR>
__global__ void k_solve_check(SolveP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix unit = t / K;
  const int c = int(t % K);
  if (unit >= G.batch * G.nseg) return;
  const int p = int(unit % G.nseg);
  if (TR ? p + 1 >= G.nseg : p == 0) return;
  const ix b = unit / G.nseg;
  const ix row = TR ? ix(p + 1) * G.seg + c : ix(p) * G.seg - K + c;
  if (row >= G.n) return;
  double sc = 0.0;
  for (int q = 0; q < K; ++q) {
    const ix r = TR ? ix(p + 1) * G.seg + q : ix(p) * G.seg - K + q;
    if (r < G.n) sc = fmax(sc, fabs(double(C.x(b, r))));
  }
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  if (!(fabs(double(C.side[unit * K + c]) - double(C.x(b, row))) <= tol * (sc + 1e-300))) C.flag[b] = 1;
}

template <class T, int K, bool TR>
__global__ void __launch_bounds__(32 * kSolveWarps) k_solve_repair(SolveP<T> C, Geo G) {
  __shared__ acc_t win[kSolveWarps][(K + 2) <= 64 ? 64 : ((K + 2) <= 128 ? 128 : 256)];
  __shared__ T ring[kSolveWarps][solve_ring<K>()][K + 2];
  const int w = threadIdx.x >> 5;
  const ix b = blockIdx.x * ix(kSolveWarps) + w;
  if (b >= G.batch || !C.flag[b]) return;  // whole warps
  solve_unit<T, K, TR>(C, b, G.n, 0, G.n, TR ? G.n - 1 : 0, nullptr, win[w], ring[w]);
}

// first (forward) / last (backward sweep reaches it first) singular pivot
template <class T>
__global__ void k_singular(Band<T> l, ix batch, int tr, int64_t* fail) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * l.n) return;
  const ix b = t / l.n, i = t % l.n;
  if (fabs(double(l.cell(b, 0, i))) < kPivotFloor) {
    if (!tr) atomicMin(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(i));
    else atomicMax(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(i + 1));
  }
}

__global__ void k_init_fail(int64_t* fail, int32_t* flag, ix batch, int64_t v) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  fail[b] = v;
  flag[b] = 0;
}

__global__ void k_status_solve(const int64_t* fail, ix batch, ix n, int tr, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix f = tr ? fail[b] - 1 : fail[b];  // backward: stored as row + 1, 0 = none
  const bool ok = tr ? f < 0 : f >= n;
  report(status, row, b, ok ? BGM_OK : BGM_ERR_SINGULAR, ok ? -1 : f);
}

// ------------------------------------------------------------------ log-det
// kernels.cpp:121-129, any bandwidth / layout: thread per (matrix, chunk of
// kLogChunk rows), then a per-matrix sum of the chunk partials in chunk order
// (deterministic).  NonPositiveDiagonal reports the first failing row.
constexpr int kLogChunk = 64;

template <class T>
__global__ void k_logdet_part(Band<T> l, ix batch, ix chunks, double* part, int64_t* fail) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, c;
  if (!split_bj(t, batch, chunks, l.s, b, c)) return;
  const ix i0 = c * kLogChunk;
  const ix i1 = i0 + kLogChunk < l.n ? i0 + kLogChunk : l.n;
  // sum of logs as one log of a product: each pivot splits into 2^e * m with
  // m in [1/sqrt2, sqrt2) (bit fields), the m multiply (|log prod| <= 23 for
  // 64 rows), so one libdevice log per chunk instead of one per row; zero,
  // negative, subnormal, inf and NaN pivots take the per-row loop
  double prod = 1.0;
  int esum = 0;
  ix bad = -1;
  bool slow = false;
#pragma unroll 8
  for (ix i = i0; i < i1; ++i) {
    const double d = double(l.cell(b, 0, i));
    const int hi = __double2hiint(d);
    const int ex = (hi >> 20) & 0x7ff;
    slow |= (hi < 0) | (ex == 0) | (ex == 0x7ff);
    // mantissa with exponent 0 (in [1, 2)); halve it above sqrt 2
    const int top = hi & 0x000fffff;
    const bool up = top >= 0x6a09e;  // 1.4142... = 0x3ff6a09e...
    const double m = __hiloint2double(top | (up ? 0x3fe00000 : 0x3ff00000), __double2loint(d));
    esum += ex - 1023 + (up ? 1 : 0);
    prod *= m;
  }
  double acc = fma(double(esum), 0.6931471805599453094, log(prod));
  if (slow) {
    acc = 0.0;
    for (ix i = i0; i < i1; ++i) {
      const double d = double(l.cell(b, 0, i));
      if (!(d > 0.0) && bad < 0) bad = i;
      acc += log(d);
    }
  }
  part[b * chunks + c] = acc;
  if (bad >= 0) atomicMin(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(bad));
}

template <class T>
__global__ void k_logdet_sum(const double* part, const int64_t* fail, ix batch, ix n, ix chunks, T* out,
                             int32_t* status, int64_t* row) {
  const ix b = (blockIdx.x * ix(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= batch) return;  // whole warps
  double acc = 0.0;
  for (ix c = lane; c < chunks; c += 32) acc += part[b * chunks + c];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane) return;
  const bool ok = fail[b] >= n;
  if (ok) out[b] = T(acc);
  report(status, row, b, ok ? BGM_OK : BGM_ERR_NONPOS_DIAG, ok ? -1 : fail[b]);
}

// ------------------------------------------------------------------ vjp_cholesky
// grad.cpp:11-36 for wide bands, one warp per (matrix, segment).  The l_bar
// window (rows [i-K, i] x cols [i-K, row]) and the matching window of L live
// in shared memory as packed lower triangles indexed (x, y) = (row - (i-K),
// col - (i-K)); per row:
//   * the row's back-substitution (q_K = 1/2 r_K / L_ii, then right-looking
//     over x2 = K-1..0: q = r'_x2 / L(j2,j2), r'_y -= q L(j2, j_y)), lanes own
//     y = lane + 32t, the pivot value travels by shuffle;
//   * l_bar(j, k) -= q_j L(i, k) fused with the shift (x, y) -> (x+1, y+1) of
//     both windows, processed in descending 32-entry chunks (each chunk loads
//     before it stores, so the in-place shift never reads a moved entry);
//   * column i-1-K of l_bar and L enters at y = 0.
template <class T>
struct VcP {
  Band<T> l, lb, qb;
  T* side;  // [unit][K][K+1] burn-in copies of q_bar rows [e, e+K)
  int32_t* flag;
};

__device__ __forceinline__ int tri_w(int a, int b) { return a * (a + 1) / 2 + b; }
__device__ __forceinline__ void untri(int idx, int& x, int& y) {
  int a = int((sqrtf(8.0f * float(idx) + 1.0f) - 1.0f) * 0.5f);
  if (tri_w(a + 1, 0) <= idx) ++a;
  if (tri_w(a, 0) > idx) --a;
  x = a;
  y = idx - tri_w(a, 0);
}

// Incremental (row, col) of a packed-triangle index stepping by +-32.
__device__ __forceinline__ void tri_next32(int& a, int& b) {
  b += 32;
  while (b > a) {
    b -= a + 1;
    ++a;
  }
}
__device__ __forceinline__ void tri_prev32(int& a, int& b) {
  b -= 32;
  while (b < 0) {
    --a;
    b += a + 1;
  }
}

template <class T, int K>
__device__ void vchol_warp(const VcP<T>& C, ix b, ix n, ix s, ix e, ix start, T* side, T* Wb, T* Lw,
                           T* sq, T* slr, T* sinv) {
  constexpr int R = (K + 1 + 31) / 32, NP = (K + 1) * (K + 2) / 2, N1 = K * (K + 1) / 2;
  const int lane = threadIdx.x & 31;
  for (int idx = lane; idx < NP; idx += 32) {
    int x, y;
    untri(idx, x, y);
    const ix r = start - K + x, c = start - K + y;
    const bool in = c >= 0 && r < n;
    Wb[idx] = in ? C.lb.cell(b, x - y, c) : T(0);
    Lw[idx] = in ? C.l.cell(b, x - y, c) : T(0);
  }
  __syncwarp();
#pragma unroll 1
  for (ix i = start; i >= s; --i) {
    T rr[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int y = lane + 32 * t;
      rr[t] = (y <= K) ? Wb[tri_w(K, y)] : T(0);
      if (y <= K) {
        slr[y] = Lw[tri_w(K, y)];
        const T d = Lw[tri_w(y, y)];
        sinv[y] = (i - K + y >= 0) ? T(1) / d : T(0);
      }
    }
    __syncwarp();
    const T qK = T(0.5) * Wb[tri_w(K, K)] / Lw[tri_w(K, K)];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int y = lane + 32 * t;
      if (y < K) rr[t] = fma(T(-2) * qK, slr[y], rr[t]);
    }
    if (lane == 0) sq[K] = qK;
#pragma unroll 1
    for (int x2 = K - 1; x2 >= 0; --x2) {
      const int slot = x2 >> 5, owner = x2 & 31;
      T v = rr[0];
#pragma unroll
      for (int t = 1; t < R; ++t)
        if (slot == t) v = rr[t];
      v = __shfl_sync(0xffffffffu, v, owner);
      const T q = v * sinv[x2];
      if (lane == owner) sq[x2] = q;
      const T* lrow = Lw + tri_w(x2, 0);  // L(j2, j_y) = Lw(x2, y)
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int y = lane + 32 * t;
        if (y < x2) rr[t] = fma(-q, lrow[y], rr[t]);
      }
    }
    __syncwarp();
    // q_bar row i: q_x at cell (K - x) of column i-K+x
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int x = lane + 32 * t;
      if (x <= K && i - K + x >= 0) {
        if (i < e) C.qb.cell(b, K - x, i - K + x) = sq[x];
        else if (side && i < e + K) side[(i - e) * (K + 1) + x] = sq[x];
      }
    }
    // update + shift, descending chunks
    {
      int cx, cy;
      untri(((N1 - 1) & ~31) + lane, cx, cy);
#pragma unroll 1
      for (int base = (N1 - 1) & ~31; base >= 0; base -= 32) {
        const int idx = base + lane;
        T wv = T(0), lv = T(0);
        const bool ok = idx < N1;
        if (ok) {
          wv = fma(-sq[cx], slr[cy], Wb[idx]);
          lv = Lw[idx];
        }
        __syncwarp();
        if (ok) {
          const int d = idx + cx + 2;  // tri(x+1, y+1)
          Wb[d] = wv;
          Lw[d] = lv;
        }
        __syncwarp();
        if (base >= 32) tri_prev32(cx, cy);
      }
    }
    const ix c = i - 1 - K;  // entering column
    for (int x = lane; x <= K; x += 32) {
      const bool in = c >= 0 && c + x < n;
      Wb[tri_w(x, 0)] = in ? C.lb.cell(b, x, c) : T(0);
      Lw[tri_w(x, 0)] = in ? C.l.cell(b, x, c) : T(0);
    }
    __syncwarp();
  }
}

template <class T, int K>
struct VcSmem {
  static constexpr int NP = (K + 1) * (K + 2) / 2;
  static constexpr size_t bytes = sizeof(T) * (2 * NP + 3 * (K + 1));
};

template <class T, int K>
__global__ void __launch_bounds__(32) k_vchol_w(VcP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  constexpr int NP = VcSmem<T, K>::NP;
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix start = e + G.burn - 1 < G.n - 1 ? e + G.burn - 1 : G.n - 1;
  vchol_warp<T, K>(C, b, G.n, s, e, start, p + 1 < G.nseg ? C.side + unit * ix(K) * (K + 1) : nullptr, sm,
                   sm + NP, sm + 2 * NP, sm + 2 * NP + (K + 1), sm + 2 * NP + 2 * (K + 1));
}

template <class T, int K>
__global__ void k_vchol_w_check(VcP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix id = t / K;
  const int c = int(t % K);
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  if (p + 1 >= G.nseg) return;
  const ix b = id / G.nseg, i = ix(p + 1) * G.seg + c;
  if (i >= G.n) return;
  const T* sd = C.side + (id * K + c) * (K + 1);
  double sc = 0.0;
  for (int x = 0; x <= K; ++x)
    if (i - K + x >= 0) sc = fmax(sc, fabs(double(C.qb.cell(b, K - x, i - K + x))));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int x = 0; x <= K; ++x)
    if (i - K + x >= 0) bad |= !(fabs(double(sd[x]) - double(C.qb.cell(b, K - x, i - K + x))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K>
__global__ void __launch_bounds__(32) k_vchol_w_repair(VcP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  constexpr int NP = VcSmem<T, K>::NP;
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  vchol_warp<T, K>(C, b, G.n, 0, G.n, G.n - 1, nullptr, sm, sm + NP, sm + 2 * NP, sm + 2 * NP + (K + 1),
                   sm + 2 * NP + 2 * (K + 1));
}

template <class T>
__global__ void k_zero_corners_w(Band<T> o, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const int K = o.lo;
  ix b, jj;
  if (!split_bj(t, batch, ix(K) * (K + 1), o.s, b, jj)) return;
  const ix j = o.n - K + jj / (K + 1);
  const int r = int(jj % (K + 1));
  if (j >= 0 && j + r >= o.n) o.cell(b, r, j) = T(0);
}

// ------------------------------------------------------------------ vjp_subset
// grad.cpp:84-143 for wide bands, one warp per (matrix, segment), forward
// over columns j.  State in shared memory:
//   B   -- the symmetric adjoint's lower cells still to be consumed, rows
//          [j, c+K] of columns c in [j-K, j], packed (y, x) = (c-(j-K), m-j);
//   bu  -- U-bar rows i in [j-K, j] (circular by i), K entries each.
// Per column: r_x = B(j, i_x) (the reference's mirror move), a forward
// substitution cur_x = r_x - sum L(i_x, i_x') scale_x' (scale = cur / L_ii,
// shuffle-broadcast), bu(i, i+d) -= S(i+d, j) cur_i, the lower cells of
// column j -= L(m, i) scale_i, then row i = j-K of bu is complete and its
// L-bar column is written (grad.cpp:130-141).  The sweep runs K columns past
// the segment so the last owned rows of bu complete from the exact state.
template <class T>
struct VsP {
  Band<T> l, s, sb, lb;
  T* side;  // [unit][K][K+2]: cur (K+1) + bvec of the K columns before the segment (burn-in)
  T* tail;  // [unit][K][K+2]: the same for the segment's last K columns (genuine)
  int32_t* flag;
};

template <class T, int K>
struct VsSmem {
  static constexpr int NP = (K + 1) * (K + 2) / 2;
  static constexpr int NU = (K + 1) * K;
  static constexpr size_t count = NP + NU + (2 * K + 1) + 4 * (K + 1);
  static constexpr size_t bytes = sizeof(T) * count;
};

template <class T, int K>
__device__ void vsub_warp(const VsP<T>& C, ix b, ix n, ix s, ix e, ix start, T* side, T* tail, T* sm) {
  using Sz = VsSmem<T, K>;
  constexpr int R = (K + 1 + 31) / 32, NP = Sz::NP, NU = Sz::NU, N1 = NP - (K + 1);
  T* Bw = sm;
  T* bu = Bw + NP;
  T* sS = bu + NU;         // S(j + t, j), t in [-K, K] at index t + K
  T* sinv = sS + 2 * K + 1;  // 1 / L(i_x, i_x)
  T* ssc = sinv + (K + 1);   // scale_x
  T* scur = ssc + (K + 1);   // cur_x
  T* sbv = scur + (K + 1);   // bvec, circular by column mod (K+1)
  const int lane = threadIdx.x & 31;
  const Band<T>& L = C.l;
  const Band<T>& S = C.s;
  // per-matrix base pointers: cell (r, c) at base[(c * w + r) << s]
  const int sh = L.s;
  const T* lbase = L.p + (((b >> sh) * n * L.w) << sh) + (b & ((ix(1) << sh) - 1));
  auto lcell = [&](ix r, ix c) -> T {
    return (c >= 0 && r < n && r - c <= K) ? lbase[(c * (K + 1) + (r - c)) << sh] : T(0);
  };
  auto scell = [&](ix r, ix c) -> T {  // symmetric S(r, c), |r - c| <= K
    if (r < 0 || c < 0 || r >= n || c >= n) return T(0);
    return r >= c ? S.cell(b, int(r - c), c) : S.cell(b, int(c - r), r);
  };
  // B for column `start`: (y, x) -> c = start-K+y, m = start+x, cell m - c = K + x - y
  for (int idx = lane; idx < NP; idx += 32) {
    int y, x;
    untri(idx, y, x);
    const ix c = start - K + y, m = start + x;
    Bw[idx] = (c >= 0 && m < n) ? C.sb.cell(b, K + x - y, c) : T(0);
  }
  for (int q = lane; q < NU; q += 32) bu[q] = T(0);
  __syncwarp();
  const ix jend = e + K < n ? e + K : n;  // K columns past the segment complete its bu rows
  auto emit = [&](ix c) {  // bu row c complete -> L-bar column c
    const int slot = int(c % (K + 1));
    const T lcc = lcell(c, c);
    const T iv = T(1) / lcc;
    T dsum = T(0);
    for (int d = lane + 1; d <= K; d += 32) {
      const T v = bu[slot * K + d - 1];
      if (c + d < n) {
        C.lb.cell(b, d, c) = v * iv;
        dsum = fma(v, lcell(c + d, c), dsum);
      } else {
        C.lb.cell(b, d, c) = T(0);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    if (lane == 0) C.lb.cell(b, 0, c) = (T(-2) * sbv[slot] * iv - dsum) * (iv * iv);
  };
#pragma unroll 1
  for (ix j = start; j < jend; ++j) {
    T rr[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int x = lane + 32 * t;
      if (x <= K) {
        const ix i = j - K + x;
        rr[t] = Bw[tri_w(x, 0)];
        sinv[x] = i >= 0 ? T(1) / lcell(i, i) : T(0);
      } else {
        rr[t] = T(0);
      }
    }
    for (int t = lane; t <= 2 * K; t += 32) sS[t] = scell(j + t - K, j);
    __syncwarp();
    // forward substitution over i_x = j-K+x
#pragma unroll 1
    for (int x = 0; x <= K; ++x) {
      const int slot = x >> 5, owner = x & 31;
      T v = rr[0];
#pragma unroll
      for (int t = 1; t < R; ++t)
        if (slot == t) v = rr[t];
      const T cur = __shfl_sync(0xffffffffu, v, owner);
      const T sc = cur * sinv[x];
      if (lane == owner) {
        scur[x] = cur;
        ssc[x] = sc;
      }
      const ix ix_ = j - K + x;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int x2 = lane + 32 * t;
        // L(i_x2, i_x) = cell x2 - x of column i_x
        if (x2 > x && x2 <= K && ix_ >= 0 && j - K + x2 < n)
          rr[t] = fma(-lbase[(ix_ * (K + 1) + (x2 - x)) << sh], sc, rr[t]);
      }
    }
    __syncwarp();
    if (lane == 0) sbv[j % (K + 1)] = scur[K];  // bvec(j): bs(j, j) when i reaches j (grad.cpp:114)
    __syncwarp();
    // burn-in / tail copies for the boundary check
    if (side && j >= s - K && j < s) {
      T* sd = side + (j - (s - K)) * (K + 2);
      for (int x = lane; x <= K; x += 32) sd[x] = scur[x];
      if (lane == 0) sd[K + 1] = sbv[j % (K + 1)];
    }
    if (tail && j >= e - K && j < e) {
      T* td = tail + (j - (e - K)) * (K + 2);
      for (int x = lane; x <= K; x += 32) td[x] = scur[x];
      if (lane == 0) td[K + 1] = sbv[j % (K + 1)];
    }
    // bu(i_x, i_x + d) -= S(i_x + d, j) cur_x, d = 1..K; row slot = i mod (K+1)
    const int jm = int(((j - K) % (K + 1) + (K + 1)) % (K + 1));
    for (int q = lane; q < NU; q += 32) {
      const int x = q / K, d = q % K + 1;
      if (j - K + x >= 0) {
        const int slot = jm + x < K + 1 ? jm + x : jm + x - (K + 1);
        T* u = bu + slot * K + d - 1;
        *u = fma(-sS[x + d], scur[x], *u);
      }
    }
    // lower cells of column j: B(j+d, j) -= sum_{x >= d} L(j+d, i_x) scale_x
    for (int d = lane + 1; d <= K; d += 32) {
      T acc = T(0);
      if (j + d < n) {
        // L(j+d, i_x) = cell K + d - x of column i_x = j - K + x
#pragma unroll 4
        for (int x = d; x <= K; ++x) {
          const ix c = j - K + x;
          if (c >= 0) acc = fma(lbase[(c * (K + 1) + (K + d - x)) << sh], ssc[x], acc);
        }
      }
      Bw[tri_w(K, d)] -= acc;
    }
    __syncwarp();
    // row j - K of bu is complete
    if (j - K >= s && j - K < e) emit(j - K);
    __syncwarp();
    if (j - K >= 0) {
      const int slot = int((j - K) % (K + 1));
      for (int d = lane; d < K; d += 32) bu[slot * K + d] = T(0);
    }
    // shift B: (y, x) -> (y-1, x-1) for x >= 1, ascending chunks
    {
      int cy, cx;
      untri(lane, cy, cx);
#pragma unroll 1
      for (int base = 0; base < NP; base += 32) {
        const int idx = base + lane;
        const bool ok = idx < NP && cx >= 1;
        T v = T(0);
        if (ok) v = Bw[idx];
        __syncwarp();
        if (ok) Bw[idx - cy - 1] = v;  // tri(y-1, x-1)
        __syncwarp();
        tri_next32(cy, cx);
      }
    }
    // new column j+1 at y = K: S-bar cells (j+1+x, j+1)
    for (int x = lane; x <= K; x += 32) {
      const ix c = j + 1, m = c + x;
      Bw[tri_w(K, x)] = (m < n) ? C.sb.cell(b, x, c) : T(0);
    }
    __syncwarp();
  }
  // rows completed only by the matrix end
  for (ix c = (n - K > s ? n - K : s); c < e; ++c)
    if (c + K >= jend && c + K >= n) emit(c);
}

template <class T, int K>
__global__ void __launch_bounds__(32) k_vsub(VsP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix start = s - G.burn > 0 ? s - G.burn : 0;
  vsub_warp<T, K>(C, b, G.n, s, e, start, p > 0 ? C.side + unit * ix(K) * (K + 2) : nullptr,
                  p + 1 < G.nseg ? C.tail + unit * ix(K) * (K + 2) : nullptr, reinterpret_cast<T*>(smraw));
}

template <class T, int K>
__global__ void k_vsub_check(VsP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix id = t / K;
  const int c = int(t % K);
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  if (p == 0) return;
  const ix b = id / G.nseg;
  const T* a = C.side + (id * K + c) * (K + 2);
  const T* r = C.tail + ((id - 1) * K + c) * (K + 2);
  double sc = 0.0;
  for (int x = 0; x < K + 2; ++x) sc = fmax(sc, fabs(double(r[x])));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int x = 0; x < K + 2; ++x) bad |= !(fabs(double(a[x]) - double(r[x])) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K>
__global__ void __launch_bounds__(32) k_vsub_repair(VsP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  vsub_warp<T, K>(C, b, G.n, 0, G.n, 0, nullptr, nullptr, reinterpret_cast<T*>(smraw));
}

// ------------------------------------------------------------------ cholesky, FP64 DMMA
// Blocked right-looking banded Cholesky on the FP64 tensor cores
// (mma.sync m8n8k4 f64, SASS DMMA), k = 64, one warp per (matrix, segment).
// The band's trailing Schur complement over rows [g, g+K+8) is held as
// 8x8 tiles (I, J), 0 <= J <= I <= K/8, in the MMA accumulator layout
// (lane: row lane/4, columns 2(lane%4) + {0,1}) -- 45 tiles, 90 doubles per
// lane, all in registers.  Per panel of 8 rows:
//   * panel column tiles (I, 0) go to shared memory, where the warp factors
//     the diagonal tile and scales the column below it (the unblocked
//     panel: 8 pivots, lane-parallel updates);
//   * L columns g..g+7 are written out from there;
//   * trailing update W_IJ -= L_I0 L_J0^T for 1 <= J <= I: 2 DMMA per tile
//     (k = 8 = 2 x 4); the A and B fragments of L_I0 / L_J0 are the same
//     (row lane/4, column 4kc + lane%4) reads of the shared panel;
//   * the tiles shift by one tile (register moves) and a fresh tile row of
//     Q enters.  Rows past n are padded with the identity.
constexpr int kDK = 64, kDT = kDK / 8 + 1, kDTiles = kDT * (kDT + 1) / 2, kDRows = kDK + 8;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__host__ __device__ constexpr int dti(int I, int J) { return I * (I + 1) / 2 + J; }

__device__ void chol_dmma_unit(const CholP<double>& C, ix b, ix n, ix s, ix e, ix i0, double* side) {
  constexpr int K = kDK;
  const int lane = threadIdx.x & 31, rr = lane >> 2, q = lane & 3, c2 = 2 * q;
  const Band<double>& Q = C.q;
  const Band<double>& L = C.l;
  auto qval = [&](ix r, ix c) -> double {  // symmetric Q(r, c), identity past n
    if (r < c) {
      const ix t = r;
      r = c;
      c = t;
    }
    if (r - c > K || c < 0) return 0.0;
    if (r >= n) return r == c ? 1.0 : 0.0;
    return Q.cell(b, int(r - c), c);
  };
  auto pick = [](const double* v, int e) -> double { return e ? v[1] : v[0]; };
  double wt[kDTiles][2];
#pragma unroll
  for (int I = 0; I < kDT; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J)
#pragma unroll
      for (int v = 0; v < 2; ++v) wt[dti(I, J)][v] = qval(i0 + 8 * I + rr, i0 + 8 * J + c2 + v);
  ix fail = n;
#pragma unroll 1
  for (ix g = i0; g < e; g += 8) {
    double* D = wt[dti(0, 0)];
    // (1) Cholesky of the diagonal tile in the fragment layout (shuffles)
    double rinv[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const double dpp = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * p + (p >> 1));
      if (lane == 0 && g + p >= s && g + p < n && !(dpp > kPivotFloor)) fail = fail < g + p ? fail : g + p;
      // 1/sqrt by the reciprocal square root, the pivot from it: one MUFU
      // sequence on the 8-step chain instead of a sqrt and a division
      const double ri = rsqrt(dpp), piv = dpp * ri;
      rinv[p] = ri;
      if (q == (p >> 1)) {
        if (rr > p) D[p & 1] *= rinv[p];
        else if (rr == p) D[p & 1] = piv;
      }
      const double lr = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * rr + (p >> 1));
      const double lc0 = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * c2 + (p >> 1));
      const double lc1 = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * (c2 + 1) + (p >> 1));
      if (c2 > p && rr >= c2) D[0] = fma(-lr, lc0, D[0]);
      if (c2 + 1 > p && rr >= c2 + 1) D[1] = fma(-lr, lc1, D[1]);
    }
    if (c2 > rr) D[0] = 0.0;
    if (c2 + 1 > rr) D[1] = 0.0;
    // (2) tiles below: X_I = W_I0 L00^-T, row by row inside each lane quad
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double l0 = __shfl_sync(0xffffffffu, pick(D, c & 1), 4 * c2 + (c >> 1));        // L00[c2][c]
      const double l1 = __shfl_sync(0xffffffffu, pick(D, c & 1), 4 * (c2 + 1) + (c >> 1));  // L00[c2+1][c]
#pragma unroll
      for (int I = 1; I < kDT; ++I) {
        double* X = wt[dti(I, 0)];
        if (q == (c >> 1)) X[c & 1] *= rinv[c];
        const double x = __shfl_sync(0xffffffffu, pick(X, c & 1), 4 * rr + (c >> 1));
        if (c2 > c) X[0] = fma(-x, l0, X[0]);
        if (c2 + 1 > c) X[1] = fma(-x, l1, X[1]);
      }
    }
    // (3) A / B fragments of the panel tiles: column 4kc + q of row rr
    double pf[kDT][2];
#pragma unroll
    for (int I = 1; I < kDT; ++I)
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const int srcl = 4 * rr + 2 * kc + (q >> 1);
        const double e0 = __shfl_sync(0xffffffffu, wt[dti(I, 0)][0], srcl);
        const double e1 = __shfl_sync(0xffffffffu, wt[dti(I, 0)][1], srcl);
        pf[I][kc] = (q & 1) ? e1 : e0;
      }
    // (4) L columns g .. g+7: lane (rr, q) holds rows 8I + rr, columns c2, c2+1
#pragma unroll
    for (int I = 0; I < kDT; ++I)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int c = c2 + v;
        const int cell = 8 * I + rr - c;
        const ix col = g + c;
        if (cell >= 0 && cell <= K && col < n) {
          const double val = (col + cell < n) ? wt[dti(I, 0)][v] : 0.0;
          if (col >= s) L.cell(b, cell, col) = val;
          else if (side && col >= s - K) side[(col - (s - K)) * (K + 1) + cell] = val;
        }
      }
    // (5) trailing update W_IJ -= X_I X_J^T on the FP64 tensor cores
#pragma unroll
    for (int I = 1; I < kDT; ++I)
#pragma unroll
      for (int J = 1; J <= I; ++J) {
        dmma(wt[dti(I, J)][0], wt[dti(I, J)][1], -pf[I][0], pf[J][0]);
        dmma(wt[dti(I, J)][0], wt[dti(I, J)][1], -pf[I][1], pf[J][1]);
      }
    // (6) shift by one tile; a fresh tile row enters: rows g2+K+rr, cols g2+8J+c2+v
#pragma unroll
    for (int I = 1; I < kDT; ++I)
#pragma unroll
      for (int J = 1; J <= I; ++J) {
        wt[dti(I - 1, J - 1)][0] = wt[dti(I, J)][0];
        wt[dti(I - 1, J - 1)][1] = wt[dti(I, J)][1];
      }
    const ix g2 = g + 8;
#pragma unroll
    for (int J = 0; J < kDT; ++J)
#pragma unroll
      for (int v = 0; v < 2; ++v) wt[dti(kDT - 1, J)][v] = qval(g2 + 8 * (kDT - 1) + rr, g2 + 8 * J + c2 + v);
  }
  if (lane == 0 && fail < n)
    atomicMin(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(fail));
}

// Multi-warp variant: the CTA's NW warps split the Schur tiles by DIAGONAL
// (tile (I, J) has d = I - J); the shift (I, J) -> (I-1, J-1) keeps d, so
// every warp keeps its tiles across panels and only the panel fragments
// travel, through shared memory.  Per panel: the owner of d = 0 factors the
// diagonal tile (shuffles) -- barrier -- the owners of the panel tiles
// (d, 0) solve them against L00 and publish their MMA fragments --
// barrier -- every warp applies its DMMA updates and shifts.
template <int K, int NW>
struct MW {
  static constexpr int T = K / 8 + 1;
  static constexpr int owner(int d) {
    const int r = d % (2 * NW);
    return r < NW ? r : 2 * NW - 1 - r;
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

template <int K, int NW>
struct MWSmem {
  double l00[8][9];
  double rinv[8];
  double pf[K / 8 + 1][2][32];
};

template <int K, int NW, int W>
__device__ void chol_mw_unit(const CholP<double>& C, ix b, ix n, ix s, ix e, ix i0, double* side,
                             MWSmem<K, NW>& sm) {
  using M = MW<K, NW>;
  constexpr int T = M::T;
  const int lane = threadIdx.x & 31, rr = lane >> 2, q = lane & 3, c2 = 2 * q;
  const Band<double>& Q = C.q;
  const Band<double>& L = C.l;
  auto qval = [&](ix r, ix c) -> double {
    if (r < c) {
      const ix t = r;
      r = c;
      c = t;
    }
    if (r - c > K || c < 0) return 0.0;
    if (r >= n) return r == c ? 1.0 : 0.0;
    return Q.cell(b, int(r - c), c);
  };
  auto pick = [](const double* v, int e) -> double { return e ? v[1] : v[0]; };
  auto store_l = [&](ix g, int I, const double* x) {  // rows 8I + rr of columns g + c2 + v
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int c = c2 + v, cell = 8 * I + rr - c;
      const ix col = g + c;
      if (cell >= 0 && cell <= K && col < n) {
        const double val = (col + cell < n) ? x[v] : 0.0;
        if (col >= s) L.cell(b, cell, col) = val;
        else if (side && col >= s - K) side[(col - (s - K)) * (K + 1) + cell] = val;
      }
    }
  };
  constexpr int NTW = M::ntiles(W) > 0 ? M::ntiles(W) : 1;
  double wt[NTW][2];
#pragma unroll
  for (int d = 0; d < T; ++d)
    if (M::owner(d) == W)
#pragma unroll
      for (int J = 0; J < T - d; ++J)
#pragma unroll
        for (int v = 0; v < 2; ++v) wt[M::slot(W, d, J)][v] = qval(i0 + 8 * (J + d) + rr, i0 + 8 * J + c2 + v);
  ix fail = n;
#pragma unroll 1
  for (ix g = i0; g < e; g += 8) {
    if (M::owner(0) == W) {  // (A) diagonal tile
      double* D = wt[M::slot(W, 0, 0)];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const double dpp = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * p + (p >> 1));
        if (lane == 0 && g + p >= s && g + p < n && !(dpp > kPivotFloor)) fail = fail < g + p ? fail : g + p;
        const double ri = rsqrt(dpp), piv = dpp * ri;  // one MUFU sequence on the chain (see k_chol_dmma)
        if (lane == 0) sm.rinv[p] = ri;
        if (q == (p >> 1)) {
          if (rr > p) D[p & 1] *= ri;
          else if (rr == p) D[p & 1] = piv;
        }
        const double lr = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * rr + (p >> 1));
        const double lc0 = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * c2 + (p >> 1));
        const double lc1 = __shfl_sync(0xffffffffu, pick(D, p & 1), 4 * (c2 + 1) + (p >> 1));
        if (c2 > p && rr >= c2) D[0] = fma(-lr, lc0, D[0]);
        if (c2 + 1 > p && rr >= c2 + 1) D[1] = fma(-lr, lc1, D[1]);
      }
      if (c2 > rr) D[0] = 0.0;
      if (c2 + 1 > rr) D[1] = 0.0;
      sm.l00[rr][c2] = D[0];
      sm.l00[rr][c2 + 1] = D[1];
      store_l(g, 0, D);
    }
    __syncthreads();
    // (B) panel tiles (d, 0), d >= 1: X = W L00^-T; publish MMA fragments
#pragma unroll
    for (int d = 1; d < T; ++d)
      if (M::owner(d) == W) {
        double* X = wt[M::slot(W, d, 0)];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (q == (c >> 1)) X[c & 1] *= sm.rinv[c];
          const double x = __shfl_sync(0xffffffffu, pick(X, c & 1), 4 * rr + (c >> 1));
          if (c2 > c) X[0] = fma(-x, sm.l00[c2][c], X[0]);
          if (c2 + 1 > c) X[1] = fma(-x, sm.l00[c2 + 1][c], X[1]);
        }
        store_l(g, d, X);
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const int srcl = 4 * rr + 2 * kc + (q >> 1);
          const double e0 = __shfl_sync(0xffffffffu, X[0], srcl);
          const double e1 = __shfl_sync(0xffffffffu, X[1], srcl);
          sm.pf[d][kc][lane] = (q & 1) ? e1 : e0;
        }
      }
    __syncthreads();
    // (C) trailing update of this warp's tiles, (D) shift and the fresh row
    const ix g2 = g + 8;
#pragma unroll
    for (int d = 0; d < T; ++d)
      if (M::owner(d) == W) {
#pragma unroll
        for (int J = 1; J < T - d; ++J) {
          double* t = wt[M::slot(W, d, J)];
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) dmma(t[0], t[1], -sm.pf[J + d][kc][lane], sm.pf[J][kc][lane]);
        }
#pragma unroll
        for (int J = 1; J < T - d; ++J) {
          wt[M::slot(W, d, J - 1)][0] = wt[M::slot(W, d, J)][0];
          wt[M::slot(W, d, J - 1)][1] = wt[M::slot(W, d, J)][1];
        }
#pragma unroll
        for (int v = 0; v < 2; ++v)
          wt[M::slot(W, d, T - 1 - d)][v] = qval(g2 + 8 * (T - 1) + rr, g2 + 8 * (T - 1 - d) + c2 + v);
      }
  }
  if (lane == 0 && fail < n)
    atomicMin(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(fail));
}

template <int K, int NW, int W>
__device__ __forceinline__ void chol_mw_dispatch(int w, const CholP<double>& C, ix b, ix n, ix s, ix e, ix i0,
                                                 double* side, MWSmem<K, NW>& sm) {
  if (w == W) chol_mw_unit<K, NW, W>(C, b, n, s, e, i0, side, sm);
  if constexpr (W + 1 < NW) chol_mw_dispatch<K, NW, W + 1>(w, C, b, n, s, e, i0, side, sm);
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_chol_mw(CholP<double> C, Geo G) {
  __shared__ MWSmem<K, NW> sm;
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix i0 = s - G.burn;
  if (i0 < 0) i0 = 0;
  i0 -= i0 % 8;
  chol_mw_dispatch<K, NW, 0>(threadIdx.x >> 5, C, b, G.n, s, e, i0,
                             p > 0 ? C.side + unit * ix(K) * (K + 1) : nullptr, sm);
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_chol_mw_repair(CholP<double> C, Geo G) {
  __shared__ MWSmem<K, NW> sm;
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  if (threadIdx.x == 0) C.fail[b] = G.n;
  __syncthreads();
  chol_mw_dispatch<K, NW, 0>(threadIdx.x >> 5, C, b, G.n, 0, G.n, 0, nullptr, sm);
}

__global__ void __launch_bounds__(32) k_chol_dmma(CholP<double> C, Geo G) {
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix i0 = s - G.burn;
  if (i0 < 0) i0 = 0;
  i0 -= i0 % 8;
  chol_dmma_unit(C, b, G.n, s, e, i0, p > 0 ? C.side + unit * ix(kDK) * (kDK + 1) : nullptr);
}

__global__ void __launch_bounds__(32) k_chol_dmma_repair(CholP<double> C, Geo G) {
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  if (threadIdx.x == 0) C.fail[b] = G.n;
  __syncwarp();
  chol_dmma_unit(C, b, G.n, 0, G.n, 0, nullptr);
}

// ------------------------------------------------------------------ subset, FP64 DMMA
// Blocked Takahashi recursion on the FP64 tensor cores, one warp per
// (matrix, segment), panels of 8 columns from the bottom up.  With the panel
// P = rows [p, p+8) and the trailing window T = the K rows below it,
// Z L = L^-T gives (block form of the column recursion in bgm_narrow.cu)
//   Z_TP = -(Z_TT L_TP) L_PP^-1,   Z_PP = (L_PP^-1 - L_TP^T Z_TP)^T L_PP^-1 .
// Z_TT lives in shared memory as 8x8 tiles, each tile diagonal d = B1 - B2 a
// ring indexed by block mod (K/8 - d), so the window slides with no copies:
// the panel's new tiles overwrite the tiles of the block leaving the window.
// Per panel: L_PP^-1 by shuffles; Y = Z_TT L_TP ((K/8)^2 x 2 DMMA);
// Z_TP = -Y L_PP^-1; H = L_TP^T Z_TP; Z_PP = (L_PP^-1 - H)^T L_PP^-1 -- all
// DMMA with operands read from padded (conflict-free) shared tiles.
template <int K>
struct TakSmem {
  static constexpr int NT = K / 8;
  static constexpr int NZ = NT * (NT + 1) / 2;
  double z[NZ][8][9];
  double lp[2][K + 8][9];
  double y[NT][8][9];
  double linv[8][9];
  double h[8][9];
};

template <int K>
__device__ __forceinline__ int tak_slot(int d, ix b2) {
  constexpr int NT = K / 8;
  return d * NT - d * (d - 1) / 2 + int(b2 % (NT - d));
}

template <int K>
__device__ void subset_dmma_unit(const SubP<double>& C, ix b, ix n, ix s, ix e, ix jend, double* side,
                                 TakSmem<K>& sm) {
  constexpr int NT = K / 8;
  const int lane = threadIdx.x & 31, rr = lane >> 2, q = lane & 3, c2 = 2 * q;
  const Band<double>& L = C.l;
  const Band<double>& S = C.s;
  const ix pb_top = (jend - 1) / 8, pb_end = s / 8;
  const bool exact_top = 8 * (pb_top + 1) >= n;  // window below the top panel is all padding
  // Z window for the top panel: identity on padded rows, else zero (burn-in)
  for (int idx = lane; idx < TakSmem<K>::NZ * 64; idx += 32) {
    const int t = idx >> 6, m = (idx >> 3) & 7, c = idx & 7;
    double v = 0.0;
    if (exact_top && t < NT && m == c) {  // diagonal ring d = 0 occupies slots [0, NT)
      v = 1.0;
    }
    sm.z[t][m][c] = v;
  }
  auto fill = [&](int buf, ix pb) {  // L rows [8pb, 8pb+K+8) x cols [8pb, 8pb+8), identity past n
    const ix c0 = 8 * pb;
    for (int idx = lane; idx < 8 * (K + 8); idx += 32) {
      const int c = idx / (K + 8), r = idx % (K + 8);
      double* dst = &sm.lp[buf][r][c];
      const ix col = c0 + c, row = c0 + r;
      const int cell = r - c;
      if (pb >= 0 && cell >= 0 && cell <= K && col < n && row < n) cpa(dst, &L.cell(b, cell, col));
      else *dst = (cell == 0 && col >= n) ? 1.0 : 0.0;
    }
    cpa_commit();
  };
  fill(0, pb_top);
  int buf = 0;
#pragma unroll 1
  for (ix pb = pb_top; pb >= pb_end; --pb) {
    cpa_wait0();
    __syncwarp();
    if (pb - 1 >= pb_end) fill(buf ^ 1, pb - 1);
    double (*lp)[9] = sm.lp[buf];
    // (1) Linv = L_PP^-1 by forward substitution in the fragment layout
    {
      double M0 = rr == c2 ? 1.0 : 0.0, M1 = rr == c2 + 1 ? 1.0 : 0.0;
      const double rme = 1.0 / lp[rr][rr];  // off the 8-step chain (see k_vsub_dmma)
      double lr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) lr[k] = rr > k ? lp[rr][k] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (rr == k) {
          M0 *= rme;
          M1 *= rme;
        }
        const double mk0 = __shfl_sync(0xffffffffu, M0, 4 * k + q);
        const double mk1 = __shfl_sync(0xffffffffu, M1, 4 * k + q);
        if (rr > k) {
          M0 = fma(-lr[k], mk0, M0);
          M1 = fma(-lr[k], mk1, M1);
        }
      }
      sm.linv[rr][c2] = M0;
      sm.linv[rr][c2 + 1] = M1;
    }
    // (2) Y_t = sum_u Z[t][u] L_TP[u]  (window blocks pb+1+t, pb+1+u)
    double yacc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      yacc[t][0] = yacc[t][1] = 0.0;
#pragma unroll
      for (int u = 0; u < NT; ++u) {
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          double a;
          if (t >= u) a = sm.z[tak_slot<K>(t - u, pb + 1 + u)][rr][4 * kc + q];
          else a = sm.z[tak_slot<K>(u - t, pb + 1 + t)][4 * kc + q][rr];
          const double bv = lp[8 + 8 * u + 4 * kc + q][rr];
          dmma(yacc[t][0], yacc[t][1], a, bv);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      sm.y[t][rr][c2] = yacc[t][0];
      sm.y[t][rr][c2 + 1] = yacc[t][1];
    }
    __syncwarp();
    // (3) Z_TP[t] = -Y_t Linv: new tiles (pb+1+t, pb) on diagonal t+1
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) dmma(z0, z1, -sm.y[t][rr][4 * kc + q], sm.linv[4 * kc + q][rr]);
      yacc[t][0] = z0;
      yacc[t][1] = z1;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      sm.y[t][rr][c2] = yacc[t][0];
      sm.y[t][rr][c2 + 1] = yacc[t][1];
      if (t + 1 < NT) {
        double (*zt)[9] = sm.z[tak_slot<K>(t + 1, pb)];
        zt[rr][c2] = yacc[t][0];
        zt[rr][c2 + 1] = yacc[t][1];
      }
    }
    __syncwarp();
    // (4) H = L_TP^T Z_TP; h = Linv - H
    {
      double h0 = 0.0, h1 = 0.0;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int kc = 0; kc < 2; ++kc)
          dmma(h0, h1, lp[8 + 8 * t + 4 * kc + q][rr], sm.y[t][4 * kc + q][rr]);
      sm.h[rr][c2] = sm.linv[rr][c2] - h0;
      sm.h[rr][c2 + 1] = sm.linv[rr][c2 + 1] - h1;
    }
    __syncwarp();
    // (5) Z_PP = h^T Linv -> tile (pb, pb) on diagonal 0
    double zp0 = 0.0, zp1 = 0.0;
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) dmma(zp0, zp1, sm.h[4 * kc + q][rr], sm.linv[4 * kc + q][rr]);
    {
      double (*zt)[9] = sm.z[tak_slot<K>(0, pb)];
      zt[rr][c2] = zp0;
      zt[rr][c2 + 1] = zp1;
    }
    // (6) S columns 8pb + c2 + v: rows from Z_PP and Z_TP
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const ix col = 8 * pb + c2 + v;
      const bool own = col >= s && col < e && col < n;
      const bool burn = side && col >= e && col < e + K && col < n;
      if (own || burn) {
        auto put = [&](int cell, double val) {
          if (cell < 0 || cell > K) return;
          const double w = (col + cell < n) ? val : 0.0;
          if (own) S.cell(b, cell, col) = w;
          else side[(col - e) * (K + 1) + cell] = w;
        };
        put(rr - c2 - v, v ? zp1 : zp0);
#pragma unroll
        for (int t = 0; t < NT; ++t) put(8 + 8 * t + rr - c2 - v, yacc[t][v]);
      }
    }
    __syncwarp();
    buf ^= 1;
  }
  cpa_wait0();
}

template <int K>
__global__ void __launch_bounds__(32) k_subset_dmma(SubP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TakSmem<K>& sm = *reinterpret_cast<TakSmem<K>*>(smraw);
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix jend = e + G.burn < G.n ? e + G.burn : G.n;  // rows [s, jend) swept, top one first
  subset_dmma_unit<K>(C, b, G.n, s, e, jend, p + 1 < G.nseg ? C.side + unit * ix(K) * (K + 1) : nullptr, sm);
}

template <int K>
__global__ void __launch_bounds__(32) k_subset_dmma_repair(SubP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TakSmem<K>& sm = *reinterpret_cast<TakSmem<K>*>(smraw);
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  subset_dmma_unit<K>(C, b, G.n, 0, G.n, G.n, nullptr, sm);
}

// ------------------------------------------------------------------ vjp_subset, FP64 DMMA
// Reverse of the blocked Takahashi recursion (see k_subset_dmma), panels of
// 8 columns from the top down, one CTA of NW warps per (matrix, segment).
// Per panel P with trailing window T (K rows), from the stored band of Z = S:
//   Linv = L_PP^-1   Y = Z_TT L_TP   Z_TP = -Y Linv   A = Linv - L_TP^T Z_TP
// and, with W the adjoint window (symmetric split of S-bar plus what the
// panels above pushed down):
//   Zb_TP = 2 W(T,P)  Zb_PP = W(P,P)
//   Ab = Linv Zb_PP^T   Linvb = A Zb_PP + Ab   Hb = -Ab
//   Ltpb = Z_TP Hb^T + Z_TT Yb   Zb_TP += L_TP Hb   Yb = -Zb_TP Linv^T
//   Linvb -= Y^T Zb_TP   W(T,T) += (Yb L_TP^T + L_TP Yb^T) / 2
//   Lppb = -Linv^T Linvb Linv^T (lower)
// L-bar(P,P) = Lppb, L-bar(T,P) = Ltpb: each band cell of L belongs to one
// panel.  Every product is a pair of m8n8k4 DMMA on 8x8 tiles in shared
// memory, stored row-major with the column XOR-swizzled by bit 1 of the row
// (conflict-free fragment reads in both orientations and 16-byte fragment
// stores).  Z and W live in per-diagonal rings of tiles; the block row
// entering at the bottom is fetched with cp.async a panel ahead.  Warps own
// the tile rows t = warp (mod NW); the 8x8 panel algebra is done redundantly
// per warp.  Checked against the scalar recursion (grad.cpp:84-143) by the
// parity tests.
__device__ __forceinline__ int sw8(int r, int c) { return r * 8 + (c ^ ((r & 2) << 1)); }

// x mod m for m <= 64 by a multiply-high with M = floor((2^32 - 1) / m) + 1
// (exact for x < 2^26: the error x (M - 2^32/m) / 2^32 stays below 1/m)
__device__ __forceinline__ unsigned mod_small(unsigned x, unsigned m, unsigned magic) {
  return x - __umulhi(x, magic) * m;
}

template <int K>
__device__ __forceinline__ int ring_slot(int d, ix b2, const unsigned* mg) {  // diagonal d holds NT+1-d tiles
  constexpr int NT = K / 8;
  const unsigned m = unsigned(NT + 1 - d);
  const int base = d * (NT + 1) - d * (d - 1) / 2;
  return m == 1 ? base : base + int(mod_small(unsigned(b2), m, mg[m]));
}

// per-matrix base of a band: cell (r, j) at p[(j w + r) << s]
struct BRow {
  double* p;
  int w, s;
  __device__ __forceinline__ double* at(int r, ix j) const { return p + ((j * w + r) << s); }
};
__device__ __forceinline__ BRow brow(const Band<double>& X, ix b) { return BRow{&X.cell(b, 0, 0), X.w, X.s}; }

// Calls f(integral_constant<int, w>) for the CTA's warp w, so a unit can resolve its warp-dependent
// indices (tile rows, transposition of a tile read, table offsets) at compile time.  NOT used by the
// kernels below: measured on the B200, eight warp-specialised copies of the subset / adjoint loops
// (WI >= 0) thrash the instruction cache -- k = 128 subset 6.3 -> 20.5 ms, adjoint 17.1 -> 66 ms,
// vjp_cholesky 7.7 -> 11.8 ms -- although each copy has ~half the instructions.  The runtime-warp
// version (WI = -1) stays; its ~10-14 instructions per DMMA (IMAD / LEA / ISETP / FSEL index math)
// are the price of one shared loop body.
template <int NW, int WI = 0, class F>
__device__ __forceinline__ void warp_dispatch(int w, F&& f) {
  if (w == WI) f(std::integral_constant<int, WI>{});
  if constexpr (WI + 1 < NW) warp_dispatch<NW, WI + 1>(w, f);
}

// L_PP^-1 in the MMA accumulator layout by forward substitution on the identity: lane (rr, q) holds
// columns 2q, 2q+1 of row rr.  The 8 steps are separate calls so a caller can interleave them with
// independent DMMAs (the shuffles' latency then hides behind the tensor pipe).
struct LinvChain {
  double M0, M1, rme, lr[8];
  int rr, q;
  __device__ __forceinline__ void init(const double* lp, int rr_, int q_) {
    rr = rr_;
    q = q_;
    M0 = rr == 2 * q ? 1.0 : 0.0;
    M1 = rr == 2 * q + 1 ? 1.0 : 0.0;
    rme = 1.0 / lp[sw8(rr, rr)];
#pragma unroll
    for (int k = 0; k < 8; ++k) lr[k] = rr > k ? lp[sw8(rr, k)] : 0.0;
  }
  __device__ __forceinline__ void step(int k) {
    if (rr == k) {
      M0 *= rme;
      M1 *= rme;
    }
    const double mk0 = __shfl_sync(0xffffffffu, M0, 4 * k + q);
    const double mk1 = __shfl_sync(0xffffffffu, M1, 4 * k + q);
    if (rr > k) {
      M0 = fma(-lr[k], mk0, M0);
      M1 = fma(-lr[k], mk1, M1);
    }
  }
};

template <int K, int NW>
struct VtSmem {
  static constexpr int NT = K / 8;
  static constexpr int NZ = NT * (NT + 3) / 2;         // Z rings, diagonals 0 .. NT-1
  static constexpr int NWT = (NT + 1) * (NT + 2) / 2;  // W rings, diagonals 0 .. NT
  double z[NZ][64];
  double w[NWT][64];
  double lp[2][(K + 8) * 8];
  double y[NT][64], zt[NT][64], yb[NT][64], gb[NT][64];
  double lin[NW][64], am[NW][64], ab[NW][64], part[NW][64], ph[NW][64], hm[64];
  int zs[NT * NT];               // element offset of Z_TT tile (t, u) in z (lower-stored)
  int ws[(NT + 1) * (NT + 1)];   // element offset of W tile (t1, t2) in w, window of the panel
  unsigned mg[NT + 2];           // mod_small multipliers
};

template <int K, int NW, int WI = -1>  // WI >= 0: the warp index as a compile-time constant
__device__ void vsub_dmma_unit(const VsP<double>& C, ix b, ix n, ix s, ix e, ix i0, double* side, double* tail,
                               VtSmem<K, NW>& sm) {
  constexpr int NT = K / 8, NTH = 32 * NW, TPW = NT / NW, NWT = VtSmem<K, NW>::NWT;
  static_assert(NT % NW == 0, "warps must divide the tile rows");
  const int tid = threadIdx.x, warp = WI >= 0 ? WI : tid >> 5, lane = tid & 31, rr = lane >> 2, q = lane & 3,
            c2 = 2 * q;
  const int o0[2] = {sw8(rr, q), sw8(rr, 4 + q)}, o1[2] = {sw8(q, rr), sw8(4 + q, rr)};
  const int oc = sw8(rr, c2);
  const Band<double>& L = C.l;
  auto mm = [&](double* acc, const double* X, bool tx, const double* Y, bool ty) {
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) dmma(acc[0], acc[1], X[tx ? o1[kc] : o0[kc]], Y[ty ? o0[kc] : o1[kc]]);
  };
  auto put = [&](double* T, double v0, double v1) { *reinterpret_cast<double2*>(T + oc) = make_double2(v0, v1); };
  auto get = [&](const double* T) { return *reinterpret_cast<const double2*>(T + oc); };
  // element (m, c) of window tile (b1, b2) of the symmetric band X: cp.async of
  // the lower-stored cell (a diagonal tile's upper half reads the mirror);
  // rows past n are identity (Z) or zero (S-bar).  W is kept as W2 = 2 W off
  // the matrix diagonal, so S-bar's cells load raw; its diagonal carries
  // S-bar_ii + 2 (pushed-down part), corrected where Zb_PP is formed.
  const BRow zrow = brow(C.s, b), grow = brow(C.sb, b), lrow = brow(L, b), orow = brow(C.lb, b);
  auto elem = [&](double* T, const BRow& X, bool ident, ix b1, ix b2, int idx) {
    const int m = idx >> 3, c = idx & 7;
    double* dst = T + sw8(m, c);
    ix r = 8 * b1 + m, cc = 8 * b2 + c;
    if (r < cc) {
      const ix t = r;
      r = cc;
      cc = t;
    }
    const int cell = int(r - cc);
    if (r < n && cell <= K) cpa(dst, X.at(cell, cc));
    else *dst = (ident && cell == 0) ? 1.0 : 0.0;
  };
  // block row bn entering a ring (tiles (bn, bn-d), d < ntile) into the slots
  // tab[d (NT+1)] / 64 of the current panel; each thread owns the element
  // (em, ec) of tiles et, et + NTH/64, ...  (NTH is a multiple of 64)
  static_assert(NTH % 64 == 0, "block size");
  const int em = tid & 7, ec = (tid & 63) >> 3, et = tid >> 6;  // lanes run down a column: 64-byte source runs
  auto row_issue = [&](double* ring, const BRow& X, bool ident, ix bn, int ntile) {
    const double* rowp = X.p + ((8 * bn * X.w) << X.s);
#pragma unroll
    for (int i = 0; i < (NT + 1 + NTH / 64 - 1) / (NTH / 64); ++i) {
      const int d = et + (NTH / 64) * i;
      if (d < ntile) {
        double* dst = ring + sm.ws[d * (NT + 1)] + sw8(em, ec);
        const bool mir = d == 0 && em < ec;
        const int cell = mir ? ec - em : 8 * d + em - ec;
        const int off = mir ? em * X.w + cell : (ec - 8 * d) * X.w + cell;
        if (8 * bn + (mir ? ec : em) < n && cell <= K) cpa(dst, rowp + (ix(off) << X.s));
        else *dst = (ident && cell == 0) ? 1.0 : 0.0;
      }
    }
  };
  auto w_init = [&](ix pb) {  // W blocks pb .. pb+NT
    for (int x = tid; x < NWT * 64; x += NTH) {
      int j = x >> 6, d = 0;
      while (j > NT - d) j -= NT + 1 - d++;
      elem(sm.w[ring_slot<K>(d, pb + j, sm.mg)], grow, false, pb + j + d, pb + j, x & 63);
    }
  };
  // L rows [8pb, 8pb+K+8) x cols [8pb, 8pb+8), identity past n
  auto fill = [&](int buf, ix pb) {  // a warp copies whole columns, lanes consecutive rows (coalesced)
#pragma unroll
    for (int c = warp; c < 8; c += NW) {
      const double* colp = lrow.at(0, 8 * pb + c);
#pragma unroll
      for (int i = 0; i < (K + 8 + 31) / 32; ++i) {
        const int r = lane + 32 * i, cell = r - c;
        if (r < K + 8) {
          double* dst = sm.lp[buf] + sw8(r, c);
          if (cell >= 0 && cell <= K && 8 * pb + r < n) cpa(dst, colp + (ix(cell) << lrow.s));
          else *dst = (cell == 0) ? 1.0 : 0.0;
        }
      }
    }
  };
  auto save_w = [&](double* dst, ix pb) {  // window of panel pb, tiles in (d, j) order
    for (int x = tid; x < NWT * 64; x += NTH) {
      int j = x >> 6, d = 0;
      while (j > NT - d) j -= NT + 1 - d++;
      dst[x] = sm.w[ring_slot<K>(d, pb + j, sm.mg)][x & 63];
    }
  };
  const ix pb0 = i0 / 8, pbe = (e + 7) / 8;
  for (int x = tid; x < NT + 2; x += NTH) sm.mg[x] = x ? 0xFFFFFFFFu / unsigned(x) + 1u : 0u;
  __syncthreads();
  for (int x = tid; x < NT * NT * 64; x += NTH) {  // Z blocks pb0+1 .. pb0+NT (lower tiles)
    const int t1 = x / (NT * 64), t2 = (x >> 6) % NT;
    if (t2 <= t1) elem(sm.z[ring_slot<K>(t1 - t2, pb0 + 1 + t2, sm.mg)], zrow, true, pb0 + 1 + t1, pb0 + 1 + t2, x & 63);
  }
  w_init(pb0);
  fill(0, pb0);
  cpa_commit();
  int buf = 0;
#pragma unroll 1
  for (ix pb = pb0; pb < pbe; ++pb) {
    cpa_wait0();
    for (int x = tid; x < NT * NT; x += NTH) {
      const int t = x / NT, u = x % NT;
      sm.zs[x] = ring_slot<K>(t > u ? t - u : u - t, pb + 1 + (t < u ? t : u), sm.mg) * 64;
    }
    for (int x = tid; x < (NT + 1) * (NT + 1); x += NTH) {
      const int t1 = x / (NT + 1), t2 = x % (NT + 1);
      if (t1 >= t2) sm.ws[x] = ring_slot<K>(t1 - t2, pb + t2, sm.mg) * 64;
    }
    __syncthreads();
    if (side && pb == s / 8) save_w(side, pb);  // burn-in state at the segment start
    row_issue(&sm.z[0][0], zrow, true, pb + NT + 1, NT);  // into the ring slots block pb has left
    const double dl0 = 8 * pb + c2 < n ? *grow.at(0, 8 * pb + c2) : 0.0;  // S-bar_ii of the panel
    const double dl1 = 8 * pb + c2 + 1 < n ? *grow.at(0, 8 * pb + c2 + 1) : 0.0;
    if (pb + 1 < pbe) fill(buf ^ 1, pb + 1);
    cpa_commit();
    const double* lp = sm.lp[buf];
    double* lin = sm.lin[warp];
    // ---- (1) Linv (per warp) and everything that does not need Y = Z_TT L_TP:
    //          Ab = Linv Zb_PP^T, G = L_TP Ab - W2(T,P) (= -Zb_TP), Yb = G Linv^T for the warp's tile rows.
    //          With Yb known first, ONE pass over the Z_TT tiles serves both big products (2): each
    //          tile's fragments are read from shared memory once instead of twice -- these kernels
    //          are bound by shared-memory bandwidth (a DMMA whose two operands come from shared memory
    //          needs 4 wavefronts per 17 clk and pipe: 93% of the bandwidth at the full tensor rate).
    {
      LinvChain ch;
      ch.init(lp, rr, q);
#pragma unroll
      for (int k = 0; k < 8; ++k) ch.step(k);
      put(lin, ch.M0, ch.M1);
      __syncwarp();
    }
    const double* wpp = &sm.w[0][0] + sm.ws[0];  // Zb_PP = (W2_PP + diag(S-bar_ii)) / 2
    {
      const double2 l2 = get(lin);
      double a[2] = {0.0, 0.0};
      mm(a, lin, false, wpp, true);
      a[0] = 0.5 * fma(l2.x, dl0, a[0]);
      a[1] = 0.5 * fma(l2.y, dl1, a[1]);
      put(sm.ab[warp], a[0], a[1]);
      if (warp == NW - 1) {  // W2_PP for the panel algebra at the end: its ring slot is refilled below
        const double2 w2 = get(wpp);
        put(sm.am[warp], w2.x, w2.y);
      }
      __syncwarp();
      double g[TPW][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        const double2 w2 = get(&sm.w[0][0] + sm.ws[(t + 1) * (NT + 1)]);
        g[i][0] = -w2.x;
        g[i][1] = -w2.y;
        mm(g[i], lp + (8 + 8 * t) * 8, false, sm.ab[warp], false);
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i) put(sm.gb[warp + NW * i], g[i][0], g[i][1]);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        g[i][0] = g[i][1] = 0.0;
        mm(g[i], sm.gb[warp + NW * i], false, lin, true);
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i) put(sm.yb[warp + NW * i], g[i][0], g[i][1]);
    }
    __syncthreads();
    // W block row pb+NT+1 enters the slots of column pb (read for the last time above)
    row_issue(&sm.w[0][0], grow, false, pb + NT + 1, NT + 1);
    cpa_commit();
    // ---- (2) Y = Z_TT L_TP and Q = Z_TT Yb in one pass (tile column outer), then Z_TP = -Y Linv,
    //          L-bar(T,P) = Q - Z_TP Ab^T, and the partial sums L_TP^T Z_TP (for A) and Y^T G (for Linvb)
    {
      double ya[TPW][2][2], qa[TPW][2][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        ya[i][0][0] = ya[i][0][1] = ya[i][1][0] = ya[i][1][1] = 0.0;
        qa[i][0][0] = qa[i][0][1] = qa[i][1][0] = qa[i][1][1] = 0.0;
      }
#pragma unroll
      for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int t = warp + NW * i;
          const double* zt = &sm.z[0][0] + sm.zs[t * NT + u];
          const double* y1 = lp + (8 + 8 * u) * 8;
          const double* y2 = sm.yb[u];
#pragma unroll
          for (int kc = 0; kc < 2; ++kc) {  // the tile's fragment is read once for both products
            const double xa = zt[t < u ? o1[kc] : o0[kc]];
            dmma(ya[i][u & 1][0], ya[i][u & 1][1], xa, y1[o1[kc]]);
            dmma(qa[i][u & 1][0], qa[i][u & 1][1], xa, y2[o1[kc]]);
          }
        }
#pragma unroll
      for (int i = 0; i < TPW; ++i) put(sm.y[warp + NW * i], ya[i][0][0] + ya[i][1][0], ya[i][0][1] + ya[i][1][1]);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        ya[i][0][0] = ya[i][0][1] = 0.0;
        mm(ya[i][0], sm.y[warp + NW * i], false, lin, false);
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i) put(sm.zt[warp + NW * i], -ya[i][0][0], -ya[i][0][1]);
      __syncwarp();
      double h[2] = {0.0, 0.0}, pa[2] = {0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        mm(h, lp + (8 + 8 * t) * 8, true, sm.zt[t], false);
        mm(pa, sm.y[t], true, sm.gb[t], false);
      }
      put(sm.ph[warp], h[0], h[1]);
      put(sm.part[warp], pa[0], pa[1]);
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        double la[2] = {0.0, 0.0};
        mm(la, sm.zt[t], false, sm.ab[warp], true);
        const double acc[2] = {qa[i][0][0] + qa[i][1][0] - la[0], qa[i][0][1] + qa[i][1][1] - la[1]};
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const ix col = 8 * pb + c2 + v;
          const int cell = 8 + 8 * t + rr - c2 - v;
          if (col >= s && col < e && cell <= K) *orow.at(cell, col) = (col + cell < n) ? acc[v] : 0.0;
        }
      }
    }
    // W2(T,T) += Yb L_TP^T + L_TP Yb^T: tile rows pp and NT-1-pp together (NT+1 tiles)
#pragma unroll 1
    for (int pp = warp; pp < NT / 2; pp += NW) {
      double wa[NT + 1][2];
#pragma unroll
      for (int j = 0; j <= NT; ++j) {
        const int t1 = j <= pp ? pp : NT - 1 - pp, t2 = j <= pp ? j : j - pp - 1;
        const double2 w2 = get(&sm.w[0][0] + sm.ws[(t1 + 1) * (NT + 1) + t2 + 1]);
        wa[j][0] = w2.x;
        wa[j][1] = w2.y;
        mm(wa[j], sm.yb[t1], false, lp + (8 + 8 * t2) * 8, true);
        mm(wa[j], lp + (8 + 8 * t1) * 8, false, sm.yb[t2], true);
      }
#pragma unroll
      for (int j = 0; j <= NT; ++j) {
        const int t1 = j <= pp ? pp : NT - 1 - pp, t2 = j <= pp ? j : j - pp - 1;
        put(&sm.w[0][0] + sm.ws[(t1 + 1) * (NT + 1) + t2 + 1], wa[j][0], wa[j][1]);
      }
    }
    __syncthreads();
    // ---- (3) the panel's own 8x8 algebra on the last warp: A = Linv - L_TP^T Z_TP,
    //          Linvb = A Zb_PP + Ab - Y^T Zb_TP, Lppb = -Linv^T (Linvb Linv^T)
    if (warp == NW - 1) {
      double h0 = 0.0, h1 = 0.0, p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) {
        const double2 hh = get(sm.ph[w2]);
        const double2 pp2 = get(sm.part[w2]);
        h0 += hh.x;
        h1 += hh.y;
        p0 += pp2.x;
        p1 += pp2.y;
      }
      const double2 l2 = get(lin);
      const double2 ab2 = get(sm.ab[warp]);
      const double am0 = l2.x - h0, am1 = l2.y - h1;
      put(sm.hm, am0, am1);
      __syncwarp();
      double v[2] = {0.0, 0.0};
      mm(v, sm.hm, false, sm.am[warp], false);  // A W2_PP (the copy taken in (1))
      v[0] = 0.5 * fma(am0, dl0, v[0]);
      v[1] = 0.5 * fma(am1, dl1, v[1]);
      __syncwarp();
      put(sm.hm, v[0] + ab2.x + p0, v[1] + ab2.y + p1);  // Linvb
      __syncwarp();
      double t2[2] = {0.0, 0.0};
      mm(t2, sm.hm, false, lin, true);
      __syncwarp();
      put(sm.hm, t2[0], t2[1]);
      __syncwarp();
      double p2[2] = {0.0, 0.0};
      mm(p2, lin, true, sm.hm, false);
#pragma unroll
      for (int v2 = 0; v2 < 2; ++v2) {
        const ix col = 8 * pb + c2 + v2;
        const int cell = rr - c2 - v2;
        if (col >= s && col < e && cell >= 0) *orow.at(cell, col) = (col + cell < n) ? -p2[v2] : 0.0;
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  cpa_wait0();
  __syncthreads();
  if (tail) save_w(tail, pbe);  // genuine state the next segment's burn-in must reproduce
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_vsub_dmma(VsP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  VtSmem<K, NW>& sm = *reinterpret_cast<VtSmem<K, NW>*>(smraw);
  constexpr int STATE = VtSmem<K, NW>::NWT * 64;
  if (G.span_rows > 0) {
    for (int k = 0; k < G.span_kmax; ++k) {
      ix b, s, e;
      if (!span_piece(G, blockIdx.x, k, b, s, e)) continue;  // uniform across the CTA
      ix i0 = s - G.burn;
      if (i0 < 0) i0 = 0;
      i0 -= i0 % 8;
      const ix slot = (ix(blockIdx.x) * G.span_kmax + k) * ix(STATE);
      vsub_dmma_unit<K, NW>(C, b, G.n, s, e, i0, s > 0 ? C.side + slot : nullptr, e < G.n ? C.tail + slot : nullptr,
                            sm);
      __syncthreads();  // the next piece reuses the shared windows
    }
    return;
  }
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  ix i0 = s - G.burn;
  if (i0 < 0) i0 = 0;
  i0 -= i0 % 8;
  vsub_dmma_unit<K, NW>(C, b, G.n, s, e, i0, p > 0 ? C.side + unit * ix(STATE) : nullptr,
                        p + 1 < G.nseg ? C.tail + unit * ix(STATE) : nullptr, sm);
}

template <int K, int NW>
__global__ void k_vsub_dmma_check(VsP<double> C, Geo G) {
  constexpr int STATE = VtSmem<K, NW>::NWT * 64;
  const ix id = (blockIdx.x * ix(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const double *a, *r;
  ix bflag;
  if (G.span_rows > 0) {  // id = CTA: its first piece, if it starts inside a matrix, against the
    ix b, s, e;           // last piece of the CTA before (same matrix)
    if (id < 1 || !span_piece(G, id, 0, b, s, e) || s == 0) return;
    const int kprev = int(b - ((id - 1) * G.span_rows) / G.n8);
    a = C.side + (id * G.span_kmax) * ix(STATE);
    r = C.tail + ((id - 1) * G.span_kmax + kprev) * ix(STATE);
    bflag = b;
  } else {
    if (id >= G.batch * G.nseg) return;
    const int p = int(id % G.nseg);
    if (p == 0) return;
    a = C.side + id * ix(STATE);
    r = C.tail + (id - 1) * ix(STATE);
    bflag = id / G.nseg;
  }
  double sc = 0.0;
  for (int i = lane; i < STATE; i += 32) sc = fmax(sc, fabs(r[i]));
#pragma unroll
  for (int o = 16; o; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
  bool bad = false;
  for (int i = lane; i < STATE; i += 32) bad |= !(fabs(a[i] - r[i]) <= kCheckTol * (sc + 1e-300));
  bad = __any_sync(0xffffffffu, bad);
  if (bad && lane == 0) C.flag[bflag] = 1;
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_vsub_dmma_repair(VsP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  VtSmem<K, NW>& sm = *reinterpret_cast<VtSmem<K, NW>*>(smraw);
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  vsub_dmma_unit<K, NW>(C, b, G.n, 0, G.n, 0, nullptr, nullptr, sm);
}

// ------------------------------------------------------------------ vjp_cholesky, FP64 DMMA
// Blocked reverse of the banded Cholesky (the scalar recursion is
// grad.cpp:20-36), panels of 8 columns from the bottom up.  With Abar the
// lower-stored adjoint of Q and G its symmetric split (G = (Abar + Abar^T)/2
// off the diagonal, Abar_ii on it), the forward panel step
//   L_PP = chol(A_PP)   L_TP = A_TP L_PP^-T   A_TT -= L_TP L_TP^T
// reverses to
//   Lb_TP = Lbar_TP - 2 G_TT L_TP        Abar_TP = Lb_TP L_PP^-1
//   Lb_PP = tril(Lbar_PP - Abar_TP^T L_TP)
//   S = L_PP^-T Phi(L_PP^T Lb_PP) L_PP^-1  (Phi: lower part, halved diagonal)
//   Abar_PP = tril(S + S^T) with diagonal S_ii, i.e. G_PP = (S + S^T) / 2,
// where G_TT holds only q-bar cells already produced by the panels below.
// One CTA of NW warps per (matrix, segment); warps own the tile rows
// t = warp (mod NW), the 8x8 panel algebra runs on the last warp.  G lives
// in diagonal rings of swizzled 8x8 tiles (see k_vsub_dmma); each panel
// writes its new tile column into slots no warp reads during the panel.
template <class T>
struct VdP {
  Band<T> l, lb, qb;
  T* side;  // [unit][NT(NT+1)/2][64] G window entering the segment's first panel (burn-in)
  T* tail;  // the same after the segment's last panel (genuine)
  int32_t* flag;
};

template <int K, int NW>
struct VdSmem {
  static constexpr int NT = K / 8;
  static constexpr int NZ = NT * (NT + 3) / 2;  // rings, diagonal d holds NT+1-d tiles
  double g[NZ][64];
  double lp[2][(K + 8) * 8];
  double lt[NT][64];
  double lin[NW][64], part[NW][64];
  double s1[64], s2[64];
  int zs[NT * NT];  // element offset of G_TT tile (t, u) in g (lower-stored)
  unsigned mg[NT + 2];
};

template <int K, int NW, int WI = -1>  // WI >= 0: the warp index as a compile-time constant
__device__ void vchol_dmma_unit(const VdP<double>& C, ix b, ix n, ix s, ix e, ix iend, double* side, double* tail,
                                VdSmem<K, NW>& sm) {
  constexpr int NT = K / 8, NTH = 32 * NW, TPW = NT / NW, NST = NT * (NT + 1) / 2;
  static_assert(NT % NW == 0, "warps must divide the tile rows");
  const int tid = threadIdx.x, warp = WI >= 0 ? WI : tid >> 5, lane = tid & 31, rr = lane >> 2, q = lane & 3,
            c2 = 2 * q;
  const int o0[2] = {sw8(rr, q), sw8(rr, 4 + q)}, o1[2] = {sw8(q, rr), sw8(4 + q, rr)};
  const int oc = sw8(rr, c2);
  const Band<double>& L = C.l;
  const BRow lrow = brow(L, b), brow_lb = brow(C.lb, b), brow_qb = brow(C.qb, b);
  auto mm = [&](double* acc, const double* X, bool tx, const double* Y, bool ty) {
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) dmma(acc[0], acc[1], X[tx ? o1[kc] : o0[kc]], Y[ty ? o0[kc] : o1[kc]]);
  };
  auto put = [&](double* Tt, double v0, double v1) { *reinterpret_cast<double2*>(Tt + oc) = make_double2(v0, v1); };
  // (kept as is: a division-free warp-per-column version of this copy measured 4% slower here)
  auto fill = [&](int buf, ix pb) {  // L rows [8pb, 8pb+K+8) x cols [8pb, 8pb+8), identity past n
    for (int x = tid; x < 8 * (K + 8); x += NTH) {
      const int c = x / (K + 8), r = x % (K + 8), cell = r - c;
      const ix col = 8 * pb + c, row = 8 * pb + r;
      double* dst = sm.lp[buf] + sw8(r, c);
      if (cell >= 0 && cell <= K && col < n && row < n) cpa(dst, lrow.at(cell, col));
      else *dst = (cell == 0) ? 1.0 : 0.0;
    }
  };
  // l-bar fragments of panel pb: rows 8pb+8+8t+rr (own t) and 8pb+rr, columns 8pb+c2+v
  auto load_lb = [&](ix pb, double (*ft)[2], double* fp) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const ix col = 8 * pb + c2 + v;
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int cell = 8 + 8 * (warp + NW * i) + rr - c2 - v;
        ft[i][v] = (pb >= 0 && cell <= K && col + cell < n) ? *brow_lb.at(cell, col) : 0.0;
      }
      const int cell = rr - c2 - v;
      fp[v] = (pb >= 0 && cell >= 0 && col + cell < n) ? *brow_lb.at(cell, col) : 0.0;
    }
  };
  auto save_g = [&](double* dst, ix b0) {  // window blocks b0 .. b0+NT-1, tiles in (d, j) order
    for (int x = tid; x < NST * 64; x += NTH) {
      int j = x >> 6, d = 0;
      while (j > NT - 1 - d) j -= NT - d++;
      dst[x] = sm.g[ring_slot<K>(d, b0 + j, sm.mg)][x & 63];
    }
  };
  const ix pb_top = (iend + 7) / 8 - 1, pb_end = s / 8;
  for (int x = tid; x < NT + 2; x += NTH) sm.mg[x] = x ? 0xFFFFFFFFu / unsigned(x) + 1u : 0u;
  __syncthreads();
  for (int x = tid; x < VdSmem<K, NW>::NZ * 64; x += NTH) (&sm.g[0][0])[x] = 0.0;
  fill(0, pb_top);
  cpa_commit();
  double lbt[TPW][2], lbp[2];
  load_lb(pb_top, lbt, lbp);
  int buf = 0;
#pragma unroll 1
  for (ix pb = pb_top; pb >= pb_end; --pb) {
    cpa_wait0();
    for (int x = tid; x < NT * NT; x += NTH) {
      const int t = x / NT, u = x % NT;
      sm.zs[x] = ring_slot<K>(t > u ? t - u : u - t, pb + 1 + (t < u ? t : u), sm.mg) * 64;
    }
    __syncthreads();
    if (side && 8 * (pb + 1) == e) save_g(side, pb + 1);  // burn-in state entering the segment
    if (pb > pb_end) fill(buf ^ 1, pb - 1);
    cpa_commit();
    double nbt[TPW][2], nbp[2];
    load_lb(pb > pb_end ? pb - 1 : -1, nbt, nbp);
    const double* lp = sm.lp[buf];
    double* lin = sm.lin[warp];
    // Linv (per warp), then Lb_TP = Lbar_TP - 2 G_TT L_TP (own tile rows).  (Interleaving the chain with
    // the products and running them tile-column outer, as the subset kernels do, was slower here:
    // 7.73 vs 7.14 ms at k = 128.)
    {
      double M0 = rr == c2 ? 1.0 : 0.0, M1 = rr == c2 + 1 ? 1.0 : 0.0;
      // this lane's row pivot reciprocal and row of L_PP, loaded / divided
      // up front: only the shuffles and FMAs stay on the 8-step chain
      const double rme = 1.0 / lp[sw8(rr, rr)];
      double lr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) lr[k] = rr > k ? lp[sw8(rr, k)] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (rr == k) {
          M0 *= rme;
          M1 *= rme;
        }
        const double mk0 = __shfl_sync(0xffffffffu, M0, 4 * k + q);
        const double mk1 = __shfl_sync(0xffffffffu, M1, 4 * k + q);
        if (rr > k) {
          M0 = fma(-lr[k], mk0, M0);
          M1 = fma(-lr[k], mk1, M1);
        }
      }
      put(lin, M0, M1);
    }
    {
      double ga[TPW][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        ga[i][0] = ga[i][1] = 0.0;
#pragma unroll
        for (int u = 0; u < NT; ++u) mm(ga[i], &sm.g[0][0] + sm.zs[t * NT + u], t < u, lp + (8 + 8 * u) * 8, false);
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i)
        put(sm.lt[warp + NW * i], fma(-2.0, ga[i][0], lbt[i][0]), fma(-2.0, ga[i][1], lbt[i][1]));
    }
    __syncwarp();
    // Abar_TP = Lb_TP Linv -> q-bar cells, G column (halved), and the partial Abar_TP^T L_TP
    {
      double aa[TPW][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        aa[i][0] = aa[i][1] = 0.0;
        mm(aa[i], sm.lt[warp + NW * i], false, lin, false);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        put(sm.lt[t], aa[i][0], aa[i][1]);
        if (t + 1 < NT) put(sm.g[ring_slot<K>(t + 1, pb, sm.mg)], 0.5 * aa[i][0], 0.5 * aa[i][1]);
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const ix col = 8 * pb + c2 + v;
          const int cell = 8 + 8 * t + rr - c2 - v;
          if (col >= s && col < e && cell <= K) *brow_qb.at(cell, col) = (col + cell < n) ? aa[i][v] : 0.0;
        }
      }
      __syncwarp();
      double pa[2] = {0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        mm(pa, sm.lt[t], true, lp + (8 + 8 * t) * 8, false);
      }
      put(sm.part[warp], pa[0], pa[1]);
    }
    __syncthreads();
    if (warp == NW - 1) {
      // Lb_PP = tril(Lbar_PP - sum of partials); X = L_PP^T Lb_PP; Phi
      double x0 = lbp[0], x1 = lbp[1];
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) {
        const double2 p2 = *reinterpret_cast<const double2*>(sm.part[w2] + oc);
        x0 -= p2.x;
        x1 -= p2.y;
      }
      put(sm.s1, c2 <= rr ? x0 : 0.0, c2 + 1 <= rr ? x1 : 0.0);
      __syncwarp();
      double xa[2] = {0.0, 0.0};
      mm(xa, lp, true, sm.s1, false);
      put(sm.s2, c2 < rr ? xa[0] : (c2 == rr ? 0.5 * xa[0] : 0.0),
          c2 + 1 < rr ? xa[1] : (c2 + 1 == rr ? 0.5 * xa[1] : 0.0));
      __syncwarp();
      double ya[2] = {0.0, 0.0};  // Phi Linv
      mm(ya, sm.s2, false, lin, false);
      put(sm.s1, ya[0], ya[1]);
      __syncwarp();
      double sa[2] = {0.0, 0.0};  // S = Linv^T (Phi Linv)
      mm(sa, lin, true, sm.s1, false);
      put(sm.s2, sa[0], sa[1]);
      __syncwarp();
      double gp[2];
#pragma unroll
      for (int v = 0; v < 2; ++v) gp[v] = 0.5 * (sa[v] + sm.s2[sw8(c2 + v, rr)]);
      put(sm.g[ring_slot<K>(0, pb, sm.mg)], gp[0], gp[1]);
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const ix col = 8 * pb + c2 + v;
        const int cell = rr - c2 - v;
        if (col >= s && col < e && cell >= 0)
          *brow_qb.at(cell, col) = (col + cell < n) ? (cell == 0 ? sa[v] : 2.0 * gp[v]) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      lbt[i][0] = nbt[i][0];
      lbt[i][1] = nbt[i][1];
    }
    lbp[0] = nbp[0];
    lbp[1] = nbp[1];
    buf ^= 1;
  }
  cpa_wait0();
  if (tail) save_g(tail, pb_end);  // genuine state leaving the segment's first column block
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_vchol_dmma(VdP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  VdSmem<K, NW>& sm = *reinterpret_cast<VdSmem<K, NW>*>(smraw);
  constexpr int NT = K / 8, STATE = NT * (NT + 1) / 2 * 64;
  if (G.span_rows > 0) {  // row spans (see Geo): the sweep runs upwards, so a piece that ENDS inside a
    for (int k = 0; k < G.span_kmax; ++k) {  // matrix burns in from below its end
      ix b, s, e;
      if (!span_piece(G, blockIdx.x, k, b, s, e)) continue;  // uniform across the CTA
      const ix iend = e + G.burn < G.n ? e + G.burn : G.n;
      const ix slot = (ix(blockIdx.x) * G.span_kmax + k) * ix(STATE);
      vchol_dmma_unit<K, NW>(C, b, G.n, s, e, iend, e < G.n ? C.side + slot : nullptr, s > 0 ? C.tail + slot : nullptr,
                             sm);
      __syncthreads();  // the next piece reuses the shared windows
    }
    return;
  }
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix iend = e + G.burn < G.n ? e + G.burn : G.n;
  vchol_dmma_unit<K, NW>(C, b, G.n, s, e, iend, p + 1 < G.nseg ? C.side + unit * ix(STATE) : nullptr,
                         p > 0 ? C.tail + unit * ix(STATE) : nullptr, sm);
}

template <int K, int NW>
__global__ void k_vchol_dmma_check(VdP<double> C, Geo G) {
  constexpr int NT = K / 8, STATE = NT * (NT + 1) / 2 * 64;
  const ix id = (blockIdx.x * ix(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const double *a, *r;
  ix bflag;
  if (G.span_rows > 0) {  // id = CTA whose first piece starts inside a matrix: its genuine state against
    ix b, s, e;           // the burn-in state of the previous CTA's last piece (same matrix)
    if (id < 1 || !span_piece(G, id, 0, b, s, e) || s == 0) return;
    const int kprev = int(b - ((id - 1) * G.span_rows) / G.n8);
    a = C.side + ((id - 1) * G.span_kmax + kprev) * ix(STATE);
    r = C.tail + (id * G.span_kmax) * ix(STATE);
    bflag = b;
  } else {
    if (id >= G.batch * G.nseg) return;
    const int p = int(id % G.nseg);
    if (p + 1 >= G.nseg) return;
    a = C.side + id * ix(STATE);
    r = C.tail + (id + 1) * ix(STATE);
    bflag = id / G.nseg;
  }
  double sc = 0.0;
  for (int i = lane; i < STATE; i += 32) sc = fmax(sc, fabs(r[i]));
#pragma unroll
  for (int o = 16; o; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
  bool bad = false;
  for (int i = lane; i < STATE; i += 32) bad |= !(fabs(a[i] - r[i]) <= kCheckTol * (sc + 1e-300));
  bad = __any_sync(0xffffffffu, bad);
  if (bad && lane == 0) C.flag[bflag] = 1;
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_vchol_dmma_repair(VdP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  VdSmem<K, NW>& sm = *reinterpret_cast<VdSmem<K, NW>*>(smraw);
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  vchol_dmma_unit<K, NW>(C, b, G.n, 0, G.n, G.n, nullptr, nullptr, sm);
}

// ------------------------------------------------------------------ subset, FP64 DMMA, multi-warp
// The blocked Takahashi recursion of k_subset_dmma on a CTA of NW warps with
// the machinery of k_vsub_dmma (swizzled tiles, rings holding NT+1-d tiles
// per diagonal, per-panel slot tables).  Warps own the tile rows
// t = warp (mod NW) of Y = Z_TT L_TP and Z_TP = -Y L_PP^-1 and their share of
// L_TP^T Z_TP; warp 0 then forms Z_PP while the other warps already start the
// next panel (its row 0 is the only consumer of Z_PP).  One barrier per
// panel: the slot tables, the partial sums and the L panel are double
// buffered, and each panel's new tiles go to slots no warp reads in it.
template <int K, int NW>
struct TakMwSmem {
  static constexpr int NT = K / 8;
  static constexpr int NZ = NT * (NT + 3) / 2;
  double z[NZ][64];
  double lp[2][(K + 8) * 8];
  double y[NT][64], zt[NT][64];
  double lin[NW][64], ph[2][NW][64], hm[64];
  int zs[2][NT * NT];
  unsigned mg[NT + 2];
};

template <int K, int NW, int WI = -1>  // WI >= 0: the warp index as a compile-time constant
__device__ void subset_mw_unit(const SubP<double>& C, ix b, ix n, ix s, ix e, ix jend, double* side,
                               TakMwSmem<K, NW>& sm) {
  constexpr int NT = K / 8, NTH = 32 * NW, TPW = NT / NW;
  static_assert(NT % NW == 0, "warps must divide the tile rows");
  const int tid = threadIdx.x, warp = WI >= 0 ? WI : tid >> 5, lane = tid & 31, rr = lane >> 2, q = lane & 3,
            c2 = 2 * q;
  const int o0[2] = {sw8(rr, q), sw8(rr, 4 + q)}, o1[2] = {sw8(q, rr), sw8(4 + q, rr)};
  const int oc = sw8(rr, c2);
  auto mm = [&](double* acc, const double* X, bool tx, const double* Y, bool ty) {
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) dmma(acc[0], acc[1], X[tx ? o1[kc] : o0[kc]], Y[ty ? o0[kc] : o1[kc]]);
  };
  auto put = [&](double* T, double v0, double v1) { *reinterpret_cast<double2*>(T + oc) = make_double2(v0, v1); };
  auto get = [&](const double* T) { return *reinterpret_cast<const double2*>(T + oc); };
  const BRow lrow = brow(C.l, b), srow = brow(C.s, b);
  const ix pb_top = (jend - 1) / 8, pb_end = s / 8;
  const bool exact_top = 8 * (pb_top + 1) >= n;  // window below the top panel is all padding
  for (int x = tid; x < NT + 2; x += NTH) sm.mg[x] = x ? 0xFFFFFFFFu / unsigned(x) + 1u : 0u;
  for (int x = tid; x < TakMwSmem<K, NW>::NZ * 64; x += NTH) {  // diagonal ring d = 0: slots [0, NT+1)
    const int t = x >> 6, m = (x >> 3) & 7, c = x & 7;
    (&sm.z[0][0])[x] = (exact_top && t <= NT && m == c) ? 1.0 : 0.0;
  }
  // L rows [8pb, 8pb+K+8) x cols [8pb, 8pb+8), identity past n: a warp copies whole columns, lanes
  // consecutive rows (coalesced)
  auto fill = [&](int buf, ix pb) {
#pragma unroll
    for (int c = warp; c < 8; c += NW) {
      const double* colp = lrow.at(0, 8 * pb + c);
#pragma unroll
      for (int i = 0; i < (K + 8 + 31) / 32; ++i) {
        const int r = lane + 32 * i, cell = r - c;
        if (r < K + 8) {
          double* dst = sm.lp[buf] + sw8(r, c);
          if (cell >= 0 && cell <= K && 8 * pb + r < n) cpa(dst, colp + (ix(cell) << lrow.s));
          else *dst = (cell == 0) ? 1.0 : 0.0;
        }
      }
    }
  };
  auto tables = [&](ix pb) {
    int* zs = sm.zs[pb & 1];
    for (int x = tid; x < NT * NT; x += NTH) {
      const int t = x / NT, u = x % NT;
      zs[x] = ring_slot<K>(t > u ? t - u : u - t, pb + 1 + (t < u ? t : u), sm.mg) * 64;
    }
  };
  // S cell (8pb + rr + rofs, 8pb + c2 + v) of this lane's fragment
  auto out = [&](ix pb, int rofs, const double* v2) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const ix col = 8 * pb + c2 + v;
      const int cell = rofs + rr - c2 - v;
      if (cell < 0 || cell > K || col >= n) continue;
      const double w = (col + cell < n) ? v2[v] : 0.0;
      if (col >= s && col < e) *srow.at(cell, col) = w;
      else if (side && col >= e && col < e + K) side[(col - e) * (K + 1) + cell] = w;
    }
  };
  __syncthreads();
  tables(pb_top);
  fill(0, pb_top);
  cpa_commit();
  cpa_wait0();
  __syncthreads();
  int buf = 0;
#pragma unroll 1
  for (ix pb = pb_top; pb >= pb_end; --pb) {
    if (pb > pb_end) fill(buf ^ 1, pb - 1);
    cpa_commit();
    const double* lp = sm.lp[buf];
    const int* zs = sm.zs[pb & 1];
    double* lin = sm.lin[warp];
    {  // Linv (per warp) interleaved with Y = Z_TT L_TP (tile column outer)
      LinvChain ch;
      ch.init(lp, rr, q);
      double ya[TPW][2][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) ya[i][0][0] = ya[i][0][1] = ya[i][1][0] = ya[i][1][1] = 0.0;
#pragma unroll
      for (int u = 0; u < NT; ++u) {
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int t = warp + NW * i;
          mm(ya[i][u & 1], &sm.z[0][0] + zs[t * NT + u], t < u, lp + (8 + 8 * u) * 8, false);
        }
        if ((u + 1) % (NT / 8) == 0) ch.step((u + 1) / (NT / 8) - 1);
      }
      put(lin, ch.M0, ch.M1);
#pragma unroll
      for (int i = 0; i < TPW; ++i) put(sm.y[warp + NW * i], ya[i][0][0] + ya[i][1][0], ya[i][0][1] + ya[i][1][1]);
      __syncwarp();
      double h[2] = {0.0, 0.0};
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + NW * i;
        double zz[2] = {0.0, 0.0};
        mm(zz, sm.y[t], false, lin, false);
        zz[0] = -zz[0];
        zz[1] = -zz[1];
        put(sm.zt[t], zz[0], zz[1]);
        if (t + 1 < NT) put(&sm.z[0][0] + ring_slot<K>(t + 1, pb, sm.mg) * 64, zz[0], zz[1]);
        out(pb, 8 + 8 * t, zz);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < TPW; ++i) mm(h, lp + (8 + 8 * (warp + NW * i)) * 8, true, sm.zt[warp + NW * i], false);
      put(sm.ph[pb & 1][warp], h[0], h[1]);
    }
    if (pb > pb_end) tables(pb - 1);
    cpa_wait0();
    __syncthreads();
    if (warp == 0) {  // Z_PP = (Linv - L_TP^T Z_TP)^T Linv -> tile (pb, pb), S cells
      double h0 = 0.0, h1 = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) {
        const double2 p2 = get(sm.ph[pb & 1][w2]);
        h0 += p2.x;
        h1 += p2.y;
      }
      const double2 l2 = get(lin);
      put(sm.hm, l2.x - h0, l2.y - h1);
      __syncwarp();
      double zp[2] = {0.0, 0.0};
      mm(zp, sm.hm, true, lin, false);
      put(&sm.z[0][0] + ring_slot<K>(0, pb, sm.mg) * 64, zp[0], zp[1]);
      out(pb, 0, zp);
      __syncwarp();
    }
    buf ^= 1;
  }
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_subset_mw(SubP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TakMwSmem<K, NW>& sm = *reinterpret_cast<TakMwSmem<K, NW>*>(smraw);
  if (G.span_rows > 0) {  // row spans (see Geo); the sweep runs upwards: a piece that ends inside a matrix
    for (int k = 0; k < G.span_kmax; ++k) {  // burns in from below its end
      ix b, s, e;
      if (!span_piece(G, blockIdx.x, k, b, s, e)) continue;  // uniform across the CTA
      const ix jend = e + G.burn < G.n ? e + G.burn : G.n;
      const ix slot = ix(blockIdx.x) * G.span_kmax + k;
      subset_mw_unit<K, NW>(C, b, G.n, s, e, jend, e < G.n ? C.side + slot * ix(K) * (K + 1) : nullptr, sm);
      __syncthreads();  // the next piece reuses the shared windows
    }
    return;
  }
  const ix unit = blockIdx.x;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  if (b >= G.batch) return;
  const ix s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix jend = e + G.burn < G.n ? e + G.burn : G.n;
  subset_mw_unit<K, NW>(C, b, G.n, s, e, jend, p + 1 < G.nseg ? C.side + unit * ix(K) * (K + 1) : nullptr, sm);
}

template <int K, int NW>
__global__ void __launch_bounds__(32 * NW) k_subset_mw_repair(SubP<double> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  TakMwSmem<K, NW>& sm = *reinterpret_cast<TakMwSmem<K, NW>*>(smraw);
  const ix b = blockIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  subset_mw_unit<K, NW>(C, b, G.n, 0, G.n, G.n, nullptr, sm);
}

int g_segment_rows = 0;

template <class T, int K, int P, int TS>
bool run_chol(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  using Sh = Shape<K, P, TS>;
  Geo G;
  G.batch = q.batch;
  G.n = q.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol<T, K, P, TS>, Sh::NT, 0);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    ix units = ix(sms) * per;
    ix nseg = units / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  seg = (seg + TS - 1) / TS * TS;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t bytes = sizeof(T) * size_t(units) * K * (K + 1) + sizeof(int64_t) * size_t(G.batch) +
                       sizeof(int32_t) * size_t(G.batch) + 64;
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), bytes, s) != cudaSuccess) return false;
  CholP<T> C;
  C.q = view<T>(q);
  C.l = view<T>(l);
  C.side = reinterpret_cast<T*>(ws);
  C.fail = reinterpret_cast<int64_t*>(ws + sizeof(T) * size_t(units) * K * (K + 1));
  C.flag = reinterpret_cast<int32_t*>(C.fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, C.flag, G.batch, G.n);
  {
    timing::Scope ts("wide_chol", s);
    k_chol<T, K, P, TS><<<unsigned(units), Sh::NT, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_check", s);
    k_chol_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_repair", s);
    k_chol_repair<T, K, P, TS><<<unsigned(G.batch), Sh::NT, 0, s>>>(C, G);
  }
  k_status<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, G.batch, G.n, st, row);
  scratch_free(ws, s);
  return true;
}


// config-4 fp64 Cholesky on the FP64 tensor cores, NW warps per unit
template <int K, int NW>
bool run_chol_mw(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  Geo G;
  G.batch = q.batch;
  G.n = q.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_mw<K, NW>, 32 * NW, 0);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
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
  const size_t sb = sizeof(double) * size_t(units) * K * (K + 1);
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), sb + 12 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  CholP<double> C;
  C.q = view<double>(q);
  C.l = view<double>(l);
  C.side = reinterpret_cast<double*>(ws);
  C.fail = reinterpret_cast<int64_t*>(ws + sb);
  C.flag = reinterpret_cast<int32_t*>(C.fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, C.flag, G.batch, G.n);
  {
    timing::Scope ts("wide_chol_dmma", s);
    k_chol_mw<K, NW><<<unsigned(units), 32 * NW, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_check", s);
    k_chol_check<double, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_repair", s);
    k_chol_mw_repair<K, NW><<<unsigned(G.batch), 32 * NW, 0, s>>>(C, G);
  }
  k_status<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, G.batch, G.n, st, row);
  scratch_free(ws, s);
  return true;
}

// config-4 k = 64 fp64 Cholesky on the FP64 tensor cores
bool run_chol_dmma(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  constexpr int K = kDK;
  Geo G;
  G.batch = q.batch;
  G.n = q.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_dmma, 32, 0);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
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
  const size_t sb = sizeof(double) * size_t(units) * K * (K + 1);
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), sb + 12 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  CholP<double> C;
  C.q = view<double>(q);
  C.l = view<double>(l);
  C.side = reinterpret_cast<double*>(ws);
  C.fail = reinterpret_cast<int64_t*>(ws + sb);
  C.flag = reinterpret_cast<int32_t*>(C.fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, C.flag, G.batch, G.n);
  {
    timing::Scope ts("wide_chol_dmma", s);
    k_chol_dmma<<<unsigned(units), 32, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_check", s);
    k_chol_check<double, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_chol_repair", s);
    k_chol_dmma_repair<<<unsigned(G.batch), 32, 0, s>>>(C, G);
  }
  k_status<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, G.batch, G.n, st, row);
  scratch_free(ws, s);
  return true;
}

// Row-span geometry (see Geo): equal runs of rows over `ctas` CTAs (BGM_WIDE_SPAN_CTAS overrides the
// count, BGM_WIDE_SPAN=0 disables).  Declined when a run would be shorter than min_rows (small
// batches keep the per-matrix segments) or when the uniform segments already fill the slots.
inline bool span_rows(Geo& G, ix ctas, ix min_rows) {
  static const int off = [] {
    const char* e = std::getenv("BGM_WIDE_SPAN");
    return e && e[0] == '0';
  }();
  if (off) return false;
  if (const char* cv = std::getenv("BGM_WIDE_SPAN_CTAS"))
    if (std::atoi(cv) >= 1) ctas = std::atoi(cv);
  const ix n8 = (G.n + 7) / 8 * 8;
  ix rows = (G.batch * n8 + ctas - 1) / ctas;
  rows = (rows + 7) / 8 * 8;
  if (rows < min_rows || rows >= G.batch * n8) return false;
  G.span_rows = rows;
  G.n8 = n8;
  G.span_kmax = int((rows + n8 - 1) / n8) + 1;
  return true;
}

// segments per matrix: fill the resident CTA slots in whole waves, burn-in
// overhead counted (the k_vsub_dmma grid is one short launch)
inline int pick_nseg(ix batch, ix n, int slots, int burn, int seg_min) {
  int best = 1;
  double best_eff = 0.0;
  for (int ns = 1; ns <= 256; ++ns) {
    const ix seg = (n + ns - 1) / ns;
    if (ns > 1 && seg < seg_min) break;
    const double units = double(batch) * ns;
    const double waves = std::ceil(units / slots);
    const double eff = units / (waves * slots) * double(seg) / double(seg + (ns > 1 ? burn : 0));
    if (eff > best_eff * 1.0001) {
      best_eff = eff;
      best = ns;
    }
  }
  return best;
}

template <int K, int NW>
bool run_vsub_dmma(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb, int32_t* st,
                   int64_t* row, cudaStream_t s) {
  const size_t smem = sizeof(VtSmem<K, NW>);
  if (smem > 227 * 1024) return false;
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_vsub_dmma<K, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_vsub_dmma_repair<K, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  constexpr int STATE = VtSmem<K, NW>::NWT * 64;
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vsub_dmma<K, NW>, 32 * NW, smem);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    const int ns = pick_nseg(G.batch, G.n, sms * per, G.burn, 2 * G.burn);
    seg = (G.n + ns - 1) / ns;
  }
  seg = (seg + 7) / 8 * 8;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  ix units = G.batch * G.nseg, slots = units;
  if (g_segment_rows <= 0 && span_rows(G, ix(sms) * per, 2 * ix(G.burn))) {
    units = (G.batch * G.n8 + G.span_rows - 1) / G.span_rows;
    slots = units * G.span_kmax;
  }
  const size_t sb_bytes = sizeof(double) * size_t(slots) * STATE;
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), 2 * sb_bytes + 12 * size_t(G.batch) + 64, s) != cudaSuccess)
    return false;
  VsP<double> C;
  C.l = view<double>(l);
  C.s = view<double>(sm);
  C.sb = view<double>(sb);
  C.lb = view<double>(lb);
  C.side = reinterpret_cast<double*>(ws);
  C.tail = reinterpret_cast<double*>(ws + sb_bytes);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + 2 * sb_bytes);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, G.n);
  k_diag_check<double><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, fail);
  {
    timing::Scope ts("wide_vjp_subset_dmma", s);
    k_vsub_dmma<K, NW><<<unsigned(units), 32 * NW, smem, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_subset_check", s);
    k_vsub_dmma_check<K, NW><<<blocks_for(units * 32, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_subset_repair", s);
    k_vsub_dmma_repair<K, NW><<<unsigned(G.batch), 32 * NW, smem, s>>>(C, G);
  }
  const ix zw = ((G.batch + l.tile - 1) / l.tile * l.tile) * K * (K + 1);
  k_zero_corners_w<double><<<blocks_for(zw, 128), 128, 0, s>>>(C.lb, G.batch);
  k_status_code<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, st, row);
  scratch_free(ws, s);
  return true;
}

template <int K>
bool run_vchol_dmma(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  constexpr int NW = K >= 128 ? 4 : 2, NT = K / 8, STATE = NT * (NT + 1) / 2 * 64;
  const size_t smem = sizeof(VdSmem<K, NW>);
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_vchol_dmma<K, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_vchol_dmma_repair<K, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vchol_dmma<K, NW>, 32 * NW, smem);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    const int ns = pick_nseg(G.batch, G.n, sms * per, G.burn, 2 * G.burn);
    seg = (G.n + ns - 1) / ns;
  }
  seg = (seg + 7) / 8 * 8;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  ix units = G.batch * G.nseg, slots = units;
  if (g_segment_rows <= 0 && span_rows(G, ix(sms) * per, 2 * ix(G.burn))) {
    units = (G.batch * G.n8 + G.span_rows - 1) / G.span_rows;
    slots = units * G.span_kmax;
  }
  const size_t sb_bytes = sizeof(double) * size_t(slots) * STATE;
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), 2 * sb_bytes + 4 * size_t(G.batch) + 64, s) != cudaSuccess)
    return false;
  VdP<double> C;
  C.l = view<double>(l);
  C.lb = view<double>(lb);
  C.qb = view<double>(qb);
  C.side = reinterpret_cast<double*>(ws);
  C.tail = reinterpret_cast<double*>(ws + sb_bytes);
  C.flag = reinterpret_cast<int32_t*>(ws + 2 * sb_bytes);
  cudaMemsetAsync(C.flag, 0, sizeof(int32_t) * size_t(G.batch), s);
  {
    timing::Scope ts("wide_vjp_chol_dmma", s);
    k_vchol_dmma<K, NW><<<unsigned(units), 32 * NW, smem, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_chol_check", s);
    k_vchol_dmma_check<K, NW><<<blocks_for(units * 32, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_chol_repair", s);
    k_vchol_dmma_repair<K, NW><<<unsigned(G.batch), 32 * NW, smem, s>>>(C, G);
  }
  const ix zw = ((G.batch + l.tile - 1) / l.tile * l.tile) * K * (K + 1);
  k_zero_corners_w<double><<<blocks_for(zw, 128), 128, 0, s>>>(C.qb, G.batch);
  scratch_free(ws, s);
  return true;
}

template <int K, int NW>
bool run_subset_mw(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  const size_t smem = sizeof(TakMwSmem<K, NW>);
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_subset_mw<K, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_subset_mw_repair<K, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  G.burn = (G.burn + 7) / 8 * 8;
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_subset_mw<K, NW>, 32 * NW, smem);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    const int ns = pick_nseg(G.batch, G.n, sms * per, G.burn, 2 * G.burn);
    seg = (G.n + ns - 1) / ns;
  }
  seg = (seg + 7) / 8 * 8;
  if (seg < K) seg = (K + 7) / 8 * 8;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  ix units = G.batch * G.nseg, slots = units;
  // Row spans are opt-in here (BGM_WIDE_SPAN_SUBSET=1, or a forced CTA count): alone the kernel gains
  // 14% (k = 128: 5.79 -> 4.96 ms), but in the config-4 suite it runs beside two other stream lanes that
  // were using the SMs its 128 CTAs leave free, and the step got 0.5 ms slower.
  const char* sv = std::getenv("BGM_WIDE_SPAN_SUBSET");
  const bool want_span = (sv && sv[0] == '1') || std::getenv("BGM_WIDE_SPAN_CTAS") != nullptr;
  if (g_segment_rows <= 0 && want_span && span_rows(G, ix(sms) * per, 2 * ix(G.burn))) {
    units = (G.batch * G.n8 + G.span_rows - 1) / G.span_rows;
    slots = units * G.span_kmax;
  }
  const size_t side_bytes = sizeof(double) * size_t(slots) * K * (K + 1);
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), side_bytes + 12 * size_t(G.batch) + 64, s) != cudaSuccess)
    return false;
  SubP<double> C;
  C.l = view<double>(l);
  C.s = view<double>(sb);
  C.side = reinterpret_cast<double*>(ws);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + side_bytes);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, G.n);
  k_diag_check<double><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, fail);
  {
    timing::Scope ts("wide_subset_mw", s);
    k_subset_mw<K, NW><<<unsigned(units), 32 * NW, smem, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_subset_check", s);
    k_subset_check<double, K><<<blocks_for(slots * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_subset_repair", s);
    k_subset_mw_repair<K, NW><<<unsigned(G.batch), 32 * NW, smem, s>>>(C, G);
  }
  k_status_code<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, st, row);
  scratch_free(ws, s);
  return true;
}

template <int K>
bool run_subset_dmma(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  const size_t smem = sizeof(TakSmem<K>);
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_subset_dmma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_subset_dmma_repair<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  G.burn = (G.burn + 7) / 8 * 8;
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_subset_dmma<K>, 32, smem);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    ix nseg = ix(sms) * per / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  seg = (seg + 7) / 8 * 8;
  if (seg < K) seg = (K + 7) / 8 * 8;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t side_bytes = sizeof(double) * size_t(units) * K * (K + 1);
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), side_bytes + 12 * size_t(G.batch) + 64, s) != cudaSuccess)
    return false;
  SubP<double> C;
  C.l = view<double>(l);
  C.s = view<double>(sb);
  C.side = reinterpret_cast<double*>(ws);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + side_bytes);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, G.n);
  k_diag_check<double><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, fail);
  {
    timing::Scope ts("wide_subset_dmma", s);
    k_subset_dmma<K><<<unsigned(units), 32, smem, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_subset_check", s);
    k_subset_check<double, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_subset_repair", s);
    k_subset_dmma_repair<K><<<unsigned(G.batch), 32, smem, s>>>(C, G);
  }
  k_status_code<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, st, row);
  scratch_free(ws, s);
  return true;
}

template <class T, int K, int P, int TS>
bool run_subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  using Sh = Shape<K, P, TS>;
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  ix seg = g_segment_rows > 0 ? ix(requested_seg(g_segment_rows, K)) : pick_seg(k_subset<T, K, P, TS>, Sh::NT, G, 2 * ix(G.burn));
  seg = (seg + TS - 1) / TS * TS;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t side_bytes = sizeof(T) * size_t(units) * K * (K + 1);
  const size_t bytes = side_bytes + sizeof(int64_t) * size_t(G.batch) + sizeof(int32_t) * size_t(G.batch) + 64;
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), bytes, s) != cudaSuccess) return false;
  SubP<T> C;
  C.l = view<T>(l);
  C.s = view<T>(sb);
  C.side = reinterpret_cast<T*>(ws);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + side_bytes);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, G.n);
  k_diag_check<T><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, fail);
  {
    timing::Scope ts("wide_subset", s);
    k_subset<T, K, P, TS><<<unsigned(units), Sh::NT, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_subset_check", s);
    k_subset_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_subset_repair", s);
    k_subset_repair<T, K, P, TS><<<unsigned(G.batch), Sh::NT, 0, s>>>(C, G);
  }
  k_status_code<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, st, row);
  scratch_free(ws, s);
  return true;
}

template <class T, int K, bool TR>
bool run_solve(const bgm_band& l, const bgm_vec& v, const bgm_vec& x, int32_t* st, int64_t* row, cudaStream_t s) {
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = (kBurnGen + 2) * K;  // a solve damps by ~sqrt(K)|L(i,m)/L(i,i)| per generation
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    int sms = 148, dev = 0, per = 1;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_solve<T, K, TR>, 32 * kSolveWarps, 0);
    ix nseg = ix(sms) * (per > 0 ? per : 1) * kSolveWarps / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  if (seg < K) seg = K;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t side_bytes = sizeof(T) * size_t(units) * K;
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), side_bytes + 12 * size_t(G.batch) + 64, s) != cudaSuccess)
    return false;
  SolveP<T> C;
  C.l = view<T>(l);
  C.v = view<T>(v);
  C.x = view<T>(x);
  C.side = reinterpret_cast<T*>(ws);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + (side_bytes + 7) / 8 * 8);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init_fail<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, TR ? 0 : G.n);
  k_singular<T><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, TR, fail);
  {
    timing::Scope ts(TR ? "wide_solve_t" : "wide_solve", s);
    k_solve<T, K, TR><<<unsigned((units + kSolveWarps - 1) / kSolveWarps), 32 * kSolveWarps, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_solve_check", s);
    k_solve_check<T, K, TR><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_solve_repair", s);
    k_solve_repair<T, K, TR><<<unsigned((G.batch + kSolveWarps - 1) / kSolveWarps), 32 * kSolveWarps, 0, s>>>(C, G);
  }
  k_status_solve<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, TR, st, row);
  scratch_free(ws, s);
  return true;
}

template <class T>
bool run_logdet(const bgm_band& l, void* out, int32_t* st, int64_t* row, cudaStream_t s) {
  const ix chunks = (l.n + kLogChunk - 1) / kLogChunk;
  char* ws = nullptr;
  const size_t pb = sizeof(double) * size_t(l.batch) * chunks;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), pb + sizeof(int64_t) * size_t(l.batch) + 64, s) != cudaSuccess)
    return false;
  double* part = reinterpret_cast<double*>(ws);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + pb);
  {
    timing::Scope ts("log_det", s);
    fill_fail<<<blocks_for(l.batch, 128), 128, 0, s>>>(fail, l.batch, l.n);
    const Band<T> L = view<T>(l);
    const ix work = ((l.batch + l.tile - 1) / l.tile * l.tile) * chunks;
    k_logdet_part<T><<<blocks_for(work, 128), 128, 0, s>>>(L, l.batch, chunks, part, fail);
    k_logdet_sum<T><<<blocks_for(l.batch * 32, 128), 128, 0, s>>>(part, fail, l.batch, l.n, chunks,
                                                                static_cast<T*>(out), st, row);
  }
  scratch_free(ws, s);
  return true;
}

template <class T, int K>
bool run_vchol(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  const size_t smem = VcSmem<T, K>::bytes;
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_vchol_w<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_vchol_w_repair<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    int sms = 148, dev = 0, per = 1;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vchol_w<T, K>, 32, smem);
    ix nseg = ix(sms) * (per > 0 ? per : 1) / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t side = sizeof(T) * size_t(units) * K * (K + 1);
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), side + 4 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  VcP<T> C;
  C.l = view<T>(l);
  C.lb = view<T>(lb);
  C.qb = view<T>(qb);
  C.side = reinterpret_cast<T*>(ws);
  C.flag = reinterpret_cast<int32_t*>(ws + (side + 7) / 8 * 8);
  cudaMemsetAsync(C.flag, 0, sizeof(int32_t) * size_t(G.batch), s);
  {
    timing::Scope ts("wide_vjp_chol", s);
    k_vchol_w<T, K><<<unsigned(units), 32, smem, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_chol_check", s);
    k_vchol_w_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_chol_repair", s);
    k_vchol_w_repair<T, K><<<unsigned(G.batch), 32, smem, s>>>(C, G);
  }
  const ix zw = ((G.batch + l.tile - 1) / l.tile * l.tile) * K * (K + 1);
  k_zero_corners_w<T><<<blocks_for(zw, 128), 128, 0, s>>>(C.qb, G.batch);
  scratch_free(ws, s);
  return true;
}

template <class T, int K>
bool run_vsub(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb, int32_t* st,
              int64_t* row, cudaStream_t s) {
  const size_t smem = VsSmem<T, K>::bytes;
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_vsub<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_vsub_repair<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = kBurnGen * K;
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  ix seg = requested_seg(g_segment_rows, K);
  if (seg <= 0) {
    int sms = 148, dev = 0, per = 1;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_vsub<T, K>, 32, smem);
    ix nseg = ix(sms) * (per > 0 ? per : 1) / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  if (seg < K) seg = K;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;
  const size_t sd = sizeof(T) * size_t(units) * K * (K + 2);
  char* ws = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&ws), 2 * sd + 12 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  VsP<T> C;
  C.l = view<T>(l);
  C.s = view<T>(sm);
  C.sb = view<T>(sb);
  C.lb = view<T>(lb);
  C.side = reinterpret_cast<T*>(ws);
  C.tail = reinterpret_cast<T*>(ws + sd);
  int64_t* fail = reinterpret_cast<int64_t*>(ws + (2 * sd + 7) / 8 * 8);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, G.n);
  k_diag_check<T><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, fail);
  {
    timing::Scope ts("wide_vjp_subset", s);
    k_vsub<T, K><<<unsigned(units), 32, smem, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_subset_check", s);
    k_vsub_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_vjp_subset_repair", s);
    k_vsub_repair<T, K><<<unsigned(G.batch), 32, smem, s>>>(C, G);
  }
  k_status_code<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, st, row);
  scratch_free(ws, s);
  return true;
}
}  // namespace

// fp32 bands on the FP64 tensor-core paths: the band is widened into an fp64
// scratch copy of the same layout, the fp64 kernel runs, the result is
// narrowed back (conversion traffic is a few MB against a compute-bound op;
// the arithmetic is then fp64, tighter than the reference's fp32 loop)
// 4 elements per thread (float4 <-> 2 x double2) when both sides are 16-byte
// aligned; the scalar tail / unaligned case element by element
__global__ void k_widen(const float* a, double* b, ix count) {
  const ix t0 = blockIdx.x * ix(blockDim.x) + threadIdx.x, st = ix(gridDim.x) * blockDim.x;
  ix done = 0;
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
    const ix q = count / 4;
    for (ix i = t0; i < q; i += st) {
      const float4 v = reinterpret_cast<const float4*>(a)[i];
      reinterpret_cast<double2*>(b)[2 * i] = make_double2(v.x, v.y);
      reinterpret_cast<double2*>(b)[2 * i + 1] = make_double2(v.z, v.w);
    }
    done = q * 4;
  }
  for (ix i = done + t0; i < count; i += st) b[i] = a[i];
}
__global__ void k_narrow(const double* a, float* b, ix count) {
  const ix t0 = blockIdx.x * ix(blockDim.x) + threadIdx.x, st = ix(gridDim.x) * blockDim.x;
  ix done = 0;
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
    const ix q = count / 4;
    for (ix i = t0; i < q; i += st) {
      const double2 u = reinterpret_cast<const double2*>(a)[2 * i];
      const double2 w = reinterpret_cast<const double2*>(a)[2 * i + 1];
      reinterpret_cast<float4*>(b)[i] = make_float4(float(u.x), float(u.y), float(w.x), float(w.y));
    }
    done = q * 4;
  }
  for (ix i = done + t0; i < count; i += st) b[i] = float(a[i]);
}

static ix band_count(const bgm_band& x) {
  return (x.batch + x.tile - 1) / x.tile * x.tile * x.n * (x.lower + x.upper + 1);
}

struct Widened {
  bgm_band d{};
  bool ok = false;
  Widened(const bgm_band& x, bool copy, cudaStream_t s) {
    d = x;
    d.dtype = BGM_F64;
    const ix cnt = band_count(x);
    if (scratch_alloc(&d.data, sizeof(double) * size_t(cnt) + 16, s) != cudaSuccess) return;
    if (copy) k_widen<<<1184, 256, 0, s>>>(static_cast<const float*>(x.data), static_cast<double*>(d.data), cnt);
    ok = true;
  }
  void narrow_into(const bgm_band& x, cudaStream_t s) const {
    k_narrow<<<1184, 256, 0, s>>>(static_cast<const double*>(d.data), static_cast<float*>(x.data), band_count(x));
  }
  void release(cudaStream_t s) {
    if (ok) scratch_free(d.data, s);
    ok = false;
  }
};

static bool wide32() {
  static const bool on = [] {
    const char* e = std::getenv("BGM_WIDE_F32_DMMA");
    const char* d = std::getenv("BGM_WIDE_DMMA");
    return !(e && e[0] == '0') && !(d && d[0] == '0');
  }();
  return on;
}

// run an fp64 entry point on widened copies of fp32 operands
template <class F>
bool via_f64(std::initializer_list<const bgm_band*> in, std::initializer_list<const bgm_band*> out, cudaStream_t s,
             F&& run) {
  Widened* w[8];
  int nw = 0;
  bool ok = true;
  for (const bgm_band* x : in) {
    w[nw] = new Widened(*x, true, s);
    ok = ok && w[nw++]->ok;
  }
  for (const bgm_band* x : out) {
    w[nw] = new Widened(*x, false, s);
    ok = ok && w[nw++]->ok;
  }
  if (ok) {
    bgm_band d[8];
    for (int i = 0; i < nw; ++i) d[i] = w[i]->d;
    ok = run(d);
    if (ok) {
      int j = int(in.size());
      for (const bgm_band* x : out) w[j++]->narrow_into(*x, s);
    }
  }
  for (int i = 0; i < nw; ++i) {
    w[i]->release(s);
    delete w[i];
  }
  return ok;
}

bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  if (q.lower != l.lower || q.upper != 0 || l.upper != 0 || q.batch == 0 || q.n == 0) return false;
  if (q.n < 4 * q.lower) return false;  // short matrices: the generic sweep is fine
  const bool f64 = q.dtype == BGM_F64;
  // fp32 storage: the look-ahead kernel reads / writes fp32 directly (fp64 arithmetic); only if it
  // declines is the band widened into an fp64 scratch copy for the fp64 DMMA kernels
  static const bool la32 = [] {
    const char* e = std::getenv("BGM_WIDE_DMMA_WARPS");
    const char* d = std::getenv("BGM_WIDE_DMMA");
    return !(e && std::atoi(e) != 0) && !(d && d[0] == '0');
  }();
  if (!f64 && (q.lower == 64 || q.lower == 128) && wide32() && la32 &&
      cholesky_la(q, l, st, row, s, g_segment_rows))
    return true;
  if (!f64 && (q.lower == 64 || q.lower == 128) && wide32() &&
      via_f64({&q}, {&l}, s, [&](bgm_band* d) { return cholesky(d[0], d[1], st, row, s); }))
    return true;
  switch (q.lower) {
    case 64: {
      static const bool use_dmma = [] {
        const char* e = std::getenv("BGM_WIDE_DMMA");
        return !(e && e[0] == '0');
      }();
      if (f64 && use_dmma) {
        static const int nw = [] {
          const char* e = std::getenv("BGM_WIDE_DMMA_WARPS");
          return e ? std::atoi(e) : 0;  // 0: look-ahead kernel
        }();
        if (nw == 0 && cholesky_la(q, l, st, row, s, g_segment_rows)) return true;
        if (nw == 2) return run_chol_mw<64, 2>(q, l, st, row, s);
        return run_chol_dmma(q, l, st, row, s);
      }
      return f64 ? run_chol<double, 64, 8, 9>(q, l, st, row, s) : run_chol<float, 64, 8, 9>(q, l, st, row, s);
    }
    case 128: {
      static const bool use_dmma = [] {
        const char* e = std::getenv("BGM_WIDE_DMMA");
        return !(e && e[0] == '0');
      }();
      if (f64 && use_dmma) {
        static const int nw = [] {
          const char* e = std::getenv("BGM_WIDE_DMMA_WARPS");
          return e ? std::atoi(e) : 0;  // 0: look-ahead kernel
        }();
        if (nw == 8) return run_chol_mw<128, 8>(q, l, st, row, s);
        if (nw == 0 && cholesky_la(q, l, st, row, s, g_segment_rows)) return true;
        if (nw == 2) return run_chol_mw<128, 2>(q, l, st, row, s);
        return run_chol_mw<128, 4>(q, l, st, row, s);
      }
      return f64 ? run_chol<double, 128, 16, 9>(q, l, st, row, s) : run_chol<float, 128, 16, 9>(q, l, st, row, s);
    }
    default: return false;
  }
}

static int subset_warps() {  // BGM_SUBSET_WARPS: 1 = single-warp kernel
  static const int w = [] {
    const char* e = std::getenv("BGM_SUBSET_WARPS");
    return e ? std::atoi(e) : 0;  // 0: 4 warps for k = 64, 8 for k = 128
  }();
  return w;
}

bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  if (l.lower != sb.lower || l.upper != 0 || sb.upper != 0 || l.batch == 0 || l.n == 0) return false;
  if (l.n < 4 * l.lower) return false;
  const bool f64 = l.dtype == BGM_F64;
  if (!f64 && (l.lower == 64 || l.lower == 128) && wide32() &&
      via_f64({&l}, {&sb}, s, [&](bgm_band* d) { return subset(d[0], d[1], st, row, s); }))
    return true;
  static const bool use_dmma = [] {
    const char* e = std::getenv("BGM_WIDE_DMMA");
    return !(e && e[0] == '0');
  }();
  switch (l.lower) {
    case 64:
      if (f64 && use_dmma) {
        const int nw = subset_warps();
        if (nw == 1) return run_subset_dmma<64>(l, sb, st, row, s);
        return nw == 2 ? run_subset_mw<64, 2>(l, sb, st, row, s) : run_subset_mw<64, 4>(l, sb, st, row, s);
      }
      return f64 ? run_subset<double, 64, 8, 9>(l, sb, st, row, s) : run_subset<float, 64, 8, 9>(l, sb, st, row, s);
    case 128:
      if (f64 && use_dmma) {
        const int nw = subset_warps();
        if (nw == 1) return run_subset_dmma<128>(l, sb, st, row, s);
        return nw == 4 ? run_subset_mw<128, 4>(l, sb, st, row, s) : run_subset_mw<128, 8>(l, sb, st, row, s);
      }
      return f64 ? run_subset<double, 128, 16, 9>(l, sb, st, row, s)
                 : run_subset<float, 128, 16, 9>(l, sb, st, row, s);
    default: return false;
  }
}

bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s) {
  if (l.upper != 0 || l.batch == 0 || l.n == 0 || l.n < 8 * l.lower) return false;
  static const bool blocked = [] {
    const char* e = std::getenv("BGM_WSOLVE_BLK");
    return !(e && e[0] == '0');
  }();
  if (blocked && solve_vec_blk(l, v, tr, x, st, row, s, g_segment_rows)) return true;
  const bool f64 = l.dtype == BGM_F64;
  switch (l.lower) {
#define BGM_SOLVE(KK)                                                                           \
  case KK:                                                                                      \
    if (f64) return tr ? run_solve<double, KK, true>(l, v, x, st, row, s) : run_solve<double, KK, false>(l, v, x, st, row, s); \
    return tr ? run_solve<float, KK, true>(l, v, x, st, row, s) : run_solve<float, KK, false>(l, v, x, st, row, s);
    BGM_SOLVE(64)
    BGM_SOLVE(128)
#undef BGM_SOLVE
    default: return false;
  }
}

bool log_det(const bgm_band& l, void* out, int32_t* st, int64_t* row, cudaStream_t s) {
  if (l.batch == 0 || l.n == 0) return false;
  return l.dtype == BGM_F64 ? run_logdet<double>(l, out, st, row, s) : run_logdet<float>(l, out, st, row, s);
}

bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  if (l.upper != 0 || lb.upper != 0 || qb.upper != 0 || lb.lower != l.lower || qb.lower != l.lower ||
      l.batch == 0 || l.n < 4 * l.lower)
    return false;
  const bool f64 = l.dtype == BGM_F64;
  if (!f64 && (l.lower == 64 || l.lower == 128) && wide32() &&
      via_f64({&l, &lb}, {&qb}, s, [&](bgm_band* d) { return vjp_cholesky(d[0], d[1], d[2], s); }))
    return true;
  static const bool use_dmma = [] {
    const char* e = std::getenv("BGM_WIDE_DMMA");
    return !(e && e[0] == '0');
  }();
  switch (l.lower) {
    case 64:
      if (f64 && use_dmma) return run_vchol_dmma<64>(l, lb, qb, s);
      return f64 ? run_vchol<double, 64>(l, lb, qb, s) : run_vchol<float, 64>(l, lb, qb, s);
    case 128:
      if (f64 && use_dmma) return run_vchol_dmma<128>(l, lb, qb, s);
      return f64 ? run_vchol<double, 128>(l, lb, qb, s) : run_vchol<float, 128>(l, lb, qb, s);
    default: return false;
  }
}

static int vsub_warps() {
  static const int w = [] {
    const char* e = std::getenv("BGM_VSUB_WARPS");
    return e ? std::atoi(e) : 0;  // 0: 4 warps for k = 64, 8 for k = 128
  }();
  return w;
}

bool vjp_subset(const bgm_band& l, const bgm_band& sm, const bgm_band& sb, const bgm_band& lb, int32_t* st,
                int64_t* row, cudaStream_t s) {
  if (l.upper != 0 || l.batch == 0 || l.n < 4 * l.lower) return false;
  const bool f64 = l.dtype == BGM_F64;
  if (!f64 && (l.lower == 64 || l.lower == 128) && wide32() &&
      via_f64({&l, &sm, &sb}, {&lb}, s, [&](bgm_band* d) { return vjp_subset(d[0], d[1], d[2], d[3], st, row, s); }))
    return true;
  static const bool use_dmma = [] {
    const char* e = std::getenv("BGM_WIDE_DMMA");
    return !(e && e[0] == '0');
  }();
  switch (l.lower) {
    case 16:
      return f64 ? run_vsub<double, 16>(l, sm, sb, lb, st, row, s) : run_vsub<float, 16>(l, sm, sb, lb, st, row, s);
    case 64:
      if (f64 && use_dmma && (vsub_warps() == 8 ? run_vsub_dmma<64, 8>(l, sm, sb, lb, st, row, s)
                                                : run_vsub_dmma<64, 4>(l, sm, sb, lb, st, row, s)))
        return true;
      return f64 ? run_vsub<double, 64>(l, sm, sb, lb, st, row, s) : run_vsub<float, 64>(l, sm, sb, lb, st, row, s);
    case 128:
      if (f64 && use_dmma && (vsub_warps() != 4 ? run_vsub_dmma<128, 8>(l, sm, sb, lb, st, row, s)
                                                : run_vsub_dmma<128, 4>(l, sm, sb, lb, st, row, s)))
        return true;
      return f64 ? run_vsub<double, 128>(l, sm, sb, lb, st, row, s) : run_vsub<float, 128>(l, sm, sb, lb, st, row, s);
    default: return false;
  }
}

void set_segment_rows(int rows) { g_segment_rows = rows; }

}  // namespace wide
}  // namespace bgm
