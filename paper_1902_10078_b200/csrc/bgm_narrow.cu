// Narrow-band (k <= 16) fast paths for the per-operator API: cholesky,
// solve_vec (L and L^T) and the Takahashi subset, tile-32 layout.
//
// Same organisation as the config-3 sweeps (bgm_mlik_t1.cu): one thread per
// (matrix, segment), a warp = the 32 matrices of one tile on one segment, so
// every band-cell access is one coalesced 256-byte warp transaction; the
// recurrence state lives in registers (solves) or in a per-thread packed
// triangle in shared memory laid out [entry][thread] (cholesky, subset),
// shifted physically as it is updated.  Segments start with a burn-in from a
// zero state; a check kernel compares each unit's burn-in copy of the K
// values / columns next to its segment with the neighbour's genuine ones and
// flagged matrices are recomputed by a single-unit sweep.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_timing.cuh"

namespace bgm {
namespace narrow {
namespace {

constexpr int kThreads = 32;     // one warp per CTA: shared memory bounds residency
// narrow solves: rows in flight per thread (shared-memory ring); measured at
// configs 1 / 3: k = 16 gains from depth (1.26 -> 1.03 ms), k = 4 does not
template <int K>
constexpr int solve_pf() {
  return K >= 16 ? 10 : 3;
}
constexpr int kBurnMin = 64;     // burn-in rows: max(kBurnMin, kBurnGen * K)
constexpr int kBurnGen = 16;
constexpr int kFewTiles = 64;     // below this many 32-matrix tiles the grid is segment-bound
constexpr double kCheckTol = 1e-12;

__host__ __device__ constexpr int tri(int a, int b) { return a * (a + 1) / 2 + b; }

struct Geo {
  ix batch, n, seg, tiles;
  int nseg, burn;
  int l2a;  // solves: L2 bulk-prefetch distance in rows (0 = off)
};

struct Unit {
  ix b, id;
  int p;
  bool live;
};
__device__ __forceinline__ Unit unit_of(const Geo& G) {
  const ix gt = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix warp = gt >> 5, tile = warp / G.nseg;
  Unit u;
  u.p = int(warp % G.nseg);
  u.b = tile * 32 + (gt & 31);
  u.live = tile < G.tiles && u.b < G.batch;
  u.id = u.b * G.nseg + u.p;
  return u;
}

// tile-32 base pointer of matrix b: cell (r, column j) at base[(j * w + r) * 32]
template <class T>
__device__ __forceinline__ T* bbase(const Band<T>& B, ix b) {
  return B.p + (b >> 5) * B.n * B.w * 32 + (b & 31);
}
template <class T>
__device__ __forceinline__ T* vbase(const Vec<T>& V, ix b) {
  return V.p + (b >> 5) * V.n * 32 + (b & 31);
}

template <class T>
__device__ __forceinline__ double dabs(T x) {
  return fabs(double(x));
}

template <class T>
__device__ __forceinline__ void cpa(T* dst, const T* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
// 1 / sqrt(x) by the reciprocal square root: the Cholesky pivot chains take
// one MUFU sequence per row instead of a square root and a division
__device__ __forceinline__ double rsq_t(double x) { return rsqrt(x); }
__device__ __forceinline__ float rsq_t(float x) { return rsqrtf(x); }

__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ------------------------------------------------------------------ cholesky
// Right-looking: the window W holds the trailing Schur complement rows
// i .. i+K-1 (packed, rows 0..K-1); row i+K enters fresh as Q(i+K, i..i+K).
template <class T>
struct CholP {
  Band<T> q, l;
  T* side;  // [unit][K][K+1]
  int64_t* fail;
  int32_t* flag;
};

template <class T, int K>
__device__ void chol_unit(const CholP<T>& C, ix b, ix n, ix s, ix e, ix i0, T* side, T* win) {
  constexpr int W = K + 1, ts = kThreads;
  auto Wr = [&](int a, int c) -> T& { return win[tri(a, c) * ts]; };
  const T* qb = bbase(C.q, b);
  T* lb = bbase(C.l, b);
  const ix cs = ix(W) * 32;  // column stride
  // window rows i0 .. i0+K-1 from Q
#pragma unroll 1
  for (int a = 0; a < K; ++a)
    for (int c = 0; c <= a; ++c)
      Wr(a, c) = (i0 + a < n) ? qb[(i0 + c) * cs + (a - c) * 32] : T(0);
  auto load_row = [&](ix r, T* out) {  // Q(r, r-K .. r) -> out[0..K] (column r-K+c)
#pragma unroll
    for (int c = 0; c <= K; ++c) out[c] = (r < n) ? qb[(r - K + c) * cs + (K - c) * 32] : T(0);
  };
  ix fail = n;
  auto emit = [&](ix i, const T* l) {
    if (i >= s) {
      T* col = lb + i * cs;
#pragma unroll
      for (int a = 0; a <= K; ++a) col[a * 32] = (i + a < n) ? l[a] : T(0);
    } else if (side && i >= s - K) {
      T* sd = side + (i - (s - K)) * W;
#pragma unroll
      for (int a = 0; a <= K; ++a) sd[a] = l[a];
    }
  };
  // ---- paired body (bgm_mlik_t1.cu's forward, without the L L^T input): rows
  // i and i+1 in one pass over the window.  The two pivots need window columns
  // 0 and 1 only; every other entry is read and written once per two rows:
  //   W''(a-2, q-2) = W(a, q) - c_a c_q - d_{a-1} d_{q-1}
  // with c, d the Cholesky columns i, i+1.  The fresh rows i+K, i+K+1 of Q
  // arrive by cp.async in a per-thread slot after the window.
  T* slot = win + (K * (K + 1) / 2) * ts;  // [2][W][thread]
  auto fetch2 = [&](ix i) {
#pragma unroll
    for (int c = 0; c <= K; ++c) {
      cpa(slot + c * ts, qb + (i + c) * cs + (K - c) * 32);  // Q(i+K, i+c)
      cpa(slot + (W + c) * ts, qb + (i + 1 + c) * cs + (K - c) * 32);  // Q(i+K+1, i+1+c)
    }
    cpa_commit();
  };
  auto pair = [&](ix i) {
    cpa_wait();
    T q0[W], q1[W];
#pragma unroll
    for (int c = 0; c <= K; ++c) {
      q0[c] = slot[c * ts];
      q1[c] = slot[(W + c) * ts];
    }
    const T d0 = Wr(0, 0);
    if (!(double(d0) > kPivotFloor) && i >= s) fail = fail < i ? fail : i;
    const T r0 = rsq_t(d0), p0 = d0 * r0;  // one MUFU sequence on the pivot chain
    T c[W];
    c[0] = p0;
#pragma unroll
    for (int a = 1; a < K; ++a) c[a] = Wr(a, 0) * r0;
    c[K] = q0[0] * r0;
    // column 0 of the window after step i
    auto v = [&](int a1) { return a1 + 1 < K ? fma(-c[a1 + 1], c[1], Wr(a1 + 1, 1)) : fma(-c[K], c[1], q0[1]); };
    const T d1 = v(0);
    if (!(double(d1) > kPivotFloor) && i + 1 >= s) fail = fail < i + 1 ? fail : i + 1;
    const T r1 = rsq_t(d1), p1 = d1 * r1;
    T dd[W];
    dd[0] = p1;
#pragma unroll
    for (int a = 1; a < K; ++a) dd[a] = v(a) * r1;
    dd[K] = q1[0] * r1;
    fetch2(i + 2);
#pragma unroll
    for (int a = 2; a < K; ++a) {
#pragma unroll
      for (int q = 2; q <= a; ++q) Wr(a - 2, q - 2) = fma(-dd[a - 1], dd[q - 1], fma(-c[a], c[q], Wr(a, q)));
    }
#pragma unroll
    for (int q = 2; q <= K; ++q) Wr(K - 2, q - 2) = fma(-dd[K - 1], dd[q - 1], fma(-c[K], c[q], q0[q]));
#pragma unroll
    for (int q = 1; q <= K; ++q) Wr(K - 1, q - 1) = fma(-dd[K], dd[q], q1[q]);
    emit(i, c);
    emit(i + 1, dd);
  };
  ix i = i0;
  if (K >= 2 && i + 1 < e && i + K + 3 < n) {
    fetch2(i);
#pragma unroll 1
    for (; i + 1 < e && i + K + 3 < n; i += 2) pair(i);
    cpa_wait();
  }
  T qn[W];
  load_row(i + K, qn);
#pragma unroll 1
  for (; i < e; ++i) {
    T q[W];
#pragma unroll
    for (int c = 0; c <= K; ++c) q[c] = qn[c];
    load_row(i + K + 1, qn);  // one row ahead
    const T d = Wr(0, 0);
    if (!(double(d) > kPivotFloor) && i >= s) fail = fail < i ? fail : i;
    const T rinv = rsq_t(d), piv = d * rinv;
    T l[W];
    l[0] = piv;
#pragma unroll
    for (int a = 1; a < K; ++a) l[a] = Wr(a, 0) * rinv;
    l[K] = (i + K < n) ? q[0] * rinv : T(0);
    emit(i, l);
#pragma unroll
    for (int a = 1; a < K; ++a) {
#pragma unroll
      for (int c = 1; c <= a; ++c) Wr(a - 1, c - 1) = fma(-l[a], l[c], Wr(a, c));
    }
#pragma unroll
    for (int c = 1; c <= K; ++c) Wr(K - 1, c - 1) = fma(-l[K], l[c], q[c]);
  }
  if (fail < n) atomicMin(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(fail));
}

template <class T, int K>
__global__ void k_chol(CholP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const Unit u = unit_of(G);
  if (!u.live) return;
  const ix s = ix(u.p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix i0 = s - G.burn > 0 ? s - G.burn : 0;
  chol_unit<T, K>(C, u.b, G.n, s, e, i0, u.p > 0 ? C.side + u.id * ix(K) * (K + 1) : nullptr,
                  sm + threadIdx.x);
}

template <class T, int K>
__global__ void k_chol_check(CholP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix id = t / K;
  const int c = int(t % K);
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  if (p == 0) return;
  const ix b = id / G.nseg, col = ix(p) * G.seg - K + c;
  const T* sd = C.side + (id * K + c) * (K + 1);
  double sc = 0.0;
  for (int r = 0; r <= K; ++r) sc = fmax(sc, dabs(C.l.cell(b, r, col)));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int r = 0; r <= K; ++r) bad |= !(fabs(double(sd[r]) - double(C.l.cell(b, r, col))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K>
__global__ void k_chol_repair(CholP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  C.fail[b] = G.n;
  chol_unit<T, K>(C, b, G.n, 0, G.n, 0, nullptr, sm + threadIdx.x);
}

// ------------------------------------------------------------------ solves
template <class T>
struct SolveP {
  Band<T> l;
  Vec<T> v, x;
  T* side;  // [unit][K]
  int32_t* flag;
  int64_t* fail;  // singular pivots (first row forward, last row + 1 backward)
};

// Forward: res[a] = residual of row i+a; x_i = res[0] / L(i,i) (the
// reference divides, kernels_serial.cpp:47).  Backward: x window x[a] =
// x_{i+1+a}; x_i = (v_i - sum_a L(i+1+a, i) x[a]) / L(i,i).
template <class T, int K, bool TR>
__device__ void solve_unit(const SolveP<T>& C, ix b, ix n, ix s, ix e, ix start, T* side, int l2a, T* ring,
                           const T* carry = nullptr) {
  constexpr int W = K + 1;
  const T* lb = bbase(C.l, b);
  const T* vb = vbase(C.v, b);
  T* xb = vbase(C.x, b);
  const ix cs = ix(W) * 32;
  auto load_col = [&](ix j, T* out, T& vv) {
    const bool in = j >= 0 && j < n;
#pragma unroll
    for (int a = 0; a <= K; ++a) out[a] = (in && j + a < n) ? lb[j * cs + a * 32] : T(0);
    const ix vr = TR ? j : j + K + 1;
    vv = (vr >= 0 && vr < n) ? vb[vr * 32] : T(0);
  };
  T win[W];
  if (!TR) {
#pragma unroll
    for (int a = 0; a <= K; ++a) win[a] = (start + a < n) ? vb[(start + a) * 32] : T(0);
    if (carry) {  // exact carry-in: x_{s-K .. s-1} known; start == s
#pragma unroll
      for (int a = 0; a <= K; ++a) {
        const ix r = start + a;
        if (r >= n) continue;
#pragma unroll
        for (int m = 0; m < K; ++m) {  // column start-K+m, row r: cell r - (start-K+m)
          const ix c = start - K + m;
          const int cell = int(r - c);
          if (c >= 0 && cell <= K) win[a] = fma(-lb[c * cs + cell * 32], carry[m], win[a]);
        }
      }
    }
  } else {
#pragma unroll
    for (int a = 0; a <= K; ++a) win[a] = (carry && a < K) ? carry[a] : T(0);
  }
  // rows stream through a ring of PF prefetched columns (static register
  // indices: the row loop is unrolled by PF); the tile's columns further
  // ahead are pulled into L2 by one bulk prefetch per PF rows (a column of
  // the 32 interleaved matrices is w * 256 contiguous bytes).
  constexpr int PF = solve_pf<K>();
  const int dir = TR ? -1 : 1;
  const ix stop = TR ? s - 1 : e;
  const ix rows = TR ? start - stop : stop - start;
  // rows stream through a per-thread shared-memory ring of PF slots
  // ([slot][cell][thread]) filled by cp.async PF rows ahead; the tile's
  // columns further ahead are pulled into L2 by one bulk prefetch per PF rows
  constexpr int ts = kThreads;
  auto issue = [&](ix j, int q) {
    if (j >= 0 && j < n) {
      T* d = ring + q * (W + 1) * ts;
#pragma unroll
      for (int a = 0; a <= K; ++a)
        if (j + a < n) cpa(d + a * ts, lb + j * cs + a * 32);
      const ix vr = TR ? j : j + K + 1;
      if (vr >= 0 && vr < n) cpa(d + W * ts, vb + vr * 32);
    }
    cpa_commit();
  };
  auto take = [&](ix j, int q, T* col, T& vv) {
    const T* d = ring + q * (W + 1) * ts;
    const bool in = j >= 0 && j < n;
#pragma unroll
    for (int a = 0; a <= K; ++a) col[a] = (in && j + a < n) ? d[a * ts] : T(0);
    const ix vr = TR ? j : j + K + 1;
    vv = (in && vr >= 0 && vr < n) ? d[W * ts] : T(0);
  };
  auto l2_ahead = [&](ix i) {
    const ix lo = TR ? i - l2a - PF + 1 : i + l2a, hi = lo + PF - 1;
    if (l2a > 0 && lo >= 0 && hi < n)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lb - (b & 31) + lo * cs),
                   "r"(unsigned(PF * cs * sizeof(T)))
                   : "memory");
  };
  int same = 0;
  ix sing = -1;  // pass 1 vets the pivots of its own rows (kernels.cpp:43-45)
  auto row = [&](ix i, const T* col, T vv) {
    T xi;
    if (!TR) {
      xi = win[0] / col[0];
#pragma unroll
      for (int a = 1; a <= K; ++a) win[a - 1] = fma(-col[a], xi, win[a]);
      win[K] = vv;  // v_{i+K+1}
    } else {
      T acc = T(0);
#pragma unroll
      for (int a = 1; a <= K; ++a) acc = fma(col[a], win[a - 1], acc);
      xi = (vv - acc) / col[0];
#pragma unroll
      for (int a = K - 1; a >= 1; --a) win[a] = win[a - 1];
      win[0] = xi;
    }
    if (i >= s && i < e) {
      if (!carry && sing < 0 && dabs(col[0]) < kPivotFloor) sing = i;  // first met: lowest forward, highest backward
      if (carry) {  // fix-up: K consecutive rows equal to pass 1 => same state => pass 1 is exact onwards
        const T old = xb[i * 32];
        same = (__double_as_longlong(double(old)) == __double_as_longlong(double(xi))) ? same + 1 : 0;
      }
      xb[i * 32] = xi;
    } else if (side) {
      const ix o = TR ? i - e : i - (s - K);
      if (o >= 0 && o < K) side[o] = xi;
    }
  };
#pragma unroll
  for (int q = 0; q < PF; ++q) issue(start + q * dir, q);
  ix i = start;
#pragma unroll 1
  for (ix blk = 0; blk < rows; blk += PF) {
    if ((threadIdx.x & 31) == 0) l2_ahead(i);
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      if (i == stop) break;
      T col[W], vv;
      asm volatile("cp.async.wait_group %0;" ::"n"(PF - 1) : "memory");  // row i's group has landed
      take(i, q, col, vv);
      issue(i + PF * dir, q);  // refill the slot PF rows ahead
      row(i, col, vv);
      i += dir;
    }
    if (carry && same >= K) break;
  }
  cpa_wait();
  if (sing >= 0) {
    if (!TR) atomicMin(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(sing));
    else atomicMax(reinterpret_cast<unsigned long long*>(C.fail + b), static_cast<unsigned long long>(sing + 1));
  }
}

template <class T, int K, bool TR>
__global__ void k_solve(SolveP<T> C, Geo G) {
  const Unit u = unit_of(G);
  if (!u.live) return;
  const ix s = ix(u.p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  ix start;
  T* side = nullptr;
  if (!TR) {
    start = s - G.burn > 0 ? s - G.burn : 0;
    if (u.p > 0) side = C.side + u.id * K;
  } else {
    start = e + G.burn - 1 < G.n - 1 ? e + G.burn - 1 : G.n - 1;
    if (u.p + 1 < G.nseg) side = C.side + u.id * K;
  }
  extern __shared__ __align__(16) unsigned char smraw[];
  solve_unit<T, K, TR>(C, u.b, G.n, s, e, start, side, G.l2a, reinterpret_cast<T*>(smraw) + threadIdx.x);
}

template <class T, int K, bool TR>
__global__ void k_solve_check(SolveP<T> C, Geo G, int32_t* uflag) {
  const ix id = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  if (TR ? p + 1 >= G.nseg : p == 0) return;
  const ix b = id / G.nseg;
  const ix r0 = TR ? ix(p + 1) * G.seg : ix(p) * G.seg - K;
  // bitwise: the fix-up of a flagged segment stops as soon as it rejoins pass 1,
  // so an exact check costs only the rows the burn-in had not yet converged
  bool bad = false;
  for (int c = 0; c < K; ++c)
    if (r0 + c < G.n) bad |= C.side[id * K + c] != C.x(b, r0 + c);
  uflag[id] = bad ? 1 : 0;
}

template <class T, int K, bool TR>
__global__ void k_solve_repair(SolveP<T> C, Geo G) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  solve_unit<T, K, TR>(C, b, G.n, 0, G.n, TR ? G.n - 1 : 0, nullptr, G.l2a, reinterpret_cast<T*>(smraw) + threadIdx.x);
}

// Fix-up of segments whose burn-in did not converge: the neighbour's genuine
// boundary values (snapshot) give the exact carry-in, and the segment is
// recomputed from it.  A re-check then confirms the snapshot the next
// segment used was itself final; anything else goes to the full repair.
template <class T, int K, bool TR>
__global__ void k_solve_snap(SolveP<T> C, Geo G, T* snap) {
  const ix id = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  const ix b = id / G.nseg, s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  for (int c = 0; c < K; ++c) {
    const ix r = TR ? s + c : e - K + c;
    snap[id * K + c] = (r >= 0 && r < G.n) ? C.x(b, r) : T(0);
  }
}

template <class T, int K, bool TR>
__global__ void k_solve_fix(SolveP<T> C, Geo G, const int32_t* uflag, const T* snap) {
  const Unit u = unit_of(G);
  if (!u.live || !uflag[u.id]) return;
  const ix s = ix(u.p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const T* carry = snap + (TR ? u.id + 1 : u.id - 1) * K;
  extern __shared__ __align__(16) unsigned char smraw[];
  solve_unit<T, K, TR>(C, u.b, G.n, s, e, TR ? e - 1 : s, nullptr, G.l2a, reinterpret_cast<T*>(smraw) + threadIdx.x,
                       carry);
}

template <class T, int K, bool TR>
__global__ void k_solve_recheck(SolveP<T> C, Geo G, const int32_t* uflag, const T* snap) {
  const ix id = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (id >= G.batch * G.nseg || !uflag[id]) return;
  const int p = int(id % G.nseg);
  if (TR ? p == 0 : p + 1 >= G.nseg) return;  // nobody downstream
  const ix b = id / G.nseg, s = ix(p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  double sc = 0.0;
  for (int c = 0; c < K; ++c) sc = fmax(sc, dabs(snap[id * K + c]));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int c = 0; c < K; ++c) {
    const ix r = TR ? s + c : e - K + c;
    if (r >= 0 && r < G.n) bad |= !(fabs(double(C.x(b, r)) - double(snap[id * K + c])) <= tol * (sc + 1e-300));
  }
  if (bad) C.flag[b] = 1;
}


// ------------------------------------------------------------------ subset
// Column-form Takahashi (see bgm_wide.cu): window S over rows j+1 .. j+K,
// packed lower triangle [entry][thread], index x <-> row j+1+x.
template <class T>
struct SubP {
  Band<T> l, s;
  T* side;  // [unit][K][K+1]
  int32_t* flag;
};

template <class T, int K>
__device__ void subset_unit(const SubP<T>& C, ix b, ix n, ix s, ix e, ix jtop, T* side, T* win) {
  constexpr int W = K + 1, ts = kThreads;
  auto Sr = [&](int x, int y) -> T& { return win[tri(x, y) * ts]; };
  const T* lb = bbase(C.l, b);
  T* sb = bbase(C.s, b);
  const ix cs = ix(W) * 32;
#pragma unroll 1
  for (int q = 0; q < K * (K + 1) / 2; ++q) win[q * ts] = T(0);
  auto load_col = [&](ix j, T* out) {
    const bool in = j >= 0 && j < n;
#pragma unroll
    for (int a = 0; a <= K; ++a) out[a] = (in && j + a < n) ? lb[j * cs + a * 32] : T(0);
  };
  T cn[W];
  load_col(jtop, cn);
#pragma unroll 1
  for (ix j = jtop; j >= s; --j) {
    T lc[W];
#pragma unroll
    for (int a = 0; a <= K; ++a) lc[a] = cn[a];
    load_col(j - 1, cn);
    const T inv = T(1) / lc[0];
    T out[K];
#pragma unroll
    for (int x = 0; x < K; ++x) out[x] = T(0);
    // out = S(window) lc(1..K); entries shifted (x,y) -> (x+1,y+1) in place
#pragma unroll
    for (int x = K - 1; x >= 0; --x) {
#pragma unroll
      for (int y = x; y >= 0; --y) {
        const T sv = Sr(x, y);
        if (x < K - 1) Sr(x + 1, y + 1) = sv;
        out[x] = fma(sv, lc[y + 1], out[x]);
        if (y != x) out[y] = fma(sv, lc[x + 1], out[y]);
      }
    }
    T dot = T(0);
#pragma unroll
    for (int x = 0; x < K; ++x) {
      out[x] = -out[x] * inv;  // S(j+1+x, j)
      dot = fma(lc[x + 1], out[x], dot);
    }
    const T sjj = inv * inv - inv * dot;
    Sr(0, 0) = sjj;
#pragma unroll
    for (int x = 1; x < K; ++x) Sr(x, 0) = out[x - 1];
    if (j < e) {
      T* col = sb + j * cs;
      col[0] = sjj;
#pragma unroll
      for (int x = 0; x < K; ++x) col[(x + 1) * 32] = (j + 1 + x < n) ? out[x] : T(0);
    } else if (side && j < e + K) {
      T* sd = side + (j - e) * W;
      sd[0] = sjj;
#pragma unroll
      for (int x = 0; x < K; ++x) sd[x + 1] = (j + 1 + x < n) ? out[x] : T(0);
    }
  }
}

template <class T, int K>
__global__ void k_subset(SubP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const Unit u = unit_of(G);
  if (!u.live) return;
  const ix s = ix(u.p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix jtop = e + G.burn - 1 < G.n - 1 ? e + G.burn - 1 : G.n - 1;
  subset_unit<T, K>(C, u.b, G.n, s, e, jtop, u.p + 1 < G.nseg ? C.side + u.id * ix(K) * (K + 1) : nullptr,
                    sm + threadIdx.x);
}

template <class T, int K>
__global__ void k_subset_check(SubP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix id = t / K;
  const int c = int(t % K);
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  if (p + 1 >= G.nseg) return;
  const ix b = id / G.nseg, col = ix(p + 1) * G.seg + c;
  if (col >= G.n) return;
  const T* sd = C.side + (id * K + c) * (K + 1);
  double sc = 0.0;
  for (int r = 0; r <= K; ++r) sc = fmax(sc, dabs(C.s.cell(b, r, col)));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int r = 0; r <= K; ++r) bad |= !(fabs(double(sd[r]) - double(C.s.cell(b, r, col))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K>
__global__ void k_subset_repair(SubP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  subset_unit<T, K>(C, b, G.n, 0, G.n, G.n - 1, nullptr, sm + threadIdx.x);
}

// First pivot below the floor per matrix: thread per (matrix, 64-row chunk),
// one index split per thread (not per element), one atomic per chunk.
template <class T>
__global__ void k_diag_small(Band<T> l, ix batch, ix chunks, int64_t* fail) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, c;
  if (!split_bj(t, batch, chunks, l.s, b, c)) return;
  const ix i1 = (c + 1) * 64 < l.n ? (c + 1) * 64 : l.n;
  ix bad = -1;
#pragma unroll 8
  for (ix i = c * 64; i < i1; ++i)
    if (bad < 0 && dabs(l.cell(b, 0, i)) < kPivotFloor) bad = i;
  if (bad >= 0) atomicMin(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(bad));
}

// ------------------------------------------------------------------ vjp_cholesky
// Reverse of the right-looking column Cholesky (the same gradient as Giles'
// row sweep of grad.cpp:11-36, in the order that reads every input once):
// the forward's column j sets L(j,j) = sqrt(A(j,j)), L(i,j) = A(i,j)/L(j,j)
// and updates the trailing K x K window A(i,i') -= L(i,j) L(i',j), so from
// the bottom up, with Ab the (lower-stored, final) q_bar window of the rows
// below j,
//   g_x = l_bar(j+1+x, j) - sum_y (Ab + Ab^T)(x, y) L(j+1+y, j)
//   q_bar(j+1+x, j) = g_x / L(j,j)
//   q_bar(j, j) = (l_bar(j,j) - sum_x g_x L(j+1+x, j) / L(j,j)) / (2 L(j,j)).
// Window: Ab over rows/cols (j, j+K], packed [entry][thread]; one pass reads
// each entry once (two FMAs) and moves it to (x+1, y+1) in memmove order, the
// new column enters at y = 0.  Input columns are read once, coalesced across
// the warp's 32 matrices.
template <class T>
struct VcholP {
  Band<T> l, lb, qb;
  int l2a;
  T* side;  // [unit][K][K+1]: burn-in q_bar columns [e, e+K)
  int32_t* flag;
};

#ifndef VCHOL_FENCE
#define VCHOL_FENCE 4
#endif

#ifndef VCHOL_SLOT
#define VCHOL_SLOT 1  // vjp_cholesky pairs: the next pair's columns by cp.async into a slot
#endif
template <class T, int K>
__device__ void vchol_unit(const VcholP<T>& C, ix b, ix n, ix s, ix e, ix start, T* side, T* win) {
  constexpr int W = K + 1, ts = kThreads;
  auto Wa = [&](int x, int y) -> T& { return win[tri(x, y) * ts]; };
  const T* lbase = bbase(C.l, b);
  const T* gbase = bbase(C.lb, b);
  T* qbase = bbase(C.qb, b);
  const ix cs = ix(W) * 32;
#pragma unroll
  for (int x = 0; x < K * (K + 1) / 2; ++x) win[x * ts] = T(0);  // burn-in (or rows past n)
  auto load = [&](ix j, T* u, T* g, T& d, T& gd) {
    const T* lc = lbase + j * cs;
    const T* gc = gbase + j * cs;
#pragma unroll
    for (int x = 0; x < K; ++x) {
      const bool in = j + 1 + x < n;
      u[x] = in ? lc[(x + 1) * 32] : T(0);
      g[x] = in ? gc[(x + 1) * 32] : T(0);
    }
    d = lc[0];
    gd = gc[0];
  };
  auto emit = [&](ix j, T ad, const T* a) {
    if (j < e) {
      T* qc = qbase + j * cs;
      qc[0] = ad;
#pragma unroll
      for (int x = 0; x < K; ++x) qc[(x + 1) * 32] = (j + 1 + x < n) ? a[x] : T(0);
    } else if (side && j < e + K) {
      T* sd = side + (j - e) * W;
      sd[0] = ad;
#pragma unroll
      for (int x = 0; x < K; ++x) sd[x + 1] = (j + 1 + x < n) ? a[x] : T(0);
    }
  };
  auto finish = [&](const T* u, const T* g, T d, T gd, T* a) {
    const T rd = T(1) / d;
#pragma unroll
    for (int x = 0; x < K; ++x) {
      a[x] = g[x] * rd;
      gd = fma(-a[x], u[x], gd);
    }
    return T(0.5) * gd * rd;
  };
  ix j = start;
  // ---- paired rows j, j-1 in one pass over the window: each entry v at
  // (x, y) feeds row j's g at (x, y) and row j-1's at (x+1, y+1), and moves
  // two places down the diagonal; row j's new column (the window's column 0
  // after row j) is folded into row j-1 after the pass.
  const int L2A = C.l2a;  // L2 bulk prefetch distance (columns) of L and L-bar, per tile (0 = off)
#if VCHOL_SLOT
  // cp.async slot after the window: [4 columns: L j, L-bar j, L j-1, L-bar j-1][W][thread]
  T* vslot = win + (K * (K + 1) / 2) * ts;
  bool slot_ready = false;
  auto fetch4 = [&](ix jj) {  // columns jj, jj-1 of L and L-bar (all in [0, n))
#pragma unroll
    for (int r = 0; r < W; ++r) {
      cpa(vslot + (0 * W + r) * ts, lbase + jj * cs + r * 32);
      cpa(vslot + (1 * W + r) * ts, gbase + jj * cs + r * 32);
      cpa(vslot + (2 * W + r) * ts, lbase + (jj - 1) * cs + r * 32);
      cpa(vslot + (3 * W + r) * ts, gbase + (jj - 1) * cs + r * 32);
    }
    cpa_commit();
  };
#endif
  const T* ltile = lbase - (b & 31);
  const T* gtile = gbase - (b & 31);
#pragma unroll 1
  for (; j - 1 >= s; j -= 2) {
    if (L2A > 0 && (threadIdx.x & 31) == 0 && j - 1 - L2A >= 0) {
      const unsigned bytes = unsigned(2 * cs * sizeof(T));
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ltile + (j - 1 - L2A) * cs), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gtile + (j - 1 - L2A) * cs), "r"(bytes) : "memory");
    }
    T u[K], g[K], u2[K], g2[K], d, gd, d2, gd2;
#if VCHOL_SLOT
    // the pair's four columns arrived by cp.async during the previous pair
    if (!slot_ready) fetch4(j);
    cpa_wait();
    auto take = [&](int c, ix jj, T* uu, T* gg, T& dd_, T& gdd) {
      const T* su = vslot + (2 * c) * W * ts;
      const T* sg = vslot + (2 * c + 1) * W * ts;
#pragma unroll
      for (int x = 0; x < K; ++x) {
        const bool in = jj + 1 + x < n;
        uu[x] = in ? su[(x + 1) * ts] : T(0);
        gg[x] = in ? sg[(x + 1) * ts] : T(0);
      }
      dd_ = su[0];
      gdd = sg[0];
    };
    take(0, j, u, g, d, gd);
    take(1, j - 1, u2, g2, d2, gd2);
    slot_ready = j - 3 >= s;
    if (slot_ready) fetch4(j - 2);
#else
    load(j, u, g, d, gd);
    load(j - 1, u2, g2, d2, gd2);
#endif
#pragma unroll
    for (int x = K - 1; x >= 0; --x) {
#pragma unroll
      for (int y = x; y >= 0; --y) {
        const T v = Wa(x, y);
        if (x == y) {
          g[x] = fma(T(-2) * v, u[x], g[x]);
          if (x + 1 < K) g2[x + 1] = fma(T(-2) * v, u2[x + 1], g2[x + 1]);
        } else {
          g[x] = fma(-v, u[y], g[x]);
          g[y] = fma(-v, u[x], g[y]);
          if (x + 1 < K) {
            g2[x + 1] = fma(-v, u2[y + 1], g2[x + 1]);
            g2[y + 1] = fma(-v, u2[x + 1], g2[y + 1]);
          }
        }
        if (x + 2 < K) Wa(x + 2, y + 2) = v;
      }
      if (x % VCHOL_FENCE == 0) asm volatile("" ::: "memory");  // bound the hoisted window loads
    }
    T a[K], a2[K];
    const T ad = finish(u, g, d, gd, a);
    // row j's column (ad, a[0..K-2]) is window column 0 when row j-1 runs
    g2[0] = fma(T(-2) * ad, u2[0], g2[0]);
#pragma unroll
    for (int x = 0; x + 1 < K; ++x) {
      g2[x + 1] = fma(-a[x], u2[0], g2[x + 1]);
      g2[0] = fma(-a[x], u2[x + 1], g2[0]);
    }
    const T ad2 = finish(u2, g2, d2, gd2, a2);
    if (K >= 2) Wa(1, 1) = ad;
#pragma unroll
    for (int x = 0; x + 2 < K; ++x) Wa(x + 2, 1) = a[x];
    Wa(0, 0) = ad2;
#pragma unroll
    for (int x = 0; x + 1 < K; ++x) Wa(x + 1, 0) = a2[x];
    emit(j, ad, a);
    emit(j - 1, ad2, a2);
  }
#if VCHOL_SLOT
  cpa_wait();
#endif
#pragma unroll 1
  for (; j >= s; --j) {
    T u[K], g[K], d, gd;
    load(j, u, g, d, gd);
#pragma unroll
    for (int x = K - 1; x >= 0; --x) {
#pragma unroll
      for (int y = x; y >= 0; --y) {
        const T v = Wa(x, y);
        if (x == y) {
          g[x] = fma(T(-2) * v, u[x], g[x]);
        } else {
          g[x] = fma(-v, u[y], g[x]);
          g[y] = fma(-v, u[x], g[y]);
        }
        if (x < K - 1) Wa(x + 1, y + 1) = v;
      }
      if (x % VCHOL_FENCE == 0) asm volatile("" ::: "memory");
    }
    T a[K];
    const T ad = finish(u, g, d, gd, a);
    Wa(0, 0) = ad;
#pragma unroll
    for (int x = 0; x + 1 < K; ++x) Wa(x + 1, 0) = a[x];
    emit(j, ad, a);
  }
}

template <class T, int K>
__global__ void k_vchol(VcholP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const Unit u = unit_of(G);
  if (!u.live) return;
  const ix s = ix(u.p) * G.seg, e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix start = e + G.burn - 1 < G.n - 1 ? e + G.burn - 1 : G.n - 1;
  vchol_unit<T, K>(C, u.b, G.n, s, e, start, u.p + 1 < G.nseg ? C.side + u.id * ix(K) * (K + 1) : nullptr,
                   sm + threadIdx.x);
}

// thread per (unit, column): q_bar columns [e, e+K) from burn-in vs genuine
template <class T, int K>
__global__ void k_vchol_check(VcholP<T> C, Geo G) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const ix id = t / K;
  const int c = int(t % K);
  if (id >= G.batch * G.nseg) return;
  const int p = int(id % G.nseg);
  if (p + 1 >= G.nseg) return;
  const ix b = id / G.nseg, j = ix(p + 1) * G.seg + c;
  if (j >= G.n) return;
  const T* sd = C.side + (id * K + c) * (K + 1);
  double sc = 0.0;
  for (int r = 0; r <= K; ++r) sc = fmax(sc, dabs(C.qb.cell(b, r, j)));
  const double tol = sizeof(T) == 8 ? kCheckTol : 1e-5;
  bool bad = false;
  for (int r = 0; r <= K; ++r) bad |= !(fabs(double(sd[r]) - double(C.qb.cell(b, r, j))) <= tol * (sc + 1e-300));
  if (bad) C.flag[b] = 1;
}

template <class T, int K>
__global__ void k_vchol_repair(VcholP<T> C, Geo G) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= G.batch || !C.flag[b]) return;
  vchol_unit<T, K>(C, b, G.n, 0, G.n, G.n - 1, nullptr, sm + threadIdx.x);
}

// corner cells (j + r >= n) of an output band are exact zeros
template <class T>
__global__ void k_zero_corners(Band<T> o, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  const int K = o.lo;
  ix b, jj;
  if (!split_bj(t, batch, ix(K) * (K + 1), o.s, b, jj)) return;
  const ix j = o.n - K + jj / (K + 1);
  const int r = int(jj % (K + 1));
  if (j >= 0 && j + r >= o.n) o.cell(b, r, j) = T(0);
}

// ------------------------------------------------------------------ common
__global__ void k_init(int64_t* fail, int32_t* flag, ix batch, int64_t v) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  fail[b] = v;
  flag[b] = 0;
}

__global__ void k_report(const int64_t* fail, ix batch, ix n, int code, int backward, int32_t* status,
                         int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix f = backward ? fail[b] - 1 : fail[b];
  const bool ok = backward ? f < 0 : f >= n;
  report(status, row, b, ok ? BGM_OK : code, ok ? -1 : f);
}

int g_segment_rows = 0;

// Solves forget their carry-in more slowly than the Cholesky Schur window
// (the error of a zero start decays with L^-1, ~0.9 per row for config-0
// factors at k = 16, and the slowest of a warp's 32 matrices sets the pace):
// a longer burn-in, and flagged segments rejoin pass 1 bitwise (early exit).
int solve_burn_rows(int K) {
  int burn = 24 * K > kBurnMin ? 24 * K : kBurnMin;
  if (const char* bv = std::getenv("BGM_NARROW_BURN"))
    if (std::atoi(bv) >= 1) burn = std::atoi(bv);
  return burn;
}

int burn_rows(int K) {
  // narrow bands forget their start state fastest: k <= 4 config-0 factors
  // converge bit-exactly within ~20 rows (the check catches anything slower)
  int burn = K <= 4 ? 32 : kBurnGen * K > kBurnMin ? kBurnGen * K : kBurnMin;
  if (const char* bv = std::getenv("BGM_NARROW_BURN"))
    if (std::atoi(bv) >= 1) burn = std::atoi(bv);
  return burn;
}

template <class KernelT>
Geo make_geo(KernelT kern, size_t smem, ix batch, ix n, int burn, int segf_default = 4) {
  Geo G;
  G.batch = batch;
  G.n = n;
  G.tiles = (batch + 31) / 32;
  G.burn = burn;
  G.l2a = 8;
  if (const char* v = std::getenv("BGM_NARROW_L2AHEAD")) G.l2a = std::atoi(v);
  int sms = 148, dev = 0, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kThreads, smem);
  if (per < 1) per = 1;
  ix seg = requested_seg(g_segment_rows, 16)  /* widest narrow band */;
  if (seg <= 0) {
    ix nseg = ix(sms) * per / G.tiles;
    if (nseg < 1) nseg = 1;
    seg = (n + nseg - 1) / nseg;
    // few tiles (a small per-GPU batch): fill the SMs with short segments
    // rather than keep segments a multiple of the burn-in (B = 512 at k = 4:
    // 0.285 -> 0.20 ms for config 1's suite)
    const char* sv = std::getenv("BGM_NARROW_SEGF");
    const int segf = sv ? std::atoi(sv) : (G.tiles < kFewTiles ? 1 : segf_default);
    if (seg < segf * ix(burn)) seg = segf * ix(burn);
  }
  if (seg < 1) seg = 1;
  G.seg = seg;
  G.nseg = int((n + seg - 1) / seg);
  return G;
}

struct Scratch {
  char* p = nullptr;
  cudaStream_t s;
  ~Scratch() {
    if (p) scratch_free(p, s);
  }
};

template <class T, int K>
bool run_chol(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  const size_t smem = sizeof(T) * (K * (K + 1) / 2 + 2 * (K + 1)) * kThreads;  // window + pair slot
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_chol<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_chol_repair<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  const int burn = burn_rows(K);
  const Geo G = make_geo(k_chol<T, K>, smem, q.batch, q.n, burn);
  const ix units = G.batch * G.nseg;
  const size_t side = sizeof(T) * size_t(units) * K * (K + 1);
  Scratch ws;
  ws.s = s;
  if (scratch_alloc(reinterpret_cast<void**>(&ws.p), side + 12 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  CholP<T> C;
  C.q = view<T>(q);
  C.l = view<T>(l);
  C.side = reinterpret_cast<T*>(ws.p);
  C.fail = reinterpret_cast<int64_t*>(ws.p + (side + 7) / 8 * 8);
  C.flag = reinterpret_cast<int32_t*>(C.fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, C.flag, G.batch, G.n);
  {
    timing::Scope t("narrow_chol", s);
    k_chol<T, K><<<unsigned(G.tiles * G.nseg), kThreads, smem, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_chol_check", s);
    k_chol_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_chol_repair", s);
    k_chol_repair<T, K><<<blocks_for(G.batch, kThreads), kThreads, smem, s>>>(C, G);
  }
  k_report<<<blocks_for(G.batch, 128), 128, 0, s>>>(C.fail, G.batch, G.n, BGM_ERR_NOT_PD, 0, st, row);
  return true;
}

template <class T, int K, bool TR>
bool run_solve(const bgm_band& l, const bgm_vec& v, const bgm_vec& x, int32_t* st, int64_t* row, cudaStream_t s) {
  int burn = solve_burn_rows(K);
  // k <= 4 with few tiles: short segments, so a 48-row burn-in (the bitwise
  // early-exit fix-up covers the rare unconverged carry-in) beats 96
  if (K <= 4 && (l.batch + 31) / 32 < kFewTiles && !std::getenv("BGM_NARROW_BURN")) burn = 48;
  const size_t smem = sizeof(T) * solve_pf<K>() * (K + 2) * kThreads;  // the per-thread row ring
  const Geo G = make_geo(k_solve<T, K, TR>, smem, l.batch, l.n, burn, 2);
  const ix units = G.batch * G.nseg;
  const size_t side = sizeof(T) * size_t(units) * K;
  Scratch ws;
  ws.s = s;
  const size_t bytes = 2 * side + sizeof(int32_t) * size_t(units) + 12 * size_t(G.batch) + 128;
  if (scratch_alloc(reinterpret_cast<void**>(&ws.p), bytes, s) != cudaSuccess) return false;
  SolveP<T> C;
  C.l = view<T>(l);
  C.v = view<T>(v);
  C.x = view<T>(x);
  C.side = reinterpret_cast<T*>(ws.p);
  T* snap = reinterpret_cast<T*>(ws.p + side);
  int64_t* fail = reinterpret_cast<int64_t*>(ws.p + (2 * side + 7) / 8 * 8);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  C.fail = fail;
  int32_t* uflag = C.flag + G.batch;
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, TR ? 0 : G.n);
  {
    timing::Scope t(TR ? "narrow_solve_t" : "narrow_solve", s);
    k_solve<T, K, TR><<<unsigned(G.tiles * G.nseg), kThreads, smem, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_solve_check", s);
    k_solve_check<T, K, TR><<<blocks_for(units, 128), 128, 0, s>>>(C, G, uflag);
    k_solve_snap<T, K, TR><<<blocks_for(units, 128), 128, 0, s>>>(C, G, snap);
  }
  {
    timing::Scope t("narrow_solve_fix", s);
    k_solve_fix<T, K, TR><<<unsigned(G.tiles * G.nseg), kThreads, smem, s>>>(C, G, uflag, snap);
    k_solve_recheck<T, K, TR><<<blocks_for(units, 128), 128, 0, s>>>(C, G, uflag, snap);
  }
  {
    timing::Scope t("narrow_solve_repair", s);
    k_solve_repair<T, K, TR><<<blocks_for(G.batch, kThreads), kThreads, smem, s>>>(C, G);
  }
  k_report<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, TR, st, row);
  return true;
}

template <class T, int K>
bool run_subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  const size_t smem = sizeof(T) * (K * (K + 1) / 2) * kThreads;
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_subset<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_subset_repair<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  const int burn = burn_rows(K);
  const Geo G = make_geo(k_subset<T, K>, smem, l.batch, l.n, burn);
  const ix units = G.batch * G.nseg;
  const size_t side = sizeof(T) * size_t(units) * K * (K + 1);
  Scratch ws;
  ws.s = s;
  if (scratch_alloc(reinterpret_cast<void**>(&ws.p), side + 12 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  SubP<T> C;
  C.l = view<T>(l);
  C.s = view<T>(sb);
  C.side = reinterpret_cast<T*>(ws.p);
  int64_t* fail = reinterpret_cast<int64_t*>(ws.p + (side + 7) / 8 * 8);
  C.flag = reinterpret_cast<int32_t*>(fail + G.batch);
  k_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, G.n);
  const ix dchunks = (G.n + 63) / 64;
  k_diag_small<T><<<blocks_for(G.tiles * 32 * dchunks, 256), 256, 0, s>>>(C.l, G.batch, dchunks, fail);
  {
    timing::Scope t("narrow_subset", s);
    k_subset<T, K><<<unsigned(G.tiles * G.nseg), kThreads, smem, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_subset_check", s);
    k_subset_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_subset_repair", s);
    k_subset_repair<T, K><<<blocks_for(G.batch, kThreads), kThreads, smem, s>>>(C, G);
  }
  k_report<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, BGM_ERR_SINGULAR, 0, st, row);
  return true;
}

template <class T, int K>
bool run_vchol(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  const size_t smem = sizeof(T) * ((K + 1) * (K + 2) / 2 + (VCHOL_SLOT ? 4 * (K + 1) : 0)) * kThreads;
  static PerDevice attr;
  if (attr.first()) {
    cudaFuncSetAttribute(k_vchol<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_vchol_repair<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr.mark();
  }
  const Geo G = make_geo(k_vchol<T, K>, smem, l.batch, l.n, kBurnGen * K > kBurnMin ? kBurnGen * K : kBurnMin);
  const ix units = G.batch * G.nseg;
  const size_t side = sizeof(T) * size_t(units) * K * (K + 1);
  Scratch ws;
  ws.s = s;
  if (scratch_alloc(reinterpret_cast<void**>(&ws.p), side + 8 * size_t(G.batch) + 64, s) != cudaSuccess) return false;
  VcholP<T> C;
  C.l = view<T>(l);
  C.lb = view<T>(lb);
  C.qb = view<T>(qb);
  C.l2a = 4;  // measured best of 0 / 4 / 16 at k = 8, 16
  if (const char* v = std::getenv("BGM_VCHOL_L2A")) C.l2a = std::atoi(v);
  C.side = reinterpret_cast<T*>(ws.p);
  C.flag = reinterpret_cast<int32_t*>(ws.p + (side + 7) / 8 * 8);
  cudaMemsetAsync(C.flag, 0, sizeof(int32_t) * size_t(G.batch), s);
  {
    timing::Scope t("narrow_vjp_chol", s);
    k_vchol<T, K><<<unsigned(G.tiles * G.nseg), kThreads, smem, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_vjp_chol_check", s);
    k_vchol_check<T, K><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope t("narrow_vjp_chol_repair", s);
    k_vchol_repair<T, K><<<blocks_for(G.batch, kThreads), kThreads, smem, s>>>(C, G);
  }
  k_zero_corners<T><<<blocks_for(G.tiles * 32 * K * (K + 1), 128), 128, 0, s>>>(C.qb, G.batch);
  return true;
}

bool shape_ok(const bgm_band& b) {
  // tile 32 (coalesced per-cell warp accesses) and long enough to segment
  return b.tile == 32 && b.upper == 0 && b.batch > 0 && b.n >= 64 && b.lower >= 1 && b.lower <= 16;
}

}  // namespace

#define BGM_NARROW_K(X) X(1) X(2) X(3) X(4) X(8) X(16)

bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  if (!shape_ok(q) || l.tile != 32 || l.lower != q.lower) return false;
  const bool f64 = q.dtype == BGM_F64;
  switch (q.lower) {
#define C_(KK) \
  case KK: return f64 ? run_chol<double, KK>(q, l, st, row, s) : run_chol<float, KK>(q, l, st, row, s);
    BGM_NARROW_K(C_)
#undef C_
    default: return false;
  }
}

bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s) {
  if (!shape_ok(l) || v.tile != 32 || x.tile != 32) return false;
  const bool f64 = l.dtype == BGM_F64;
  switch (l.lower) {
#define S_(KK)                                                                                              \
  case KK:                                                                                                  \
    if (f64) return tr ? run_solve<double, KK, true>(l, v, x, st, row, s) : run_solve<double, KK, false>(l, v, x, st, row, s); \
    return tr ? run_solve<float, KK, true>(l, v, x, st, row, s) : run_solve<float, KK, false>(l, v, x, st, row, s);
    BGM_NARROW_K(S_)
#undef S_
    default: return false;
  }
}

bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  if (!shape_ok(l) || sb.tile != 32 || sb.lower != l.lower) return false;
  const bool f64 = l.dtype == BGM_F64;
  switch (l.lower) {
#define U_(KK) \
  case KK: return f64 ? run_subset<double, KK>(l, sb, st, row, s) : run_subset<float, KK>(l, sb, st, row, s);
    BGM_NARROW_K(U_)
#undef U_
    default: return false;
  }
}

bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  if (!shape_ok(l) || lb.tile != 32 || qb.tile != 32 || lb.lower != l.lower || qb.lower != l.lower ||
      lb.upper != 0 || qb.upper != 0)
    return false;
  const bool f64 = l.dtype == BGM_F64;
  switch (l.lower) {
#define V_(KK) \
  case KK: return f64 ? run_vchol<double, KK>(l, lb, qb, s) : run_vchol<float, KK>(l, lb, qb, s);
    BGM_NARROW_K(V_)
#undef V_
    default: return false;
  }
}

void set_segment_rows(int rows) { g_segment_rows = rows; }

}  // namespace narrow
}  // namespace bgm
