// Blocked wide-band triangular solves (k = 64, 128; reference layout), one warp
// per (matrix, segment): L x = v forward, L^T x = v backward
// (kernels_serial.cpp:34-60).  Replaces the row-at-a-time kernels of
// bgm_wide.cu (three warp barriers, a shared-memory window update and a
// butterfly sum per ROW: ~1200 clk per row, 0.18-0.3 of the HBM roofline).
//
// Panels of 8 columns.  A panel is 8 (K+1)-cell columns, contiguous in the
// reference layout, so it arrives as ONE bulk copy (cp.async.bulk, mbarrier
// completion) into a ring kD panels deep.  Per panel the row-to-row
// dependency chain is confined to two 8x8 blocks that every lane evaluates
// redundantly from broadcast shared-memory reads (no shuffles, no barriers):
//   forward   x_P = L_PP^-1 r_P (substitution with reciprocals taken a panel
//             ahead), then the NEXT panel's 8 residuals r -= L_NP x_P;
//   backward  rhs_P = v_P - far_P - L_NP^T x_N with x_N the previous panel's
//             solution in registers, then substitution with L_PP^T.
// Everything else is off the chain and lane-parallel: forward, the residual
// window rows beyond the next panel take their rank-8 update in shared
// memory; backward, the dot products of the panel's columns with the solution
// window beyond the previous panel are formed ONE PANEL AHEAD (8 partial sums
// per lane, a 9-shuffle transpose reduction) and parked in shared memory.
// Long matrices are cut into segments with a burn-in, a check of the burn-in
// copies against the neighbour's genuine values, and an exact single-unit
// recomputation of flagged matrices, as in bgm_wide.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_timing.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace wide {
namespace {

constexpr double kCheckTol = 1e-12;  // as bgm_wide.cu
constexpr int kBurnGen = 6;
constexpr int kD = 4;  // panels in the ring (3 in flight)

struct Geo {
  ix batch, n, seg;
  int nseg, burn;
};

template <class T>
struct SolveP {
  Band<T> l;
  Vec<T> v, x;
  T* side;  // [unit][K] burn-in copies of the K solution values next to the segment
  int32_t* flag;
};

template <class T, int K>
struct SolveSmem {
  static constexpr int W = K + 1, CELLS = 8 * W, M = K + 16 <= 128 ? 128 : 256;
  static_assert((CELLS * sizeof(T)) % 16 == 0, "a panel is a whole number of 16-byte units");
  alignas(16) T ring[kD][CELLS];
  alignas(16) T pv[kD][8];
  alignas(16) double win[M];     // forward: residuals; backward: solution values (row mod M)
  alignas(16) double far[2][8];  // backward: far dot products of the next panel
  alignas(8) unsigned long long bar[kD];
};

__device__ __forceinline__ unsigned sptr(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra WAIT_DONE;\n"
      "bra WAIT_LOOP;\n"
      "WAIT_DONE:\n"
      "}" ::"r"(sptr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sptr(dst)),
               "l"(src), "r"(bytes), "r"(sptr(b))
               : "memory");
}
template <class T>
__device__ __forceinline__ void cpa(T* dst, const T* src) {
  if (sizeof(T) == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sptr(dst)), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sptr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// lane c (< 8) takes -1 / L(g+c, g+c) of the panel in `P` (negated: the substitution then needs no
// negation on its chain); every lane gets all eight
template <class T, int K>
__device__ __forceinline__ void recips(const T* P, int lane, double* ri) {
  const double d = double(P[(lane & 7) * (K + 1)]);
  const double rc = -1.0 / d;
#pragma unroll
  for (int c = 0; c < 8; ++c) ri[c] = __shfl_sync(0xffffffffu, rc, c);
}

// ---------------------------------------------------------------- forward, L x = v
template <class T, int K>
__device__ void fwd_unit(const SolveP<T>& C, ix b, int n, int s, int e, int start, T* side, SolveSmem<T, K>& sm) {
  using S = SolveSmem<T, K>;
  constexpr int W = S::W, M = S::M, R = (K - 8 + 31) / 32;
  const int lane = threadIdx.x & 31;
  const T* lb = &C.l.cell(b, 0, 0);
  const T* vb = &C.v(b, 0);
  T* xb = &C.x(b, 0);
  const int npan = (e - start) / 8;
  auto issue = [&](int k) {
    if (k < npan) {
      const int slot = k % kD, g = start + 8 * k;
      if (lane == 0) {  // the slot's readers passed a warp barrier; no proxy fence needed for the overwrite
        mbar_expect_tx(&sm.bar[slot], unsigned(S::CELLS * sizeof(T)));
        bulk_g2s(sm.ring[slot], lb + ix(g) * W, unsigned(S::CELLS * sizeof(T)), &sm.bar[slot]);
      }
      if (lane < 8) {
        const int vr = g + K + 8 + lane;
        if (vr < n) cpa(&sm.pv[slot][lane], vb + vr);
        else sm.pv[slot][lane] = T(0);
      }
    }
    cpa_commit();
  };
  for (int p = lane; p < M; p += 32) sm.win[p] = 0.0;
  __syncwarp();
  for (int a = lane; a < K + 8; a += 32)
    if (start + a < n) sm.win[(start + a) & (M - 1)] = double(vb[start + a]);
  for (int k = 0; k < kD - 1; ++k) issue(k);
  __syncwarp();
  double rn[8], ri[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) rn[a] = sm.win[(start + a) & (M - 1)];
  mbar_wait(&sm.bar[0], 0);
  recips<T, K>(sm.ring[0], lane, ri);
#pragma unroll 1
  for (int k = 0; k < npan; ++k) {
    const int slot = k % kD, g = start + 8 * k;
    issue(k + kD - 1);
    const T* P = sm.ring[slot];
    // (1) x_P by substitution, right-looking (every lane, broadcast reads); as soon as x_c is known
    // it also goes into (2) the next panel's residuals, rows g+8+a: L(g+8+a, g+c) x_c, and (3) the
    // far rows g+16 .. g+7+K of the residual window (lane-parallel, cells 16 + t - c of column g + c).
    // All loops run column-major so consecutive FMAs are independent.
    double x[8], nx[8], fr[R];
    int fp[R];
#pragma unroll
    for (int a = 0; a < 8; ++a) nx[a] = sm.win[(g + 8 + a) & (M - 1)];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int t = lane + 32 * q, row = g + 16 + t;
      fp[q] = (t < K - 8 && row < n) ? t : -1;
      fr[q] = sm.win[row & (M - 1)];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double mx = rn[c] * ri[c];  // -x_c
      x[c] = -mx;
#pragma unroll
      for (int j = c + 1; j < 8; ++j) rn[j] = fma(double(P[c * W + (j - c)]), mx, rn[j]);
#pragma unroll
      for (int a = 0; a < 8; ++a) nx[a] = fma(double(P[c * W + (8 + a - c)]), mx, nx[a]);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int t = fp[q];  // cells past K (short columns) and rows past n contribute nothing
        const bool on = t >= 0 && 16 + t - c <= K;
        const double lv = double(P[c * W + (on ? 16 + t - c : 0)]);
        fr[q] = fma(on ? lv : 0.0, mx, fr[q]);
      }
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) rn[a] = nx[a];
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (fp[q] >= 0) sm.win[(g + 16 + fp[q]) & (M - 1)] = fr[q];
    if (k + 1 < npan) {  // reciprocals of the next panel's pivots, off the chain
      mbar_wait(&sm.bar[(k + 1) % kD], unsigned((k + 1) / kD) & 1u);
      recips<T, K>(sm.ring[(k + 1) % kD], lane, ri);
    }
    // (4) outputs; the rows entering the window start from v
    asm volatile("cp.async.wait_group %0;" ::"n"(kD - 1) : "memory");
    if (lane < 8) {
      double xo = x[0];
#pragma unroll
      for (int c = 1; c < 8; ++c)
        if (lane == c) xo = x[c];
      const int row = g + lane;
      if (row >= s) xb[row] = T(xo);
      else if (side && row >= s - K) side[row - (s - K)] = T(xo);
      sm.win[(g + K + 8 + lane) & (M - 1)] = double(sm.pv[slot][lane]);
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------- backward, L^T x = v
// Sum over the lanes of eight per-lane values; lane l ends with the total of value (l >> 2) & 7.
__device__ __forceinline__ double reduce8(double* v, int lane) {
  // halve the value set three times (16, 8, 4 apart), then finish over lanes 2 and 1 apart
  double a[4], bq[2], c1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 16;
    const double give = hi ? v[i] : v[i + 4], keep = hi ? v[i + 4] : v[i];
    a[i] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 8;
    const double give = hi ? a[i] : a[i + 2], keep = hi ? a[i + 2] : a[i];
    bq[i] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
  }
  {
    const bool hi = lane & 4;
    const double give = hi ? bq[0] : bq[1], keep = hi ? bq[1] : bq[0];
    c1 = keep + __shfl_xor_sync(0xffffffffu, give, 4);
  }
  c1 += __shfl_xor_sync(0xffffffffu, c1, 2);
  c1 += __shfl_xor_sync(0xffffffffu, c1, 1);
  return c1;  // value index = 4 * bit4 + 2 * bit3 + bit2 of the lane = (lane >> 2) & 7 read as (16, 8, 4)
}

template <class T, int K>
__device__ void bwd_unit(const SolveP<T>& C, ix b, int n, int s, int e, int top, T* side, SolveSmem<T, K>& sm) {
  using S = SolveSmem<T, K>;
  constexpr int W = S::W, M = S::M, R = (K - 8 + 31) / 32;
  const int lane = threadIdx.x & 31;
  const T* lb = &C.l.cell(b, 0, 0);
  const T* vb = &C.v(b, 0);
  T* xb = &C.x(b, 0);
  const int npan = (top - s) / 8;  // panel k covers rows top - 8 (k + 1) .. top - 8 k - 1
  auto issue = [&](int k) {
    if (k < npan) {
      const int slot = k % kD, g = top - 8 * (k + 1);
      if (lane == 0) {
        mbar_expect_tx(&sm.bar[slot], unsigned(S::CELLS * sizeof(T)));
        bulk_g2s(sm.ring[slot], lb + ix(g) * W, unsigned(S::CELLS * sizeof(T)), &sm.bar[slot]);
      }
      if (lane < 8) cpa(&sm.pv[slot][lane], vb + g + lane);
    }
    cpa_commit();
  };
  for (int p = lane; p < M; p += 32) sm.win[p] = 0.0;  // x = 0 above the unit's first row
  if (lane < 8) sm.far[0][lane] = 0.0;
  for (int k = 0; k < kD - 1; ++k) issue(k);
  __syncwarp();
  double xp[8], ri[8];  // the previous (higher) panel's solution
#pragma unroll
  for (int a = 0; a < 8; ++a) xp[a] = 0.0;
  mbar_wait(&sm.bar[0], 0);
  recips<T, K>(sm.ring[0], lane, ri);
#pragma unroll 1
  for (int k = 0; k < npan; ++k) {
    const int slot = k % kD, g = top - 8 * (k + 1);
    issue(k + kD - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kD - 1) : "memory");
    __syncwarp();
    const T* P = sm.ring[slot];
    // (1) right-hand sides: v - far dots (formed a panel ahead) - L_NP^T x_N, every lane
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = double(sm.pv[slot][c]) - sm.far[k & 1][c];
    if (k > 0) {  // rows g+8+t of the previous panel: cells 8 + t - c of column g + c (row-major: independent FMAs)
#pragma unroll
      for (int t = 7; t >= 0; --t) {
        const double mx = -xp[t];
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(double(P[c * W + (8 + t - c)]), mx, x[c]);
      }
    }
    // (2) substitution with L_PP^T, last row first, right-looking
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      const double mx = x[j] * ri[j];  // -x_j
      x[j] = -mx;
#pragma unroll
      for (int c = 0; c < j; ++c) x[c] = fma(double(P[c * W + (j - c)]), mx, x[c]);
    }
    // (3) one panel ahead: far dots of the next (lower) panel g' = g - 8 with the rows beyond THIS panel,
    //     i.e. rows g + 8 + t, t in [0, K - 8): cells 16 + t - c of column g' + c; all known already
    if (k + 1 < npan) {
      mbar_wait(&sm.bar[(k + 1) % kD], unsigned((k + 1) / kD) & 1u);
      const T* Pn = sm.ring[(k + 1) % kD];
      recips<T, K>(Pn, lane, ri);
      double part[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) part[c] = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int t = lane + 32 * q, row = g + 8 + t;
        const bool in = t < K - 8 && row < n;
        const double xv = in ? sm.win[row & (M - 1)] : 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const bool on = in && 16 + t - c <= K;
          const double lv = double(Pn[c * W + (on ? 16 + t - c : 0)]);
          part[c] = fma(on ? lv : 0.0, xv, part[c]);
        }
      }
      const double tot = reduce8(part, lane);
      if ((lane & 3) == 0) {
        const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        sm.far[(k + 1) & 1][vi] = tot;
      }
    }
    // (4) outputs, the solution window
    if (lane < 8) {
      double xo = x[0];
#pragma unroll
      for (int c = 1; c < 8; ++c)
        if (lane == c) xo = x[c];
      const int row = g + lane;
      if (row < e) xb[row] = T(xo);
      else if (side && row < e + K) side[row - e] = T(xo);
      sm.win[row & (M - 1)] = xo;
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) xp[a] = x[a];
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// repair != 0: one warp per flagged matrix, a single exact unit
template <class T, int K, bool TR>
__global__ void __launch_bounds__(32) k_solve_blk(SolveP<T> C, Geo G, int repair) {
  extern __shared__ __align__(16) unsigned char raw[];
  SolveSmem<T, K>& sm = *reinterpret_cast<SolveSmem<T, K>*>(raw);
  ix b;
  int s, e, from;
  T* side = nullptr;
  if (repair) {
    b = blockIdx.x;
    if (b >= G.batch || !C.flag[b]) return;
    s = 0, e = int(G.n), from = TR ? int(G.n) : 0;
  } else {
    const ix unit = blockIdx.x;
    b = unit / G.nseg;
    const int p = int(unit % G.nseg);
    if (b >= G.batch) return;
    s = int(ix(p) * G.seg);
    e = int(s + G.seg < G.n ? s + G.seg : G.n);
    if (!TR) {
      from = s - G.burn > 0 ? s - G.burn : 0;
      from -= from % 8;
      if (p > 0) side = C.side + unit * K;
    } else {
      from = e + G.burn < G.n ? e + G.burn : int(G.n);
      from = (from + 7) / 8 * 8;
      if (from > G.n) from = int(G.n);
      if (p + 1 < G.nseg) side = C.side + unit * K;
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kD; ++i) mbar_init(&sm.bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (!TR) fwd_unit<T, K>(C, b, int(G.n), s, e, from, side, sm);
  else bwd_unit<T, K>(C, b, int(G.n), s, e, from, side, sm);
}

// thread per (unit, value): burn-in copy vs the neighbour's genuine values
template <class T, int K, bool TR>
__global__ void k_solve_blk_check(SolveP<T> C, Geo G) {
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

// first (forward) / last (backward sweep reaches it first) singular pivot
template <class T>
__global__ void k_blk_singular(Band<T> l, ix batch, int tr, int64_t* fail) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (t >= batch * l.n) return;
  const ix b = t / l.n, i = t % l.n;
  if (fabs(double(l.cell(b, 0, i))) < kPivotFloor) {
    if (!tr) atomicMin(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(i));
    else atomicMax(reinterpret_cast<unsigned long long*>(fail + b), static_cast<unsigned long long>(i + 1));
  }
}

__global__ void k_blk_init(int64_t* fail, int32_t* flag, ix batch, int64_t v) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  fail[b] = v;
  flag[b] = 0;
}

__global__ void k_blk_status(const int64_t* fail, ix batch, ix n, int tr, int32_t* status, int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  const ix f = tr ? fail[b] - 1 : fail[b];  // backward: stored as row + 1, 0 = none
  const bool ok = tr ? f < 0 : f >= n;
  report(status, row, b, ok ? BGM_OK : BGM_ERR_SINGULAR, ok ? -1 : f);
}

template <class T, int K, bool TR>
bool run_solve_blk(const bgm_band& l, const bgm_vec& v, const bgm_vec& x, int32_t* st, int64_t* row, cudaStream_t s,
                   int segment_rows) {
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = (kBurnGen + 2) * K;  // a solve damps by ~sqrt(K)|L(i,m)/L(i,i)| per generation
  if (const char* bv = std::getenv("BGM_WIDE_BURN"))
    if (std::atoi(bv) >= 1) G.burn = std::atoi(bv);
  G.burn = (G.burn + 7) / 8 * 8;
  const size_t smem = sizeof(SolveSmem<T, K>);
  cudaFuncSetAttribute(k_solve_blk<T, K, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  ix seg = requested_seg(segment_rows, K);
  if (seg <= 0) {
    // units per SM: enough warps to overlap the per-panel latency, few enough to keep the burn-in share small
    int sms = 148, dev = 0, upsm = K <= 64 ? 10 : 5;  // measured: a lone warp per sub-partition is latency-bound
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char* uv = std::getenv("BGM_WSOLVE_UNITS"))
      if (std::atoi(uv) >= 1) upsm = std::atoi(uv);
    ix nseg = (ix(sms) * upsm + G.batch - 1) / (G.batch > 0 ? G.batch : 1);
    if (nseg < 1) nseg = 1;
    seg = (G.n + nseg - 1) / nseg;
    if (seg < 2 * ix(G.burn)) seg = 2 * ix(G.burn);
  }
  if (seg < K) seg = K;
  seg = (seg + 7) / 8 * 8;
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
  k_blk_init<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, C.flag, G.batch, TR ? 0 : G.n);
  k_blk_singular<T><<<blocks_for(G.batch * G.n, 256), 256, 0, s>>>(C.l, G.batch, TR, fail);
  {
    timing::Scope ts(TR ? "wide_solve_t" : "wide_solve", s);
    k_solve_blk<T, K, TR><<<unsigned(units), 32, smem, s>>>(C, G, 0);
  }
  {
    timing::Scope ts("wide_solve_check", s);
    k_solve_blk_check<T, K, TR><<<blocks_for(units * K, 128), 128, 0, s>>>(C, G);
  }
  {
    timing::Scope ts("wide_solve_repair", s);
    k_solve_blk<T, K, TR><<<unsigned(G.batch), 32, smem, s>>>(C, G, 1);
  }
  k_blk_status<<<blocks_for(G.batch, 128), 128, 0, s>>>(fail, G.batch, G.n, TR, st, row);
  scratch_free(ws, s);
  return true;
}

}  // namespace

bool solve_vec_blk(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
                   cudaStream_t s, int segment_rows) {
  // reference layout (one matrix per block), whole panels, 16-byte aligned panels, 32-bit row indices
  if (l.tile != 1 || v.tile != 1 || x.tile != 1 || l.upper != 0 || l.n % 8 != 0 || l.n < 8 * l.lower) return false;
  if (l.n >= (ix(1) << 30)) return false;
  const size_t esz = l.dtype == BGM_F64 ? 8 : 4;
  if ((size_t(l.n) * size_t(l.lower + 1) * esz) % 16 != 0 || reinterpret_cast<size_t>(l.data) % 16 != 0) return false;
  const bool f64 = l.dtype == BGM_F64;
  switch (l.lower) {
#define BGM_SOLVE_BLK(KK)                                                                                   \
  case KK:                                                                                                  \
    if (f64)                                                                                                \
      return tr ? run_solve_blk<double, KK, true>(l, v, x, st, row, s, segment_rows)                        \
                : run_solve_blk<double, KK, false>(l, v, x, st, row, s, segment_rows);                      \
    return tr ? run_solve_blk<float, KK, true>(l, v, x, st, row, s, segment_rows)                           \
              : run_solve_blk<float, KK, false>(l, v, x, st, row, s, segment_rows);
    BGM_SOLVE_BLK(64)
    BGM_SOLVE_BLK(128)
#undef BGM_SOLVE_BLK
    default: return false;
  }
}

}  // namespace wide
}  // namespace bgm
