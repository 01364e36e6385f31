// Segment-parallel config-3 sweeps, bandwidth 16, fp64, tile-1 layout.
//
// The reference factors one matrix row by row (kernels_serial.cpp:12-32,
// grad.cpp:11-36): a length-n dependency chain.  At config 3 (B = 256
// matrices, n = 65536) one chain per matrix leaves a B200 idle, so every
// matrix is split into P segments and each (matrix, segment) pair becomes an
// independent "unit" run by a 16-lane team (2 units per warp):
//
//   forward : unit p starts `burn` rows before its segment from a zero
//             window (the Riccati/Schur recursion forgets its initial state
//             geometrically), then factors its own rows exactly as the
//             sequential sweep would.  The last 16 burn-in factor columns
//             are saved; check_fwd compares them with the columns unit p-1
//             produced for real.  Any mismatch beyond 1e-12 (relative to the
//             column scale) flags the matrix and repair_fwd reruns it as a
//             single exact unit -- so results never depend on convergence.
//   reverse : same scheme run downwards (Takahashi recursion on the factor
//             plus the back-solve), burning in from `burn` rows above the
//             segment; the boundary window state is compared with the one
//             unit p+1 produced, with the same repair.
//
// Team layout (forward): lane t owns the window column c = t (mod 16) and
// keeps the full column of the symmetric (k+1)x(k+1) Schur window in 16
// registers (rows indexed by absolute row mod 16).  Per row: rank-1 "+l l^T"
// (forming A = L L^T + tau^-2 I on the fly) and "-c c^T" updates, pivot via
// one rsqrt, the column c and the L column are exchanged through shared
// memory.  Reverse: lane t owns window row r = t (mod 16) of S = band(A^-1)
// and u = A^-1 y; per row a 16-term mat-vec for S(., j), one for the
// L_bar column, and a 4-value butterfly for the diagonal terms.
// Scratch Lp keeps 1/Lp(i,i) in storage row 0 (the reverse sweep only ever
// divides by the pivot).
#include <cuda_runtime.h>

#include <utility>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_mlik.cuh"
#include "bgm_timing.cuh"

namespace bgm {
namespace {

constexpr int K = 16;
constexpr int WS = K + 1;  // storage rows per column
constexpr int WARPS = 4;
constexpr int THREADS = 32 * WARPS;
constexpr int UNITS_PER_BLOCK = 2 * WARPS;
constexpr unsigned FULL = 0xffffffffu;
constexpr double kLn2 = 0.69314718055994530942;
constexpr double kLog2Pi = 1.8378770664093454836;  // inference.cpp:15
constexpr double kCheckTol = 1e-12;
constexpr int SIDE = 16 * 18;  // forward side buffer per unit: 16 columns x (17 + w)
constexpr int STATE = 16 * 17;  // reverse boundary state per unit: 16 lanes x (16 S + u)

template <class F, int... Us>
__device__ __forceinline__ void unroll_up(F&& f, std::integer_sequence<int, Us...>) {
  (f(std::integral_constant<int, Us>{}), ...);
}
template <class F, int... Us>
__device__ __forceinline__ void unroll_down(F&& f, std::integer_sequence<int, Us...>) {
  (f(std::integral_constant<int, 15 - Us>{}), ...);
}

struct Geo {
  ix batch, n, seg;  // segment rows (multiple of 16)
  int nseg, burn;    // segments per matrix, burn-in rows (multiple of 16)
};

struct FwdP {
  const double* L;
  const double* y;
  double* lp;    // Lp scratch, tile-1, storage row 0 = 1/Lp(i,i)
  double* w;     // w = Lp^-1 y
  double* side;  // [unit][16][18]
  double* part;  // [unit][4]: log|Lp|, log|L|, y'y, w'w
  int64_t* fail;  // [batch]: first non-PD row (n = none)
  double sigma;  // 1/tau2
};

struct BwdP {
  const double* L;
  const double* lp;
  const double* w;
  double* lbar;
  double* entry;  // [unit][16][17] burn-in boundary state
  double* exitb;  // [unit][16][17] genuine boundary state
  double* part;   // [unit][2]: tr S, u'u
  double c4;      // 1/tau2^2
};

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// Matrices re-run by the exact single-unit path (burn-in did not converge).
__device__ unsigned long long g_repairs = 0;

// ------------------------------------------------------------------ forward
// One unit: rows [s, e) owned, sweep starts at i0 (multiple of 16, <= s).
// `side` (nullable) receives the burn-in columns [s-16, s).
__device__ void fwd_sweep(const FwdP& P, const Geo& G, ix b, ix s, ix e, ix i0, double* side,
                          double* part, int t, double* sm, unsigned mask) {
  const ix n = G.n;
  const double* Lb = P.L + b * n * WS;
  const double* yb = P.y + b * n;
  double* lpb = P.lp + b * n * WS;
  double* wb = P.w + b * n;
  double W[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) W[q] = 0.0;
  // window columns at i0: c = i0 + t; residual for row c
  double res = (i0 + t < n) ? ldg(yb + i0 + t) : 0.0;
  double yy = 0.0, ww = 0.0, prodp = 1.0, prodl = 1.0;
  int ep = 0, el = 0;
  if (i0 == s) {  // exact start: rows [s, s+16) enter now, count their y'y
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const ix r = s + q;
      const double v = (r < e) ? ldg(yb + r) : 0.0;
      yy += v * v;
    }
  }
  ix fail_row = n;
  // prefetch registers, distance 8 steps: my L cell + (lane 0: L(i+16,i), lane 1: y(i+16))
  double pa[8], pb[8];
  auto issue = [&](ix ii, int U) {
    const int crn = (t - U) & 15;
    double a = 0.0, x = 0.0;
    if (ii < n) {
      a = ldg(Lb + ii * WS + crn);
      if (t == 0) x = ldg(Lb + ii * WS + 16);
      if (t == 1 && ii + 16 < n) x = ldg(yb + ii + 16);
    }
    pa[U & 7] = a;
    pb[U & 7] = x;
  };
  // prime: steps i0 .. i0+7
#pragma unroll
  for (int q = 0; q < 8; ++q) issue(i0 + q, q);

  const ix i_end = (e + 15) / 16 * 16;
  for (ix base = i0; base < i_end; base += 16) {
    unroll_up(
        [&](auto UC) {
          constexpr int U = decltype(UC)::value;
          const ix i = base + U;
          const int cr = (t - U) & 15;
          const bool pl = (t == U);
          const double lv = pa[U & 7];
          const double xv = pb[U & 7];
          issue(i + 8, (U + 8) & 15);
          double* lb = sm + (U & 1) * 36;  // [0..16] l, [17] y(i+16), [18..34] c
          lb[cr] = lv;
          if (t == 0) lb[16] = xv;
          if (t == 1) lb[17] = xv;
          __syncwarp(mask);
          const double l0 = lb[0];
          const double l16 = lb[16];
          const double yn = lb[17];
          W[U] = fma(l0, lv, W[U] + (pl ? P.sigma : 0.0));
          const double d = __shfl_sync(mask, W[U], U, 16);
          const double rs = rsqrt(d);
          const double cmy = W[U] * rs;
          const double c16 = l0 * l16 * rs;
          lb[18 + cr] = cmy;
          if (t == 0) lb[34] = c16;
          const double rp = __shfl_sync(mask, res, U, 16);
          const double wi = rp * rs;
          const bool own = i >= s && i < e;
          if (own) {
            lpb[i * WS + cr] = cr == 0 ? rs : cmy;
            if (t == 0) {
              lpb[i * WS + 16] = c16;
              wb[i] = wi;
            }
            const double piv = d * rs;
            if (!(d > kPivotFloor) && i < fail_row) fail_row = i;
            if (!(fabs(l0) > kPivotFloor) && i < fail_row) fail_row = i;
            prodp *= piv;
            prodl *= fabs(l0);
            ww += wi * wi;
          } else if (side && i >= s - 16 && i < s) {
            double* sd = side + (i - (s - 16)) * 18;
            sd[cr] = cr == 0 ? rs : cmy;
            if (t == 0) {
              sd[16] = c16;
              sd[17] = wi;
            }
          }
          if (i + 16 >= s && i + 16 < e) yy += yn * yn;
          const double ccol = pl ? c16 : cmy;
          const double lcol = pl ? l16 : lv;
          res = fma(-ccol, wi, pl ? yn : res);
          __syncwarp(mask);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (q == U) {
              W[q] = fma(l16, lcol, -c16 * ccol);
            } else {
              const int rel = (q - U) & 15;
              const double old = pl ? 0.0 : W[q];
              W[q] = fma(lb[rel], lcol, fma(-lb[18 + rel], ccol, old));
            }
          }
        },
        std::make_integer_sequence<int, 16>{});
    int x;
    prodp = frexp(prodp, &x);
    ep += x;
    prodl = frexp(prodl, &x);
    el += x;
  }
  if (t == 0) {
    part[0] = log(prodp) + ep * kLn2;
    part[1] = log(prodl) + el * kLn2;
    part[2] = yy;
    part[3] = ww;
    if (fail_row < n) atomicMin(reinterpret_cast<unsigned long long*>(P.fail + b),
                                static_cast<unsigned long long>(fail_row));
  }
}

__global__ void __launch_bounds__(THREADS) k_fwd(FwdP P, Geo G) {
  __shared__ double smem[UNITS_PER_BLOCK][72];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp * 2 + (lane >> 4);
  const int t = lane & 15;
  const ix unit = ix(blockIdx.x) * UNITS_PER_BLOCK + slot;
  const ix units = G.batch * G.nseg;
  if (unit >= units) return;  // whole half-warps exit together
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix i0 = s - G.burn > 0 ? s - G.burn : 0;
  fwd_sweep(P, G, b, s, e, i0, p > 0 ? P.side + unit * SIDE : nullptr, P.part + unit * 4, t,
            smem[slot], 0xffffu << (lane & 16));
}

// One thread per (matrix, segment > 0): burn-in columns vs the real ones.
__global__ void k_check_fwd(FwdP P, Geo G, int32_t* flag) {
  const ix unit = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (unit >= G.batch * G.nseg) return;
  const int p = int(unit % G.nseg);
  if (p == 0) return;
  const ix b = unit / G.nseg, n = G.n;
  const ix s = ix(p) * G.seg;
  const double* sd = P.side + unit * SIDE;
  bool bad = false;
  double wscale = 0.0;
  for (int c = 0; c < 16; ++c) wscale = fmax(wscale, fabs(P.w[b * n + s - 16 + c]));
  for (int c = 0; c < 16 && !bad; ++c) {
    const double* real = P.lp + (b * n + s - 16 + c) * WS;
    double sc = 0.0;
    for (int r = 0; r < WS; ++r) sc = fmax(sc, fabs(real[r]));
    for (int r = 0; r < WS; ++r)
      if (!(fabs(sd[c * 18 + r] - real[r]) <= kCheckTol * sc)) bad = true;
    if (!(fabs(sd[c * 18 + 17] - P.w[b * n + s - 16 + c]) <= kCheckTol * (wscale + 1e-300)))
      bad = true;
  }
  if (bad) flag[b] = 1;
}

// One team per matrix: flagged matrices rerun the forward as one exact unit.
__global__ void __launch_bounds__(THREADS) k_repair_fwd(FwdP P, Geo G, const int32_t* flag) {
  __shared__ double smem[UNITS_PER_BLOCK][72];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp * 2 + (lane >> 4);
  const ix b = ix(blockIdx.x) * UNITS_PER_BLOCK + slot;
  if (b >= G.batch || !flag[b]) return;
  const int t = lane & 15;
  double* part0 = P.part + b * G.nseg * 4;
  if (t == 0) {
    atomicAdd(&g_repairs, 1ull);
    P.fail[b] = G.n;
    for (int q = 4; q < G.nseg * 4; ++q) part0[q] = 0.0;
  }
  __syncwarp(0xffffu << (lane & 16));
  fwd_sweep(P, G, b, 0, G.n, 0, nullptr, part0, t, smem[slot], 0xffffu << (lane & 16));
}

// ------------------------------------------------------------------ reverse
__device__ void bwd_sweep(const BwdP& P, const Geo& G, ix b, ix s, ix e, ix jtop, double* entry,
                          double* exitb, double* part, int t, double* sm, unsigned mask) {
  const ix n = G.n;
  const double* Lb = P.L + b * n * WS;
  const double* lpb = P.lp + b * n * WS;
  const double* wb = P.w + b * n;
  double* lbb = P.lbar + b * n * WS;
  double S[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) S[q] = 0.0;
  double um = 0.0, tr = 0.0, uu = 0.0;
  // prefetch: lp cell, L cell, and (lane 0: 1/Lp(j,j), lane 1: L(j,j), lane 2: w_j)
  double pa[8], pb[8], pc[8];
  auto issue = [&](ix jj, int U) {
    const int rel = ((t - U - 1) & 15) + 1;
    double a = 0.0, c = 0.0, x = 0.0;
    if (jj >= 0 && jj < n) {
      a = ldg(lpb + jj * WS + rel);
      c = ldg(Lb + jj * WS + rel);
      if (t == 0) x = ldg(lpb + jj * WS);
      if (t == 1) x = ldg(Lb + jj * WS);
      if (t == 2) x = ldg(wb + jj);
    }
    pa[U & 7] = a;
    pb[U & 7] = c;
    pc[U & 7] = x;
  };
  const ix top_base = jtop / 16 * 16;
  // prime steps top_base+15 .. top_base+8
#pragma unroll
  for (int q = 0; q < 8; ++q) issue(top_base + 15 - q, 15 - q);
  bool entry_saved = (entry == nullptr);
  for (ix base = top_base; base >= s; base -= 16) {
    unroll_down(
        [&](auto UC) {
          constexpr int U = decltype(UC)::value;
          const ix j = base + U;
          const double lpm = pa[U & 7], lm = pb[U & 7], xv = pc[U & 7];
          issue(j - 8, (U + 8) & 15);
          if (j > jtop) return;  // above the sweep start (uniform across the team)
          if (!entry_saved && j == e - 1) {
            // boundary state at e (window [e, e+16)), produced by burn-in
#pragma unroll
            for (int q = 0; q < 16; ++q) entry[t * 17 + q] = S[q];
            entry[t * 17 + 16] = um;
            entry_saved = true;
          }
          const int rel = ((t - U - 1) & 15) + 1;
          const bool ent = (t == U);
          double* sb = sm + (U & 1) * 54;  // [0..16] lp col, [18..34] L col, [36..52] S(.,j)
          sb[rel] = lpm;
          sb[18 + rel] = lm;
          if (t == 0) sb[0] = xv;
          if (t == 1) sb[18] = xv;
          if (t == 2) sb[36] = xv;
          __syncwarp(mask);
          const double inv = sb[0], ljj = sb[18], wj = sb[36];
          double acc = 0.0, accl = 0.0;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int cs = ((q - U - 1) & 15) + 1;
            acc = fma(S[q], sb[cs], acc);
            accl = fma(S[q], sb[18 + cs], accl);
          }
          const double out = acc * inv;
          const double snew = -out;
          double ra = lpm * out, rb = lpm * um, rc = um * lm, rd = out * lm;
#pragma unroll
          for (int m = 8; m >= 1; m >>= 1) {
            ra += __shfl_xor_sync(mask, ra, m, 16);
            rb += __shfl_xor_sync(mask, rb, m, 16);
            rc += __shfl_xor_sync(mask, rc, m, 16);
            rd += __shfl_xor_sync(mask, rd, m, 16);
          }
          const double sjj = inv * inv + inv * ra;
          const double uj = (wj - rb) * inv;
          const double ul = uj * ljj + rc;
          const bool own = j >= s && j < e;
          if (own) {
            const double lbm = -(accl + snew * ljj) - P.c4 * um * ul;
            lbb[j * WS + rel] = (j + rel < n) ? lbm : 0.0;
            if (ent) lbb[j * WS] = rd - sjj * ljj - P.c4 * uj * ul + __drcp_rn(ljj);
            tr += sjj;
            uu += uj * uj;
          }
          sb[36 + rel] = snew;
          S[U] = snew;
          __syncwarp(mask);
          if (ent) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (q != U) S[q] = sb[36 + (((q - U - 1) & 15) + 1)];
            S[U] = sjj;
            um = uj;
          }
        },
        std::make_integer_sequence<int, 16>{});
  }
  if (exitb) {
#pragma unroll
    for (int q = 0; q < 16; ++q) exitb[t * 17 + q] = S[q];
    exitb[t * 17 + 16] = um;
  }
  if (t == 0) {
    part[0] = tr;
    part[1] = uu;
  }
}

__global__ void __launch_bounds__(THREADS) k_bwd(BwdP P, Geo G) {
  __shared__ double smem[UNITS_PER_BLOCK][108];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp * 2 + (lane >> 4);
  const int t = lane & 15;
  const ix unit = ix(blockIdx.x) * UNITS_PER_BLOCK + slot;
  if (unit >= G.batch * G.nseg) return;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix jtop = e + G.burn - 1;
  if (jtop > G.n - 1) jtop = G.n - 1;
  bwd_sweep(P, G, b, s, e, jtop, p + 1 < G.nseg ? P.entry + unit * STATE : nullptr,
            p > 0 ? P.exitb + unit * STATE : nullptr, P.part + unit * 2, t, smem[slot],
            0xffffu << (lane & 16));
}

__global__ void k_check_bwd(BwdP P, Geo G, int32_t* flag) {
  const ix unit = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (unit >= G.batch * G.nseg) return;
  const int p = int(unit % G.nseg);
  if (p + 1 >= G.nseg) return;
  const ix b = unit / G.nseg;
  const double* a = P.entry + unit * STATE;
  const double* r = P.exitb + (unit + 1) * STATE;
  double ss = 0.0, us = 0.0;
  for (int q = 0; q < 16; ++q) {
    for (int c = 0; c < 16; ++c) ss = fmax(ss, fabs(r[q * 17 + c]));
    us = fmax(us, fabs(r[q * 17 + 16]));
  }
  bool bad = false;
  for (int q = 0; q < 16; ++q) {
    for (int c = 0; c < 16; ++c)
      if (!(fabs(a[q * 17 + c] - r[q * 17 + c]) <= kCheckTol * (ss + 1e-300))) bad = true;
    if (!(fabs(a[q * 17 + 16] - r[q * 17 + 16]) <= kCheckTol * (us + 1e-300))) bad = true;
  }
  if (bad) flag[b] = 1;
}

__global__ void __launch_bounds__(THREADS) k_repair_bwd(BwdP P, Geo G, const int32_t* flag,
                                                        const int64_t* fail) {
  __shared__ double smem[UNITS_PER_BLOCK][108];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp * 2 + (lane >> 4);
  const ix b = ix(blockIdx.x) * UNITS_PER_BLOCK + slot;
  if (b >= G.batch || !flag[b] || fail[b] < G.n) return;
  const int t = lane & 15;
  double* part0 = P.part + b * G.nseg * 2;
  if (t == 0) {
    atomicAdd(&g_repairs, 1ull);
    for (int q = 2; q < G.nseg * 2; ++q) part0[q] = 0.0;
  }
  __syncwarp(0xffffu << (lane & 16));
  bwd_sweep(P, G, b, 0, G.n, G.n - 1, nullptr, nullptr, part0, t, smem[slot], 0xffffu << (lane & 16));
}

__global__ void k_finalize(const double* pf, const double* pb, const int64_t* fail, Geo G,
                           double tau2, double* loss, double* tau2_bar, int32_t* status,
                           int64_t* row) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= G.batch) return;
  double ldp = 0, ldl = 0, yy = 0, ww = 0, tr = 0, uu = 0;
  for (int p = 0; p < G.nseg; ++p) {
    const double* f = pf + (b * G.nseg + p) * 4;
    ldp += f[0];
    ldl += f[1];
    yy += f[2];
    ww += f[3];
    tr += pb[(b * G.nseg + p) * 2];
    uu += pb[(b * G.nseg + p) * 2 + 1];
  }
  const double nn = double(G.n), inv = 1.0 / tau2, c4 = inv * inv;
  // log|Lp| = sum log Lp(i,i); log|L_Q| = sum log|L(i,i)| (chol(L L^T) = L)
  loss[b] = -0.5 * nn * kLog2Pi - ldp + ldl - 0.5 * nn * log(tau2) - 0.5 * yy * inv + 0.5 * ww * c4;
  tau2_bar[b] = -nn * 0.5 * inv + 0.5 * yy * c4 + 0.5 * c4 * tr - ww * c4 * inv + 0.5 * uu * c4 * c4;
  const bool ok = fail[b] >= G.n;
  if (status) status[b] = ok ? BGM_OK : BGM_ERR_NOT_PD;
  if (row) row[b] = ok ? -1 : fail[b];
}

__global__ void k_init_fail(int64_t* fail, int32_t* flag, ix batch, ix n) {
  const ix b = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  if (b >= batch) return;
  fail[b] = n;
  flag[b] = 0;
  flag[batch + b] = 0;
}

}  // namespace

int mlik_repairs(int64_t* count, int reset) {
  unsigned long long v = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&v, g_repairs, sizeof v);
  if (e != cudaSuccess) return set_error(e);
  if (count) *count = int64_t(v);
  if (reset) {
    v = 0;
    e = cudaMemcpyToSymbol(g_repairs, &v, sizeof v);
    if (e != cudaSuccess) return set_error(e);
  }
  return BGM_OK;
}

int mlik_fast(const bgm_band& l, const bgm_vec& y, double tau2, double* loss, const bgm_band& lbar,
              double* tau2_bar, int32_t* status, int64_t* row, int segment_rows, cudaStream_t s) {
  if (fast::disabled()) return -1;
  if (l.lower != K || l.tile != 1 || y.tile != 1 || lbar.tile != 1) return -1;
  Geo G;
  G.batch = l.batch;
  G.n = l.n;
  G.burn = 32;
  // Units to fill the chip: ~12 resident warps (24 units) per SM.
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  ix seg = segment_rows;
  if (seg <= 0) {
    const ix target_units = ix(sms) * 24;
    ix per = (target_units + G.batch - 1) / G.batch;
    if (per < 1) per = 1;
    seg = (G.n + per - 1) / per;
    if (seg < 8 * G.burn) seg = 8 * G.burn;
  }
  seg = (seg + 15) / 16 * 16;
  if (seg < 16) seg = 16;
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;

  // scratch: Lp, w, side, fwd parts, states, bwd parts, fail, flags
  const size_t nb = size_t(G.batch) * size_t(G.n);
  const size_t bytes = sizeof(double) * (nb * WS + nb + size_t(units) * (SIDE + 4 + 2 * STATE + 2)) +
                       sizeof(int64_t) * size_t(G.batch) + sizeof(int32_t) * 2 * size_t(G.batch) + 256;
  char* ws = nullptr;
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, s);
  if (err != cudaSuccess) return set_error(err);
  double* dp = reinterpret_cast<double*>(ws);
  FwdP F;
  F.L = static_cast<const double*>(l.data);
  F.y = static_cast<const double*>(y.data);
  F.lp = dp;
  dp += nb * WS;
  F.w = dp;
  dp += nb;
  F.side = dp;
  dp += size_t(units) * SIDE;
  F.part = dp;
  dp += size_t(units) * 4;
  BwdP Bp;
  Bp.entry = dp;
  dp += size_t(units) * STATE;
  Bp.exitb = dp;
  dp += size_t(units) * STATE;
  Bp.part = dp;
  dp += size_t(units) * 2;
  F.fail = reinterpret_cast<int64_t*>(dp);
  int32_t* flags = reinterpret_cast<int32_t*>(F.fail + G.batch);
  F.sigma = 1.0 / tau2;
  Bp.L = F.L;
  Bp.lp = F.lp;
  Bp.w = F.w;
  Bp.lbar = static_cast<double*>(lbar.data);
  Bp.c4 = F.sigma * F.sigma;

  const unsigned ublocks = unsigned((units + UNITS_PER_BLOCK - 1) / UNITS_PER_BLOCK);
  const unsigned mblocks = unsigned((G.batch + UNITS_PER_BLOCK - 1) / UNITS_PER_BLOCK);
  const unsigned cblocks = unsigned((units + 127) / 128);
  k_init_fail<<<blocks_for(G.batch, 128), 128, 0, s>>>(F.fail, flags, G.batch, G.n);
  {
    timing::Scope ts("mlik_seg_fwd", s);
    k_fwd<<<ublocks, THREADS, 0, s>>>(F, G);
  }
  {
    timing::Scope ts("mlik_seg_check", s);
    k_check_fwd<<<cblocks, 128, 0, s>>>(F, G, flags);
    k_repair_fwd<<<mblocks, THREADS, 0, s>>>(F, G, flags);
  }
  {
    timing::Scope ts("mlik_seg_bwd", s);
    k_bwd<<<ublocks, THREADS, 0, s>>>(Bp, G);
  }
  {
    timing::Scope ts("mlik_seg_check", s);
    k_check_bwd<<<cblocks, 128, 0, s>>>(Bp, G, flags + G.batch);
    k_repair_bwd<<<mblocks, THREADS, 0, s>>>(Bp, G, flags + G.batch, F.fail);
    k_finalize<<<blocks_for(G.batch, 128), 128, 0, s>>>(F.part, Bp.part, F.fail, G, tau2, loss,
                                                        tau2_bar, status, row);
  }
  err = cudaGetLastError();
  cudaFreeAsync(ws, s);
  return err == cudaSuccess ? BGM_OK : set_error(err);
}

}  // namespace bgm
