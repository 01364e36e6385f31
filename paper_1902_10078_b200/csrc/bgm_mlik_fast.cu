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

#include <cstdio>
#include <cstdlib>
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
  int debug;         // BGM_DEBUG=1: report check mismatches
  int team;          // lanes per unit (8 or 16)
};

struct FwdP {
  const double* L;
  const double* y;
  double* lp;    // Lp scratch, tile-1, storage row 0 = 1/Lp(i,i)
  double* w;     // w = Lp^-1 y
  double* side;  // [unit][16][18]
  double* part;  // [unit][4]: log|Lp|, log|L|, y'y, w'w
  int64_t* fail;  // [batch]: first non-PD row (n = none)
  double* sink;   // write target of padding teams (one matrix worth)
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
  double* sink;
  double c4;      // 1/tau2^2
};

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// Matrices re-run by the exact single-unit path (burn-in did not converge).
__device__ unsigned long long g_repairs = 0;
// Largest burn-in deviation seen by the checks (bits of a non-negative double).
__device__ unsigned long long g_maxdev = 0;

__device__ __forceinline__ void note_dev(double rel) {
  if (rel >= 0.0) atomicMax(&g_maxdev, static_cast<unsigned long long>(__double_as_longlong(rel)));
}

// ------------------------------------------------------------------ helpers
// 1/sqrt(d) and 1/x from a float seed + two Newton steps (relative error a
// few ulp); the exact libdevice routines outside the float range.
__device__ __forceinline__ double fast_rsqrt(double d) {
  if (!(d > 1e-30 && d < 1e30)) return rsqrt(d);
  double r = double(rsqrtf(float(d)));
  const double h = 0.5 * d;
  r = r * fma(-h * r, r, 1.5);
  r = r * fma(-h * r, r, 1.5);
  return r;
}
__device__ __forceinline__ double fast_rcp(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-30 && ax < 1e30)) return __drcp_rn(x);
  double r = double(__frcp_rn(float(x)));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

template <int TEAM>
struct Team {
  static constexpr int CPL = 16 / TEAM;        // window columns (rows) per lane
  static constexpr int UPB = (32 / TEAM) * WARPS;  // units per block
  // Every lane of a warp always runs a unit (padding units are "dummies"
  // that compute but write nothing), so team collectives use the full mask.
  __device__ static constexpr unsigned mask(int) { return FULL; }
};

// Per-block phases of a sweep: BURN (no outputs), OWN (outputs, no bounds
// checks), GEN (everything checked: segment edges, matrix tail, side buffer).
enum { PH_BURN = 0, PH_OWN = 1, PH_GEN = 2 };

// ------------------------------------------------------------------ forward
struct FwdCtx {
  const double* Lb;  // this matrix's L (tile 1)
  const double* yb;
  double* lpb;
  double* wb;
  double* side;  // nullable: burn-in columns [s-16, s)
  ix n, s, e;
  double sigma;
};

template <int TEAM>
struct FwdSt {
  static constexpr int CPL = Team<TEAM>::CPL;
  double W[CPL][16];  // W[m][q]: window row (absolute = q mod 16) of my m-th column
  double res[CPL];
  double pa[CPL][8];  // prefetched L cells (distance 8 rows)
  double pb[8];       // prefetched aux value (lane 0: L(i+16,i), lane 1: y(i+16))
  double yy, ww, prodp, prodl;
  int ep, el;
  ix fail;
};

template <int TEAM, int PH>
__device__ __forceinline__ void fwd_block(FwdSt<TEAM>& S, const FwdCtx& C, ix base, int t,
                                          double* sm, unsigned mask) {
  constexpr int CPL = Team<TEAM>::CPL;
  const ix n = C.n;
  const double* Lblk = C.Lb + base * WS;
  // aux pointer: lane 1 streams y(i+16), every other lane L(i+16, i)
  const double* auxp = (t == 1) ? C.yb + base + 16 : Lblk + 16;
  const int auxs = (t == 1) ? 1 : WS;
  const int aux_slot = 16 + (t < 2 ? t : 2);
  unroll_up(
      [&](auto UC) {
        constexpr int U = decltype(UC)::value;
        constexpr int PT = U % TEAM;  // pivot lane
        constexpr int PM = U / TEAM;  // pivot lane's column slot
        const ix i = base + U;
        const bool pl = (t == PT);
        int cr[CPL];
        double lv[CPL];
#pragma unroll
        for (int m = 0; m < CPL; ++m) {
          cr[m] = (t + TEAM * m - U) & 15;
          lv[m] = S.pa[m][U & 7];
        }
        const double xv = S.pb[U & 7];
        // prefetch row i + 8
        {
          const ix ii = i + 8;
#pragma unroll
          for (int m = 0; m < CPL; ++m) {
            const int crn = (t + TEAM * m - U - 8) & 15;
            double a;
            if (PH == PH_GEN)
              a = ii < n ? ldg(C.Lb + ii * WS + crn) : 0.0;
            else
              a = ldg(Lblk + (U + 8) * WS + crn);
            S.pa[m][U & 7] = a;
          }
          double x;
          if (PH == PH_GEN) {
            const bool ok = (t == 1) ? (ii + 16 < n) : (ii < n);
            x = ok ? ldg(auxp + (U + 8) * auxs) : 0.0;
          } else {
            x = ldg(auxp + (U + 8) * auxs);
          }
          S.pb[U & 7] = x;
        }
        double* lb = sm + (U & 1) * 40;  // [0..16] l, [17] y(i+16), [18] scratch, [20..36] c
#pragma unroll
        for (int m = 0; m < CPL; ++m) lb[cr[m]] = lv[m];
        lb[aux_slot] = xv;
        __syncwarp(mask);
        const double l0 = lb[0], l16 = lb[16], yn = lb[17];
#pragma unroll
        for (int m = 0; m < CPL; ++m)
          S.W[m][U] = fma(l0, lv[m], S.W[m][U] + ((m == PM && pl) ? C.sigma : 0.0));
        const double d = __shfl_sync(mask, S.W[PM][U], PT, TEAM);
        const double rs = fast_rsqrt(d);
        double cmy[CPL];
#pragma unroll
        for (int m = 0; m < CPL; ++m) {
          cmy[m] = S.W[m][U] * rs;
          lb[20 + cr[m]] = cmy[m];
        }
        const double c16 = l0 * l16 * rs;
        lb[36] = c16;
        const double rp = __shfl_sync(mask, S.res[PM], PT, TEAM);
        const double wi = rp * rs;
        bool own = true;
        if (PH == PH_GEN) own = (i >= C.s && i < C.e);
        if (PH != PH_BURN && own) {
          double* lpi = C.lpb + i * WS;
#pragma unroll
          for (int m = 0; m < CPL; ++m) lpi[cr[m]] = (m == PM && pl) ? rs : cmy[m];
          double* o2 = (t == 1) ? C.wb + i : lpi + 16;
          *o2 = (t == 1) ? wi : c16;
          if (!(d > kPivotFloor) || !(fabs(l0) > kPivotFloor)) S.fail = i < S.fail ? i : S.fail;
          S.prodp *= d * rs;
          S.prodl *= fabs(l0);
          S.ww += wi * wi;
        }
        if (PH == PH_GEN && C.side && i >= C.s - 16 && i < C.s) {
          double* sd = C.side + (i - (C.s - 16)) * 18;
#pragma unroll
          for (int m = 0; m < CPL; ++m) sd[cr[m]] = (m == PM && pl) ? rs : cmy[m];
          sd[t == 1 ? 17 : 16] = (t == 1) ? wi : c16;
        }
        if (PH != PH_BURN) {
          const ix r16 = i + 16;
          if (PH == PH_OWN ? (r16 < C.e) : (r16 >= C.s && r16 < C.e)) S.yy += yn * yn;
        }
        double ccol[CPL], lcol[CPL];
#pragma unroll
        for (int m = 0; m < CPL; ++m) {
          const bool me = (m == PM && pl);
          ccol[m] = me ? c16 : cmy[m];
          lcol[m] = me ? l16 : lv[m];
          S.res[m] = fma(-ccol[m], wi, me ? yn : S.res[m]);
        }
        __syncwarp(mask);
        // window update: W += l l^T - c c^T on my columns; the pivot lane's
        // column is dead after this row and restarts as column i+16
#pragma unroll
        for (int m = 0; m < CPL; ++m) {
          const bool me = (m == PM && pl);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (q == U) {
              S.W[m][U] = fma(l16, lcol[m], -c16 * ccol[m]);
            } else {
              const int rel = (q - U) & 15;
              S.W[m][q] = fma(lb[rel], lcol[m], fma(-lb[20 + rel], ccol[m], me ? 0.0 : S.W[m][q]));
            }
          }
        }
      },
      std::make_integer_sequence<int, 16>{});
}

// One unit: rows [s, e) owned, sweep starts at i0 (multiple of 16, <= s).
template <int TEAM>
__device__ void fwd_sweep(const FwdP& P, const Geo& G, ix b, ix s, ix e, ix i0, double* side,
                          double* part, int t, double* sm, unsigned mask, bool dummy = false) {
  constexpr int CPL = Team<TEAM>::CPL;
  const ix n = G.n;
  FwdCtx C;
  C.Lb = P.L + b * n * WS;
  C.yb = P.y + b * n;
  C.lpb = dummy ? P.lp : P.lp + b * n * WS;  // dummies write into the sink
  C.wb = dummy ? P.w : P.w + b * n;
  C.side = side;
  C.n = n;
  C.s = s;
  C.e = e;
  C.sigma = P.sigma;
  FwdSt<TEAM> S;
#pragma unroll
  for (int m = 0; m < CPL; ++m) {
#pragma unroll
    for (int q = 0; q < 16; ++q) S.W[m][q] = 0.0;
    const ix c = i0 + t + TEAM * m;  // my window column at i0
    S.res[m] = c < n ? ldg(C.yb + c) : 0.0;
  }
  S.yy = 0.0;
  S.ww = 0.0;
  S.prodp = 1.0;
  S.prodl = 1.0;
  S.ep = 0;
  S.el = 0;
  S.fail = n;
  if (i0 == s) {  // exact start: rows [s, s+16) enter now
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const ix r = s + q;
      const double v = r < e ? ldg(C.yb + r) : 0.0;
      S.yy += v * v;
    }
  }
  // prime the prefetch ring with rows i0 .. i0+7
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const ix ii = i0 + q;
#pragma unroll
    for (int m = 0; m < CPL; ++m) {
      const int crn = (t + TEAM * m - q) & 15;
      S.pa[m][q] = ii < n ? ldg(C.Lb + ii * WS + crn) : 0.0;
    }
    const bool ok = (t == 1) ? (ii + 16 < n) : (ii < n);
    S.pb[q] = ok ? ((t == 1) ? ldg(C.yb + ii + 16) : ldg(C.Lb + ii * WS + 16)) : 0.0;
  }
  for (ix base = i0; base < e; base += 16) {
    const bool inb = base + 40 <= n;  // block rows and their prefetch stay inside the matrix
    if (inb && base + 16 <= s - 16)
      fwd_block<TEAM, PH_BURN>(S, C, base, t, sm, mask);
    else if (inb && base >= s && base + 16 <= e)
      fwd_block<TEAM, PH_OWN>(S, C, base, t, sm, mask);
    else
      fwd_block<TEAM, PH_GEN>(S, C, base, t, sm, mask);
    int x;
    S.prodp = frexp(S.prodp, &x);
    S.ep += x;
    S.prodl = frexp(S.prodl, &x);
    S.el += x;
  }
  if (t == 0) {
    part[0] = log(S.prodp) + S.ep * kLn2;
    part[1] = log(S.prodl) + S.el * kLn2;
    part[2] = S.yy;
    part[3] = S.ww;
    if (S.fail < n)
      atomicMin(reinterpret_cast<unsigned long long*>(P.fail + b),
                static_cast<unsigned long long>(S.fail));
  }
}

template <int TEAM>
__global__ void __launch_bounds__(THREADS, 3) k_fwd(FwdP P, Geo G) {
  constexpr int UPB = Team<TEAM>::UPB;
  __shared__ __align__(16) double smem[UPB][80];
  const int lane = threadIdx.x & 31;
  const int slot = threadIdx.x / TEAM;
  const int t = lane & (TEAM - 1);
  ix unit = ix(blockIdx.x) * UPB + slot;
  const bool dummy = unit >= G.batch * G.nseg;
  if (dummy) unit = 0;  // padding team: recompute unit 0 into the dummy sinks
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  const ix i0 = s - G.burn > 0 ? s - G.burn : 0;
  FwdP Q = P;
  if (dummy) {
    Q.lp = P.sink;
    Q.w = P.sink;
    Q.fail = reinterpret_cast<int64_t*>(P.sink);
  }
  fwd_sweep<TEAM>(Q, G, b, s, e, i0, (p > 0 && !dummy) ? P.side + unit * SIDE : nullptr,
                  dummy ? P.sink : P.part + unit * 4, t, smem[slot], Team<TEAM>::mask(lane), dummy);
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
  double dev = 0.0;
  double wscale = 0.0;
  for (int c = 0; c < 16; ++c) wscale = fmax(wscale, fabs(P.w[b * n + s - 16 + c]));
  for (int c = 0; c < 16 && !bad; ++c) {
    const double* real = P.lp + (b * n + s - 16 + c) * WS;
    double sc = 0.0;
    for (int r = 0; r < WS; ++r) sc = fmax(sc, fabs(real[r]));
    for (int r = 0; r < WS; ++r) dev = fmax(dev, fabs(sd[c * 18 + r] - real[r]) / (sc + 1e-300));
    dev = fmax(dev, fabs(sd[c * 18 + 17] - P.w[b * n + s - 16 + c]) / (wscale + 1e-300));
    for (int r = 0; r < WS; ++r)
      if (!(fabs(sd[c * 18 + r] - real[r]) <= kCheckTol * sc)) {
        if (G.debug == 1 && !bad)
          printf("fwd check b=%lld p=%d col=%lld r=%d burn=%.17g real=%.17g\n", (long long)b, p,
                 (long long)(s - 16 + c), r, sd[c * 18 + r], real[r]);
        bad = true;
      }
    if (!(fabs(sd[c * 18 + 17] - P.w[b * n + s - 16 + c]) <= kCheckTol * (wscale + 1e-300))) {
      if (G.debug == 1 && !bad)
        printf("fwd check w b=%lld p=%d row=%lld burn=%.17g real=%.17g\n", (long long)b, p,
               (long long)(s - 16 + c), sd[c * 18 + 17], P.w[b * n + s - 16 + c]);
      bad = true;
    }
  }
  if (G.debug) note_dev(dev);
  if (bad) flag[b] = 1;
}

// One team per matrix: flagged matrices rerun the forward as one exact unit.
template <int TEAM>
__global__ void __launch_bounds__(THREADS, 3) k_repair_fwd(FwdP P, Geo G, const int32_t* flag) {
  constexpr int UPB = Team<TEAM>::UPB;
  __shared__ __align__(16) double smem[UPB][80];
  const int lane = threadIdx.x & 31;
  const int slot = threadIdx.x / TEAM;
  const ix b0 = ix(blockIdx.x) * UPB + slot;
  const bool work = b0 < G.batch && flag[b0];
  // whole warps skip when none of their teams has work; otherwise idle teams
  // run as dummies so the team collectives stay converged
  if (!__any_sync(FULL, work)) return;
  const ix b = work ? b0 : 0;
  const int t = lane & (TEAM - 1);
  FwdP Q = P;
  double* part0 = P.part + b * G.nseg * 4;
  if (work) {
    if (t == 0) {
      atomicAdd(&g_repairs, 1ull);
      P.fail[b] = G.n;
      for (int q = 4; q < G.nseg * 4; ++q) part0[q] = 0.0;
    }
  } else {
    Q.lp = P.sink;
    Q.w = P.sink;
    Q.fail = reinterpret_cast<int64_t*>(P.sink);
    part0 = P.sink;
  }
  __syncwarp();
  fwd_sweep<TEAM>(Q, G, b, 0, G.n, 0, nullptr, part0, t, smem[slot], Team<TEAM>::mask(lane), !work);
}

// ------------------------------------------------------------------ reverse
struct BwdCtx {
  const double* Lb;
  const double* lpb;
  const double* wb;
  double* lbb;
  ix n, s, e, jtop;
  double c4;
};

template <int TEAM>
struct BwdSt {
  static constexpr int RPL = Team<TEAM>::CPL;
  double S[RPL][16];  // S[m][q]: my m-th window row, column (absolute = q mod 16)
  double um[RPL];
  double pa[RPL][4], pb[RPL][4];  // prefetched Lp / L cells (distance 4 rows)
  double pc[4];                   // aux: lane 0 1/Lp(j,j), lane 1 L(j,j), lane 2 w_j
  double tr, uu;
};

// Sum of 4 values over the team, result identical on every lane:
// reduce-scatter over the top two levels, butterfly below, allgather via smem.
template <int TEAM>
__device__ __forceinline__ void team_sum4(double& a, double& b, double& c, double& d, int t,
                                          double* red, unsigned mask) {
  constexpr int H = TEAM / 2, Q = TEAM / 4;
  const bool hi = t & H;
  double k0, k1;
  {
    const double s0 = hi ? a : c, s1 = hi ? b : d;
    const double r0 = __shfl_xor_sync(mask, s0, H, TEAM);
    const double r1 = __shfl_xor_sync(mask, s1, H, TEAM);
    k0 = (hi ? c : a) + r0;
    k1 = (hi ? d : b) + r1;
  }
  const bool q1 = t & Q;
  double k = (q1 ? k1 : k0) + __shfl_xor_sync(mask, q1 ? k0 : k1, Q, TEAM);
#pragma unroll
  for (int o = Q / 2; o >= 1; o >>= 1) k += __shfl_xor_sync(mask, k, o, TEAM);
  red[t / Q] = k;  // (hi, q1) -> a, b, c, d
  __syncwarp(mask);
  a = red[0];
  b = red[1];
  c = red[2];
  d = red[3];
}

template <int TEAM, int PH>
__device__ __forceinline__ void bwd_block(BwdSt<TEAM>& S, const BwdCtx& C, ix base, int t,
                                          double* sm, unsigned mask) {
  constexpr int RPL = Team<TEAM>::CPL;
  const ix n = C.n;
  const double* auxp = (t == 2) ? C.wb : (t == 1 ? C.Lb : C.lpb);
  const int auxs = (t == 2) ? 1 : WS;
  const int aux_slot = t == 0 ? 0 : t == 1 ? 18 : t == 2 ? 36 : 54;
  unroll_down(
      [&](auto UC) {
        constexpr int U = decltype(UC)::value;
        constexpr int ET = U % TEAM;  // lane whose row j+16 leaves and row j enters
        constexpr int EM = U / TEAM;
        const ix j = base + U;
        const bool ent = (t == ET);
        int rel[RPL];
        double lpm[RPL], lm[RPL];
#pragma unroll
        for (int m = 0; m < RPL; ++m) {
          rel[m] = ((t + TEAM * m - U - 1) & 15) + 1;
          lpm[m] = S.pa[m][U & 3];
          lm[m] = S.pb[m][U & 3];
        }
        const double xv = S.pc[U & 3];
        {  // prefetch row j - 4
          const ix jj = j - 4;
          const bool ok = (PH != PH_GEN) || (jj >= 0 && jj < n);
#pragma unroll
          for (int m = 0; m < RPL; ++m) {
            const int reln = ((t + TEAM * m - U + 4 - 1) & 15) + 1;
            S.pa[m][U & 3] = ok ? ldg(C.lpb + jj * WS + reln) : 0.0;
            S.pb[m][U & 3] = ok ? ldg(C.Lb + jj * WS + reln) : 0.0;
          }
          S.pc[U & 3] = ok ? ldg(auxp + jj * auxs) : 0.0;
        }
        if (PH == PH_GEN && j > C.jtop) return;
        double* sb = sm + (U & 1) * 64;  // [0] 1/Lp(j,j) [1..16] Lp col, [18] L(j,j) [19..34] L col,
                                         // [36] w_j [37..52] S(.,j), [54] scratch, [56..59] sums
#pragma unroll
        for (int m = 0; m < RPL; ++m) {
          sb[rel[m]] = lpm[m];
          sb[18 + rel[m]] = lm[m];
        }
        sb[aux_slot] = xv;
        __syncwarp(mask);
        const double inv = sb[0], ljj = sb[18], wj = sb[36];
        double out[RPL], accl[RPL];
#pragma unroll
        for (int m = 0; m < RPL; ++m) {
          double a0 = 0.0, a1 = 0.0, l0 = 0.0, l1 = 0.0;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int cs = ((q - U - 1) & 15) + 1;
            if (q & 1) {
              a1 = fma(S.S[m][q], sb[cs], a1);
              l1 = fma(S.S[m][q], sb[18 + cs], l1);
            } else {
              a0 = fma(S.S[m][q], sb[cs], a0);
              l0 = fma(S.S[m][q], sb[18 + cs], l0);
            }
          }
          out[m] = (a0 + a1) * inv;
          accl[m] = l0 + l1;
        }
        double ra = 0.0, rb = 0.0, rc = 0.0, rd = 0.0;
#pragma unroll
        for (int m = 0; m < RPL; ++m) {
          ra = fma(lpm[m], out[m], ra);
          rb = fma(lpm[m], S.um[m], rb);
          rc = fma(S.um[m], lm[m], rc);
          rd = fma(out[m], lm[m], rd);
        }
        team_sum4<TEAM>(ra, rb, rc, rd, t, sb + 56, mask);
        const double sjj = inv * inv + inv * ra;
        const double uj = (wj - rb) * inv;
        const double ul = uj * ljj + rc;
        bool own = true;
        if (PH == PH_GEN) own = (j >= C.s && j < C.e);
        if (PH == PH_BURN) own = false;
        if (own) {
          double* lbj = C.lbb + j * WS;
#pragma unroll
          for (int m = 0; m < RPL; ++m) {
            const double v = -(accl[m] - out[m] * ljj) - C.c4 * S.um[m] * ul;
            lbj[rel[m]] = (PH == PH_GEN && j + rel[m] >= n) ? 0.0 : v;
          }
          const double dj = rd - sjj * ljj - C.c4 * uj * ul + fast_rcp(ljj);
          if (ent) lbj[0] = dj;
          S.tr += sjj;
          S.uu += uj * uj;
        }
#pragma unroll
        for (int m = 0; m < RPL; ++m) {
          sb[36 + rel[m]] = -out[m];
          S.S[m][U] = -out[m];
        }
        __syncwarp(mask);
        if (ent) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q != U) S.S[EM][q] = sb[36 + (((q - U - 1) & 15) + 1)];
          S.S[EM][U] = sjj;
          S.um[EM] = uj;
        }
      },
      std::make_integer_sequence<int, 16>{});
}

template <int TEAM>
__device__ void bwd_sweep(const BwdP& P, const Geo& G, ix b, ix s, ix e, ix jtop, double* entry,
                          double* exitb, double* part, int t, double* sm, unsigned mask,
                          bool dummy = false) {
  constexpr int RPL = Team<TEAM>::CPL;
  const ix n = G.n;
  BwdCtx C;
  C.Lb = P.L + b * n * WS;
  C.lpb = P.lp + b * n * WS;
  C.wb = P.w + b * n;
  C.lbb = dummy ? P.lbar : P.lbar + b * n * WS;
  C.n = n;
  C.s = s;
  C.e = e;
  C.jtop = jtop;
  C.c4 = P.c4;
  BwdSt<TEAM> S;
#pragma unroll
  for (int m = 0; m < RPL; ++m) {
#pragma unroll
    for (int q = 0; q < 16; ++q) S.S[m][q] = 0.0;
    S.um[m] = 0.0;
  }
  S.tr = 0.0;
  S.uu = 0.0;
  const ix top_base = jtop / 16 * 16;
  const double* auxp = (t == 2) ? C.wb : (t == 1 ? C.Lb : C.lpb);
  const int auxs = (t == 2) ? 1 : WS;
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // rows top_base+15 .. top_base+12
    const int U = 15 - q;
    const ix jj = top_base + U;
    const bool ok = jj < n;
#pragma unroll
    for (int m = 0; m < RPL; ++m) {
      const int rl = ((t + TEAM * m - U - 1) & 15) + 1;
      S.pa[m][U & 3] = ok ? ldg(C.lpb + jj * WS + rl) : 0.0;
      S.pb[m][U & 3] = ok ? ldg(C.Lb + jj * WS + rl) : 0.0;
    }
    S.pc[U & 3] = ok ? ldg(auxp + jj * auxs) : 0.0;
  }
  for (ix base = top_base; base >= s; base -= 16) {
    if (entry && base + 16 == e) {  // boundary window [e, e+16) reached by burn-in
#pragma unroll
      for (int m = 0; m < RPL; ++m) {
        double* en = entry + (t + TEAM * m) * 17;
#pragma unroll
        for (int q = 0; q < 16; ++q) en[q] = S.S[m][q];
        en[16] = S.um[m];
      }
    }
    const bool inb = base >= 16 && base + 31 < n && base + 15 <= jtop;
    if (inb && base >= e)
      bwd_block<TEAM, PH_BURN>(S, C, base, t, sm, mask);
    else if (inb && base >= s && base + 16 <= e)
      bwd_block<TEAM, PH_OWN>(S, C, base, t, sm, mask);
    else
      bwd_block<TEAM, PH_GEN>(S, C, base, t, sm, mask);
  }
  if (exitb) {
#pragma unroll
    for (int m = 0; m < RPL; ++m) {
      double* ex = exitb + (t + TEAM * m) * 17;
#pragma unroll
      for (int q = 0; q < 16; ++q) ex[q] = S.S[m][q];
      ex[16] = S.um[m];
    }
  }
  if (t == 0) {
    part[0] = S.tr;
    part[1] = S.uu;
  }
}

template <int TEAM>
__global__ void __launch_bounds__(THREADS, 3) k_bwd(BwdP P, Geo G) {
  constexpr int UPB = Team<TEAM>::UPB;
  __shared__ __align__(16) double smem[UPB][128];
  const int lane = threadIdx.x & 31;
  const int slot = threadIdx.x / TEAM;
  const int t = lane & (TEAM - 1);
  ix unit = ix(blockIdx.x) * UPB + slot;
  const bool dummy = unit >= G.batch * G.nseg;
  if (dummy) unit = 0;
  const ix b = unit / G.nseg;
  const int p = int(unit % G.nseg);
  const ix s = ix(p) * G.seg;
  const ix e = s + G.seg < G.n ? s + G.seg : G.n;
  ix jtop = e + G.burn - 1;
  if (jtop > G.n - 1) jtop = G.n - 1;
  BwdP Q = P;
  if (dummy) Q.lbar = P.sink;
  bwd_sweep<TEAM>(Q, G, b, s, e, jtop, (p + 1 < G.nseg && !dummy) ? P.entry + unit * STATE : nullptr,
                  (p > 0 && !dummy) ? P.exitb + unit * STATE : nullptr,
                  dummy ? P.sink : P.part + unit * 2, t, smem[slot], Team<TEAM>::mask(lane), dummy);
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
  double dev = 0.0;
  for (int q = 0; q < 16; ++q) {
    for (int c = 0; c < 17; ++c) {
      const double sc = c < 16 ? ss : us;
      dev = fmax(dev, fabs(a[q * 17 + c] - r[q * 17 + c]) / (sc + 1e-300));
      if (!(fabs(a[q * 17 + c] - r[q * 17 + c]) <= kCheckTol * (sc + 1e-300))) {
        if (G.debug == 1 && !bad)
          printf("bwd check b=%lld p=%d lane=%d slot=%d burn=%.17g real=%.17g\n", (long long)b, p, q,
                 c, a[q * 17 + c], r[q * 17 + c]);
        bad = true;
      }
    }
  }
  if (G.debug) note_dev(dev);
  if (bad) flag[b] = 1;
}

template <int TEAM>
__global__ void __launch_bounds__(THREADS, 3) k_repair_bwd(BwdP P, Geo G, const int32_t* flag,
                                                           const int64_t* fail) {
  constexpr int UPB = Team<TEAM>::UPB;
  __shared__ __align__(16) double smem[UPB][128];
  const int lane = threadIdx.x & 31;
  const int slot = threadIdx.x / TEAM;
  const ix b0 = ix(blockIdx.x) * UPB + slot;
  const bool work = b0 < G.batch && flag[b0] && fail[b0] >= G.n;
  if (!__any_sync(FULL, work)) return;
  const ix b = work ? b0 : 0;
  const int t = lane & (TEAM - 1);
  BwdP Q = P;
  double* part0 = P.part + b * G.nseg * 2;
  if (work) {
    if (t == 0) {
      atomicAdd(&g_repairs, 1ull);
      for (int q = 2; q < G.nseg * 2; ++q) part0[q] = 0.0;
    }
  } else {
    Q.lbar = P.sink;
    part0 = P.sink;
  }
  __syncwarp();
  bwd_sweep<TEAM>(Q, G, b, 0, G.n, G.n - 1, nullptr, nullptr, part0, t, smem[slot],
                  Team<TEAM>::mask(lane), !work);
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

int mlik_repairs(int64_t* count, double* max_dev, int reset) {
  unsigned long long v = 0, d = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&v, g_repairs, sizeof v);
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(&d, g_maxdev, sizeof d);
  if (e != cudaSuccess) return set_error(e);
  if (count) *count = int64_t(v);
  if (max_dev) *max_dev = __builtin_bit_cast(double, d);
  if (reset) {
    v = 0;
    e = cudaMemcpyToSymbol(g_repairs, &v, sizeof v);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_maxdev, &v, sizeof v);
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
  G.burn = 128;  // window errors ride ~16 rows to the pivot before damping (~1e-2-1e-3 per 16 rows)
  {
    const char* dbg = std::getenv("BGM_DEBUG");
    G.debug = dbg ? (dbg[0] == '1' ? 2 : dbg[0] == '2' ? 1 : 0) : 0;  // 1: printf + dev, 2: dev only
  }
  // Team size: BGM_TEAM=8|16 (default 16).
  int team = 16;
  {
    const char* e = std::getenv("BGM_TEAM");
    if (e && std::atoi(e) == 8) team = 8;
  }
  // One wave: as many units as fit resident on the chip.
  int sms = 148, bpm = 1;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int bf = 1, bb = 1;
    if (team == 8) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bf, k_fwd<8>, THREADS, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bb, k_bwd<8>, THREADS, 0);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bf, k_fwd<16>, THREADS, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bb, k_bwd<16>, THREADS, 0);
    }
    bpm = bf < bb ? bf : bb;
    if (bpm < 1) bpm = 1;
  }
  const int upb = (32 / team) * WARPS;
  ix seg = segment_rows;
  if (seg <= 0) {
    const ix capacity = ix(sms) * bpm * upb;
    ix per = capacity / G.batch;
    if (per < 1) per = 1;
    seg = (G.n + per - 1) / per;
    seg = (seg + 15) / 16 * 16;
    if (seg < 4 * G.burn) seg = 4 * G.burn;
  }
  G.seg = seg;
  G.nseg = int((G.n + seg - 1) / seg);
  const ix units = G.batch * G.nseg;

  // scratch: Lp, w, side, fwd parts, states, bwd parts, fail, flags
  const size_t nb = size_t(G.batch) * size_t(G.n);
  const size_t sink_len = size_t(G.n) * WS + 64;
  const size_t bytes = sizeof(double) * (nb * WS + nb + size_t(units) * (SIDE + 4 + 2 * STATE + 2) + sink_len) +
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
  F.sink = dp;
  Bp.sink = dp;
  dp += sink_len;
  F.fail = reinterpret_cast<int64_t*>(dp);
  int32_t* flags = reinterpret_cast<int32_t*>(F.fail + G.batch);
  F.sigma = 1.0 / tau2;
  Bp.L = F.L;
  Bp.lp = F.lp;
  Bp.w = F.w;
  Bp.lbar = static_cast<double*>(lbar.data);
  Bp.c4 = F.sigma * F.sigma;

  const unsigned ublocks = unsigned((units + upb - 1) / upb);
  const unsigned mblocks = unsigned((G.batch + upb - 1) / upb);
  const unsigned cblocks = unsigned((units + 127) / 128);
  k_init_fail<<<blocks_for(G.batch, 128), 128, 0, s>>>(F.fail, flags, G.batch, G.n);
  {
    timing::Scope ts("mlik_seg_fwd", s);
    if (team == 8)
      k_fwd<8><<<ublocks, THREADS, 0, s>>>(F, G);
    else
      k_fwd<16><<<ublocks, THREADS, 0, s>>>(F, G);
  }
  {
    timing::Scope ts("mlik_seg_check", s);
    k_check_fwd<<<cblocks, 128, 0, s>>>(F, G, flags);
    if (team == 8)
      k_repair_fwd<8><<<mblocks, THREADS, 0, s>>>(F, G, flags);
    else
      k_repair_fwd<16><<<mblocks, THREADS, 0, s>>>(F, G, flags);
  }
  {
    timing::Scope ts("mlik_seg_bwd", s);
    if (team == 8)
      k_bwd<8><<<ublocks, THREADS, 0, s>>>(Bp, G);
    else
      k_bwd<16><<<ublocks, THREADS, 0, s>>>(Bp, G);
  }
  {
    timing::Scope ts("mlik_seg_check", s);
    k_check_bwd<<<cblocks, 128, 0, s>>>(Bp, G, flags + G.batch);
    if (team == 8)
      k_repair_bwd<8><<<mblocks, THREADS, 0, s>>>(Bp, G, flags + G.batch, F.fail);
    else
      k_repair_bwd<16><<<mblocks, THREADS, 0, s>>>(Bp, G, flags + G.batch, F.fail);
    k_finalize<<<blocks_for(G.batch, 128), 128, 0, s>>>(F.part, Bp.part, F.fail, G, tau2, loss,
                                                        tau2_bar, status, row);
  }
  err = cudaGetLastError();
  cudaFreeAsync(ws, s);
  return err == cudaSuccess ? BGM_OK : set_error(err);
}

}  // namespace bgm
