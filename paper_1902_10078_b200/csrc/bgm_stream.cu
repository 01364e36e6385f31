// Staged band x band products and the fused product VJP for the 32-matrix
// interleaved layout (tile 32): kernels_detail.hpp:16-28 (product_column),
// kernels.cpp:72-90 (product_band_band / _restricted), grad.cpp:145-151
// (vjp_product_band_band).
//
// The band products are HBM streams: every operand column is read from HBM
// once and reused by the 2k+1 output columns around it.  Here the reuse
// happens in shared memory instead of L1:
//
//  * one persistent CTA per SM walks a contiguous run of output columns of
//    one tile (32 matrices) -- or of one lane group of LN matrices of it;
//  * each operand has a ring of RC columns in shared memory, filled by TMA
//    tensor copies (cp.async.bulk.tensor.3d over lanes x cells x columns; box = LN lanes x W storage rows,
//    i.e. one band column of LN matrices) that complete on an mbarrier;
//    loads run D steps (D*CJ columns) ahead of the compute;
//  * a thread's window of H+1 columns (H = the operand's column halo) wraps
//    at most once around the ring: one compare-select per column, and every
//    shared-memory read within a column has a compile-time offset;
//  * thread = (matrix lane, output column): it loads op(Y)(., j) once into
//    registers, accumulates each output cell over its exact k range with
//    one LDS + a multiply and an add per term, in the reference's k order
//    without FMA contraction (kernels_detail.hpp:22-24: s += a(i,k) b(k,j)),
//    so fp64 results are bitwise the reference's (the k = 16 shapes of config
//    3 use FMA instead: FP64-bound otherwise); fp64 accumulation for fp32,
//    and stores the column with coalesced 8-byte stores (LN lanes x 8 B);
//  * the fused VJP stages P-bar, A and B once and produces both A-bar and
//    B-bar columns from them (grad.cpp:148-149), so P-bar is read from HBM
//    once instead of twice.
//
// Columns outside [0, n) and corner cells are never trusted: steps whose
// windows touch either matrix end run a predicated variant; interior steps
// run unpredicated.  Shapes are compile-time (the benchmarked band shapes of
// configs 2 and 3); anything else returns false and runs bgm_product.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "bgm_common.cuh"
#include "bgm_timing.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace stream {
namespace {

constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }

// One product C = op(X) op(Y) restricted to C's band.  X, Y stored bands
// (XL, XU), (YL, YU); TX / TY = read transposed; output band (CL, CU).
template <int TX_, int TY_, int XL_, int XU_, int YL_, int YU_, int CL_, int CU_>
struct PS {
  static constexpr int TX = TX_, TY = TY_, XL = XL_, XU = XU_, YL = YL_, YU = YU_, CL = CL_, CU = CU_;
  static constexpr int CW = CL + CU + 1;
  static constexpr int OXL = TX ? XU : XL, OXU = TX ? XL : XU;
  static constexpr int OYL = TY ? YU : YL, OYU = TY ? YL : YU;
  // k - j over all terms of output column j, and i - j of cells with terms
  static constexpr int EMIN = cmax(-OYU, -CU - OXL), EMAX = cmin(OYL, CL + OXU);
  static constexpr int DMIN = cmax(-CU, -OYU - OXU), DMAX = cmin(CL, OYL + OXL);
  // stored-column offsets (relative to j) read from X and from Y
  static constexpr int XLO = TX ? DMIN : EMIN, XHI = TX ? DMAX : EMAX;
  static constexpr int YLO = TY ? EMIN : 0, YHI = TY ? EMAX : 0;
  static constexpr int MARGIN = cmax(cmax(-EMIN, EMAX), cmax(CU, CL));
};

struct NoP {
  static constexpr int XLO = 0, XHI = 0, YLO = 0, YHI = 0, MARGIN = 0;
};

// Up to three staged operands (widths W0..W2) and one or two products
// reading them (operand indices X1, Y1, X2, Y2).
template <int NOP_, int W0, int W1, int W2, class P1_, int X1_, int Y1_, class P2_ = NoP, int X2_ = 0, int Y2_ = 0,
          bool FMA_ = false>
struct Spec {
  static constexpr int NOP = NOP_;
  // FMA: contract each term into one fused multiply-add.  Off (the default),
  // terms are a separate multiply and add in the reference's order, and fp64
  // results are bitwise the reference's; on for the k = 16 shapes, whose
  // doubled fp64 instruction count would otherwise make them FP64-bound.
  static constexpr bool FMA = FMA_;
  using P1 = P1_;
  using P2 = P2_;
  static constexpr int X1 = X1_, Y1 = Y1_, X2 = X2_, Y2 = Y2_;
  static constexpr bool TWO = !std::is_same<P2_, NoP>::value;
  static constexpr int W(int o) { return o == 0 ? W0 : o == 1 ? W1 : W2; }
  static constexpr int lo(int o) {
    return cmin(cmin(X1 == o ? P1::XLO : 0, Y1 == o ? P1::YLO : 0),
                cmin(TWO && X2 == o ? P2::XLO : 0, TWO && Y2 == o ? P2::YLO : 0));
  }
  static constexpr int hi(int o) {
    return cmax(cmax(X1 == o ? P1::XHI : 0, Y1 == o ? P1::YHI : 0),
                cmax(TWO && X2 == o ? P2::XHI : 0, TWO && Y2 == o ? P2::YHI : 0));
  }
  static constexpr int H(int o) { return hi(o) - lo(o); }
  static constexpr int MARGIN = cmax(cmax(P1::MARGIN, P2::MARGIN),
                                     cmax(cmax(-lo(0), hi(0)), cmax(cmax(-lo(1), hi(1)), cmax(-lo(2), hi(2)))));
};

// Ring geometry of operand o for lane-group width LN, CJ columns per step
// and D steps of prefetch.  A ring slot holds one band column of LN
// matrices: WP >= W cells (the TMA box pads the column with out-of-bounds
// zero cells so every slot starts on a 128-byte boundary), SS = WP * LN
// elements.  RC = ring columns (a multiple of CJ: step loads land on
// CJ-aligned slots as one box).  MIR: the ring keeps a copy of its first H
// slots after its end (PH = physical slots), so windows never wrap (no
// per-column select) at the cost of H more slots.
// Consumer threads = LN * CJ * NPART (NPART = 2: the two products of a
// fused VJP, or the two halves of one product's cells); one producer warp.
template <class T, int LN, int CJ, int D, int NPART, class S, bool MIR>
struct Geom {
  static constexpr int WP(int o) {
    return (S::W(o) * LN * int(sizeof(T))) % 128 == 0 ? S::W(o)
           : (S::W(o) + 1) * LN * int(sizeof(T)) % 128 == 0 ? S::W(o) + 1
           : (S::W(o) + 2) * LN * int(sizeof(T)) % 128 == 0 ? S::W(o) + 2
                                                             : S::W(o) + 3;
  }
  static constexpr int SS(int o) { return WP(o) * LN; }
  static constexpr int RC(int o) { return ((D + 1) * CJ + S::H(o) + CJ - 1) / CJ * CJ; }
  static constexpr int PH(int o) { return RC(o) + (MIR ? (S::H(o) + CJ - 1) / CJ * CJ : 0); }
  // ring size seen by a window: with the mirror a window never wraps
  static constexpr int WRC(int o) { return MIR ? (1 << 30) : RC(o); }
  static constexpr int OFF(int o) { return o == 0 ? 0 : o == 1 ? PH(0) * SS(0) : PH(0) * SS(0) + PH(1) * SS(1); }
  static constexpr int ELEMS = OFF(2) + (S::NOP > 2 ? PH(2) * SS(2) : 0);
  static constexpr size_t SMEM = size_t(ELEMS) * sizeof(T) + 16 * (D + 1);
  static constexpr int NC = LN * CJ * NPART;
  static constexpr int THREADS = NC + 32;
};

// per operand: box of CJ columns (step loads) and of one column (run starts)
struct Maps {
  CUtensorMap step[3];
  CUtensorMap col[3];
};

struct SGeo {
  ix n;
  ix nchunks;  // ceil(n / CJ)
  ix plane;    // tiles * nchunks: work units of one lane group
  ix per;      // units per CTA
  int groups;  // 32 / LN; CTA c serves lane group c % groups
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_init_n(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
// box at (lane x, cell 0, column z) of the (lanes, cells, columns) tensor
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* map, int x, int z, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(0), "r"(z), "r"(bar)
      : "memory");
}

// Output column j of one product from the staged windows.  A window points
// at the thread's lane in the slot s of stored column j + LO; stored column
// j + LO + q sits q slots further, wrapping once at RC (one compare-select
// per column; the row offsets within a column are immediates).
template <int SS, int RC>
struct Win {
  const void* b;
  int s;
  template <class T>
  __device__ __forceinline__ const T* col(int q) const {
    const T* p = static_cast<const T*>(b);
    return s + q >= RC ? p + (q - RC) * SS : p + q * SS;
  }
};

template <class T, int LN, class P, class WX, class WY, int LOX, int LOY, int R0, int R1, bool EDGE, bool FMA>
__device__ __forceinline__ void prod_col(WX wx, WY wy, ix j, ix n, T* __restrict__ out) {
  constexpr int NE = P::EMAX - P::EMIN + 1;
  acc_t yv[NE];
  bool kv[NE];
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    const int e = P::EMIN + q;
    const T* p = P::TY ? wy.template col<T>(e - LOY) + (P::YU - e) * LN : wy.template col<T>(0 - LOY) + (e + P::YU) * LN;
    kv[q] = !EDGE || (j + e >= 0 && j + e < n);
    yv[q] = acc_t(*p);
  }
#pragma unroll
  for (int r = R0; r < R1; ++r) {
    const int d = r - P::CU;
    const int elo = cmax(d - P::OXL, P::EMIN), ehi = cmin(d + P::OXU, P::EMAX);
    acc_t acc = 0;
#pragma unroll
    for (int q = 0; q < NE; ++q) {
      const int e = P::EMIN + q;
      if (e < elo || e > ehi) continue;
      const T* p = P::TX ? wx.template col<T>(d - LOX) + (e - d + P::XU) * LN
                         : wx.template col<T>(e - LOX) + (d - e + P::XU) * LN;
      if (!EDGE || kv[q])  // FMA off: no contraction, the reference's s += a * b
        acc = FMA ? fma(acc_t(*p), yv[q], acc) : __dadd_rn(acc, __dmul_rn(acc_t(*p), yv[q]));
    }
    T v = T(acc);
    if (EDGE && (j + d < 0 || j + d >= n)) v = T(0);
    out[r * 32] = v;
  }
}

// Consumer part PART of NPART (warp-uniform): the product it serves (the
// two products of a fused VJP split the parts) and its share of that
// product's output cells.
template <class T, int LN, class Gm, class S, int NPART, int PART>
__device__ __forceinline__ void do_part(const T* const* b, const int* sl, ix j, ix n, bool interior, T* o1, T* o2) {
  constexpr int NSUB = S::TWO ? NPART / 2 : NPART;
  constexpr int PI = S::TWO ? PART / NSUB : 0;
  constexpr int SUB = PART % NSUB;
  using P = std::conditional_t<PI == 0, typename S::P1, typename S::P2>;
  constexpr int X = PI == 0 ? S::X1 : S::X2, Y = PI == 0 ? S::Y1 : S::Y2;
  constexpr int R0 = P::CW * SUB / NSUB, R1 = P::CW * (SUB + 1) / NSUB;
  using WX = Win<Gm::SS(X), Gm::WRC(X)>;
  using WY = Win<Gm::SS(Y), Gm::WRC(Y)>;
  T* o = PI == 0 ? o1 : o2;
  if (interior)
    prod_col<T, LN, P, WX, WY, S::lo(X), S::lo(Y), R0, R1, false, S::FMA>(WX{b[X], sl[X]}, WY{b[Y], sl[Y]}, j, n, o);
  else
    prod_col<T, LN, P, WX, WY, S::lo(X), S::lo(Y), R0, R1, true, S::FMA>(WX{b[X], sl[X]}, WY{b[Y], sl[Y]}, j, n, o);
}

// Producer warp: one lane walks the CTA's runs and issues, for every step,
// the TMA copies of the operand columns new at that step (the whole first
// window at a run start), after the consumers released the ring slots they
// overwrite (empty barrier of the step NB earlier; a full drain at run
// starts, where the column -> slot mapping restarts).  Consumers wait on the
// step's full barrier, compute their output columns, and release the step.
template <class T, int LN, int CJ, int D, int NPART, class S, bool MIR>
__global__ void __launch_bounds__(LN* CJ* NPART + 32) k_stream(const __grid_constant__ Maps maps, T* __restrict__ c1,
                                                              T* __restrict__ c2, SGeo G) {
  using Gm = Geom<T, LN, CJ, D, NPART, S, MIR>;
  constexpr int NB = D + 1;
  constexpr int NC = Gm::NC;
  static_assert((LN * CJ) % 32 == 0, "a consumer part must be whole warps");
  static_assert(NPART == 1 || NPART == 2 || NPART == 4, "parts");
  static_assert(!S::TWO || NPART >= 2, "a fused VJP needs a part per product");
  static_assert(CJ <= 256 && LN * sizeof(T) % 16 == 0, "TMA box limits");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + size_t(Gm::ELEMS) * sizeof(T));
  uint64_t* empty = full + NB;
  const int tid = threadIdx.x;
  if (tid == NC) {
    for (int i = 0; i < NB; ++i) {
      bar_init_n(smem_u32(&full[i]), 1);
      bar_init_n(smem_u32(&empty[i]), NC / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const ix n = G.n;
  const int grp = int(blockIdx.x % unsigned(G.groups));
  const int lane0 = grp * LN;
  const ix ubeg = ix(blockIdx.x / unsigned(G.groups)) * G.per;
  const ix uend = ubeg + G.per < G.plane ? ubeg + G.per : G.plane;

  if (tid >= NC) {  // ---- producer warp
    if (tid != NC) return;
    for (int o = 0; o < S::NOP; ++o) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.step[o]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.col[o]) : "memory");
    }
    uint32_t g = 0;
    for (ix u = ubeg; u < uend;) {
      const ix tile = u / G.nchunks, c0 = u % G.nchunks;
      const int steps = int((c0 + (uend - u) < G.nchunks ? c0 + (uend - u) : G.nchunks) - c0);
      u += steps;
      const int zf = int(tile * n + c0 * CJ);  // global column index of the run start
      // drain: every step of the previous run released
      for (uint32_t q = g >= uint32_t(NB) ? g - NB : 0; q < g; ++q) bar_wait(smem_u32(&empty[q % NB]), (q / NB) & 1);
      for (int l = 0; l < steps; ++l) {
        const uint32_t m = g + l;
        if (l >= NB) bar_wait(smem_u32(&empty[m % NB]), ((m - NB) / NB) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bar = smem_u32(&full[m % NB]);
        // run-relative column rel sits in slot (rel - hi) mod RC: step l's new
        // columns [l CJ + hi, (l+1) CJ + hi) are the CJ-aligned slots from l CJ mod RC
        uint32_t bytes = 0;
#pragma unroll
        for (int o = 0; o < S::NOP; ++o) {
          const uint32_t colb = uint32_t(Gm::SS(o) * sizeof(T));
          bytes += colb * CJ * (MIR && (l * CJ) % Gm::RC(o) < S::H(o) ? 2u : 1u);
          if (l == 0) bytes += colb * S::H(o) * (MIR && Gm::RC(o) - S::H(o) < S::H(o) ? 2u : 1u);
        }
        bar_expect(bar, bytes);
#pragma unroll
        for (int o = 0; o < S::NOP; ++o) {
          const int lo = S::lo(o), hi = S::hi(o), RCo = Gm::RC(o);
          T* base = ring + Gm::OFF(o);
          if (l == 0) {  // the halo [lo, hi) before the first step's columns
            for (int rel = lo; rel < hi; ++rel) {
              const int slot = rel - hi + RCo;
              tma_load(smem_u32(base + slot * Gm::SS(o)), &maps.col[o], lane0, zf + rel, bar);
              if (MIR && slot < S::H(o))
                tma_load(smem_u32(base + (slot + RCo) * Gm::SS(o)), &maps.col[o], lane0, zf + rel, bar);
            }
          }
          const int slot = (l * CJ) % RCo;
          const int z = zf + l * CJ + hi;
          tma_load(smem_u32(base + slot * Gm::SS(o)), &maps.step[o], lane0, z, bar);
          if (MIR && slot < S::H(o)) tma_load(smem_u32(base + (slot + RCo) * Gm::SS(o)), &maps.step[o], lane0, z, bar);
        }
      }
      g += steps;
    }
    return;
  }

  // ---- consumers
  constexpr int PT = LN * CJ;
  const int part = tid / PT;
  const int lane = tid % LN, cj = (tid % PT) / LN;
  uint32_t g = 0;
  for (ix u = ubeg; u < uend;) {
    const ix tile = u / G.nchunks, c0 = u % G.nchunks;
    const int steps = int((c0 + (uend - u) < G.nchunks ? c0 + (uend - u) : G.nchunks) - c0);
    u += steps;
    const ix jf = c0 * CJ;
    for (int l = 0; l < steps; ++l) {
      const uint32_t m = g + l;
      bar_wait(smem_u32(&full[m % NB]), (m / NB) & 1);
      const ix jt = jf + ix(l) * CJ;
      const ix j = jt + cj;
      if (j < n) {
        const int rel = l * CJ + cj;  // column j relative to the run start; window starts at rel + lo
        int sl[3];
        const T* b[3];
#pragma unroll
        for (int o = 0; o < 3; ++o) {
          sl[o] = o < S::NOP ? (rel + Gm::RC(o) - S::H(o)) % Gm::RC(o) : 0;
          b[o] = o < S::NOP ? ring + Gm::OFF(o) + sl[o] * Gm::SS(o) + lane : ring;
        }
        const bool interior = jt >= S::MARGIN && jt + CJ - 1 + S::MARGIN <= n - 1;
        T* o1 = c1 + ((tile * n + j) * S::P1::CW) * 32 + lane0 + lane;
        T* o2 = nullptr;
        if constexpr (S::TWO) o2 = c2 + ((tile * n + j) * S::P2::CW) * 32 + lane0 + lane;
        switch (part) {
          case 0:
            do_part<T, LN, Gm, S, NPART, 0>(b, sl, j, n, interior, o1, o2);
            break;
          case 1:
            if constexpr (NPART > 1) do_part<T, LN, Gm, S, NPART, 1>(b, sl, j, n, interior, o1, o2);
            break;
          case 2:
            if constexpr (NPART > 2) do_part<T, LN, Gm, S, NPART, 2>(b, sl, j, n, interior, o1, o2);
            break;
          default:
            if constexpr (NPART > 3) do_part<T, LN, Gm, S, NPART, 3>(b, sl, j, n, interior, o1, o2);
            break;
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) bar_arrive(smem_u32(&empty[m % NB]));
    }
    g += steps;
  }
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Whole band array as a 3-D tensor (32 lanes, w cells, tiles * n columns);
// box = (LN lanes, WP cells, ncol columns), cells w.. WP-1 out of bounds
// (zero-filled) so that each column fills a 128-byte-aligned slot.
template <class T>
bool make_map(CUtensorMap* m, const bgm_band& d, int LN, int WP, int ncol) {
  auto enc = encoder();
  if (!enc) return false;
  const int w = d.lower + d.upper + 1;
  const ix tiles = (d.batch + 31) / 32;
  cuuint64_t dims[3] = {32, cuuint64_t(w), cuuint64_t(tiles * d.n)};
  cuuint64_t strides[2] = {32 * sizeof(T), cuuint64_t(w) * 32 * sizeof(T)};
  cuuint32_t box[3] = {cuuint32_t(LN), cuuint32_t(WP), cuuint32_t(ncol)};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d.data, dims,
             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             // promote to the box row only: a wider promotion fetches the other lane
             // groups' halves, which their own CTAs re-read later
             LN * sizeof(T) >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
             : LN * sizeof(T) >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool usable(const bgm_band& d) {
  const ix tiles = (d.batch + 31) / 32;
  return d.tile == 32 && (reinterpret_cast<uintptr_t>(d.data) & 15) == 0 && tiles * d.n < (ix(1) << 31);
}

template <class T, int LN, int CJ, int D, int NPART, class S, bool MIR>
bool run(const bgm_band* ops, const bgm_band& c1, const bgm_band* c2, const char* name, cudaStream_t s) {
  using Gm = Geom<T, LN, CJ, D, NPART, S, MIR>;
  static_assert(Gm::SMEM <= 227 * 1024, "ring does not fit in shared memory");
  static_assert(Gm::THREADS <= 1024, "block too large");
  auto kern = k_stream<T, LN, CJ, D, NPART, S, MIR>;
  const ix n = c1.n;
  if (n < 4 * (S::MARGIN + CJ)) return false;
  for (int o = 0; o < S::NOP; ++o)
    if (!usable(ops[o]) || ops[o].lower + ops[o].upper + 1 != S::W(o)) return false;
  if (!usable(c1) || (c2 && !usable(*c2))) return false;
  Maps maps;
  for (int o = 0; o < S::NOP; ++o)
    if (!make_map<T>(&maps.step[o], ops[o], LN, Gm::WP(o), CJ) || !make_map<T>(&maps.col[o], ops[o], LN, Gm::WP(o), 1))
      return false;
  static PerDeviceInt occ_cache;
  int occ = occ_cache.get();
  if (occ < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::SMEM));
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, Gm::THREADS, Gm::SMEM);
    occ = per;
    occ_cache.set(per);
  }
  if (occ < 1) return false;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  SGeo G;
  G.n = n;
  G.nchunks = (n + CJ - 1) / CJ;
  G.groups = 32 / LN;
  G.plane = (c1.batch + 31) / 32 * G.nchunks;
  ix per_plane = ix(sms) * occ / G.groups;
  if (per_plane < 1) per_plane = 1;
  G.per = (G.plane + per_plane - 1) / per_plane;
  per_plane = (G.plane + G.per - 1) / G.per;
  timing::Scope t(name, s);
  kern<<<unsigned(per_plane * G.groups), Gm::THREADS, Gm::SMEM, s>>>(
      maps, static_cast<T*>(c1.data), c2 ? static_cast<T*>(c2->data) : nullptr, G);
  return cudaPeekAtLastError() == cudaSuccess;
}

// Configurations are given for fp64 (lane-group width LN, CJ columns per
// step).  fp32 rows are half as wide: twice the lanes and half the columns
// per step when LN < 32 (same thread count, same TMA row bytes).
template <class T, int LN, int CJ, int D, int NPART, class S, bool MIR>
bool run_cfg(const bgm_band* ops, const bgm_band& c1, const bgm_band* c2, const char* name, cudaStream_t s) {
  constexpr bool widen = sizeof(T) == 4 && LN < 32 && CJ % 2 == 0;
  return run<T, widen ? 2 * LN : LN, widen ? CJ / 2 : CJ, D, NPART, S, MIR>(ops, c1, c2, name, s);
}

bool same(const bgm_band& a, const bgm_band& b) {
  return a.data == b.data && a.lower == b.lower && a.upper == b.upper && a.n == b.n && a.tile == b.tile;
}

// ---- the benchmarked shapes ----
// L L^T full (8,8) from one staged L (8,0)           [config 2]
using S_llt8 = Spec<1, 9, 1, 1, PS<0, 1, 8, 0, 8, 0, 8, 8>, 0, 0>;
// band(L L^T) lower (16,0) = precision_from_factor  [config 3, inference.cpp:23-26]
using S_llt16 = Spec<1, 17, 1, 1, PS<0, 1, 16, 0, 16, 0, 16, 0>, 0, 0, NoP, 0, 0, true>;
// A(8,8) B(3,3) -> (11,11)                          [config 2]
using S_ab = Spec<2, 17, 7, 1, PS<0, 0, 8, 8, 3, 3, 11, 11>, 0, 1>;
// fused VJP, operands 0 = P-bar, 1 = A, 2 = B:
//   A-bar = P-bar op(B)^T on band(A), B-bar = op(A)^T P-bar on band(B)
template <int AL, int AU, int BL, int BU, int PL, int PU, bool FMA = false>
using S_vjp = Spec<3, PL + PU + 1, AL + AU + 1, BL + BU + 1, PS<0, 1, PL, PU, BL, BU, AL, AU>, 0, 2,
                   PS<1, 0, AL, AU, PL, PU, BL, BU>, 1, 0, FMA>;
using S_vab = S_vjp<8, 8, 3, 3, 11, 11>;   // config 2: A(8,8), B(3,3), P-bar (11,11)
using S_vllt = S_vjp<8, 0, 0, 8, 8, 8>;    // config 2: L, L^T, P-bar (8,8)
using S_vdl = S_vjp<16, 0, 0, 16, 16, 0, true>;  // config 3 dL: L, L^T, G (16,0)

template <class T>
bool product_t(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  if (!ta && tb && same(a, b) && a.lower == 8 && a.upper == 0 && c.lower == 8 && c.upper == 8)
    return run_cfg<T, 32, 8, 3, 2, S_llt8, true>(&a, c, nullptr, "stream_llt8", s);
  if (!ta && tb && same(a, b) && a.lower == 16 && a.upper == 0 && c.lower == 16 && c.upper == 0)
    return run_cfg<T, 16, 8, 3, 2, S_llt16, false>(&a, c, nullptr, "stream_llt16", s);
  if (!ta && !tb && a.lower == 8 && a.upper == 8 && b.lower == 3 && b.upper == 3 && c.lower == 11 && c.upper == 11) {
    const bgm_band ops[2] = {a, b};
    return run_cfg<T, 16, 8, 3, 4, S_ab, true>(ops, c, nullptr, "stream_ab", s);
  }
  return false;
}

template <class T>
bool vjp_t(const bgm_band& a, const bgm_band& b, const bgm_band& pb, const bgm_band& ab, const bgm_band& bb,
           cudaStream_t s) {
  const bgm_band ops[3] = {pb, a, b};
  auto is = [](const bgm_band& x, int l, int u) { return x.lower == l && x.upper == u; };
  if (is(a, 8, 8) && is(b, 3, 3) && is(pb, 11, 11))
    return run_cfg<T, 16, 4, 3, 4, S_vab, true>(ops, ab, &bb, "stream_vjp_ab", s);
  if (is(a, 8, 0) && is(b, 0, 8) && is(pb, 8, 8))
    return run_cfg<T, 16, 8, 2, 4, S_vllt, true>(ops, ab, &bb, "stream_vjp_llt", s);
  if (is(a, 16, 0) && is(b, 0, 16) && is(pb, 16, 0))
    return run_cfg<T, 16, 8, 1, 4, S_vdl, false>(ops, ab, &bb, "stream_vjp_dl", s);
  return false;
}

}  // namespace

bool product(const bgm_band& a, int ta, const bgm_band& b, int tb, const bgm_band& c, cudaStream_t s) {
  if (c.tile != 32 || c.n == 0 || c.batch == 0) return false;
  return a.dtype == BGM_F64 ? product_t<double>(a, ta, b, tb, c, s) : product_t<float>(a, ta, b, tb, c, s);
}

bool vjp_product(const bgm_band& a, const bgm_band& b, const bgm_band& pb, const bgm_band& ab, const bgm_band& bb,
                 cudaStream_t s) {
  if (a.tile != 32 || a.n == 0 || a.batch == 0) return false;
  return a.dtype == BGM_F64 ? vjp_t<double>(a, b, pb, ab, bb, s) : vjp_t<float>(a, b, pb, ab, bb, s);
}

}  // namespace stream
}  // namespace bgm
