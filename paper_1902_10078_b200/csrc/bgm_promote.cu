// Promotion of bands the fast paths do not take directly.
//
// The segment-parallel kernels are compiled for lower bandwidths
// {1, 2, 3, 4, 8, 16} in the 32-matrix interleave (bgm_narrow.cu) and for
// {64, 128} in the reference layout (bgm_wide.cu, plus the k = 16 adjoint
// of the inverse subset).  Any other lower band -- a bandwidth in between,
// or a narrow band handed over in the reference layout (the C++ drop-in
// passes single matrices that way) -- would otherwise run the one-thread-
// per-matrix reference loops.  Here such an operand is staged into scratch
// as a band of the next compiled bandwidth K' >= k, zero-padded, in the
// layout that path reads; the fast kernel runs; the result is cropped back.
//
// Zero padding is exact for these operators: a factor whose extra diagonals
// are zero has zero extra diagonals in its Cholesky factor (every extra
// cell is (0 - sum of products with a zero factor) / pivot), the extra
// terms the kernels add to in-band sums are exact zeros, and the in-band
// entries of the inverse subset are entries of the same inverse.  The
// adjoints' in-band cells are the gradients of the same functions (the
// extra cells are constants held at zero, and their cotangents are zero).
// Results match the unpadded computation to rounding (tests:
// test_promote_gpu.py); pivot-failure rows are unchanged.
#include <cuda_runtime.h>

#include "bgm_common.cuh"
#include "bgm_fast.cuh"
#include "bgm_timing.cuh"
#include "bgm_wide.cuh"

namespace bgm {
namespace promote {
namespace {

// dst cell (r, j) of every matrix <- src entry (j + r - dst.up, j) if src
// holds it, else 0 (corner cells included).  Thread per (matrix, column),
// split with the destination's tile bits fastest so tile-32 writes coalesce.
template <class T>
__global__ void k_copy_band(Band<T> src, Band<T> dst, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, j;
  if (dst.n == 0 || !split_bj(t, batch, dst.n, dst.s > src.s ? dst.s : src.s, b, j)) return;
  for (int r = 0; r < dst.w; ++r) {
    const ix i = j + r - dst.up;
    dst.cell(b, r, j) = src.in_band(i, j) ? src.at(b, i, j) : T(0);
  }
}

template <class T>
__global__ void k_copy_vec(Vec<T> src, Vec<T> dst, ix batch) {
  const ix t = blockIdx.x * ix(blockDim.x) + threadIdx.x;
  ix b, i;
  if (dst.n == 0 || !split_bj(t, batch, dst.n, dst.s > src.s ? dst.s : src.s, b, i)) return;
  dst(b, i) = src(b, i);
}

int tile_bits(int tile) { return tile == 32 ? 5 : 0; }
ix rounded(ix batch, int tile) { return (batch + tile - 1) / tile * tile; }
size_t esize(int dtype) { return dtype == BGM_F64 ? 8 : 4; }

// The compiled bandwidth and layout a lower band of bandwidth k goes to.
bool target(const bgm_band& b, int& K, int& tile) {
  if (b.upper != 0 || b.batch <= 0 || b.lower < 1 || b.lower > 128) return false;
  const int k = b.lower;
  if (k <= 16) {
    K = k <= 4 ? k : (k <= 8 ? 8 : 16);
    tile = 32;
  } else {
    K = k <= 64 ? 64 : 128;
    tile = 1;
  }
  if (K == k && tile == b.tile) return false;  // the direct path already declined it
  // long enough for the segmented kernels (bgm_narrow.cu shape_ok, bgm_wide.cu)
  return b.n >= (tile == 32 ? 64 : 8 * ix(K)) && K < b.n;
}

// A scratch band / vector in the promoted shape.
struct Staged {
  void* mem = nullptr;
  cudaStream_t s = nullptr;
  bool ok = false;
  Staged() = default;
  Staged(const Staged&) = delete;
  Staged& operator=(const Staged&) = delete;
  ~Staged() {
    if (mem) scratch_free(mem, s);
  }
  bool alloc(size_t bytes, cudaStream_t st) {
    s = st;
    ok = scratch_alloc(&mem, bytes ? bytes : 8, st) == cudaSuccess;
    return ok;
  }
};

struct SBand : Staged {
  bgm_band d{};
  bool make(const bgm_band& like, int K, int tile, cudaStream_t st) {
    d = like;
    d.lower = K;
    d.upper = 0;
    d.tile = tile;
    if (!alloc(esize(like.dtype) * size_t(rounded(like.batch, tile)) * size_t(like.n) * size_t(K + 1), st))
      return false;
    d.data = mem;
    return true;
  }
};

struct SVec : Staged {
  bgm_vec d{};
  bool make(const bgm_vec& like, int tile, cudaStream_t st) {
    d = like;
    d.tile = tile;
    if (!alloc(esize(like.dtype) * size_t(rounded(like.batch, tile)) * size_t(like.n), st)) return false;
    d.data = mem;
    return true;
  }
};

template <class T>
void copy_band(const bgm_band& src, const bgm_band& dst, cudaStream_t s) {
  const Band<T> a = view<T>(src), b = view<T>(dst);
  const int sh = tile_bits(src.tile) > tile_bits(dst.tile) ? tile_bits(src.tile) : tile_bits(dst.tile);
  const ix work = rounded(dst.batch, 1 << sh) * dst.n;
  if (work) k_copy_band<T><<<blocks_for(work, 256), 256, 0, s>>>(a, b, dst.batch);
}
void copy_band(const bgm_band& src, const bgm_band& dst, cudaStream_t s) {
  if (src.dtype == BGM_F64)
    copy_band<double>(src, dst, s);
  else
    copy_band<float>(src, dst, s);
}
template <class T>
void copy_vec(const bgm_vec& src, const bgm_vec& dst, cudaStream_t s) {
  const Vec<T> a = view<T>(src), b = view<T>(dst);
  const int sh = tile_bits(src.tile) > tile_bits(dst.tile) ? tile_bits(src.tile) : tile_bits(dst.tile);
  const ix work = rounded(dst.batch, 1 << sh) * dst.n;
  if (work) k_copy_vec<T><<<blocks_for(work, 256), 256, 0, s>>>(a, b, dst.batch);
}
void copy_vec(const bgm_vec& src, const bgm_vec& dst, cudaStream_t s) {
  if (src.dtype == BGM_F64)
    copy_vec<double>(src, dst, s);
  else
    copy_vec<float>(src, dst, s);
}

bool stage_in(SBand& x, const bgm_band& src, int K, int tile, cudaStream_t s) {
  if (!x.make(src, K, tile, s)) return false;
  copy_band(src, x.d, s);
  return true;
}
bool stage_in(SVec& x, const bgm_vec& src, int tile, cudaStream_t s) {
  if (!x.make(src, tile, s)) return false;
  copy_vec(src, x.d, s);
  return true;
}

// The fast path for an already promoted shape (never promotes again).
bool direct_cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  return narrow::cholesky(q, l, st, row, s) || wide::cholesky(q, l, st, row, s);
}
bool direct_solve(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
                  cudaStream_t s) {
  return narrow::solve_vec(l, v, tr, x, st, row, s) || wide::solve_vec(l, v, tr, x, st, row, s);
}
bool direct_subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  return narrow::subset(l, sb, st, row, s) || wide::subset(l, sb, st, row, s);
}
bool direct_vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  return narrow::vjp_cholesky(l, lb, qb, s) || wide::vjp_cholesky(l, lb, qb, s);
}

}  // namespace

bool cholesky(const bgm_band& q, const bgm_band& l, int32_t* st, int64_t* row, cudaStream_t s) {
  int K, tile;
  if (!target(q, K, tile) || l.lower != q.lower || l.upper != 0) return false;
  timing::Scope ts("promote", s);
  SBand qs, ls;
  if (!stage_in(qs, q, K, tile, s) || !ls.make(l, K, tile, s)) return false;
  if (!direct_cholesky(qs.d, ls.d, st, row, s)) return false;
  copy_band(ls.d, l, s);  // crop
  return true;
}

bool solve_vec(const bgm_band& l, const bgm_vec& v, int tr, const bgm_vec& x, int32_t* st, int64_t* row,
               cudaStream_t s) {
  int K, tile;
  if (!target(l, K, tile)) return false;
  timing::Scope ts("promote", s);
  SBand ls;
  SVec vs, xs;
  if (!stage_in(ls, l, K, tile, s) || !stage_in(vs, v, tile, s) || !xs.make(x, tile, s)) return false;
  if (!direct_solve(ls.d, vs.d, tr, xs.d, st, row, s)) return false;
  copy_vec(xs.d, x, s);
  return true;
}

bool subset(const bgm_band& l, const bgm_band& sb, int32_t* st, int64_t* row, cudaStream_t s) {
  int K, tile;
  if (!target(l, K, tile) || sb.lower != l.lower || sb.upper != 0) return false;
  timing::Scope ts("promote", s);
  SBand ls, ss;
  if (!stage_in(ls, l, K, tile, s) || !ss.make(sb, K, tile, s)) return false;
  if (!direct_subset(ls.d, ss.d, st, row, s)) return false;
  copy_band(ss.d, sb, s);
  return true;
}

bool vjp_cholesky(const bgm_band& l, const bgm_band& lb, const bgm_band& qb, cudaStream_t s) {
  int K, tile;
  if (!target(l, K, tile) || lb.lower != l.lower || qb.lower != l.lower || lb.upper != 0 || qb.upper != 0)
    return false;
  SBand ls, lbs, qbs;
  timing::Scope ts("promote", s);
  if (!stage_in(ls, l, K, tile, s) || !stage_in(lbs, lb, K, tile, s) || !qbs.make(qb, K, tile, s)) return false;
  if (!direct_vjp_cholesky(ls.d, lbs.d, qbs.d, s)) return false;
  copy_band(qbs.d, qb, s);
  return true;
}

bool vjp_subset(const bgm_band& l, const bgm_band& sm, const bgm_band& sbar, const bgm_band& lbar, int32_t* st,
                int64_t* row, cudaStream_t s) {
  // compiled adjoints of the inverse subset: k = 16 (tile 32 here), 64, 128
  // (reference layout).  The adjoint on the wider pattern needs the inverse
  // on that pattern, which the caller's S (k diagonals) does not hold: it is
  // recomputed from the staged factor -- the same values the caller's S has
  // on the k diagonals when S = sparse_inverse_subset(L), the reference's
  // contract for this call (grad.hpp:46-47).
  if (l.upper != 0 || l.batch <= 0 || l.lower < 1 || l.lower > 128 || sm.lower != l.lower ||
      sbar.lower != l.lower || lbar.lower != l.lower)
    return false;
  const int k = l.lower;
  const int K = k <= 16 ? 16 : (k <= 64 ? 64 : 128), tile = K == 16 ? 32 : 1;
  if ((K == k && tile == l.tile) || l.n < 8 * ix(K) || K >= l.n) return false;
  timing::Scope ts("promote", s);
  SBand ls, ss, sbs, lbs;
  if (!stage_in(ls, l, K, tile, s) || !ss.make(sm, K, tile, s) || !stage_in(sbs, sbar, K, tile, s) ||
      !lbs.make(lbar, K, tile, s))
    return false;
  if (!direct_subset(ls.d, ss.d, st, row, s)) return false;
  if (!wide::vjp_subset(ls.d, ss.d, sbs.d, lbs.d, st, row, s)) return false;
  copy_band(lbs.d, lbar, s);
  return true;
}

}  // namespace promote
}  // namespace bgm
