// Shared device-side layout helpers for the bandgm_b200 kernels.
//
// Device layout (include/bandgm_b200.h): batch-interleaved band storage,
//   element (b, r, j) -> ((b >> s) * n * w + j * w + r) << s | (b & (2^s - 1))
// with interleave width 2^s in {1, 32}.  r = i - j + upper is the reference
// storage row of matrix entry (i, j) (banded.hpp:1-11).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include <cmath>

#include "bandgm_b200.h"

namespace bgm {

using ix = int64_t;

constexpr double kPivotFloor = 1e-300;  // kernels.hpp:20

// Accumulator of the HBM-bound dot products (band x band, band x vector): fp64
// for both storage types.  fp32 x fp32 products are exact in fp64, so an fp32
// output is the correctly rounded value of the exact dot up to the fp64 sum's
// rounding -- no fp32 cancellation -- at no cost on a memory-bound kernel.
using acc_t = double;

template <class T>
struct Band {
  T* p;
  ix n;
  int lo, up, w, s;  // s = log2(tile)

  __host__ __device__ __forceinline__ ix off(ix b, int r, ix j) const {
    return ((((b >> s) * n + j) * w + r) << s) + (b & ((ix(1) << s) - 1));
  }
  __device__ __forceinline__ T& cell(ix b, int r, ix j) const { return p[off(b, r, j)]; }
  // Unchecked in-band accessor (banded.hpp:64-65).
  __device__ __forceinline__ T& at(ix b, ix i, ix j) const {
    return p[off(b, int(i - j + up), j)];
  }
  __device__ __forceinline__ bool in_band(ix i, ix j) const {
    const ix d = i - j;
    return i >= 0 && i < n && j >= 0 && j < n && d >= -up && d <= lo;
  }
  // banded.hpp:69-71
  __device__ __forceinline__ T at_or_zero(ix b, ix i, ix j) const {
    return in_band(i, j) ? p[off(b, int(i - j + up), j)] : T(0);
  }
  // Mirrored read of a symmetric lower store (banded.hpp:129).
  __device__ __forceinline__ T sym(ix b, ix i, ix j) const { return i >= j ? at(b, i, j) : at(b, j, i); }
  // Writes all w cells of column j: in-band cells from `f(i)`, corners 0.
  template <class F>
  __device__ __forceinline__ void write_column(ix b, ix j, F&& f) const {
    for (int r = 0; r < w; ++r) {
      const ix i = r - up + j;
      cell(b, r, j) = (i >= 0 && i < n) ? f(i) : T(0);
    }
  }
};

template <class T>
struct Vec {
  T* p;
  ix n;
  int s;
  __host__ __device__ __forceinline__ ix off(ix b, ix i) const {
    return (((b >> s) * n + i) << s) + (b & ((ix(1) << s) - 1));
  }
  __device__ __forceinline__ T& operator()(ix b, ix i) const { return p[off(b, i)]; }
};

inline int tile_shift(int tile) { return tile == 32 ? 5 : 0; }

template <class T>
inline Band<T> view(const bgm_band& d) {
  return Band<T>{static_cast<T*>(d.data), d.n, d.lower, d.upper, d.lower + d.upper + 1,
                 tile_shift(d.tile)};
}
template <class T>
inline Vec<T> view(const bgm_vec& d) {
  return Vec<T>{static_cast<T*>(d.data), d.n, tile_shift(d.tile)};
}

// Host-side validation of descriptors.
inline bool valid(const bgm_band& d) {
  if (d.batch < 0 || d.n < 0 || d.lower < 0 || d.upper < 0) return false;
  if (d.n > 0 && (d.lower >= d.n || d.upper >= d.n)) return false;
  if (d.tile != 1 && d.tile != 32) return false;
  if (d.dtype != BGM_F64 && d.dtype != BGM_F32) return false;
  if (d.batch > 0 && d.n > 0 && d.data == nullptr) return false;
  return true;
}
inline bool valid(const bgm_vec& d) {
  if (d.batch < 0 || d.n < 0) return false;
  if (d.tile != 1 && d.tile != 32) return false;
  if (d.dtype != BGM_F64 && d.dtype != BGM_F32) return false;
  if (d.batch > 0 && d.n > 0 && d.data == nullptr) return false;
  return true;
}

__device__ __forceinline__ void report(int32_t* status, int64_t* row, ix b, int st, ix r) {
  if (status) status[b] = st;
  if (row) row[b] = r;
}

inline unsigned blocks_for(ix work, int threads) {
  ix b = (work + threads - 1) / threads;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

// Thread -> (matrix b, index j) with the tile's low bits fastest, so a warp
// touches 32 interleaved matrices of one column (tile 32) or 32 consecutive
// columns of one matrix (tile 1).
__device__ __forceinline__ bool split_bj(ix t, ix batch, ix n, int s, ix& b, ix& j) {
  const ix lanes = ix(1) << s;
  const ix lo = t & (lanes - 1);
  const ix rest = t >> s;
  j = rest % n;
  b = (rest / n) * lanes + lo;
  return b < batch;
}

int set_error(cudaError_t e);

// Kernel attributes (the > 48 KB dynamic shared-memory opt-in) and the
// occupancy derived from them belong to a device context: cache them per
// device ordinal, safely from any host thread (a repeated set is harmless).
struct PerDevice {
  std::atomic<unsigned long long> done{0};
  static unsigned long long bit() {
    int d = 0;
    cudaGetDevice(&d);
    return 1ull << (d & 63);
  }
  bool first() const { return !(done.load(std::memory_order_acquire) & bit()); }
  void mark() { done.fetch_or(bit(), std::memory_order_acq_rel); }
};
// A caller-requested segment length (bgm_set_segment_rows; 0 = automatic),
// clamped so every segment start s >= bandwidth: the boundary checks read
// the k columns before s.
inline long long requested_seg(long long rows, int k) { return rows > 0 && rows < k + 1 ? k + 1 : rows; }

struct PerDeviceInt {  // value + 1 per device ordinal, 0 = not yet known
  std::atomic<int> v[64] = {};
  static int dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  int get() const { return v[dev()].load(std::memory_order_acquire) - 1; }
  void set(int x) { v[dev()].store(x + 1, std::memory_order_release); }
};

// Stream-ordered scratch from the library's private pool (bgm_scratch.cu).
cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t s);
cudaError_t scratch_free(void* ptr, cudaStream_t s);

}  // namespace bgm
