// FP64 peak microbenchmarks: the denominators of the FP64 side of every
// roofline this library reports (BASELINE.md §2 asks for them to be
// measured on the box, not taken from the nominal 37.2 TF).
//
//   k_dfma_peak: every thread runs 16 independent DFMA chains (enough to
//                cover the DFMA latency at 8 warps per SMSP).
//   k_dmma_peak: every warp runs 8 independent mma.sync.m8n8k4.f64 (DMMA)
//                accumulators, 512 flops per instruction.
//
// Both are timed with CUDA events on the caller's stream after one warm-up
// launch; the grid is 4 CTAs x 256 threads per SM (persistent, one wave).
#include <cuda_runtime.h>

#include "bandgm_b200.h"
#include "bgm_common.cuh"

namespace bgm {
namespace {

constexpr int kChains = 16;
constexpr int kMma = 8;

__global__ void __launch_bounds__(256) k_dfma_peak(double* sink, int iters, double m, double c) {
  double a[kChains];
#pragma unroll
  for (int q = 0; q < kChains; ++q) a[q] = 1e-3 * (threadIdx.x + q);
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int q = 0; q < kChains; ++q) a[q] = fma(a[q], m, c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += a[q];
  if (s == 1.2345e-300) sink[blockIdx.x] = s;  // never true; keeps the chains live
}

__global__ void __launch_bounds__(256) k_dmma_peak(double* sink, int iters) {
  const int lane = threadIdx.x & 31;
  double a = 1e-3 * lane, b = 2e-3 * lane;
  double c0[kMma], c1[kMma];
#pragma unroll
  for (int q = 0; q < kMma; ++q) c0[q] = c1[q] = 0.0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int q = 0; q < kMma; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0[q]), "+d"(c1[q])
                     : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kMma; ++q) s += c0[q] + c1[q];
  if (s == 1.2345e-300) sink[blockIdx.x] = s;
}

}  // namespace
}  // namespace bgm

extern "C" int bgm_fp64_peak(double* dfma_tflops, double* dmma_tflops, bgm_stream stream) {
  using namespace bgm;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(cudaGetLastError());
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned blocks = unsigned(sms) * 4, threads = 256;
  double* sink = nullptr;
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&sink), sizeof(double) * blocks, s);
  if (err != cudaSuccess) return set_error(err);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  // DFMA: iters x 8 x kChains FMAs per thread
  const int it_f = 4096;
  k_dfma_peak<<<blocks, threads, 0, s>>>(sink, 64, 0.999999, 1e-7);
  cudaEventRecord(e0, s);
  k_dfma_peak<<<blocks, threads, 0, s>>>(sink, it_f, 0.999999, 1e-7);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (dfma_tflops)
    *dfma_tflops = 2.0 * double(blocks) * threads * it_f * 8 * kChains / (double(ms) * 1e-3) / 1e12;
  // DMMA: iters x 4 x kMma instructions per warp, 512 flops each
  const int it_m = 2048;
  k_dmma_peak<<<blocks, threads, 0, s>>>(sink, 64);
  cudaEventRecord(e0, s);
  k_dmma_peak<<<blocks, threads, 0, s>>>(sink, it_m);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (dmma_tflops)
    *dmma_tflops = 512.0 * double(blocks) * (threads / 32) * it_m * 4 * kMma / (double(ms) * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, s);
  err = cudaGetLastError();
  return err == cudaSuccess ? BGM_OK : set_error(err);
}
