// Dependent-chain latencies and single-warp throughputs of the instructions
// the wide (DMMA) and narrow (DFMA + shared window) kernels are built from,
// measured with clock64 on one warp (and one 4-warp CTA for the barrier).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench scripts/ubench_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int N = 256;

__global__ void k_lat(long long* out, double* sink, double seed) {
  __shared__ double sm[1024];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = double((i * 8 + 8) % 1024);  // pointer chase
  __syncthreads();
  double a = seed + lane * 1e-3, b = 1.0 - 1e-9 * lane;
  long long t0, t1;
  int r = 0;
  // 0: dependent DMMA chain
  {
    double d0 = a, d1 = b;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) dmma(d0, d1, a, b);
    t1 = clock64();
    sink[lane] += d0 + d1;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 1: 8 independent DMMA accumulators (N/8 rounds)
  {
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j][0] = a + j, d[j][1] = b + j;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N / 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(d[j][0], d[j][1], a, b);
    t1 = clock64();
#pragma unroll
    for (int j = 0; j < 8; ++j) sink[lane] += d[j][0] + d[j][1];
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 2: dependent DFMA chain
  {
    double x = a;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = fma(x, b, a);
    t1 = clock64();
    sink[lane] += x;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 3: 8 independent DFMA chains
  {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = a + j;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N / 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], b, a);
    t1 = clock64();
#pragma unroll
    for (int j = 0; j < 8; ++j) sink[lane] += x[j];
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 4: dependent shuffle chain (64-bit value = two SHFL)
  {
    double x = a;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    t1 = clock64();
    sink[lane] += x;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 5: dependent rsqrt(double) chain
  {
    double x = a + 2.0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = rsqrt(x) + 1.5;
    t1 = clock64();
    sink[lane] += x;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 6: dependent sqrt + division chain
  {
    double x = a + 2.0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = 1.0 / sqrt(x) + 1.5;
    t1 = clock64();
    sink[lane] += x;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 7: dependent LDS.64 chain
  {
    int idx = lane;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) idx = int(sm[idx & 1023]);
    t1 = clock64();
    sink[lane] += idx;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 8: __syncthreads round trips
  {
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 9: STS -> barrier -> LDS round trip (publish a value to the CTA)
  {
    double x = a;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
      if (threadIdx.x == (i & 127)) sm[5] = x + 1.0;
      __syncthreads();
      x = sm[5];
      __syncthreads();
    }
    t1 = clock64();
    sink[lane] += x;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 10: dependent DMUL chain
  {
    double x = a;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = x * b;
    t1 = clock64();
    sink[lane] += x;
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
  // 11: pairs of dependent DMMAs over 8 accumulators (kc = 0, 1 back to back)
  {
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j][0] = a + j, d[j][1] = b + j;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N / 16; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dmma(d[j][0], d[j][1], a, b);
        dmma(d[j][0], d[j][1], b, a);
      }
    t1 = clock64();
#pragma unroll
    for (int j = 0; j < 8; ++j) sink[lane] += d[j][0] + d[j][1];
    if (threadIdx.x == 0) out[r] = t1 - t0;
    ++r;
  }
}

int main() {
  long long* out;
  double* sink;
  cudaMallocManaged(&out, 64 * sizeof(long long));
  cudaMalloc(&sink, 1024 * sizeof(double));
  cudaMemset(sink, 0, 1024 * sizeof(double));
  const char* names[] = {"DMMA dependent",      "DMMA 8 independent", "DFMA dependent",   "DFMA 8 independent",
                         "SHFL.64 dependent",   "rsqrt(double) dep",  "1/sqrt(double) dep", "LDS.64 dependent",
                         "__syncthreads",       "STS+bar+LDS+bar",    "DMUL dependent",   "DMMA pairs x8"};
  for (int threads : {32, 128}) {
    for (int rep = 0; rep < 2; ++rep) {
      k_lat<<<1, threads>>>(out, sink, 1.25);
      cudaDeviceSynchronize();
    }
    printf("-- %d threads per CTA, clocks per instruction (N = %d)\n", threads, N);
    for (int i = 0; i < 12; ++i) printf("%-22s %8.1f\n", names[i], double(out[i]) / N);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
