// Library-private, stream-ordered scratch memory.
//
// The default CUDA memory pool hands freed memory back to the driver at every
// synchronisation (release threshold 0), so a multi-GB workspace allocated
// per call would be re-mapped on every call.  The sweeps instead draw from a
// per-device pool owned by this library whose release threshold is
// unbounded: after the first call the workspace is recycled in stream order
// at no cost, and the host application's own pools are left untouched.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "bgm_common.cuh"

namespace bgm {

namespace {
constexpr int kMaxDevices = 64;
std::mutex g_mu;
cudaMemPool_t g_pools[kMaxDevices] = {};
}  // namespace

static cudaMemPool_t pool_for_current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    g_pools[dev] = p;
  }
  return g_pools[dev];
}

cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t s) {
  cudaMemPool_t p = pool_for_current_device();
  if (!p) return cudaMallocAsync(ptr, bytes, s);
  return cudaMallocFromPoolAsync(ptr, bytes, p, s);
}

cudaError_t scratch_free(void* ptr, cudaStream_t s) { return cudaFreeAsync(ptr, s); }

}  // namespace bgm
