// Optional per-kernel CUDA-event timing (bench.py's roofline attribution).
// Off by default; when enabled every instrumented launch records an event
// pair on its own stream, aggregated per kernel name.
#pragma once

#include <cuda_runtime.h>

namespace bgm {
namespace timing {

bool enabled();
// Records the start event; returns a slot id (or -1 when disabled).
int begin(const char* name, cudaStream_t s);
void end(int slot, cudaStream_t s);

struct Scope {
  int slot;
  cudaStream_t s;
  Scope(const char* name, cudaStream_t st) : slot(begin(name, st)), s(st) {}
  ~Scope() { end(slot, s); }
};

}  // namespace timing
}  // namespace bgm
