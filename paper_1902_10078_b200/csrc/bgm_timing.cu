#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bandgm_b200.h"
#include "bgm_timing.cuh"

namespace bgm {
namespace timing {
namespace {
struct Rec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
struct Agg {
  std::string name;
  double ms;
  long count;
};
std::vector<Agg> g_agg;

void drain_locked() {
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& a : g_agg)
      if (a.name == r.name) {
        a.ms += ms;
        ++a.count;
        found = true;
        break;
      }
    if (!found) g_agg.push_back({r.name, ms, 1});
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_recs.clear();
}
}  // namespace

bool enabled() { return g_on; }

int begin(const char* name, cudaStream_t s) {
  if (!g_on) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec r{name, nullptr, nullptr};
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
  g_recs.push_back(r);
  return int(g_recs.size()) - 1;
}

void end(int slot, cudaStream_t s) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (slot < int(g_recs.size())) cudaEventRecord(g_recs[slot].b, s);
}

}  // namespace timing
}  // namespace bgm

using namespace bgm::timing;

extern "C" {

int bgm_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  drain_locked();
  g_agg.clear();
  g_on = on != 0;
  return BGM_OK;
}

int bgm_timing_read(int idx, char* name, int name_len, double* total_ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(g_mu);
  drain_locked();
  if (idx < 0 || idx >= int(g_agg.size())) return int(g_agg.size());
  if (name && name_len > 0) {
    std::strncpy(name, g_agg[idx].name.c_str(), size_t(name_len - 1));
    name[name_len - 1] = 0;
  }
  if (total_ms) *total_ms = g_agg[idx].ms;
  if (count) *count = g_agg[idx].count;
  return int(g_agg.size());
}

}  // extern "C"
