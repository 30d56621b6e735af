// Opt-in kernel timing for the bench (tnb_timing_enable / tnb_timing_read):
// CUDA events recorded around libtnb's own launches on their streams.
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace tnb {
namespace {
std::atomic<bool> g_on{false};
std::mutex g_mu;
struct Acc {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  double ms = 0.0;
  int64_t n = 0;
};
std::map<std::string, Acc>& table() {
  static std::map<std::string, Acc> t;
  return t;
}
}  // namespace

bool timing_on() { return g_on.load(std::memory_order_relaxed); }

void timing_push(const char* name, cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> lk(g_mu);
  table()[name].pending.emplace_back(a, b);
}

}  // namespace tnb

extern "C" int tnb_timing_enable(int32_t on) {
  using namespace tnb;
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& kv : table())
    for (auto& e : kv.second.pending) {
      cudaEventSynchronize(e.second);
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
  table().clear();
  g_on.store(on != 0);
  return TNB_OK;
}

extern "C" int tnb_timing_read(const char* kernel, double* total_ms, int64_t* launches) {
  using namespace tnb;
  if (!kernel) return set_error(TNB_EINVAL, "null kernel name");
  std::lock_guard<std::mutex> lk(g_mu);
  Acc& acc = table()[kernel];
  for (auto& e : acc.pending) {
    int rc = check_cuda(cudaEventSynchronize(e.second), "timing sync");
    if (rc) return rc;
    float ms = 0.f;
    rc = check_cuda(cudaEventElapsedTime(&ms, e.first, e.second), "timing elapsed");
    if (rc) return rc;
    acc.ms += ms;
    acc.n += 1;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  acc.pending.clear();
  if (total_ms) *total_ms = acc.ms;
  if (launches) *launches = acc.n;
  return TNB_OK;
}
