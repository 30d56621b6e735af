// Host transport codec for index matrices on the end-to-end path
// (tnb_narrow_indices_host; device side: tnb_widen_indices in codec.cu).
//
// The reference's entries() takes an int64 index matrix (core.py:394-416,
// reached from t[idx], indexing.py:120-130).  When that matrix lives in host
// memory, moving it to the GPU over PCIe is the whole cost of a call: 80 B
// per sample at cfg2 against a few ns of GPU time.  Every cfg index is
// below 128, so the values travel as int8 (or int16) and are widened back
// to int64 on the device.  The narrowing is a pure RANGE CHECK on the raw
// values (does x fit the narrow type?): wrapping negatives, the per-mode
// bounds check and the lowest-OOB-mode report all stay in the device prep
// kernel, which sees exactly the values the caller passed.  A matrix with a
// value that does not fit is sent as int64 unchanged.
//
// Plain C++ (no CUDA): compiled by g++ with per-ISA clones so the same .so
// uses AVX-512 on the GPU box's Xeons and AVX2 / SSE elsewhere.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "tnb.h"

namespace tnb {
int set_error(int code, const char* fmt, ...);  // abi.cu: thread-local tnb_last_error()
}

namespace {

template <typename N, int64_t LO, int64_t SPAN>
__attribute__((target_clones("arch=skylake-avx512", "avx2", "default")))
uint64_t narrow_range(const int64_t* __restrict in, N* __restrict out, int64_t n) {
  // bad accumulates every bit of (x - LO) above the narrow type's span: zero
  // iff all LO <= x < LO + SPAN (branch-free, so the loop vectorises)
  uint64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = in[i];
    bad |= ((uint64_t)(x - LO)) & ~(uint64_t)(SPAN - 1);
    out[i] = (N)x;
  }
  return bad;
}

int hw_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

// A persistent pool of hw_threads() - 1 workers (the caller is worker 0):
// spawning 15 threads per 2^21-row chunk cost ~0.6 ms, a third of the
// chunk's narrowing time.  One job at a time (callers serialise on `call`);
// workers sleep on a condition variable between jobs.
class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool(hw_threads() - 1);  // never destroyed: workers outlive static teardown
    return *p;
  }
  int size() const { return (int)workers_.size() + 1; }
  // runs f(0..n-1) with n <= size(), f(0) on the calling thread
  void run(int n, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> call(call_);
    n = std::max(1, std::min(n, size()));
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      active_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
    for (auto& t : workers_) t.detach();
  }
  void loop(int id) {
    int64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (id >= active_) continue;
        job = job_;
      }
      (*job)(id);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int active_ = 0, pending_ = 0;
  int64_t gen_ = 0;
};

}  // namespace

extern "C" int tnb_narrow_indices_host(const int64_t* idx, int64_t count, int32_t width, void* out,
                                       int32_t nthreads, int32_t* fits) {
  if (!fits || count < 0 || (count > 0 && (!idx || !out)) || (width != 1 && width != 2))
    return tnb::set_error(TNB_EINVAL, "narrow_indices: bad arguments (width must be 1 or 2)");
  *fits = 1;
  if (count == 0) return TNB_OK;
  int nt = nthreads > 0 ? nthreads : hw_threads();
  // >= 1 MiB of input per thread: below that, waking workers costs more than it saves
  const int64_t per_min = (1 << 20) / 8;
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, count / per_min));
  std::vector<uint64_t> bad(nt, 0);
  const std::function<void(int)> work = [&](int t) {
    // 64-value aligned ranges: no two threads share an output cache line
    const int64_t blk = ((count + nt - 1) / nt + 63) & ~(int64_t)63;
    const int64_t lo = std::min<int64_t>(count, (int64_t)t * blk);
    const int64_t hi = std::min<int64_t>(count, lo + blk);
    if (hi <= lo) return;
    if (width == 1)
      bad[t] = narrow_range<int8_t, -128, 256>(idx + lo, static_cast<int8_t*>(out) + lo, hi - lo);
    else
      bad[t] = narrow_range<int16_t, -32768, 65536>(idx + lo, static_cast<int16_t*>(out) + lo, hi - lo);
  };
  if (nt == 1) {
    work(0);
  } else if (nt <= Pool::get().size()) {
    Pool::get().run(nt, work);
  } else {  // more threads than the hardware has (explicit request): one-off threads
    std::vector<std::thread> extra;
    for (int t = 1; t < nt; ++t) extra.emplace_back(work, t);
    work(0);
    for (auto& th : extra) th.join();
  }
  uint64_t any = 0;
  for (uint64_t b : bad) any |= b;
  *fits = any ? 0 : 1;
  return TNB_OK;
}

extern "C" int tnb_host_threads(void) { return hw_threads(); }
