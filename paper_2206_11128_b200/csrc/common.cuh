// Shared definitions of libtnb (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "tnb.h"

namespace tnb {

// Modes a single fused launch can carry in its parameter block.
constexpr int kMaxModes = 128;

// Device view of one repacked mode (see TNB_LAYOUT_* in tnb.h).
struct ModeDev {
  const float* s;   // slices of batch element 0
  int64_t bstride;  // floats between batch elements (0 when unbatched)
  int32_t layout;   // TNB_LAYOUT_DENSE / TNB_LAYOUT_DIAG
  int32_t J;
  int32_t rl;
  int32_t rr;
};

struct ChainDev {
  int32_t n;
  int32_t rmax;
  int64_t batch;  // >= 1 (1 when unbatched)
  ModeDev m[kMaxModes];
};

// ---------------------------------------------------------------------------
// host-side error plumbing (thread-local message, status codes only)
int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
inline int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// Validates a chain descriptor and fills a ChainDev (n <= kMaxModes).
int make_chain_dev(const tnb_chain* c, ChainDev* out, bool need_fused);
int64_t mode_floats(const tnb_mode& m);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Opt-in per-kernel timing (tnb_timing_enable): brackets a launch with CUDA
// events on its stream; a no-op unless enabled.
bool timing_on();
void timing_push(const char* name, cudaEvent_t a, cudaEvent_t b);
struct KTimer {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  KTimer(const char* n, cudaStream_t s) : name(n), st(s) {
    if (timing_on() && cudaEventCreate(&a) == cudaSuccess) cudaEventRecord(a, st);
  }
  ~KTimer() {
    cudaEvent_t b;
    if (a && cudaEventCreate(&b) == cudaSuccess) {
      cudaEventRecord(b, st);
      timing_push(name, a, b);
    }
  }
};

// Number of SMs of the current device (cached per device).
int num_sms();

// ---------------------------------------------------------------------------
// device helpers
__device__ __forceinline__ float ldg_f(const float* p) { return __ldg(p); }

// Normalises one raw index (negative wrap, core.py:411-413) and reports an
// out-of-bounds value by lowering *err to the mode number (core.py:414-415).
__device__ __forceinline__ int32_t norm_index(int64_t raw, int32_t J, int32_t k, int32_t* err) {
  // one unsigned compare covers both v < 0 and v >= J
  uint64_t v = (uint64_t)(raw < 0 ? raw + J : raw);
  if (v >= (uint64_t)J) {
    atomicMin(err, k);
    v = 0;
  }
  return (int32_t)v;
}

}  // namespace tnb

// launchers implemented across translation units
namespace tnb {
// elt: element size in bytes, 4 (fp32, the hot path) or 8 (float64, the
// reference's dtype; generic kernels only)
int launch_repack(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes,
                  cudaStream_t st, int elt);
int launch_tt_core(const ChainDev& ch, int k, void* out, cudaStream_t st, int elt);
int launch_promote_cp(const tnb_node* node, int position, int64_t batch, void* out,
                      cudaStream_t st, int elt);
int64_t entries_workspace(const tnb_chain* c, int64_t m, int algo, int elt);
int entries_plan(const tnb_chain* c, int64_t m, int algo, tnb_entries_info* info);
int launch_entries(const tnb_chain* c, const int64_t* idx, int64_t m, void* out, int32_t* err,
                   int algo, void* ws, int64_t ws_bytes, cudaStream_t st, int elt);
int64_t full_workspace(const tnb_chain* c, int64_t lo, int64_t hi, int elt);
int launch_full(const tnb_chain* c, int64_t lo, int64_t hi, void* out, void* ws,
                int64_t ws_bytes, cudaStream_t st, int elt);
int launch_dot(const tnb_chain* a, const tnb_chain* b, void* out, bool is_norm, cudaStream_t st, int elt);
}  // namespace tnb
