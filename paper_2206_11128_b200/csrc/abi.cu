// extern "C" entry points of libtnb: argument validation, status codes and
// dispatch to the kernels.  See include/tnb.h for the contract and the
// reference interface (file:line) each entry point replaces.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>

#include "common.cuh"

namespace tnb {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return TNB_OK;
  return set_error(TNB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int64_t mode_floats(const tnb_mode& m) {
  int64_t j = m.phys;
  if (m.layout == TNB_LAYOUT_DIAG) return j * m.r_left;
  return j * (int64_t)m.r_left * m.r_right;
}

int make_chain_dev(const tnb_chain* c, ChainDev* out, bool need_fused) {
  if (!c || !c->modes) return set_error(TNB_EINVAL, "null chain");
  if (c->n_modes < 1) return set_error(TNB_EINVAL, "a tensor needs at least one mode");
  if (need_fused && c->n_modes > kMaxModes)
    return set_error(TNB_EINVAL, "fused kernels support at most %d modes, got %d", kMaxModes,
                     c->n_modes);
  if (c->batch < 0) return set_error(TNB_EINVAL, "batch must be >= 0");
  out->n = c->n_modes;
  out->batch = c->batch > 0 ? c->batch : 1;
  int rmax = 1;
  const int nn = c->n_modes < kMaxModes ? c->n_modes : kMaxModes;
  for (int k = 0; k < c->n_modes; ++k) {
    const tnb_mode& m = c->modes[k];
    if (m.phys < 0 || m.r_left < 0 || m.r_right < 0)
      return set_error(TNB_EINVAL, "mode %d: negative size", k);
    if (m.layout == TNB_LAYOUT_DIAG && m.r_left != m.r_right)
      return set_error(TNB_EINVAL, "mode %d: diagonal layout needs equal ranks", k);
    if (m.layout != TNB_LAYOUT_DIAG && m.layout != TNB_LAYOUT_DENSE)
      return set_error(TNB_EINVAL, "mode %d: unknown layout %d", k, m.layout);
    if (k + 1 < c->n_modes && m.r_right != c->modes[k + 1].r_left)
      return set_error(TNB_EINVAL, "rank mismatch between modes %d and %d: %d vs %d", k, k + 1,
                       m.r_right, c->modes[k + 1].r_left);
    if (m.r_left > rmax) rmax = m.r_left;
    if (m.r_right > rmax) rmax = m.r_right;
    if (k < nn) {
      ModeDev& d = out->m[k];
      d.s = m.slices;
      d.bstride = c->batch > 0 ? mode_floats(m) : 0;
      d.layout = m.layout;
      d.J = m.phys;
      d.rl = m.r_left;
      d.rr = m.r_right;
    }
  }
  if (c->modes[0].r_left != 1 || c->modes[c->n_modes - 1].r_right != 1)
    return set_error(TNB_EINVAL, "boundary ranks must be 1, got %d, %d", c->modes[0].r_left,
                     c->modes[c->n_modes - 1].r_right);
  out->rmax = rmax;
  return TNB_OK;
}

int num_sms() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

}  // namespace tnb

using namespace tnb;

extern "C" {

const char* tnb_version(void) { return "tnb 0.1.0 (sm_100a)"; }

const char* tnb_last_error(void) { return g_err; }

int tnb_device_check(void) {
  int dev = 0;
  int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10)
    return set_error(TNB_ECUDA, "libtnb is built for sm_100a; device %d is sm_%d%d", dev, major,
                     minor);
  return TNB_OK;
}

int tnb_plan_modes(const tnb_node* nodes, int32_t n, tnb_mode* modes) {
  if (!nodes || !modes) return set_error(TNB_EINVAL, "null argument");
  if (n < 1) return set_error(TNB_EINVAL, "a tensor needs at least one mode");
  for (int k = 0; k < n; ++k) {
    const tnb_node& nd = nodes[k];
    tnb_mode& m = modes[k];
    if (nd.internal < 0 || nd.phys < 0 || nd.r_left < 0 || nd.r_right < 0)
      return set_error(TNB_EINVAL, "node %d: negative size", k);
    if (!nd.factor && nd.phys != nd.internal)
      return set_error(TNB_EINVAL, "node %d: phys != internal without a factor", k);
    m.phys = nd.phys;
    m.slices = nullptr;
    if (nd.kind == TNB_KIND_TT) {
      m.layout = TNB_LAYOUT_DENSE;
      m.r_left = nd.r_left;
      m.r_right = nd.r_right;
    } else if (nd.kind == TNB_KIND_CP) {
      // _node_ranks (core.py:244-251): R inside, 1 outward at chain ends
      if (nd.r_left != nd.r_right)
        return set_error(TNB_EINVAL, "node %d: CP rank must be given as r_left == r_right", k);
      const int R = nd.r_left;
      if (n == 1) {
        m.layout = TNB_LAYOUT_DENSE;
        m.r_left = m.r_right = 1;
      } else if (k == 0) {
        m.layout = TNB_LAYOUT_DENSE;
        m.r_left = 1;
        m.r_right = R;
      } else if (k == n - 1) {
        m.layout = TNB_LAYOUT_DENSE;
        m.r_left = R;
        m.r_right = 1;
      } else {
        m.layout = TNB_LAYOUT_DIAG;
        m.r_left = m.r_right = R;
      }
    } else {
      return set_error(TNB_EINVAL, "unknown node kind %d", nd.kind);
    }
  }
  for (int k = 0; k + 1 < n; ++k)
    if (modes[k].r_right != modes[k + 1].r_left)
      return set_error(TNB_EINVAL, "rank mismatch between modes %d and %d: %d vs %d", k, k + 1,
                       modes[k].r_right, modes[k + 1].r_left);
  if (modes[0].r_left != 1 || modes[n - 1].r_right != 1)
    return set_error(TNB_EINVAL, "boundary ranks must be 1, got %d, %d", modes[0].r_left,
                     modes[n - 1].r_right);
  return TNB_OK;
}

int64_t tnb_mode_floats(const tnb_mode* mode, int64_t batch) {
  if (!mode) return -1;
  return mode_floats(*mode) * (batch > 0 ? batch : 1);
}

static int repack_any(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes, void* stream,
                      int elt) {
  if (!nodes || !modes || n < 1) return set_error(TNB_EINVAL, "null argument");
  if (batch < 0) return set_error(TNB_EINVAL, "batch must be >= 0");
  for (int k = 0; k < n; ++k) {
    if (!modes[k].slices && mode_floats(modes[k]) > 0)
      return set_error(TNB_EINVAL, "mode %d: null slices", k);
    if (!nodes[k].core) return set_error(TNB_EINVAL, "node %d: null core", k);
  }
  return launch_repack(nodes, n, batch, modes, (cudaStream_t)stream, elt);
}

static int tt_core_any(const tnb_chain* chain, int32_t k, void* out, void* stream, int elt) {
  static thread_local ChainDev ch;
  int rc = make_chain_dev(chain, &ch, true);
  if (rc) return rc;
  if (k < 0 || k >= chain->n_modes) return set_error(TNB_EINVAL, "mode %d out of range", k);
  if (!out) return set_error(TNB_EINVAL, "null output");
  return launch_tt_core(ch, k, out, (cudaStream_t)stream, elt);
}

static int promote_any(const tnb_node* node, int32_t position, int64_t batch, void* out, void* stream, int elt) {
  if (!node || !out) return set_error(TNB_EINVAL, "null argument");
  if (node->kind != TNB_KIND_CP) return set_error(TNB_EINVAL, "promote_cp_node expects a CP node");
  if (position < TNB_POS_INTERIOR || position > TNB_POS_SINGLE)
    return set_error(TNB_EINVAL, "unknown position %d", position);
  return launch_promote_cp(node, position, batch, out, (cudaStream_t)stream, elt);
}

static int entries_any(const tnb_chain* chain, const int64_t* idx, int64_t m, void* out, int32_t* err_mode,
                       int32_t algo, void* ws, int64_t ws_bytes, void* stream, int elt) {
  if (m < 0) return set_error(TNB_EINVAL, "negative sample count");
  if (!err_mode) return set_error(TNB_EINVAL, "null err_mode");
  if (m > 0 && (!idx || !out)) return set_error(TNB_EINVAL, "null index or output");
  return launch_entries(chain, idx, m, out, err_mode, algo, ws, ws_bytes, (cudaStream_t)stream, elt);
}

int tnb_repack_f32(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes,
                   void* stream) {
  return repack_any(nodes, n, batch, modes, stream, 4);
}

int tnb_tt_core_f32(const tnb_chain* chain, int32_t k, float* out, void* stream) {
  return tt_core_any(chain, k, out, stream, 4);
}

int tnb_promote_cp_f32(const tnb_node* node, int32_t position, int64_t batch, float* out,
                       void* stream) {
  return promote_any(node, position, batch, out, stream, 4);
}

int64_t tnb_entries_workspace_bytes(const tnb_chain* chain, int64_t m, int32_t algo) {
  return entries_workspace(chain, m, algo, 4);
}

int tnb_entries_f32(const tnb_chain* chain, const int64_t* idx, int64_t m, float* out,
                    int32_t* err_mode, int32_t algo, void* ws, int64_t ws_bytes, void* stream) {
  return entries_any(chain, idx, m, out, err_mode, algo, ws, ws_bytes, stream, 4);
}

int64_t tnb_full_workspace_bytes(const tnb_chain* chain, int64_t lo, int64_t hi) {
  return full_workspace(chain, lo, hi, 4);
}

int tnb_full_f32(const tnb_chain* chain, int64_t lo, int64_t hi, float* out, void* ws,
                 int64_t ws_bytes, void* stream) {
  return launch_full(chain, lo, hi, out, ws, ws_bytes, (cudaStream_t)stream, 4);
}

int tnb_dot_f32(const tnb_chain* a, const tnb_chain* b, float* out, void* stream) {
  if (!out) return set_error(TNB_EINVAL, "null output");
  return launch_dot(a, b, out, false, (cudaStream_t)stream, 4);
}

int tnb_norm_f32(const tnb_chain* t, float* out, void* stream) {
  if (!out) return set_error(TNB_EINVAL, "null output");
  return launch_dot(t, t, out, true, (cudaStream_t)stream, 4);
}

// ---- float64 instantiation (the generic kernels in double) ----------------
int tnb_repack_f64(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes,
                   void* stream) {
  return repack_any(nodes, n, batch, modes, stream, 8);
}

int tnb_tt_core_f64(const tnb_chain* chain, int32_t k, double* out, void* stream) {
  return tt_core_any(chain, k, out, stream, 8);
}

int tnb_promote_cp_f64(const tnb_node* node, int32_t position, int64_t batch, double* out,
                       void* stream) {
  return promote_any(node, position, batch, out, stream, 8);
}

int64_t tnb_entries_workspace_bytes_f64(const tnb_chain* chain, int64_t m, int32_t algo) {
  return entries_workspace(chain, m, algo, 8);
}

int tnb_entries_f64(const tnb_chain* chain, const int64_t* idx, int64_t m, double* out,
                    int32_t* err_mode, int32_t algo, void* ws, int64_t ws_bytes, void* stream) {
  return entries_any(chain, idx, m, out, err_mode, algo, ws, ws_bytes, stream, 8);
}

int64_t tnb_full_workspace_bytes_f64(const tnb_chain* chain, int64_t lo, int64_t hi) {
  return full_workspace(chain, lo, hi, 8);
}

int tnb_full_f64(const tnb_chain* chain, int64_t lo, int64_t hi, double* out, void* ws,
                 int64_t ws_bytes, void* stream) {
  return launch_full(chain, lo, hi, out, ws, ws_bytes, (cudaStream_t)stream, 8);
}

int tnb_dot_f64(const tnb_chain* a, const tnb_chain* b, double* out, void* stream) {
  if (!out) return set_error(TNB_EINVAL, "null output");
  return launch_dot(a, b, out, false, (cudaStream_t)stream, 8);
}

int tnb_norm_f64(const tnb_chain* t, double* out, void* stream) {
  if (!out) return set_error(TNB_EINVAL, "null output");
  return launch_dot(t, t, out, true, (cudaStream_t)stream, 8);
}

}  // extern "C"

extern "C" int tnb_entries_plan(const tnb_chain* chain, int64_t m, int32_t algo, tnb_entries_info* info) {
  return tnb::entries_plan(chain, m, algo, info);
}
