// K1: batched multi-index entry evaluation (reference: entries,
// core.py:394-460, reached from t[idx] via indexing.py:120-130).
//
// Three algorithms share one contract (tnb.h):
//   LAYERED  - one launch per mode over a global [m][B][r] state buffer; any
//              rank, any number of modes (the reference's own mode-by-mode
//              structure, core.py:419-429).  Needs a workspace.
//   CHAIN    - one thread per (sample, batch element); the r-vector state
//              lives in registers for the whole chain, cores are read through
//              L1/L2.  Ranks <= 32.
//   BUCKETED - entries_bucketed.cu: the performance kernel (cfg2 / cfg5).
// Index handling is identical in all three: negatives wrap, any value outside
// [-J, J) lowers *err to its mode number (core.py:409-416), and the kernel
// keeps going with a clamped index so no out-of-range address is formed.
#include "common.cuh"

namespace tnb {
int launch_entries_bucketed(const ChainDev& ch, const int64_t* idx, int64_t m, float* out,
                            int32_t* err, void* ws, int64_t ws_bytes, cudaStream_t st, bool reuse_records = false);
bool bucketed_supported(const ChainDev& ch);
int64_t bucketed_workspace(const ChainDev& ch, int64_t m);
void bucketed_info(const ChainDev& ch, int64_t m, tnb_entries_info* info);
double chain_entry_flops(const ChainDev& ch);
bool two_table_ok(const ChainDev& ch, int64_t m);
// entries_gsort.cuh: the global-sort tcgen05 path
bool gsort_ok(const ChainDev& ch, int64_t m, bool batched);
bool gsort_auto(const ChainDev& ch, int64_t m, bool batched);
int64_t gsort_workspace(const ChainDev& ch, int64_t m, bool batched);
void gsort_info(const ChainDev& ch, int64_t m, tnb_entries_info* info, bool batched);
int launch_entries_gsort(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                         int64_t ws_bytes, cudaStream_t st);
int64_t gsort_table_bytes(const ChainDev& ch, int64_t m, bool batched);
int gsort_tables(const ChainDev& ch, int64_t m, bool batched, void* table_ws, cudaStream_t st, int slot,
                 cudaEvent_t* done);
int gsort_compute(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                  int64_t ws_bytes, void* table_ws, cudaStream_t st, bool batched, bool reuse_records,
                  cudaEvent_t tables);
int64_t two_table_workspace(const ChainDev& ch, int64_t m);
void two_table_info(const ChainDev& ch, int64_t m, tnb_entries_info* info);
int launch_two_table(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                     int64_t ws_bytes, cudaStream_t st);

namespace {

__device__ __forceinline__ float fmat(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }

// T = float (the hot path) or double (the reference's dtype)
template <typename T, int RMAX>
__global__ void __launch_bounds__(256) entries_chain_kernel(const __grid_constant__ ChainDev ch,
                                                            const int64_t* __restrict__ idx,
                                                            int64_t m, T* __restrict__ out,
                                                            int32_t* err) {
  const int64_t B = ch.batch;
  const int N = ch.n;
  const int64_t total = m * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / B;
    const int64_t e = t - s * B;
    const int64_t* row = idx + s * N;
    T v[RMAX];
#pragma unroll
    for (int a = 0; a < RMAX; ++a) v[a] = (a == 0) ? T(1) : T(0);
    for (int k = 0; k < N; ++k) {
      const ModeDev& md = ch.m[k];
      const int j = norm_index(row[k], md.J, k, err);
      if (md.J == 0) continue;
      const T* g = reinterpret_cast<const T*>(md.s) + e * md.bstride;
      if (md.layout == TNB_LAYOUT_DIAG) {
        g += (int64_t)j * md.rl;
#pragma unroll
        for (int a = 0; a < RMAX; ++a)
          if (a < md.rl) v[a] *= __ldg(g + a);
      } else {
        const int rl = md.rl, rr = md.rr;
        g += (int64_t)j * rl * rr;
        T w[RMAX];
#pragma unroll
        for (int c = 0; c < RMAX; ++c) w[c] = T(0);
#pragma unroll
        for (int a = 0; a < RMAX; ++a) {
          if (a < rl) {
            const T va = v[a];
            const T* ga = g + a * rr;
#pragma unroll
            for (int c = 0; c < RMAX; ++c)
              if (c < rr) w[c] = fmat(va, __ldg(ga + c), w[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < RMAX; ++c) v[c] = w[c];
      }
    }
    out[t] = v[0];
  }
}

// One mode of the layered algorithm: thread per (sample, batch element, c).
template <typename T>
__global__ void entries_layer_kernel(ModeDev md, int k, int N, int64_t B,
                                     const int64_t* __restrict__ idx, int64_t m,
                                     const T* __restrict__ vin, T* __restrict__ vout,
                                     int stride, T* __restrict__ out, int last,
                                     int32_t* err) {
  const int rl = md.rl, rr = md.rr;
  const int64_t total = m * B * rr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t se = t / rr;
    const int c = (int)(t - se * rr);
    const int64_t s = se / B;
    const int64_t e = se - s * B;
    const int j = norm_index(idx[s * N + k], md.J, k, err);
    T acc = 0;
    if (md.J > 0) {
      const T* g = reinterpret_cast<const T*>(md.s) + e * md.bstride;
      const T* vi = vin ? vin + se * stride : nullptr;
      if (md.layout == TNB_LAYOUT_DIAG) {
        acc = (vi ? vi[c] : T(1)) * __ldg(g + (int64_t)j * rl + c);
      } else {
        const T* gj = g + (int64_t)j * rl * rr + c;
        for (int a = 0; a < rl; ++a) acc = fmat(vi ? vi[a] : T(1), __ldg(gj + (int64_t)a * rr), acc);
      }
    }
    if (last)
      out[se] = acc;
    else
      vout[se * stride + c] = acc;
  }
}

inline int grid_for(int64_t total, int threads) {
  int64_t g = ceil_div(total, threads);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

int pick_algo(const tnb_chain* c, int algo, int rmax) {
  if (algo != TNB_ALGO_AUTO) return algo;
  if (c->n_modes > kMaxModes || rmax > 32) return TNB_ALGO_LAYERED;
  return TNB_ALGO_CHAIN;
}

// float64 AUTO: the layered kernels beat the register chain once m is large
// (cfg2 chain, 2^20 tuples: 7.7 vs 25.4 ms; cfg5: 3.0 vs 7.1 ms -- in double
// the chain kernel's per-thread slice reads are L2-bound)
int pick_algo_f64(const tnb_chain* c, int algo, int rmax, int64_t m) {
  if (algo == TNB_ALGO_AUTO && m >= (1 << 12)) return TNB_ALGO_LAYERED;
  return pick_algo(c, algo, rmax);
}

int chain_rmax(const tnb_chain* c) {
  int r = 1;
  for (int k = 0; k < c->n_modes; ++k) {
    if (c->modes[k].r_left > r) r = c->modes[k].r_left;
    if (c->modes[k].r_right > r) r = c->modes[k].r_right;
  }
  return r;
}

// Batched chains (core.py:425-429, _step_entries_batched core.py:447-460)
// on the bucketed kernels: batch element b is the unbatched chain whose
// modes point b * bstride into the repacked slices.  Every element shares
// the index matrix, so the prep / sort tile records are built once (element
// 0) and reused; each element builds its own tables and runs the compute
// kernel into a [B][m] scratch, which one transpose kernel turns into the
// reference's [m][B] output.
ChainDev element_chain(const ChainDev& ch, int64_t b) {
  ChainDev e = ch;
  e.batch = 1;
  for (int k = 0; k < ch.n; ++k) {
    e.m[k].s = ch.m[k].s + b * ch.m[k].bstride;
    e.m[k].bstride = 0;
  }
  return e;
}

// out[s][b] = tmp[b][s]: thread = sample, B consecutive floats per thread
__global__ void batch_transpose_kernel(const float* __restrict__ tmp, int64_t m, int64_t B, float* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x)
    for (int64_t b = 0; b < B; ++b) out[s * B + b] = __ldcs(tmp + b * m + s);
}

int64_t batched_tmp_offset(const ChainDev& ch, int64_t m) {
  return (bucketed_workspace(element_chain(ch, 0), m) + 255) & ~(int64_t)255;
}

}  // namespace

bool bucketed_ok(const ChainDev& ch) {
  return ch.batch > 1 ? bucketed_supported(element_chain(ch, 0)) : bucketed_supported(ch);
}

// AUTO: chains that merge into a prefix and a suffix table (any rank) run
// the fused two-table kernel
bool use_two_table(const tnb_chain* c, const ChainDev& ch, int64_t m, int algo) {
  return algo == TNB_ALGO_AUTO && c->n_modes <= kMaxModes && m >= (1 << 12) && two_table_ok(ch, m);
}

// AUTO: large unbatched calls whose merged chain is first . dense . [diag] . last
// run the global-sort tcgen05 path (TNB_ENTRIES_GSORT=0 turns that off)
// (batched chains: one element at a time over the records sorted once)
bool use_gsort(const ChainDev& ch, int64_t m, int algo) {
  if (algo == TNB_ALGO_GSORT) return true;
  if (algo != TNB_ALGO_AUTO) return false;
  return ch.batch > 1 ? gsort_auto(element_chain(ch, 0), m, true) : gsort_auto(ch, m, false);
}

bool gsort_ok_any(const ChainDev& ch, int64_t m) {
  return ch.batch > 1 ? gsort_ok(element_chain(ch, 0), m, true) : gsort_ok(ch, m, false);
}

// batched workspace: [element workspace (its head holds the tables of the even
// elements)] [a second table region for the odd elements] [tmp: B x m results]
int64_t gsort_tab2_offset(const ChainDev& ch, int64_t m) {
  return (gsort_workspace(element_chain(ch, 0), m, true) + 255) & ~(int64_t)255;
}

int64_t gsort_tmp_offset(const ChainDev& ch, int64_t m) {
  return gsort_tab2_offset(ch, m) + ((gsort_table_bytes(element_chain(ch, 0), m, true) + 255) & ~(int64_t)255);
}

int64_t gsort_workspace_any(const ChainDev& ch, int64_t m) {
  if (ch.batch <= 1) return gsort_workspace(ch, m, false);
  return gsort_tmp_offset(ch, m) + ch.batch * m * (int64_t)sizeof(float);
}

int launch_gsort_any(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                     int64_t ws_bytes, cudaStream_t st) {
  if (ch.batch <= 1) return launch_entries_gsort(ch, idx, m, out, err, ws, ws_bytes, st);
  const int64_t off2 = gsort_tab2_offset(ch, m), off = gsort_tmp_offset(ch, m);
  const int64_t need = off + ch.batch * m * (int64_t)sizeof(float);
  if (!ws || ws_bytes < need)
    return set_error(TNB_EWORKSPACE, "batched global-sort entries needs %lld workspace bytes, got %lld",
                     (long long)need, (long long)ws_bytes);
  unsigned char* w = static_cast<unsigned char*>(ws);
  float* tmp = reinterpret_cast<float*>(w + off);
  // element b's tables live in region b & 1; element b + 1's are built (side
  // stream) while element b's index passes / compute kernel run: the fork
  // waits for what is queued on st, i.e. compute b - 1, the region's last reader
  auto region = [&](int64_t b) { return (b & 1) ? w + off2 : w; };
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int rc = gsort_tables(element_chain(ch, 0), m, true, region(0), st, 0, &ev[0]);
  for (int64_t b = 0; b < ch.batch && !rc; ++b) {
    if (b + 1 < ch.batch) rc = gsort_tables(element_chain(ch, b + 1), m, true, region(b + 1), st, (b + 1) & 1, &ev[(b + 1) & 1]);
    if (rc) {
      if (ev[b & 1]) cudaStreamWaitEvent(st, ev[b & 1], 0);
      break;
    }
    rc = gsort_compute(element_chain(ch, b), idx, m, tmp + b * m, err, ws, off2, region(b), st, true, b > 0, ev[b & 1]);
    if (rc && b + 1 < ch.batch && ev[(b + 1) & 1]) cudaStreamWaitEvent(st, ev[(b + 1) & 1], 0);
  }
  if (rc) return rc;
  int64_t g = (m + 255) / 256;
  if (g > (int64_t)num_sms() * 16) g = (int64_t)num_sms() * 16;
  batch_transpose_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, st>>>(tmp, m, ch.batch, out);
  return check_launch("batch_transpose");
}

bool use_bucketed(const ChainDev& ch, int64_t m, int algo) {
  if (algo == TNB_ALGO_BUCKETED) return true;
  return algo == TNB_ALGO_AUTO && m >= (1 << 16) && bucketed_ok(ch);
}

int launch_bucketed_any(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                        int64_t ws_bytes, cudaStream_t st) {
  if (!bucketed_ok(ch)) return set_error(TNB_EINVAL, "bucketed algorithm does not support this chain");
  if (ch.batch <= 1) return launch_entries_bucketed(ch, idx, m, out, err, ws, ws_bytes, st);
  const int64_t off = batched_tmp_offset(ch, m);
  const int64_t need = off + ch.batch * m * (int64_t)sizeof(float);
  if (!ws || ws_bytes < need)
    return set_error(TNB_EWORKSPACE, "batched bucketed entries needs %lld workspace bytes, got %lld",
                     (long long)need, (long long)ws_bytes);
  float* tmp = reinterpret_cast<float*>(static_cast<unsigned char*>(ws) + off);
  for (int64_t b = 0; b < ch.batch; ++b) {
    const int rc = launch_entries_bucketed(element_chain(ch, b), idx, m, tmp + b * m, err, ws, off, st, b > 0);
    if (rc) return rc;
  }
  int64_t g = (m + 255) / 256;
  if (g > (int64_t)num_sms() * 16) g = (int64_t)num_sms() * 16;
  batch_transpose_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, st>>>(tmp, m, ch.batch, out);
  return check_launch("batch_transpose");
}

int64_t entries_workspace(const tnb_chain* c, int64_t m, int algo, int elt) {
  if (!c || !c->modes || c->n_modes < 1 || m < 0) return -1;
  const int rmax = chain_rmax(c);
  if (elt == 8) {
    if (pick_algo_f64(c, algo, rmax, m) != TNB_ALGO_LAYERED) return 0;
    const int64_t B = c->batch > 0 ? c->batch : 1;
    return 2 * m * B * (int64_t)rmax * 8;
  }
  if (c->n_modes <= kMaxModes && (algo == TNB_ALGO_AUTO || algo == TNB_ALGO_BUCKETED || algo == TNB_ALGO_GSORT)) {
    static thread_local ChainDev ch;
    if (make_chain_dev(c, &ch, true) == TNB_OK && use_two_table(c, ch, m, algo)) return two_table_workspace(ch, m);
    if (make_chain_dev(c, &ch, true) == TNB_OK && use_gsort(ch, m, algo)) return gsort_workspace_any(ch, m);
    if (make_chain_dev(c, &ch, true) == TNB_OK && use_bucketed(ch, m, algo) && bucketed_ok(ch))
      return ch.batch > 1 ? batched_tmp_offset(ch, m) + ch.batch * m * (int64_t)sizeof(float)
                          : bucketed_workspace(ch, m);
  }
  if (pick_algo(c, algo, rmax) != TNB_ALGO_LAYERED) return 0;
  const int64_t B = c->batch > 0 ? c->batch : 1;
  return 2 * m * B * (int64_t)rmax * (int64_t)sizeof(float);
}

// per-entry kernel flops of a chain: 2*r_l*r_r per interior dense step, R
// per diagonal (CP) step, 2*r_l for the closing dot; the first mode is a copy
double chain_entry_flops(const ChainDev& ch) {
  double f = 0.0;
  for (int k = 1; k < ch.n; ++k) {
    const ModeDev& md = ch.m[k];
    if (md.layout == TNB_LAYOUT_DIAG) f += md.rl;
    else f += 2.0 * md.rl * md.rr;
  }
  return f * (double)ch.batch;
}

int entries_plan(const tnb_chain* c, int64_t m, int algo, tnb_entries_info* info) {
  static thread_local ChainDev ch;
  if (!c || !c->modes || !info || m < 0) return set_error(TNB_EINVAL, "null argument");
  const int use = pick_algo(c, algo, chain_rmax(c));
  int rc = make_chain_dev(c, &ch, use != TNB_ALGO_LAYERED);
  if (rc) return rc;
  info->algo = use;
  info->n_virtual = ch.n;
  info->prefix_modes = info->suffix_modes = 1;
  info->prefix_rows = info->suffix_rows = 0;
  info->table_flops = 0.0;
  info->diag_tables = info->table_launches = 0;
  info->compute_kernel = info->tile = 0;
  info->tensor_flops = 0.0;
  if (c->n_modes <= kMaxModes && use_two_table(c, ch, m, algo)) {
    info->algo = TNB_ALGO_BUCKETED;
    two_table_info(ch, m, info);
    return TNB_OK;
  }
  if (use_gsort(ch, m, algo)) {
    if (!gsort_ok_any(ch, m)) return set_error(TNB_EINVAL, "the global-sort algorithm does not support this chain");
    info->algo = TNB_ALGO_GSORT;
    gsort_info(ch.batch > 1 ? element_chain(ch, 0) : ch, m, info, ch.batch > 1);
    // batched: B elements, each its own tables and compute launch
    info->kernel_flops *= (double)ch.batch;
    info->tensor_flops *= (double)ch.batch;
    info->table_flops *= (double)ch.batch;
    info->table_launches *= (int32_t)ch.batch;
    return TNB_OK;
  }
  if (use_bucketed(ch, m, algo) && bucketed_ok(ch)) {
    info->algo = TNB_ALGO_BUCKETED;
    bucketed_info(ch.batch > 1 ? element_chain(ch, 0) : ch, m, info);
    // batched: B elements, each its own tables and compute launch
    info->kernel_flops *= (double)ch.batch;
    info->tensor_flops *= (double)ch.batch;
    info->table_flops *= (double)ch.batch;
    info->table_launches *= (int32_t)ch.batch;
    return TNB_OK;
  }
  info->kernel_flops = chain_entry_flops(ch) * (double)m;
  return TNB_OK;
}

template <typename T>
int entries_generic(const tnb_chain* c, const ChainDev& ch, int use, const int64_t* idx, int64_t m, T* out,
                    int32_t* err, void* ws, int64_t ws_bytes, cudaStream_t st) {
  const int64_t B = ch.batch;
  int rc;
  if (use == TNB_ALGO_CHAIN) {
    const int64_t total = m * B;
    const int g = grid_for(total, 256);
    if (ch.rmax <= 8)
      entries_chain_kernel<T, 8><<<g, 256, 0, st>>>(ch, idx, m, out, err);
    else if (ch.rmax <= 16)
      entries_chain_kernel<T, 16><<<g, 256, 0, st>>>(ch, idx, m, out, err);
    else if (ch.rmax <= 32)
      entries_chain_kernel<T, 32><<<g, 256, 0, st>>>(ch, idx, m, out, err);
    else
      return set_error(TNB_EINVAL, "chain algorithm supports ranks <= 32, got %d", ch.rmax);
    return check_launch("entries_chain");
  }
  if (use != TNB_ALGO_LAYERED) return set_error(TNB_EINVAL, "unknown entries algorithm %d", use);
  const int64_t need = 2 * m * B * (int64_t)ch.rmax * (int64_t)sizeof(T);
  if (!ws || ws_bytes < need)
    return set_error(TNB_EWORKSPACE, "entries needs %lld workspace bytes, got %lld",
                     (long long)need, (long long)ws_bytes);
  T* buf[2] = {(T*)ws, (T*)ws + m * B * ch.rmax};
  const T* vin = nullptr;
  for (int k = 0; k < c->n_modes; ++k) {
    const tnb_mode& mm = c->modes[k];
    ModeDev md;
    md.s = mm.slices;
    md.bstride = c->batch > 0 ? mode_floats(mm) : 0;
    md.layout = mm.layout;
    md.J = mm.phys;
    md.rl = mm.r_left;
    md.rr = mm.r_right;
    const int last = (k == c->n_modes - 1);
    T* vout = buf[k & 1];
    const int64_t total = m * B * md.rr;
    if (total > 0)
      entries_layer_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(md, k, c->n_modes, B, idx, m, vin, vout,
                                                                    ch.rmax, out, last, err);
    rc = check_launch("entries_layer");
    if (rc) return rc;
    vin = vout;
  }
  return TNB_OK;
}

int launch_entries(const tnb_chain* c, const int64_t* idx, int64_t m, void* out_v, int32_t* err,
                   int algo, void* ws, int64_t ws_bytes, cudaStream_t st, int elt) {
  static thread_local ChainDev ch;
  if (!c || !c->modes) return set_error(TNB_EINVAL, "null chain");
  const int rmax0 = chain_rmax(c);
  const int use = pick_algo(c, algo, rmax0);
  int rc = make_chain_dev(c, &ch, use != TNB_ALGO_LAYERED);
  if (rc) return rc;
  // "no error" sentinel 0x7f7f7f7f >= n_modes
  rc = check_cuda(cudaMemsetAsync(err, 0x7f, sizeof(int32_t), st), "memset err");
  if (rc || m == 0) return rc;
  if (elt == 8) {  // float64: the generic algorithms only
    if (use == TNB_ALGO_BUCKETED || use == TNB_ALGO_GSORT)
      return set_error(TNB_EINVAL, "the bucketed / global-sort algorithms are fp32 only");
    const int use64 = pick_algo_f64(c, algo, rmax0, m);
    return entries_generic<double>(c, ch, use64, idx, m, static_cast<double*>(out_v), err, ws, ws_bytes, st);
  }
  float* out = static_cast<float*>(out_v);
  if (use_two_table(c, ch, m, algo)) return launch_two_table(ch, idx, m, out, err, ws, ws_bytes, st);
  if (use_gsort(ch, m, algo)) {
    if (!gsort_ok_any(ch, m)) return set_error(TNB_EINVAL, "the global-sort algorithm does not support this chain");
    return launch_gsort_any(ch, idx, m, out, err, ws, ws_bytes, st);
  }
  if ((algo == TNB_ALGO_AUTO && use_bucketed(ch, m, algo)) || use == TNB_ALGO_BUCKETED)
    return launch_bucketed_any(ch, idx, m, out, err, ws, ws_bytes, st);
  return entries_generic<float>(c, ch, use, idx, m, out, err, ws, ws_bytes, st);
}

}  // namespace tnb
