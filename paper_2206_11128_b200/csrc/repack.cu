// K0: per-node preparation, run once per tensor instead of once per call.
//
// Reference: node_tt_core (core.py:307-327) promotes CP nodes
// (promote_cp_node, core.py:266-296) and absorbs Tucker factors
// (apply_factor, einsum "ji,rik->rjk", core.py:330-334) on EVERY entries /
// full / chain_dot call.  Here it happens once, into the layout the hot
// kernels read:
//   TT            -> dense  [B?][J][r_l][r_r]   (contiguous r_l x r_r tiles)
//   CP interior   -> diag   [B?][J][R]          (copy tensor kept implicit)
//   CP left/right -> dense  [B?][J][1][R] / [B?][J][R][1]  (same bytes as the
//                                                 [J][R] table)
//   CP one-mode   -> dense  [B?][J][1][1]       (sum over R, core.py:316-320)
// The work is tiny (J*I*r_l*r_r MACs per mode) and HBM/latency bound.
#include "common.cuh"

namespace tnb {
namespace {

// fp32 kernels use fmaf; the float64 instantiation (the reference's dtype,
// SURVEY §8(f) row 4) uses fma
__device__ __forceinline__ float fmat(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }

// TT: out[b][j][a][c] = sum_i F[b][j][i] * core[b][a][i][c]  (or core[b][a][j][c])
template <typename T>
__global__ void repack_tt_kernel(const T* __restrict__ core, const T* __restrict__ fac,
                                 int64_t B, int I, int J, int rl, int rr,
                                 T* __restrict__ out) {
  const int64_t per = (int64_t)J * rl * rr;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    int64_t r = t - b * per;
    const int j = (int)(r / ((int64_t)rl * rr));
    r -= (int64_t)j * rl * rr;
    const int a = (int)(r / rr);
    const int c = (int)(r - (int64_t)a * rr);
    const T* cb = core + b * (int64_t)rl * I * rr + (int64_t)a * I * rr + c;
    T v;
    if (fac) {
      const T* fr = fac + b * (int64_t)J * I + (int64_t)j * I;
      T acc = 0;
      for (int i = 0; i < I; ++i) acc = fmat(__ldg(fr + i), __ldg(cb + (int64_t)i * rr), acc);
      v = acc;
    } else {
      v = __ldg(cb + (int64_t)j * rr);
    }
    out[t] = v;
  }
}

// CP: U'[b][j][a] = sum_i F[b][j][i] U[b][i][a]; single-mode chains store the
// sum over a (the reference sums first, then applies the factor).
template <typename T>
__global__ void repack_cp_kernel(const T* __restrict__ core, const T* __restrict__ fac,
                                 int64_t B, int I, int J, int R, int single,
                                 T* __restrict__ out) {
  const int ro = single ? 1 : R;
  const int64_t per = (int64_t)J * ro;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    const int64_t r = t - b * per;
    const int j = (int)(r / ro);
    const int a = (int)(r - (int64_t)j * ro);
    const T* ub = core + b * (int64_t)I * R;
    T v = 0;
    if (fac) {
      const T* fr = fac + b * (int64_t)J * I + (int64_t)j * I;
      for (int i = 0; i < I; ++i) {
        T u;
        if (single) {
          u = 0;
          for (int q = 0; q < R; ++q) u += __ldg(ub + (int64_t)i * R + q);
        } else {
          u = __ldg(ub + (int64_t)i * R + a);
        }
        v = fmat(__ldg(fr + i), u, v);
      }
    } else if (single) {
      for (int q = 0; q < R; ++q) v += __ldg(ub + (int64_t)j * R + q);
    } else {
      v = __ldg(ub + (int64_t)j * R + a);
    }
    out[t] = v;
  }
}

// Repacked mode -> reference layout [B?][r_l][J][r_r] (node_tt_core output).
template <typename T>
__global__ void tt_core_kernel(ModeDev md, int64_t B, T* __restrict__ out) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int64_t per = (int64_t)rl * J * rr;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    int64_t r = t - b * per;
    const int a = (int)(r / ((int64_t)J * rr));
    r -= (int64_t)a * J * rr;
    const int j = (int)(r / rr);
    const int c = (int)(r - (int64_t)j * rr);
    const T* s = reinterpret_cast<const T*>(md.s) + b * md.bstride;
    T v;
    if (md.layout == TNB_LAYOUT_DIAG)
      v = (a == c) ? s[(int64_t)j * rl + a] : T(0);
    else
      v = s[((int64_t)j * rl + a) * rr + c];
    out[t] = v;
  }
}

// promote_cp_node (core.py:266-296), no factor: reference layout output.
template <typename T>
__global__ void promote_cp_kernel(const T* __restrict__ u, int64_t B, int I, int R, int pos,
                                  T* __restrict__ out) {
  int rl, rr;
  if (pos == TNB_POS_LEFT) { rl = 1; rr = R; }
  else if (pos == TNB_POS_RIGHT) { rl = R; rr = 1; }
  else if (pos == TNB_POS_SINGLE) { rl = 1; rr = 1; }
  else { rl = R; rr = R; }
  const int64_t per = (int64_t)rl * I * rr;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    int64_t r = t - b * per;
    const int a = (int)(r / ((int64_t)I * rr));
    r -= (int64_t)a * I * rr;
    const int i = (int)(r / rr);
    const int c = (int)(r - (int64_t)i * rr);
    const T* ub = u + b * (int64_t)I * R + (int64_t)i * R;
    T v;
    if (pos == TNB_POS_LEFT) v = ub[c];
    else if (pos == TNB_POS_RIGHT) v = ub[a];
    else if (pos == TNB_POS_SINGLE) {
      v = 0;
      for (int q = 0; q < R; ++q) v += ub[q];
    } else v = (a == c) ? ub[a] : T(0);
    out[t] = v;
  }
}

inline int grid_for(int64_t total) {
  int64_t g = ceil_div(total, 256);
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

template <typename T>
int repack_t(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes, cudaStream_t st) {
  const int64_t B = batch > 0 ? batch : 1;
  for (int k = 0; k < n; ++k) {
    const tnb_node& nd = nodes[k];
    const tnb_mode& m = modes[k];
    const int64_t total = mode_floats(m) * B;
    if (total == 0) continue;
    if (nd.kind == TNB_KIND_TT) {
      if (m.r_left != nd.r_left || m.r_right != nd.r_right || m.layout != TNB_LAYOUT_DENSE)
        return set_error(TNB_EINVAL, "mode %d: plan does not match node", k);
      repack_tt_kernel<T><<<grid_for(total), 256, 0, st>>>(
          reinterpret_cast<const T*>(nd.core), reinterpret_cast<const T*>(nd.factor), B, nd.internal, nd.phys,
          nd.r_left, nd.r_right, reinterpret_cast<T*>(const_cast<float*>(m.slices)));
    } else {
      const int single = (n == 1);
      repack_cp_kernel<T><<<grid_for(total), 256, 0, st>>>(
          reinterpret_cast<const T*>(nd.core), reinterpret_cast<const T*>(nd.factor), B, nd.internal, nd.phys,
          nd.r_left, single, reinterpret_cast<T*>(const_cast<float*>(m.slices)));
    }
    int rc = check_launch("repack");
    if (rc) return rc;
  }
  return TNB_OK;
}

template int repack_t<float>(const tnb_node*, int32_t, int64_t, const tnb_mode*, cudaStream_t);
template int repack_t<double>(const tnb_node*, int32_t, int64_t, const tnb_mode*, cudaStream_t);

int launch_repack(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes, cudaStream_t st,
                  int elt) {
  return elt == 8 ? repack_t<double>(nodes, n, batch, modes, st) : repack_t<float>(nodes, n, batch, modes, st);
}

int launch_tt_core(const ChainDev& ch, int k, void* out, cudaStream_t st, int elt) {
  const ModeDev& md = ch.m[k];
  const int64_t total = (int64_t)md.rl * md.J * md.rr * ch.batch;
  if (total == 0) return TNB_OK;
  if (elt == 8)
    tt_core_kernel<double><<<grid_for(total), 256, 0, st>>>(md, ch.batch, static_cast<double*>(out));
  else
    tt_core_kernel<float><<<grid_for(total), 256, 0, st>>>(md, ch.batch, static_cast<float*>(out));
  return check_launch("tt_core");
}

int launch_promote_cp(const tnb_node* node, int position, int64_t batch, void* out, cudaStream_t st,
                      int elt) {
  const int64_t B = batch > 0 ? batch : 1;
  const int R = node->r_left, I = node->internal;
  int rl = R, rr = R;
  if (position == TNB_POS_LEFT) rl = 1;
  if (position == TNB_POS_RIGHT) rr = 1;
  if (position == TNB_POS_SINGLE) rl = rr = 1;
  const int64_t total = (int64_t)rl * I * rr * B;
  if (total == 0) return TNB_OK;
  if (elt == 8)
    promote_cp_kernel<double><<<grid_for(total), 256, 0, st>>>(reinterpret_cast<const double*>(node->core), B, I, R,
                                                               position, static_cast<double*>(out));
  else
    promote_cp_kernel<float><<<grid_for(total), 256, 0, st>>>(node->core, B, I, R, position,
                                                              static_cast<float*>(out));
  return check_launch("promote_cp");
}

}  // namespace tnb
