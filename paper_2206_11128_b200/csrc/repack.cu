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

// TT: out[b][j][a][c] = sum_i F[b][j][i] * core[b][a][i][c]  (or core[b][a][j][c])
__global__ void repack_tt_kernel(const float* __restrict__ core, const float* __restrict__ fac,
                                 int64_t B, int I, int J, int rl, int rr,
                                 float* __restrict__ out) {
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
    const float* cb = core + b * (int64_t)rl * I * rr + (int64_t)a * I * rr + c;
    float v;
    if (fac) {
      const float* fr = fac + b * (int64_t)J * I + (int64_t)j * I;
      float acc = 0.f;
      for (int i = 0; i < I; ++i) acc = fmaf(__ldg(fr + i), __ldg(cb + (int64_t)i * rr), acc);
      v = acc;
    } else {
      v = __ldg(cb + (int64_t)j * rr);
    }
    out[t] = v;
  }
}

// CP: U'[b][j][a] = sum_i F[b][j][i] U[b][i][a]; single-mode chains store the
// sum over a (the reference sums first, then applies the factor).
__global__ void repack_cp_kernel(const float* __restrict__ core, const float* __restrict__ fac,
                                 int64_t B, int I, int J, int R, int single,
                                 float* __restrict__ out) {
  const int ro = single ? 1 : R;
  const int64_t per = (int64_t)J * ro;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / per;
    const int64_t r = t - b * per;
    const int j = (int)(r / ro);
    const int a = (int)(r - (int64_t)j * ro);
    const float* ub = core + b * (int64_t)I * R;
    float v = 0.f;
    if (fac) {
      const float* fr = fac + b * (int64_t)J * I + (int64_t)j * I;
      for (int i = 0; i < I; ++i) {
        float u;
        if (single) {
          u = 0.f;
          for (int q = 0; q < R; ++q) u += __ldg(ub + (int64_t)i * R + q);
        } else {
          u = __ldg(ub + (int64_t)i * R + a);
        }
        v = fmaf(__ldg(fr + i), u, v);
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
__global__ void tt_core_kernel(ModeDev md, int64_t B, float* __restrict__ out) {
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
    const float* s = md.s + b * md.bstride;
    float v;
    if (md.layout == TNB_LAYOUT_DIAG)
      v = (a == c) ? s[(int64_t)j * rl + a] : 0.f;
    else
      v = s[((int64_t)j * rl + a) * rr + c];
    out[t] = v;
  }
}

// promote_cp_node (core.py:266-296), no factor: reference layout output.
__global__ void promote_cp_kernel(const float* __restrict__ u, int64_t B, int I, int R, int pos,
                                  float* __restrict__ out) {
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
    const float* ub = u + b * (int64_t)I * R + (int64_t)i * R;
    float v;
    if (pos == TNB_POS_LEFT) v = ub[c];
    else if (pos == TNB_POS_RIGHT) v = ub[a];
    else if (pos == TNB_POS_SINGLE) {
      v = 0.f;
      for (int q = 0; q < R; ++q) v += ub[q];
    } else v = (a == c) ? ub[a] : 0.f;
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

int launch_repack(const tnb_node* nodes, int32_t n, int64_t batch, const tnb_mode* modes,
                  cudaStream_t st) {
  const int64_t B = batch > 0 ? batch : 1;
  for (int k = 0; k < n; ++k) {
    const tnb_node& nd = nodes[k];
    const tnb_mode& m = modes[k];
    const int64_t total = mode_floats(m) * B;
    if (total == 0) continue;
    if (nd.kind == TNB_KIND_TT) {
      if (m.r_left != nd.r_left || m.r_right != nd.r_right || m.layout != TNB_LAYOUT_DENSE)
        return set_error(TNB_EINVAL, "mode %d: plan does not match node", k);
      repack_tt_kernel<<<grid_for(total), 256, 0, st>>>(nd.core, nd.factor, B, nd.internal,
                                                         nd.phys, nd.r_left, nd.r_right,
                                                         m.slices);
    } else {
      const int single = (n == 1);
      repack_cp_kernel<<<grid_for(total), 256, 0, st>>>(nd.core, nd.factor, B, nd.internal,
                                                         nd.phys, nd.r_left, single, m.slices);
    }
    int rc = check_launch("repack");
    if (rc) return rc;
  }
  return TNB_OK;
}

int launch_tt_core(const ChainDev& ch, int k, float* out, cudaStream_t st) {
  const ModeDev& md = ch.m[k];
  const int64_t total = (int64_t)md.rl * md.J * md.rr * ch.batch;
  if (total == 0) return TNB_OK;
  tt_core_kernel<<<grid_for(total), 256, 0, st>>>(md, ch.batch, out);
  return check_launch("tt_core");
}

int launch_promote_cp(const tnb_node* node, int position, int64_t batch, float* out,
                      cudaStream_t st) {
  const int64_t B = batch > 0 ? batch : 1;
  const int R = node->r_left, I = node->internal;
  int rl = R, rr = R;
  if (position == TNB_POS_LEFT) rl = 1;
  if (position == TNB_POS_RIGHT) rr = 1;
  if (position == TNB_POS_SINGLE) rl = rr = 1;
  const int64_t total = (int64_t)rl * I * rr * B;
  if (total == 0) return TNB_OK;
  promote_cp_kernel<<<grid_for(total), 256, 0, st>>>(node->core, B, I, R, position, out);
  return check_launch("promote_cp");
}

}  // namespace tnb
