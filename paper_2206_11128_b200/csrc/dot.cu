// K3: chain inner product and norm (reference: chain_dot core.py:362-384,
// norm core.py:387-391, arithmetic.dot arithmetic.py:189-193).
//
// Per batch element (pair) the r_a x r_b transfer matrix M is propagated core
// by core:  M'[c][d] = sum_{j,a,b} M[a][b] A_j[a][c] B_j[b][d], evaluated as
// the two-stage contraction numpy's einsum path picks for the reference
// (Y = M B_j, then M' += A_j^T Y).  One CTA per pair; the
// transfer matrices live in shared memory, core slices stream from HBM once.
#include "common.cuh"

namespace tnb {
bool dot_fast_supported(const ChainDev& a, const ChainDev& b);
int launch_dot_fast(const ChainDev& a, const ChainDev& b, float* out, bool is_norm, cudaStream_t st);

namespace {

__device__ __forceinline__ float fmat(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float sqrt_pos(float v) { return sqrtf(fmaxf(v, 0.f)); }
__device__ __forceinline__ double sqrt_pos(double v) { return sqrt(fmax(v, 0.0)); }

// T = float (generic fp32 path) or double (the reference's dtype)
template <typename T>
__global__ void __launch_bounds__(256) dot_kernel(const __grid_constant__ ChainDev A,
                                                  const __grid_constant__ ChainDev Bc,
                                                  T* __restrict__ out, int is_norm, int cap) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T* sm = reinterpret_cast<T*>(sm_raw);
  T* M = sm;
  T* Y = sm + cap;
  T* Mn = sm + 2 * cap;
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) M[0] = T(1);
  __syncthreads();
  for (int k = 0; k < A.n; ++k) {
    const ModeDev& ma = A.m[k];
    const ModeDev& mb = Bc.m[k];
    const int ral = ma.rl, rar = ma.rr, rbl = mb.rl, rbr = mb.rr;
    const T* ga = reinterpret_cast<const T*>(ma.s) + e * ma.bstride;
    const T* gb = reinterpret_cast<const T*>(mb.s) + e * mb.bstride;
    for (int t = tid; t < rar * rbr; t += nt) Mn[t] = T(0);
    for (int j = 0; j < ma.J; ++j) {
      // Y[a][d] = sum_b M[a][b] B_j[b][d]
      for (int t = tid; t < ral * rbr; t += nt) {
        const int a = t / rbr, d = t - (t / rbr) * rbr;
        T acc;
        if (mb.layout == TNB_LAYOUT_DIAG) {
          acc = M[a * rbl + d] * __ldg(gb + (int64_t)j * rbl + d);
        } else {
          const T* bj = gb + (int64_t)j * rbl * rbr + d;
          acc = 0;
          for (int b = 0; b < rbl; ++b) acc = fmat(M[a * rbl + b], __ldg(bj + b * rbr), acc);
        }
        Y[t] = acc;
      }
      __syncthreads();
      // M'[c][d] += sum_a A_j[a][c] Y[a][d]
      for (int t = tid; t < rar * rbr; t += nt) {
        const int c = t / rbr, d = t - (t / rbr) * rbr;
        T acc = Mn[t];
        if (ma.layout == TNB_LAYOUT_DIAG) {
          acc = fmat(__ldg(ga + (int64_t)j * ral + c), Y[c * rbr + d], acc);
        } else {
          const T* aj = ga + (int64_t)j * ral * rar + c;
          for (int a = 0; a < ral; ++a) acc = fmat(__ldg(aj + a * rar), Y[a * rbr + d], acc);
        }
        Mn[t] = acc;
      }
      __syncthreads();
    }
    for (int t = tid; t < rar * rbr; t += nt) M[t] = Mn[t];
    __syncthreads();
  }
  if (tid == 0) {
    const T v = M[0];
    out[e] = is_norm ? sqrt_pos(v) : v;
  }
}

}  // namespace

int launch_dot(const tnb_chain* a, const tnb_chain* b, void* out, bool is_norm, cudaStream_t st, int elt) {
  static thread_local ChainDev ca, cb;
  int rc = make_chain_dev(a, &ca, true);
  if (rc) return rc;
  rc = make_chain_dev(b, &cb, true);
  if (rc) return rc;
  if (a->n_modes != b->n_modes) return set_error(TNB_EINVAL, "shape mismatch: %d vs %d modes",
                                                 a->n_modes, b->n_modes);
  for (int k = 0; k < a->n_modes; ++k)
    if (a->modes[k].phys != b->modes[k].phys)
      return set_error(TNB_EINVAL, "shape mismatch on mode %d: %d vs %d", k, a->modes[k].phys,
                       b->modes[k].phys);
  if (a->batch != b->batch) return set_error(TNB_EINVAL, "operands must agree on batching");
  KTimer kt("dot", st);
  const char* gen = getenv("TNB_DOT_GENERIC");
  if (elt == 4 && !(gen && gen[0] == '1') && dot_fast_supported(ca, cb))
    return launch_dot_fast(ca, cb, static_cast<float*>(out), is_norm, st);
  int cap = 1;
  for (int k = 0; k < a->n_modes; ++k) {
    const int ral = a->modes[k].r_left, rar = a->modes[k].r_right;
    const int rbl = b->modes[k].r_left, rbr = b->modes[k].r_right;
    const int s[3] = {ral * rbl, ral * rbr, rar * rbr};
    for (int q = 0; q < 3; ++q) cap = s[q] > cap ? s[q] : cap;
  }
  const size_t smem = 3 * (size_t)cap * (size_t)elt;
  if (smem > 200 * 1024) return set_error(TNB_EINVAL, "ranks too large for dot (r_a*r_b=%d)", cap);
  const int64_t B = ca.batch;
  if (B > 0x7fffffff) return set_error(TNB_EINVAL, "batch too large");
  if (elt == 8) {
    if (smem > 48 * 1024) {
      rc = check_cuda(cudaFuncSetAttribute(dot_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "dot smem attr");
      if (rc) return rc;
    }
    dot_kernel<double><<<(unsigned)B, 256, smem, st>>>(ca, cb, static_cast<double*>(out), is_norm ? 1 : 0, cap);
  } else {
    if (smem > 48 * 1024) {
      rc = check_cuda(cudaFuncSetAttribute(dot_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "dot smem attr");
      if (rc) return rc;
    }
    dot_kernel<float><<<(unsigned)B, 256, smem, st>>>(ca, cb, static_cast<float*>(out), is_norm ? 1 : 0, cap);
  }
  return check_launch("dot");
}

}  // namespace tnb
