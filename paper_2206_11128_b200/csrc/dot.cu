// K3: chain inner product and norm (reference: chain_dot core.py:362-384,
// norm core.py:387-391, arithmetic.dot arithmetic.py:189-193).
//
// Per batch element (pair) the r_a x r_b transfer matrix M is propagated core
// by core:  M'[c][d] = sum_{j,a,b} M[a][b] A_j[a][c] B_j[b][d], evaluated as
// the two-stage contraction numpy's einsum path picks for the reference
// (Y = M B_j, then M' += A_j^T Y).  One CTA per pair; the
// transfer matrices live in shared memory, core slices stream from HBM once.
#include <algorithm>

#include "common.cuh"

namespace tnb {
bool dot_fast_supported(const ChainDev& a, const ChainDev& b);
int launch_dot_fast(const ChainDev& a, const ChainDev& b, float* out, bool is_norm, cudaStream_t st);
int dot_mma_rank(const ChainDev& a, const ChainDev& b);
int launch_dot_mma(const ChainDev& a, const ChainDev& b, float* out, bool is_norm, cudaStream_t st);

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

// Chunked kernel for dense chains of any rank (the rank-16 mma.sync kernel
// covers r = 16 fp32 only): per mode, CH slices of A and B at a time are
// staged in shared memory with coalesced 16-byte loads, then
//   Y_j[a][d] = sum_b M[a][b] B_j[b][d]          (all CH slices)
//   M'[c][d] += sum_{j in chunk, a} A_j[a][c] Y_j[a][d]
// each thread computing VW consecutive d (one 16-byte shared load of B / Y
// per VW FMAs; A and M entries broadcast).  Three barriers per CH slices
// instead of two per slice; persistent CTAs, several per SM.
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using V = float4;
  static constexpr int W = 4;
  __device__ static void fma(const float s, const V& b, float* acc) {
    acc[0] = fmaf(s, b.x, acc[0]);
    acc[1] = fmaf(s, b.y, acc[1]);
    acc[2] = fmaf(s, b.z, acc[2]);
    acc[3] = fmaf(s, b.w, acc[3]);
  }
};
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int W = 2;
  __device__ static void fma(const double s, const V& b, double* acc) {
    acc[0] = ::fma(s, b.x, acc[0]);
    acc[1] = ::fma(s, b.y, acc[1]);
  }
};

template <typename T>
__device__ __forceinline__ void stage(T* dst, const T* __restrict__ src, int64_t count, int tid, int nt) {
  // 16-byte pieces (both ends 16-byte aligned by construction), scalar tail
  using V = typename Vec<T>::V;
  constexpr int W = Vec<T>::W;
  const int64_t nv = count / W;
  for (int64_t i = tid; i < nv; i += nt) reinterpret_cast<V*>(dst)[i] = __ldg(reinterpret_cast<const V*>(src) + i);
  for (int64_t i = nv * W + tid; i < count; i += nt) dst[i] = __ldg(src + i);
}

// asynchronous staging (cp.async, 16-byte pieces + element tail), one commit
// group per call; the caller waits with cp.async.wait_group
template <typename T>
__device__ __forceinline__ void stage_async(T* dst, const T* __restrict__ src, int64_t count, int tid, int nt) {
  constexpr int W = 16 / (int)sizeof(T);
  const int64_t nv = count / W;
  for (int64_t i = tid; i < nv; i += nt)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + i * W)),
                 "l"(src + i * W)
                 : "memory");
  for (int64_t i = nv * W + tid; i < count; i += nt) {
    if constexpr (sizeof(T) == 8)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + i)),
                   "l"(src + i)
                   : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + i)),
                   "l"(src + i)
                   : "memory");
  }
}

__device__ __forceinline__ int chunk_slices(int scap, int sa, int sb, int sy, int J) {
  const int mx = sa > sb ? (sa > sy ? sa : sy) : (sb > sy ? sb : sy);
  int ch = scap / mx;
  return ch < 1 ? 1 : (ch > J ? J : ch);
}

template <typename T>
__global__ void __launch_bounds__(256) dot_chunk_kernel(const __grid_constant__ ChainDev A,
                                                        const __grid_constant__ ChainDev Bc, T* __restrict__ out,
                                                        int is_norm, int mcap, int scap) {
  using V = typename Vec<T>::V;
  constexpr int W = Vec<T>::W;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  T* M = reinterpret_cast<T*>(sm_raw);   // [ral][rbl]
  T* Mt = M + mcap;                      // M transposed [rbl][ral] (W x W register tiles of Y)
  T* Mn = Mt + mcap;                     // next M, [rar][rbr]
  T* Ps = Mn + mcap;                     // per-thread W x W partials of M' (tiled modes), [nt][W][W]
  T* Asb[2] = {Ps + 256 * W * W, Ps + 256 * W * W + scap};  // double-buffered slice chunks
  T* Bsb[2] = {Asb[1] + scap, Asb[1] + 2 * scap};
  T* Ys = Bsb[1] + scap;
  const int tid = threadIdx.x, nt = blockDim.x;
  // The next (pair, mode, chunk) item is staged with cp.async while the
  // current one is computed: chunks run ahead across modes and pairs.
  auto issue = [&](int64_t e, int k, int j0, int buf) {
    if (e < A.batch) {
      const ModeDev& ma = A.m[k];
      const ModeDev& mb = Bc.m[k];
      const int sa = ma.rl * ma.rr, sb = mb.rl * mb.rr, sy = ma.rl * mb.rr;
      const int ch = chunk_slices(scap, sa, sb, sy, ma.J);
      const int nj = ma.J - j0 < ch ? ma.J - j0 : ch;
      stage_async(Asb[buf], reinterpret_cast<const T*>(ma.s) + e * ma.bstride + (int64_t)j0 * sa, (int64_t)nj * sa,
                  tid, nt);
      stage_async(Bsb[buf], reinterpret_cast<const T*>(mb.s) + e * mb.bstride + (int64_t)j0 * sb, (int64_t)nj * sb,
                  tid, nt);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  issue(blockIdx.x, 0, 0, 0);
  for (int64_t e = blockIdx.x; e < A.batch; e += gridDim.x) {
    if (tid == 0) M[0] = Mt[0] = T(1);
    __syncthreads();
    for (int k = 0; k < A.n; ++k) {
      const ModeDev& ma = A.m[k];
      const ModeDev& mb = Bc.m[k];
      const int ral = ma.rl, rar = ma.rr, rbl = mb.rl, rbr = mb.rr, J = ma.J;
      const T* ga = reinterpret_cast<const T*>(ma.s) + e * ma.bstride;
      const T* gb = reinterpret_cast<const T*>(mb.s) + e * mb.bstride;
      const int sa = ral * rar, sb = rbl * rbr, sy = ral * rbr;
      const int CH = chunk_slices(scap, sa, sb, sy, J);
      // W x W register tiles when every dimension they span is a multiple of
      // W (interior modes); the rank-1 boundary modes take the scalar rows
      const bool tiled = (ral % W == 0) && (rar % W == 0) && (rbr % W == 0);
      const int ta = ral / W, td = rbr / W, tc = rar / W;
      // M' reduction split: og output tiles x nsplit slices of the (j, a) pairs
      const int og = tc * td;
      // kept: the M' tiles fit one per thread (else each chunk's tiles are
      // looped over and added into Mn)
      const bool kept = tiled && og <= nt;
      const int nsplit = kept ? nt / og : 1;
      for (int t = tid; t < rar * rbr; t += nt) Mn[t] = T(0);
      // tiled: this thread's M' tile (output tile o, reduction slice rs) in
      // registers across the whole mode, reduced in a fixed order at its end
      const int o = kept ? tid % og : 0, rs = kept ? tid / og : 0;
      const int c0 = kept ? (o / td) * W : 0, dd0 = kept ? (o % td) * W : 0;
      T macc[W][W];
#pragma unroll
      for (int i = 0; i < W; ++i)
#pragma unroll
        for (int q = 0; q < W; ++q) macc[i][q] = T(0);
      for (int j0 = 0; j0 < J; j0 += CH) {
        const int nj = J - j0 < CH ? J - j0 : CH;
        // stage the following item into the other buffer (its previous
        // contents were consumed before the barrier that ended the last chunk)
        if (j0 + CH < J) issue(e, k, j0 + CH, buf ^ 1);
        else if (k + 1 < A.n) issue(e, k + 1, 0, buf ^ 1);
        else issue(e + gridDim.x, 0, 0, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // this chunk's copies (this thread's) landed
        __syncthreads();  // ... everyone's; previous chunk done with Ys (and Mn zeroed)
        const T* As = Asb[buf];
        const T* Bs = Bsb[buf];
        if (tiled) {
          // Y_j[a0..a0+W)[d0..d0+W) = sum_b Mt[b][a0..] x B_j[b][d0..]
          const int groups = nj * ta * td;
          for (int g = tid; g < groups; g += nt) {
            const int j = g / (ta * td), r = g - j * (ta * td), a0 = (r / td) * W, d0 = (r % td) * W;
            T acc[W][W];
#pragma unroll
            for (int i = 0; i < W; ++i)
#pragma unroll
              for (int q = 0; q < W; ++q) acc[i][q] = T(0);
            const T* bj = Bs + j * sb + d0;
            for (int b = 0; b < rbl; ++b) {
              const V mv = *reinterpret_cast<const V*>(Mt + b * ral + a0);
              const V bv = *reinterpret_cast<const V*>(bj + b * rbr);
              const T* mp = reinterpret_cast<const T*>(&mv);
#pragma unroll
              for (int i = 0; i < W; ++i) Vec<T>::fma(mp[i], bv, acc[i]);
            }
#pragma unroll
            for (int i = 0; i < W; ++i)
              *reinterpret_cast<V*>(Ys + j * sy + (a0 + i) * rbr + d0) = *reinterpret_cast<V*>(acc[i]);
          }
        } else {
          for (int t = tid; t < nj * sy; t += nt) {
            const int j = t / sy, r = t - j * sy, a = r / rbr, d = r - a * rbr;
            T acc = T(0);
            for (int b = 0; b < rbl; ++b) acc = fmat(M[a * rbl + b], Bs[j * sb + b * rbr + d], acc);
            Ys[j * sy + r] = acc;
          }
        }
        __syncthreads();
        if (tiled && !kept) {
          for (int oo = tid; oo < og; oo += nt) {
            const int cc = (oo / td) * W, d0 = (oo % td) * W;
            T acc[W][W];
#pragma unroll
            for (int i = 0; i < W; ++i)
#pragma unroll
              for (int q = 0; q < W; ++q) acc[i][q] = T(0);
            for (int ja = 0; ja < nj * ral; ++ja) {
              const int j = ja / ral, a = ja - j * ral;
              const V av = *reinterpret_cast<const V*>(As + j * sa + a * rar + cc);
              const V yv = *reinterpret_cast<const V*>(Ys + j * sy + a * rbr + d0);
              const T* ap = reinterpret_cast<const T*>(&av);
#pragma unroll
              for (int i = 0; i < W; ++i) Vec<T>::fma(ap[i], yv, acc[i]);
            }
#pragma unroll
            for (int i = 0; i < W; ++i)
#pragma unroll
              for (int q = 0; q < W; ++q) Mn[(cc + i) * rbr + d0 + q] += acc[i][q];
          }
        } else if (tiled) {
          // M'[c0..][d0..] += sum over this thread's slice of (j, a) of A_j[a][c0..] x Y_j[a][d0..]
          if (tid < og * nsplit) {
            for (int ja = rs; ja < nj * ral; ja += nsplit) {
              const int j = ja / ral, a = ja - j * ral;
              const V av = *reinterpret_cast<const V*>(As + j * sa + a * rar + c0);
              const V yv = *reinterpret_cast<const V*>(Ys + j * sy + a * rbr + dd0);
              const T* ap = reinterpret_cast<const T*>(&av);
#pragma unroll
              for (int i = 0; i < W; ++i) Vec<T>::fma(ap[i], yv, macc[i]);
            }
          }
        } else {
          for (int t = tid; t < rar * rbr; t += nt) {
            const int c = t / rbr, d = t - c * rbr;
            T acc = T(0);
            for (int j = 0; j < nj; ++j)
              for (int a = 0; a < ral; ++a) acc = fmat(As[j * sa + a * rar + c], Ys[j * sy + a * rbr + d], acc);
            Mn[t] += acc;
          }
        }
        __syncthreads();  // As / Bs [buf] and Ys consumed: the next issue may refill them
        buf ^= 1;
      }
      if (kept) {
        // fixed-order reduction of the nsplit partial tiles (deterministic)
        if (tid < og * nsplit) {
#pragma unroll
          for (int i = 0; i < W; ++i)
#pragma unroll
            for (int q = 0; q < W; ++q) Ps[(tid * W + i) * W + q] = macc[i][q];
        }
        __syncthreads();
        for (int t = tid; t < rar * rbr; t += nt) {
          const int c = t / rbr, d = t - c * rbr;
          const int oo = (c / W) * td + d / W, i = c % W, q = d % W;
          T v = T(0);
          for (int r2 = 0; r2 < nsplit; ++r2) v += Ps[((r2 * og + oo) * W + i) * W + q];
          Mn[t] = v;
        }
      }
      __syncthreads();
      for (int t = tid; t < rar * rbr; t += nt) {
        const int c = t / rbr, d = t - c * rbr;
        M[t] = Mn[t];
        Mt[d * rar + c] = Mn[t];
      }
      __syncthreads();
    }
    if (tid == 0) {
      const T v = M[0];
      out[e] = is_norm ? sqrt_pos(v) : v;
    }
    __syncthreads();
  }
}

bool chunk_ok(const ChainDev& a, const ChainDev& b, int elt) {
  for (int k = 0; k < a.n; ++k) {
    const ModeDev &ma = a.m[k], &mb = b.m[k];
    if (ma.layout != TNB_LAYOUT_DENSE || mb.layout != TNB_LAYOUT_DENSE) return false;
    // 16-byte staging: slice runs, batch strides and chunk starts 16-byte aligned
    if ((reinterpret_cast<uintptr_t>(ma.s) & 15) || (reinterpret_cast<uintptr_t>(mb.s) & 15)) return false;
    if (((ma.bstride * elt) & 15) || ((mb.bstride * elt) & 15)) return false;
    if (ma.J > 1 && (((int64_t)ma.rl * ma.rr * elt) & 15)) return false;
    if (mb.J > 1 && (((int64_t)mb.rl * mb.rr * elt) & 15)) return false;
  }
  return true;
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
  if (elt == 4 && !(gen && gen[0] == '1') && dot_mma_rank(ca, cb))
    return launch_dot_mma(ca, cb, static_cast<float*>(out), is_norm, st);
  const char* chk = getenv("TNB_DOT_CHUNK");
  if (!(chk && chk[0] == '0') && chunk_ok(ca, cb, elt)) {
    int mcap = 1, scap_min = 1;
    for (int k = 0; k < a->n_modes; ++k) {
      const tnb_mode &x = a->modes[k], &y = b->modes[k];
      const int s4[4] = {x.r_left * y.r_left, x.r_right * y.r_right, x.r_left * x.r_right, y.r_left * y.r_right};
      mcap = std::max(mcap, std::max(s4[0], s4[1]));
      scap_min = std::max(scap_min, std::max(std::max(s4[2], s4[3]), x.r_left * y.r_right));
    }
    mcap = (mcap + 3) & ~3;
    // staged operand capacity: ~16 KB of fp32 (8 KB of fp64 values -- 16 KB) per operand, at least one slice
    const int scap = ((std::max(scap_min, 16384 / 4) + 3) & ~3);
    const size_t smem = ((size_t)3 * mcap + 256 * 16 / (elt / 4) + 5 * (size_t)scap) * (size_t)elt;
    if (smem <= 200 * 1024) {
      const int64_t B = ca.batch;
      int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)(227 * 1024) / (smem + 1024)));
      const int64_t slots = (int64_t)num_sms() * per_sm;
      const int grid = (int)(B < slots ? B : slots);
      if (elt == 8) {
        rc = check_cuda(cudaFuncSetAttribute(dot_chunk_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem), "dot smem attr");
        if (rc) return rc;
        dot_chunk_kernel<double><<<grid, 256, smem, st>>>(ca, cb, static_cast<double*>(out), is_norm ? 1 : 0, mcap,
                                                          scap);
      } else {
        rc = check_cuda(cudaFuncSetAttribute(dot_chunk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem), "dot smem attr");
        if (rc) return rc;
        dot_chunk_kernel<float><<<grid, 256, smem, st>>>(ca, cb, static_cast<float*>(out), is_norm ? 1 : 0, mcap,
                                                         scap);
      }
      return check_launch("dot_chunk");
    }
  }
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
