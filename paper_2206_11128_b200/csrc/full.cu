// K2: dense decompression (reference: full, core.py:337-359).
//
// The reference accumulates the chain left to right through 2-D unfoldings,
// m = m @ g.reshape(r_l, J*r_r) (core.py:345-351).  Here the chain is split at
// a rank edge p: a left partial L = G_0..G_{p-1} of shape (prod_{k<p} J_k, r_p)
// and a right partial R = G_p..G_{N-1} of shape (r_p, prod_{k>=p} J_k) are
// built by small step kernels, and ONE GEMM out = L @ R produces the C-order
// output.  That last GEMM is the whole cost: it writes prod(J) floats and is
// bound by HBM write bandwidth when its FLOPs run on tensor cores
// (full_tc.cu); the SIMT GEMM below is the generic path.
// A slab [lo, hi) of the leading mode restricts L's rows, which is the
// reference's own full(t[lo:hi]) (indexing.py:132-137); it is also how the
// multi-GPU runner shards full() across devices.
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace tnb {
// tcgen05 3xTF32 GEMM (full_tc.cu); returns false when the shape is unsupported
bool tc_gemm_supported(int64_t M, int64_t N, int K, int64_t lda, int64_t ldb, int64_t ldc);
int64_t tc_gemm_workspace(int64_t M);
int launch_tc_gemm(const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb,
                   int64_t sB, float* C, int64_t ldc, int64_t sC, int64_t M, int64_t N, int K,
                   int64_t batch, void* ws, cudaStream_t st);

namespace {

struct Step {
  int k;
  int64_t rows;  // left: P rows of the input; right: columns n of the input
};

struct FullPlan {
  int n = 0;
  int p = 0;            // split edge, 1 <= p <= n
  int64_t slab_rows = 0;
  int64_t rowsL = 0;    // rows of L
  int64_t colsR = 0;    // columns of R
  int64_t l_buf = 0;    // floats per batch element per L ping-pong buffer
  int64_t r_buf = 0;    // floats per batch element per R ping-pong buffer
  int64_t out_per = 0;  // floats per batch element of the output slab
  int64_t tc_bytes = 0; // tensor-core GEMM workspace (split L tiles)
};

__device__ __forceinline__ float fmat(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }

int make_plan(const tnb_chain* c, int64_t lo, int64_t hi, FullPlan* P, int elt) {
  if (!c || !c->modes || c->n_modes < 1) return set_error(TNB_EINVAL, "null chain");
  const int n = c->n_modes;
  const tnb_mode* m = c->modes;
  if (lo < 0 || hi < lo || hi > m[0].phys)
    return set_error(TNB_EINVAL, "slab [%lld, %lld) outside leading mode of size %d",
                     (long long)lo, (long long)hi, m[0].phys);
  P->n = n;
  P->slab_rows = hi - lo;
  // out size per batch element
  int64_t out_per = P->slab_rows;
  for (int k = 1; k < n; ++k) out_per *= m[k].phys;
  P->out_per = out_per;
  // choose p by a weighted FMA count (step kernels ~4x less efficient than
  // the final GEMM) with a memory tie-break
  double best = -1;
  for (int p = 1; p <= n; ++p) {
    double cost = 0, mem = 0;
    double rows = (double)P->slab_rows;
    for (int k = 1; k < p; ++k) {
      const double f = (m[k].layout == TNB_LAYOUT_DIAG) ? 1.0 : (double)m[k].r_right;
      const double w = (k == n - 1 && p == n) ? 1.0 : 4.0;  // last step writes out
      cost += w * rows * m[k].phys * m[k].r_left * f;
      rows *= m[k].phys;
      mem += rows * m[k].r_right;
    }
    double cols = 1;
    if (p < n) {
      cols = m[n - 1].phys;
      for (int k = n - 2; k >= p; --k) {
        const double f = (m[k].layout == TNB_LAYOUT_DIAG) ? 1.0 : (double)m[k].r_right;
        cost += 4.0 * cols * m[k].phys * m[k].r_left * f;
        cols *= m[k].phys;
        mem += cols * m[k].r_left;
      }
      cost += rows * cols * m[p].r_left;  // final GEMM
    }
    const double score = cost + 1e-3 * mem;
    if (best < 0 || score < best) {
      best = score;
      P->p = p;
    }
  }
  // TNB_FULL_SPLIT=p pins the split edge (tests reach every step shape with it)
  if (const char* e = getenv("TNB_FULL_SPLIT")) {
    const int pin = atoi(e);
    if (pin >= 1 && pin <= n) P->p = pin;
  }
  // buffer sizes for the chosen p
  const int p = P->p;
  int64_t rows = P->slab_rows, lmax = 0;
  for (int k = 1; k < p; ++k) {
    rows *= m[k].phys;
    const bool writes_out = (p == n && k == n - 1);
    if (!writes_out) lmax = rows * m[k].r_right > lmax ? rows * m[k].r_right : lmax;
  }
  P->rowsL = rows;
  int64_t cols = 1, rmax = 0;
  if (p < n) {
    cols = m[n - 1].phys;
    rmax = cols * m[n - 1].r_left;
    for (int k = n - 2; k >= p; --k) {
      cols *= m[k].phys;
      const int64_t s = cols * m[k].r_left;
      rmax = s > rmax ? s : rmax;
    }
  }
  P->colsR = cols;
  P->l_buf = lmax;
  P->r_buf = rmax;
  P->tc_bytes = 0;
  if (elt == 4 && p < n && tc_gemm_supported(P->rowsL, cols, m[p].r_left, m[p].r_left, cols, cols))
    P->tc_bytes = tc_gemm_workspace(P->rowsL);
  return TNB_OK;
}

// left step: out[e][(p*J + j)*rr + c] = sum_a in[e][p*rl + a] * G_e(j, a, c)
template <typename T>
__global__ void full_left_step(ModeDev md, int64_t B, const T* __restrict__ in, int64_t in_bs,
                               int64_t P, T* __restrict__ out, int64_t out_bs) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int64_t per = P * J * rr;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / per;
    int64_t r = t - e * per;
    const int64_t p = r / ((int64_t)J * rr);
    r -= p * J * rr;
    const int j = (int)(r / rr);
    const int c = (int)(r - (int64_t)j * rr);
    const T* g = reinterpret_cast<const T*>(md.s) + e * md.bstride;
    const T* x = in + e * in_bs + p * rl;
    T acc;
    if (md.layout == TNB_LAYOUT_DIAG) {
      acc = x[c] * __ldg(g + (int64_t)j * rl + c);
    } else {
      acc = 0;
      const T* gj = g + (int64_t)j * rl * rr + c;
      for (int a = 0; a < rl; ++a) acc = fmat(x[a], __ldg(gj + (int64_t)a * rr), acc);
    }
    out[e * out_bs + r + p * J * rr] = acc;
  }
}

// R of the last mode: out[e][a*J + j] = G_e(j, a, 0)
template <typename T>
__global__ void full_right_first(ModeDev md, int64_t B, T* __restrict__ out, int64_t out_bs) {
  const int J = md.J, rl = md.rl;
  const int64_t per = (int64_t)rl * J;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / per;
    const int64_t r = t - e * per;
    const int a = (int)(r / J);
    const int j = (int)(r - (int64_t)a * J);
    out[e * out_bs + r] = __ldg(reinterpret_cast<const T*>(md.s) + e * md.bstride + (int64_t)j * rl + a);
  }
}

// right step: out[e][a][j*n + x] = sum_c G_e(j, a, c) * in[e][c][x]
template <typename T>
__global__ void full_right_step(ModeDev md, int64_t B, const T* __restrict__ in,
                                int64_t in_bs, int64_t n, T* __restrict__ out,
                                int64_t out_bs) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int64_t per = (int64_t)rl * J * n;
  const int64_t total = per * B;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / per;
    int64_t r = t - e * per;
    const int a = (int)(r / ((int64_t)J * n));
    const int64_t rem = r - (int64_t)a * J * n;
    const int j = (int)(rem / n);
    const int64_t x = rem - (int64_t)j * n;
    const T* g = reinterpret_cast<const T*>(md.s) + e * md.bstride;
    const T* y = in + e * in_bs + x;
    T acc;
    if (md.layout == TNB_LAYOUT_DIAG) {
      acc = __ldg(g + (int64_t)j * rl + a) * y[(int64_t)a * n];
    } else {
      acc = 0;
      const T* ga = g + ((int64_t)j * rl + a) * rr;
      for (int c = 0; c < rr; ++c) acc = fmat(__ldg(ga + c), y[(int64_t)c * n], acc);
    }
    out[e * out_bs + r] = acc;
  }
}

// Generic SIMT GEMM C[e] = A[e] (MxK) @ B[e] (KxN), row-major, fp32.
// 128x128 tile, BK=8, 256 threads, 8x8 outputs per thread (two 4x4 quads per
// axis so shared-memory reads and global stores are float4 and coalesced).
constexpr int GBM = 128, GBN = 128, GBK = 8;
#ifndef TNB_FULL_RIGHT_GEMM
#define TNB_FULL_RIGHT_GEMM 1
#endif
template <typename T>
__global__ void __launch_bounds__(256) gemm_kernel(const T* __restrict__ A, int64_t lda,
                                                   int64_t sA, const T* __restrict__ Bm,
                                                   int64_t ldb, int64_t sB,
                                                   T* __restrict__ C, int64_t ldc, int64_t sC,
                                                   int64_t M, int64_t N, int K, int remap_rl,
                                                   int64_t remap_J) {
  __shared__ __align__(16) T As[GBK][GBM];
  __shared__ __align__(16) T Bs[GBK][GBN];
  const int64_t e = blockIdx.z;
  A += e * sA;
  Bm += e * sB;
  C += e * sC;
  // M tiles on grid.x (2^31 - 1 blocks), N tiles on grid.y
  const int64_t m0 = (int64_t)blockIdx.x * GBM, n0 = (int64_t)blockIdx.y * GBN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  T acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += GBK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int l = tid + i * 256;
      const int r = l / GBK, kk = l % GBK;
      const int64_t gm = m0 + r;
      As[kk][r] = (gm < M && k0 + kk < K) ? __ldg(A + gm * lda + k0 + kk) : T(0);
      const int kb = l / GBN, cb = l % GBN;
      const int64_t gn = n0 + cb;
      Bs[kb][cb] = (k0 + kb < K && gn < N) ? __ldg(Bm + (int64_t)(k0 + kb) * ldb + gn) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      T av[8], bv[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[kk][ty * 4 + q];
        av[4 + q] = As[kk][64 + ty * 4 + q];
        bv[q] = Bs[kk][tx * 4 + q];
        bv[4 + q] = Bs[kk][64 + tx * 4 + q];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmat(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const bool vec = (ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (gm >= M) continue;
    // remap_rl > 0: A's rows are (j, a) pairs, C's rows (a, j) (right step)
    const int64_t om = remap_rl > 0 ? (gm % remap_rl) * remap_J + gm / remap_rl : gm;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t gn = n0 + h * 64 + tx * 4;
      T* dst = C + om * ldc + gn;
      if constexpr (std::is_same<T, float>::value) {
        if (vec && gn + 3 < N) {
          __stcs(reinterpret_cast<float4*>(dst),
                 make_float4(acc[i][h * 4], acc[i][h * 4 + 1], acc[i][h * 4 + 2], acc[i][h * 4 + 3]));
          continue;
        }
      }
      {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (gn + q < N) dst[q] = acc[i][h * 4 + q];
      }
    }
  }
}

inline int grid_for(int64_t total) {
  int64_t g = ceil_div(total, 256);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// byte offset of the tensor-core workspace (256-byte aligned)
int64_t tc_offset(const FullPlan& P, int64_t B, int elt) {
  return ((2 * P.l_buf + 2 * P.r_buf) * B * (int64_t)elt + 255) & ~(int64_t)255;
}

ModeDev mode_dev(const tnb_chain* c, int k) {
  const tnb_mode& mm = c->modes[k];
  ModeDev md;
  md.s = mm.slices;
  md.bstride = c->batch > 0 ? mode_floats(mm) : 0;
  md.layout = mm.layout;
  md.J = mm.phys;
  md.rl = mm.r_left;
  md.rr = mm.r_right;
  return md;
}

}  // namespace

// C[e] = A[e] @ B[e] (+ the right-step row remap), chunked so that any M,
// any N and any batch fit the grid limits (x: 2^31 - 1, y / z: 65535).
template <typename T>
int launch_gemm_remap(const T* A, int64_t lda, int64_t sA, const T* B, int64_t ldb, int64_t sB,
                      T* C, int64_t ldc, int64_t sC, int64_t M, int64_t N, int K, int64_t batch,
                      int remap_rl, int64_t remap_J, cudaStream_t st) {
  if (M == 0 || N == 0 || batch == 0) return TNB_OK;
  if (ceil_div(M, GBM) > INT32_MAX) return set_error(TNB_EINVAL, "gemm M too large");
  constexpr int64_t kMaxY = 65535, kMaxZ = 65535;
  for (int64_t e0 = 0; e0 < batch; e0 += kMaxZ) {
    const int64_t nb = batch - e0 < kMaxZ ? batch - e0 : kMaxZ;
    for (int64_t c0 = 0; c0 < N; c0 += kMaxY * GBN) {
      const int64_t nc = N - c0 < kMaxY * GBN ? N - c0 : kMaxY * GBN;
      const dim3 grid((unsigned)ceil_div(M, GBM), (unsigned)ceil_div(nc, GBN), (unsigned)nb);
      gemm_kernel<T><<<grid, 256, 0, st>>>(A + e0 * sA, lda, sA, B + e0 * sB + c0, ldb, sB,
                                           C + e0 * sC + c0, ldc, sC, M, nc, K, remap_rl, remap_J);
      const int rc = check_launch("gemm");
      if (rc) return rc;
    }
  }
  return TNB_OK;
}

template <typename T>
int launch_gemm(const T* A, int64_t lda, int64_t sA, const T* B, int64_t ldb, int64_t sB,
                T* C, int64_t ldc, int64_t sC, int64_t M, int64_t N, int K, int64_t batch,
                cudaStream_t st) {
  return launch_gemm_remap<T>(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, batch, 0, 0, st);
}

// fp32 tiled SIMT GEMM for other translation units (the entries table
// builder's rank > 32 levels)
int gemm_f32(const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb, int64_t sB, float* C,
             int64_t ldc, int64_t sC, int64_t M, int64_t N, int K, int64_t batch, cudaStream_t st) {
  return launch_gemm<float>(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, batch, st);
}

int64_t full_workspace(const tnb_chain* c, int64_t lo, int64_t hi, int elt) {
  FullPlan P;
  if (make_plan(c, lo, hi, &P, elt)) return -1;
  const int64_t B = c->batch > 0 ? c->batch : 1;
  return tc_offset(P, B, elt) + P.tc_bytes;
}

template <typename T>
int full_t(const tnb_chain* c, int64_t lo, int64_t hi, T* out, void* ws, int64_t ws_bytes, cudaStream_t st) {
  constexpr int elt = (int)sizeof(T);
  FullPlan P;
  int rc = make_plan(c, lo, hi, &P, elt);
  if (rc) return rc;
  ChainDev tmp;
  rc = make_chain_dev(c, &tmp, false);  // validates ranks
  if (rc) return rc;
  const int64_t B = c->batch > 0 ? c->batch : 1;
  if (P.out_per == 0) return TNB_OK;
  if (!out) return set_error(TNB_EINVAL, "null output");
  const int64_t need = tc_offset(P, B, elt) + P.tc_bytes;
  if (need > 0 && (!ws || ws_bytes < need))
    return set_error(TNB_EWORKSPACE, "full needs %lld workspace bytes, got %lld",
                     (long long)need, (long long)ws_bytes);
  T* lb[2] = {(T*)ws, (T*)ws + P.l_buf * B};
  T* rb[2] = {(T*)ws + 2 * P.l_buf * B, (T*)ws + 2 * P.l_buf * B + P.r_buf * B};
  const int n = P.n, p = P.p;

  // ---- left partial: L0 is a view of mode 0's slices (rows lo..hi) ----
  const ModeDev m0 = mode_dev(c, 0);
  const T* L = reinterpret_cast<const T*>(m0.s) + lo * (int64_t)m0.rl * m0.rr;  // dense, rl == 1
  int64_t L_bs = m0.bstride;
  int64_t rows = P.slab_rows;
  if (n == 1) {
    // out[e][j] = G_e(lo + j, 0, 0)
    for (int64_t e = 0; e < B; ++e) {
      rc = check_cuda(cudaMemcpyAsync(out + e * P.out_per, L + e * L_bs,
                                      P.out_per * sizeof(T), cudaMemcpyDeviceToDevice, st),
                      "copy");
      if (rc) return rc;
    }
    return TNB_OK;
  }
  for (int k = 1; k < p; ++k) {
    const ModeDev md = mode_dev(c, k);
    const bool writes_out = (p == n && k == n - 1);
    T* dst = writes_out ? out : lb[k & 1];
    const int64_t dst_bs = writes_out ? P.out_per : P.l_buf;
    const int64_t total = rows * md.J * md.rr * B;
    if (total > 0)
      full_left_step<T><<<grid_for(total), 256, 0, st>>>(md, B, L, L_bs, rows, dst, dst_bs);
    rc = check_launch("full_left_step");
    if (rc) return rc;
    L = dst;
    L_bs = dst_bs;
    rows *= md.J;
  }
  if (p == n) return TNB_OK;

  // ---- right partial ----
  const ModeDev ml = mode_dev(c, n - 1);
  T* R = rb[0];
  int64_t cols = ml.J;
  {
    const int64_t total = (int64_t)ml.rl * ml.J * B;
    if (total > 0) full_right_first<T><<<grid_for(total), 256, 0, st>>>(ml, B, R, P.r_buf);
    rc = check_launch("full_right_first");
    if (rc) return rc;
  }
  int which = 0;
  for (int k = n - 2; k >= p; --k) {
    const ModeDev md = mode_dev(c, k);
    T* dst = rb[which ^ 1];
    const int64_t total = (int64_t)md.rl * md.J * cols * B;
    const int64_t gm_rows = (int64_t)md.J * md.rl;
    if (TNB_FULL_RIGHT_GEMM && total > 0 && md.layout == TNB_LAYOUT_DENSE && md.rr >= 8 && cols >= 64) {
      // dense right step as a GEMM over the (j, a) rows of the core: the same
      // sequential sum over c per output, rows stored in (a, j) order
      rc = launch_gemm_remap<T>(reinterpret_cast<const T*>(md.s), md.rr, md.bstride, R, cols, P.r_buf, dst,
                                cols, P.r_buf, gm_rows, cols, md.rr, B, md.rl, md.J, st);
      if (rc) return rc;
    } else if (total > 0)
      full_right_step<T><<<grid_for(total), 256, 0, st>>>(md, B, R, P.r_buf, cols, dst, P.r_buf);
    rc = check_launch("full_right_step");
    if (rc) return rc;
    R = dst;
    which ^= 1;
    cols *= md.J;
  }
  // ---- out = L @ R ----
  KTimer kt("full_gemm", st);
  const int K = c->modes[p].r_left;
  if (K == 0) return check_cuda(cudaMemsetAsync(out, 0, P.out_per * B * sizeof(T), st), "memset");
  if constexpr (std::is_same<T, float>::value) {
    if (P.tc_bytes > 0) {
      void* tcw = (unsigned char*)ws + tc_offset(P, B, elt);
      return launch_tc_gemm(L, K, L_bs, R, cols, P.r_buf, out, cols, P.out_per, rows, cols, K, B, tcw, st);
    }
  }
  return launch_gemm<T>(L, K, L_bs, R, cols, P.r_buf, out, cols, P.out_per, rows, cols, K, B, st);
}

int launch_full(const tnb_chain* c, int64_t lo, int64_t hi, void* out, void* ws, int64_t ws_bytes,
                cudaStream_t st, int elt) {
  if (elt == 8) return full_t<double>(c, lo, hi, static_cast<double*>(out), ws, ws_bytes, st);
  return full_t<float>(c, lo, hi, static_cast<float*>(out), ws, ws_bytes, st);
}

}  // namespace tnb
