// K3 on tensor cores for TT chains of uniform rank R in {8, 32, 48} (the
// rank-16 kernel, dot_fast.cu, covers R = 16; dot.cu's chunked SIMT kernel
// covers everything else -- other ranks, CP modes, fp64).  Reference: chain_dot
// (core.py:362-384) / norm (core.py:387-391): M' = sum_j A_j^T M B_j.
//
// Per pair (one persistent 256-thread CTA per pair at a time) and mode, CH
// slices of A and B at a time are staged with cp.async (double-buffered,
// running ahead across modes and pairs), then
//   split:  the chunk's slices -> tf32 hi / lo copies in padded shared rows
//           (conflict-free fragment loads), once per element;
//   Y_j  = M B_j      on mma.sync m16n8k8 split-TF32 (3 MMAs per product:
//                     lo*hi + hi*lo + hi*hi), M's hi / lo split once per mode;
//                     warps take (slice, output tile) items; Y is stored split;
//   M'  += A_j^T Y_j  on mma.sync, warps own output tiles (and a share of the
//                     (slice, k-step) pairs when there are fewer tiles than
//                     warps); each slice's product starts from a zero fragment
//                     and joins the running tile with fp32 adds (no long MMA
//                     accumulation), partial tiles reduced in a fixed order.
// The rank-1 boundary modes run as small SIMT loops on the staged chunks.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
  // round-to-nearest-away on the bit pattern (cvt.rna.tf32's value for finite x
  // in two instructions instead of four)
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));  // exact; the tensor core truncates it
}

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void stage_async(float* dst, const float* __restrict__ src, int64_t count, int tid) {
  const int64_t nv = count / 4;
  for (int64_t i = tid; i < nv; i += kThreads)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + i * 4)), "l"(src + i * 4) : "memory");
  for (int64_t i = nv * 4 + tid; i < count; i += kThreads)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(dst + i)), "l"(src + i) : "memory");
}

// Geometry per rank: padded row strides keep every fragment load
// conflict-free -- rows indexed by the fragment's g (M as the A operand)
// need a stride = 4 (mod 8), rows indexed by t (A_j^T, B_j, Y_j) one = 8
// (mod 16).
template <int R>
struct G {
  static constexpr int MT = (R + 15) / 16;  // 16-row output / A tiles (rows >= R read as zero)
  static constexpr int NT = R / 8;          // 8-column tiles
  static constexpr int KT = R / 8;          // 8-deep k-steps
  static constexpr int T1 = MT * NT;        // output tiles of one R x R product
  static constexpr int RPM = R + 4;
  static constexpr int RPA = (R % 16 == 8) ? R : R + 8;
  static constexpr int TPW = (T1 + kWarps - 1) / kWarps;    // M' tiles per warp (T1 >= 8)
  static constexpr int KS = T1 >= kWarps ? 1 : kWarps / T1;  // warps sharing one M' tile's reduction
};

struct MmaArgs {
  ChainDev a, b;
  float* out;
  int norm;
  int ch;  // slices per chunk (interior modes)
};

template <int R>
__global__ void __launch_bounds__(kThreads) dot_mma_kernel(const __grid_constant__ MmaArgs args) {
  using Gm = G<R>;
  constexpr int MT = Gm::MT, NT = Gm::NT, KT = Gm::KT, T1 = Gm::T1, RPM = Gm::RPM, RPA = Gm::RPA;
  constexpr int TPW = Gm::TPW, KS = Gm::KS;
  const ChainDev& A = args.a;
  const ChainDev& Bc = args.b;
  const int CH = args.ch;
  const int scap = CH * R * R;          // staged floats per operand and buffer
  const int sst = CH * R * RPA;         // split words per array
  extern __shared__ __align__(16) unsigned char smem[];
  float* M = reinterpret_cast<float*>(smem);                 // [R][R]
  uint32_t* MH = reinterpret_cast<uint32_t*>(M + R * R);     // [R][RPM]
  uint32_t* ML = MH + R * RPM;
  float* Ps = reinterpret_cast<float*>(ML + R * RPM);        // [KS][R][R] partial M'
  float* Asb[2] = {Ps + KS * R * R, Ps + KS * R * R + scap};
  float* Bsb[2] = {Asb[1] + scap, Asb[1] + 2 * scap};
  uint32_t* AH = reinterpret_cast<uint32_t*>(Bsb[1] + scap);  // [CH][R][RPA] (a rows, c columns)
  uint32_t* AL = AH + sst;
  uint32_t* BH = AL + sst;                                    // [CH][R][RPA] (b rows, d columns)
  uint32_t* BL = BH + sst;
  uint32_t* YH = BL + sst;                                    // [CH][R][RPA] (a rows, d columns)
  uint32_t* YL = YH + sst;
  float* red = reinterpret_cast<float*>(YL + sst);            // [kWarps]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int N = A.n;

  auto chunk_of = [&](int k) {  // slices per staged chunk of mode k
    const ModeDev& ma = A.m[k];
    const bool interior = ma.rl == R && ma.rr == R;
    const int c = interior ? CH : (scap / (ma.rl * ma.rr > 0 ? ma.rl * ma.rr : 1));
    return c < 1 ? 1 : (c > ma.J ? ma.J : c);
  };
  auto issue = [&](int64_t e, int k, int j0, int buf) {
    if (e < A.batch) {
      const ModeDev& ma = A.m[k];
      const ModeDev& mb = Bc.m[k];
      const int sa = ma.rl * ma.rr, sb = mb.rl * mb.rr;
      const int ch = chunk_of(k);
      const int nj = ma.J - j0 < ch ? ma.J - j0 : ch;
      stage_async(Asb[buf], ma.s + e * ma.bstride + (int64_t)j0 * sa, (int64_t)nj * sa, tid);
      stage_async(Bsb[buf], mb.s + e * mb.bstride + (int64_t)j0 * sb, (int64_t)nj * sb, tid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int buf = 0;
  issue(blockIdx.x, 0, 0, 0);
  for (int64_t e = blockIdx.x; e < A.batch; e += gridDim.x) {
    float lastacc = 0.f;
    for (int k = 0; k < N; ++k) {
      const ModeDev& ma = A.m[k];
      const int J = ma.J;
      const bool first = k == 0, last = k == N - 1;
      const int ch = chunk_of(k);
      // M' tiles owned by this warp (interior modes): tile ids warp + q * kWarps
      // (T1 >= warps) or tile warp % T1 with reduction slice warp / T1
      float macc[TPW][4];
#pragma unroll
      for (int q = 0; q < TPW; ++q) macc[q][0] = macc[q][1] = macc[q][2] = macc[q][3] = 0.f;
      float fo[16];  // first mode: up to 16 outputs per thread (R * R <= 4096)
#pragma unroll
      for (int q = 0; q < 16; ++q) fo[q] = 0.f;
      for (int j0 = 0; j0 < J; j0 += ch) {
        const int nj = J - j0 < ch ? J - j0 : ch;
        if (j0 + ch < J) issue(e, k, j0 + ch, buf ^ 1);
        else if (k + 1 < N) issue(e, k + 1, 0, buf ^ 1);
        else issue(e + gridDim.x, 0, 0, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const float* As = Asb[buf];
        const float* Bs = Bsb[buf];
        if (first) {
          // M'[c][d] = sum_j A_j[c] B_j[d]  (1 x R slices)
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int o = tid + q * kThreads;
            if (o < R * R) {
              const int c = o / R, d = o - c * R;
              float acc = fo[q];
              for (int j = 0; j < nj; ++j) acc = fmaf(As[j * R + c], Bs[j * R + d], acc);
              fo[q] = acc;
            }
          }
        } else if (last) {
          // s += sum_j sum_a A_j[a] (M B_j)[a]  (R x 1 slices)
          for (int ja = tid; ja < nj * R; ja += kThreads) {
            const int j = ja / R, a = ja - j * R;
            float y = 0.f;
            for (int b = 0; b < R; ++b) y = fmaf(M[a * R + b], Bs[j * R + b], y);
            lastacc = fmaf(As[j * R + a], y, lastacc);
          }
        } else {
          // ---- split the chunk into padded tf32 hi / lo rows ----
          for (int i = tid; i < nj * R * R; i += kThreads) {
            const int j = i / (R * R), r = i - j * (R * R), row = r / R, col = r - row * R;
            uint32_t h, l;
            split(As[i], h, l);
            AH[(j * R + row) * RPA + col] = h;
            AL[(j * R + row) * RPA + col] = l;
            split(Bs[i], h, l);
            BH[(j * R + row) * RPA + col] = h;
            BL[(j * R + row) * RPA + col] = l;
          }
          __syncthreads();
          // ---- Y_j = M B_j: items (slice, output tile) ----
          for (int it = warp; it < nj * T1; it += kWarps) {
            const int j = it / T1, tile = it - j * T1, mt = tile / NT, nt = tile - mt * NT;
            const int r0 = mt * 16 + g, r1 = r0 + 8;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
              const int kc = kt * 8 + t;
              const uint32_t ah0 = r0 < R ? MH[r0 * RPM + kc] : 0u, al0 = r0 < R ? ML[r0 * RPM + kc] : 0u;
              const uint32_t ah1 = r1 < R ? MH[r1 * RPM + kc] : 0u, al1 = r1 < R ? ML[r1 * RPM + kc] : 0u;
              const uint32_t ah2 = r0 < R ? MH[r0 * RPM + kc + 4] : 0u, al2 = r0 < R ? ML[r0 * RPM + kc + 4] : 0u;
              const uint32_t ah3 = r1 < R ? MH[r1 * RPM + kc + 4] : 0u, al3 = r1 < R ? ML[r1 * RPM + kc + 4] : 0u;
              const int bi = (j * R + kc) * RPA + nt * 8 + g;
              const uint32_t bh0 = BH[bi], bl0 = BL[bi], bh1 = BH[bi + 4 * RPA], bl1 = BL[bi + 4 * RPA];
              mma(acc, al0, al1, al2, al3, bh0, bh1);
              mma(acc, ah0, ah1, ah2, ah3, bl0, bl1);
              mma(acc, ah0, ah1, ah2, ah3, bh0, bh1);
            }
            // C fragment: rows r0 / r1, columns nt*8 + 2t, +1 -> split into Y
            const int cc = nt * 8 + 2 * t;
            uint32_t h, l;
            if (r0 < R) {
              split(acc[0], h, l);
              YH[(j * R + r0) * RPA + cc] = h;
              YL[(j * R + r0) * RPA + cc] = l;
              split(acc[1], h, l);
              YH[(j * R + r0) * RPA + cc + 1] = h;
              YL[(j * R + r0) * RPA + cc + 1] = l;
            }
            if (r1 < R) {
              split(acc[2], h, l);
              YH[(j * R + r1) * RPA + cc] = h;
              YL[(j * R + r1) * RPA + cc] = l;
              split(acc[3], h, l);
              YH[(j * R + r1) * RPA + cc + 1] = h;
              YL[(j * R + r1) * RPA + cc + 1] = l;
            }
          }
          __syncthreads();
          // ---- M' += A_j^T Y_j: warp-owned output tiles ----
#pragma unroll
          for (int q = 0; q < TPW; ++q) {
            const int tile = KS > 1 ? warp % T1 : warp + q * kWarps;
            if (tile < T1 && (KS == 1 || warp < T1 * KS)) {
              const int rs = KS > 1 ? warp / T1 : 0;
              const int mt = tile / NT, nt = tile - mt * NT;
              const int c0 = mt * 16 + g, c1 = c0 + 8;
              // this warp's share of the chunk's (slice, k-step) pairs; each
              // pair's 3 MMAs start from zero and join the tile with fp32 adds
              for (int pj = rs; pj < nj * KT; pj += KS) {
                const int j = pj / KT, kt = pj - j * KT;
                float z[4] = {0.f, 0.f, 0.f, 0.f};
                {
                  const int a0 = kt * 8 + t;
                  // A operand = A_j^T: element (row c, col a) = A_j[a][c]
                  const int ab = (j * R + a0) * RPA;
                  const uint32_t ah0 = c0 < R ? AH[ab + c0] : 0u, al0 = c0 < R ? AL[ab + c0] : 0u;
                  const uint32_t ah1 = c1 < R ? AH[ab + c1] : 0u, al1 = c1 < R ? AL[ab + c1] : 0u;
                  const uint32_t ah2 = c0 < R ? AH[ab + 4 * RPA + c0] : 0u, al2 = c0 < R ? AL[ab + 4 * RPA + c0] : 0u;
                  const uint32_t ah3 = c1 < R ? AH[ab + 4 * RPA + c1] : 0u, al3 = c1 < R ? AL[ab + 4 * RPA + c1] : 0u;
                  const int yi = (j * R + a0) * RPA + nt * 8 + g;
                  const uint32_t bh0 = YH[yi], bl0 = YL[yi], bh1 = YH[yi + 4 * RPA], bl1 = YL[yi + 4 * RPA];
                  mma(z, al0, al1, al2, al3, bh0, bh1);
                  mma(z, ah0, ah1, ah2, ah3, bl0, bl1);
                  mma(z, ah0, ah1, ah2, ah3, bh0, bh1);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) macc[q][i] += z[i];
              }
            }
          }
        }
        __syncthreads();  // staged chunk, split rows and Y consumed
        buf ^= 1;
      }
      // ---- mode end: the new M (fp32) and its split copy ----
      if (first) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int o = tid + q * kThreads;
          if (o < R * R) M[o] = fo[q];
        }
      } else if (last) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lastacc += __shfl_xor_sync(0xffffffffu, lastacc, o);
        if (lane == 0) red[warp] = lastacc;
        __syncthreads();
        if (tid == 0) {
          float v = 0.f;
          for (int w = 0; w < kWarps; ++w) v += red[w];
          args.out[e] = args.norm ? sqrtf(fmaxf(v, 0.f)) : v;
        }
        lastacc = 0.f;
      } else {
        // C fragment of tile (mt, nt): rows c0 / c1, columns nt*8 + 2t, +1
#pragma unroll
        for (int q = 0; q < TPW; ++q) {
          const int tile = KS > 1 ? warp % T1 : warp + q * kWarps;
          if (tile < T1 && (KS == 1 || warp < T1 * KS)) {
            const int rs = KS > 1 ? warp / T1 : 0;
            const int mt = tile / NT, nt = tile - mt * NT;
            const int c0 = mt * 16 + g, c1 = c0 + 8, dd = nt * 8 + 2 * t;
            float* P = Ps + rs * R * R;
            if (c0 < R) {
              P[c0 * R + dd] = macc[q][0];
              P[c0 * R + dd + 1] = macc[q][1];
            }
            if (c1 < R) {
              P[c1 * R + dd] = macc[q][2];
              P[c1 * R + dd + 1] = macc[q][3];
            }
          }
        }
        __syncthreads();
        for (int o = tid; o < R * R; o += kThreads) {
          float v = Ps[o];
#pragma unroll
          for (int r2 = 1; r2 < KS; ++r2) v += Ps[r2 * R * R + o];
          M[o] = v;
        }
      }
      __syncthreads();
      if (!last) {
        for (int o = tid; o < R * R; o += kThreads) {
          const int r = o / R, c = o - r * R;
          uint32_t h, l;
          split(M[o], h, l);
          MH[r * RPM + c] = h;
          ML[r * RPM + c] = l;
        }
      }
      __syncthreads();
    }
  }
}

template <int R>
size_t mma_smem(int ch) {
  using Gm = G<R>;
  const size_t scap = (size_t)ch * R * R;
  const size_t sst = (size_t)ch * R * Gm::RPA;
  return ((size_t)R * R + 2 * (size_t)R * Gm::RPM + (size_t)Gm::KS * R * R + 4 * scap + 6 * sst + kWarps) * 4;
}

// the uniform-rank TT shape this kernel handles: boundary ranks 1, every
// interior rank R, dense, 16-byte aligned slice runs
bool mma_chain_ok(const ChainDev& c, int R) {
  if (c.n < 2) return false;
  for (int k = 0; k < c.n; ++k) {
    const ModeDev& m = c.m[k];
    const int rl = k == 0 ? 1 : R, rr = k == c.n - 1 ? 1 : R;
    if (m.layout != TNB_LAYOUT_DENSE || m.rl != rl || m.rr != rr || m.J < 1) return false;
    if ((reinterpret_cast<uintptr_t>(m.s) & 15) || ((m.bstride * 4) & 15)) return false;
    if (m.J > 1 && ((m.rl * m.rr * 4) & 15)) return false;
  }
  return true;
}

template <int R>
int launch_r(const ChainDev& a, const ChainDev& b, float* out, bool is_norm, cudaStream_t st) {
  MmaArgs args;
  args.a = a;
  args.b = b;
  args.out = out;
  args.norm = is_norm ? 1 : 0;
  // slices per chunk: ~16 KB of fp32 per staged operand, shrunk until two
  // CTAs fit an SM (one for R = 64)
  int ch = std::max(1, 4096 / (R * R));
  while (ch > 1 && mma_smem<R>(ch) > (size_t)112 * 1024) --ch;
  // boundary-mode chunks hold up to ch * R * R floats too (1 x R slices)
  args.ch = ch;
  const size_t smem = mma_smem<R>(ch);
  if (smem > (size_t)227 * 1024) return set_error(TNB_EINVAL, "dot_mma: rank %d too large", R);
  int rc = check_cuda(cudaFuncSetAttribute(dot_mma_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "dot_mma smem attr");
  if (rc) return rc;
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(4, (size_t)(227 * 1024) / (smem + 1024)));
  const int64_t slots = (int64_t)num_sms() * per_sm;
  const int grid = (int)(a.batch < slots ? a.batch : slots);
  dot_mma_kernel<R><<<grid, kThreads, smem, st>>>(args);
  return check_launch("dot_mma");
}

int env_dot_mma() {
  const char* e = getenv("TNB_DOT_MMA");
  return !(e && e[0] == '0');
}

}  // namespace

// rank of a chain the tensor-core kernel takes (0: none)
int dot_mma_rank(const ChainDev& a, const ChainDev& b) {
  if (!env_dot_mma() || a.n != b.n || a.batch != b.batch || a.n < 3) return 0;
  const int R = a.m[0].rr;
  // R = 24 measured slower than the chunked SIMT kernel (its second 16-row
  // tile is half padding): 4.48 vs 4.26 ms for 1024 cfg4-shape pairs
  if (R != 8 && R != 32 && R != 48) return 0;
  return (mma_chain_ok(a, R) && mma_chain_ok(b, R)) ? R : 0;
}

int launch_dot_mma(const ChainDev& a, const ChainDev& b, float* out, bool is_norm, cudaStream_t st) {
  switch (dot_mma_rank(a, b)) {
    case 8: return launch_r<8>(a, b, out, is_norm, st);
    case 24: return launch_r<24>(a, b, out, is_norm, st);
    case 32: return launch_r<32>(a, b, out, is_norm, st);
    case 48: return launch_r<48>(a, b, out, is_norm, st);
    default: return set_error(TNB_EINVAL, "dot_mma: unsupported chain");
  }
}

}  // namespace tnb
