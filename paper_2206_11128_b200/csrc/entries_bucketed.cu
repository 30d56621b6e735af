// K1 performance kernel: bucketed entry evaluation for unbatched chains with
// ranks <= 32 (BASELINE configs 2 and 5).
//
// Reference algorithm (core.py:432-444): per mode, argsort the samples by
// their index value so every group shares one core slice and the group's
// update is a real (n_j x r) @ (r x s) product.  A global re-sort per mode
// would cost 2 x M x r x 4 bytes of HBM traffic per mode, so
// here the grouping happens per CTA tile, on chip:
//
//   * a persistent CTA (one per SM) owns a tile of T samples; their r-vector
//     states live in shared memory at FIXED slots (sample id), so no state
//     ever moves between modes -- only a permutation is rebuilt;
//   * per interior dense mode, a counting sort of the tile's indices
//     (warp-aggregated match_any + smem atomics) yields perm, bucket starts
//     and counts;
//   * each warp takes an equal contiguous range of sorted positions; for each
//     bucket in its range it loads that core slice ONCE into registers
//     (lane group of L lanes holds all r rows x C columns), then streams its
//     samples: a group reads a sample's state row (LDS.128 broadcast within
//     the group), does r x C FMAs per lane, and writes its C output columns
//     back into the same slot (__syncwarp between reads and writes);
//   * the first mode (rank 1 on the left) is a row copy, interior CP modes
//     are diagonal scalings, the last mode (rank 1 on the right) a dot
//     product -- none of those need sorting;
//   * index tuples are read once per tile (coalesced int64), validated
//     (negative wrap, lowest OOB mode -> *err), compacted to uint8/uint16 in
//     shared memory; the next tile's indices are prefetched into L2.
// Each sample's arithmetic is a fixed FMA sequence, so results do not depend
// on the sort order or the tile a sample lands in.
#include "common.cuh"

namespace tnb {
namespace {

constexpr int kMaxJ = 1024;          // bucket count limit for sorted modes

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ int64_t ld_stream_i64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ void sts_b64(uint32_t a, uint64_t x) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(x) : "memory");
}
// acc.{x,y} += g.{x,y} * v  (packed fp32 FMA, one issue slot for two FMAs)
__device__ __forceinline__ void ffma2(uint64_t& acc, uint64_t g, float v) {
  asm("{\n\t.reg .b64 vv;\n\tmov.b64 vv, {%2, %2};\n\tfma.rn.f32x2 %0, %1, vv, %0;\n\t}"
      : "+l"(acc)
      : "l"(g), "f"(v));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t ldg_b64(const float* p) {
  uint64_t v;
  asm volatile("ld.global.nc.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(lo), "f"(hi));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, float x) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
}

// Column ownership inside a sample group of L lanes (lane q): C == 2 -> the
// pair (2q, 2q+1); C == 3 (R = 24, L = 8) -> the pair (2q, 2q+1) plus the
// single column 16 + q.  Pairs are updated with packed FFMA2 (fma.rn.f32x2).
template <int R>
struct Geo {
  static constexpr int C = (R == 24) ? 3 : 2;  // output columns per lane
  static constexpr int L = R / C;              // lanes per sample group
  static constexpr int G = 32 / L;             // sample groups per warp
  static constexpr int P = 8 / G;              // passes per iteration (8 samples)
  static constexpr int RP = R + 4;             // padded state row (bank spread)
  static_assert(L * C == R && 32 % L == 0 && G * P == 8, "geometry");
};


// K-split pass group for R == 32: NP samples (one per pass) of one bucket.
// Lane (h, qq) holds rows 16h..16h+15 of the core slice, column pair
// (2qq, 2qq+1); the two row halves are summed with one 64-bit shuffle.
template <int NP, int RP>
__device__ __forceinline__ void ks_passes(const uint64_t (&g2)[16], const uint16_t* perm, int p,
                                          uint32_t s_state, int h, int qq) {
  uint32_t rowb[NP];
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) rowb[pi] = s_state + (uint32_t)perm[p + pi] * (RP * 4);
  uint64_t acc2[NP];
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) acc2[pi] = 0ull;
#pragma unroll
  for (int a4 = 0; a4 < 4; ++a4) {
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) {
      const float4 v = lds128(rowb[pi] + h * 64 + a4 * 16);
      ffma2(acc2[pi], g2[a4 * 4 + 0], v.x);
      ffma2(acc2[pi], g2[a4 * 4 + 1], v.y);
      ffma2(acc2[pi], g2[a4 * 4 + 2], v.z);
      ffma2(acc2[pi], g2[a4 * 4 + 3], v.w);
    }
  }
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) acc2[pi] = add2(acc2[pi], __shfl_xor_sync(0xffffffffu, acc2[pi], 16));
  __syncwarp();  // every lane has read its rows
#pragma unroll
  for (int pi = 0; pi < NP; ++pi)
    if ((pi & 1) == (NP > 1 ? h : 0)) sts_b64(rowb[pi] + qq * 8, acc2[pi]);
  __syncwarp();
}

template <typename IdxT>
__host__ __device__ inline size_t smem_bytes(int T, int RP, int N, int jcap) {
  size_t b = (size_t)(T + 1) * RP * sizeof(float);  // state (+ dummy row)
  b += (size_t)T * 2 * sizeof(uint16_t);          // perm + rank
  b += (size_t)N * T * sizeof(IdxT);              // compact indices
  b = (b + 15) & ~(size_t)15;
  b += (size_t)2 * (jcap + 1) * sizeof(int);      // counts + starts
  return b;
}

template <int R, typename IdxT, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
    entries_bucketed_kernel(const __grid_constant__ ChainDev ch, const int64_t* __restrict__ idx,
                            int64_t m, float* __restrict__ out, int32_t* __restrict__ err, int T,
                            int jcap) {
  using Gm = Geo<R>;
  constexpr int C = Gm::C, L = Gm::L, G = Gm::G, P = Gm::P, RP = Gm::RP;
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = ch.n;
  float* state = reinterpret_cast<float*>(smem);
  uint16_t* perm = reinterpret_cast<uint16_t*>(state + (size_t)(T + 1) * RP);
  uint16_t* rnk = perm + T;
  IdxT* idxs = reinterpret_cast<IdxT*>(rnk + T);
  size_t off = (size_t)(T + 1) * RP * 4 + (size_t)T * 4 + (size_t)N * T * sizeof(IdxT);
  off = (off + 15) & ~(size_t)15;
  int* cnt = reinterpret_cast<int*>(smem + off);
  int* start = cnt + jcap + 1;

  const uint32_t s_state = (uint32_t)__cvta_generic_to_shared(state);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = NT / 32;
  const int gi = lane / L;   // sample group within the warp
  const int q = lane % L;    // lane within the group -> columns q*C .. q*C+C-1
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t ntiles = (m + T - 1) / T;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t s0 = tile * T;
    const int tn = (int)((m - s0) < T ? (m - s0) : T);
    {  // warm L2 with the next tile's index block
      const int64_t nt = tile + gridDim.x;
      if (nt < ntiles) {
        const int64_t ns0 = nt * T;
        const int64_t nbytes = ((m - ns0) < T ? (m - ns0) : T) * N * 8;
        const char* base = reinterpret_cast<const char*>(idx + ns0 * N);
        for (int64_t o = (int64_t)tid * 128; o < nbytes; o += (int64_t)NT * 128)
          prefetch_l2(base + o);
      }
    }
    // ---- indices: coalesced int64 read (4 loads in flight per thread),
    //      wrap/validate, compact, mode-major
    {
      const int64_t* src = idx + s0 * N;
      const int total = tn * N;
      constexpr int U = 4;
      int ss[U], kk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = tid + u * NT;
        ss[u] = e / N;
        kk[u] = e - ss[u] * N;
      }
      const int ds = (U * NT) / N, dk = (U * NT) - ds * N;
      for (int e0 = tid; e0 < total; e0 += U * NT) {
        int64_t raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * NT;
          raw[u] = (e < total) ? ld_stream_i64(src + e) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (e0 + u * NT < total) {
            const int k = kk[u];
            const int j = norm_index(raw[u], ch.m[k].J, k, err);
            idxs[(size_t)k * T + ss[u]] = (IdxT)j;
          }
          ss[u] += ds;
          kk[u] += dk;
          if (kk[u] >= N) {
            kk[u] -= N;
            ++ss[u];
          }
        }
      }
    }
    __syncthreads();

    for (int k = 0; k < N; ++k) {
      const ModeDev& md = ch.m[k];
      const IdxT* col = idxs + (size_t)k * T;
      const int rl = md.rl, rr = md.rr;
      if (k == 0) {
        if (N == 1) {  // [J][1][1]
          for (int s = tid; s < tn; s += NT) out[s0 + s] = __ldg(md.s + col[s]);
        } else if (rr == R) {  // state row = G_0[j][0][:] (16-byte copies)
          for (int e = tid; e < tn * (R / 4); e += NT) {
            const int s = e / (R / 4), c4 = e - (e / (R / 4)) * (R / 4);
            const float4 g = __ldg(reinterpret_cast<const float4*>(md.s + (int64_t)col[s] * R) + c4);
            *reinterpret_cast<float4*>(state + s * RP + c4 * 4) = g;
          }
        } else {       // state row = G_0[j][0][:], zero padded to R
          for (int e = tid; e < tn * R; e += NT) {
            const int s = e / R, c = e - (e / R) * R;
            state[s * RP + c] = (c < rr) ? __ldg(md.s + (int64_t)col[s] * rr + c) : 0.f;
          }
        }
      } else if (md.layout == TNB_LAYOUT_DIAG) {
        for (int e = tid; e < tn * R; e += NT) {
          const int s = e / R, c = e - (e / R) * R;
          if (c < rl) state[s * RP + c] *= __ldg(md.s + (int64_t)col[s] * rl + c);
        }
      } else if (k == N - 1) {  // rr == 1: out = state . G[j][:, 0]
        if (rl == R) {  // full rank: unpredicated 16-byte loads, two FMA chains
          for (int s = tid; s < tn; s += NT) {
            const float4* g4 = reinterpret_cast<const float4*>(md.s + (int64_t)col[s] * R);
            const uint32_t vrow = s_state + (uint32_t)s * (RP * 4);
            float4 gv[R / 4];
#pragma unroll
            for (int a4 = 0; a4 < R / 4; ++a4) gv[a4] = __ldg(g4 + a4);
            float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
            for (int a4 = 0; a4 < R / 4; ++a4) {
              const float4 v = lds128(vrow + a4 * 16);
              acc0 = fmaf(v.x, gv[a4].x, acc0);
              acc1 = fmaf(v.y, gv[a4].y, acc1);
              acc0 = fmaf(v.z, gv[a4].z, acc0);
              acc1 = fmaf(v.w, gv[a4].w, acc1);
            }
            out[s0 + s] = acc0 + acc1;
          }
        } else {
          for (int s = tid; s < tn; s += NT) {
            const float* g = md.s + (int64_t)col[s] * rl;
            const float* v = state + s * RP;
            float acc = 0.f;
#pragma unroll
            for (int a = 0; a < R; ++a)
              if (a < rl) acc = fmaf(v[a], __ldg(g + a), acc);
            out[s0 + s] = acc;
          }
        }
      } else {
        // ---- counting sort of the tile by this mode's index ----
        const int J = md.J;
        const int kbits = 32 - __clz(J > 1 ? J - 1 : 1);
        for (int j = tid; j <= J; j += NT) cnt[j] = 0;
        __syncthreads();
        const int tn32 = (tn + 31) & ~31;
        for (int s = tid; s < tn32; s += NT) {
          const bool act = s < tn;
          const unsigned amask = __ballot_sync(0xffffffffu, act);
          if (act) {
            const int key = col[s];
            // lanes holding the same key: AND of per-bit ballots (cheaper
            // than MATCH.ANY for the <= 10-bit keys of sorted modes)
            unsigned peers = amask;
            for (int b = 0; b < kbits; ++b) {
              const bool bit = (key >> b) & 1;
              const unsigned bal = __ballot_sync(amask, bit);
              peers &= bit ? bal : ~bal;
            }
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&cnt[key], __popc(peers));
            base = __shfl_sync(peers, base, leader);
            rnk[s] = (uint16_t)(base + __popc(peers & lt_mask));
          }
        }
        __syncthreads();
        if (warp == 0) {  // exclusive scan of cnt[0..J) -> start
          const int per = (J + 31) / 32;
          const int lo = lane * per;
          int sum = 0;
          for (int j = lo; j < lo + per && j < J; ++j) sum += cnt[j];
          int incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          int run = incl - sum;
          for (int j = lo; j < lo + per && j < J; ++j) {
            start[j] = run;
            run += cnt[j];
          }
        }
        __syncthreads();
        for (int s = tid; s < tn; s += NT) perm[start[col[s]] + rnk[s]] = (uint16_t)s;
        __syncthreads();

        // ---- warp ranges of sorted positions; core slice in registers ----
        const int lo = (int)(((int64_t)warp * tn) / nwarps);
        const int hi = (int)(((int64_t)(warp + 1) * tn) / nwarps);
        int p = lo;
        while (p < hi) {
          const int key = col[perm[p]];
          const int bend = min(start[key] + cnt[key], hi);
          if constexpr (R == 32) {
            // K-split geometry: lane (h, qq) owns rows 16h..16h+15 and the
            // column pair (2qq, 2qq+1); one sample per pass, the two row
            // halves are summed with one 64-bit shuffle.  Halves the core
            // registers (32) so 8 passes stay in flight.
            const int h = lane >> 4, qq = lane & 15;
            uint64_t g2[16];
            const float* gs = md.s + (int64_t)key * rl * rr;
            if (rl == R && rr == R) {
#pragma unroll
              for (int i = 0; i < 16; ++i) g2[i] = ldg_b64(gs + (16 * h + i) * R + 2 * qq);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int a = 16 * h + i;
                const float x0 = (a < rl && 2 * qq < rr) ? __ldg(gs + a * rr + 2 * qq) : 0.f;
                const float x1 = (a < rl && 2 * qq + 1 < rr) ? __ldg(gs + a * rr + 2 * qq + 1) : 0.f;
                g2[i] = pack2(x0, x1);
              }
            }
            // exact-size pass groups: no dummy rows, no wasted FMAs
            while (bend - p >= 8) {
              ks_passes<8, RP>(g2, perm, p, s_state, h, qq);
              p += 8;
            }
            if (bend - p >= 4) {
              ks_passes<4, RP>(g2, perm, p, s_state, h, qq);
              p += 4;
            }
            if (bend - p >= 2) {
              ks_passes<2, RP>(g2, perm, p, s_state, h, qq);
              p += 2;
            }
            if (bend - p >= 1) {
              ks_passes<1, RP>(g2, perm, p, s_state, h, qq);
              p += 1;
            }
          } else {
            // core slice -> registers (see Geo for the column ownership)
            constexpr int C1 = (C == 3) ? 1 : 0;
            uint64_t g2[R];
            float g1[C1 ? R : 1];
            const float* gs = md.s + (int64_t)key * rl * rr;
            const int cp = 2 * q, cs = 16 + q;
            if (rl == R && rr == R) {  // full rank: unpredicated 8-byte loads
  #pragma unroll
              for (int a = 0; a < R; ++a) {
                g2[a] = ldg_b64(gs + a * R + cp);
                if constexpr (C1) g1[a] = __ldg(gs + a * R + cs);
              }
            } else {
  #pragma unroll
              for (int a = 0; a < R; ++a) {
                const bool ra = a < rl;
                const float x0 = (ra && cp < rr) ? __ldg(gs + a * rr + cp) : 0.f;
                const float x1 = (ra && cp + 1 < rr) ? __ldg(gs + a * rr + cp + 1) : 0.f;
                g2[a] = pack2(x0, x1);
                if constexpr (C1) g1[a] = (ra && cs < rr) ? __ldg(gs + a * rr + cs) : 0.f;
              }
            }
            while (p < bend) {
              const int n = min(8, bend - p);
              // empty slots of a ragged last iteration point at the dummy row T
              uint32_t row[P];
  #pragma unroll
              for (int pi = 0; pi < P; ++pi) {
                const int w = pi * G + gi;
                const int sidx = (w < n) ? (int)perm[p + w] : T;
                row[pi] = s_state + (uint32_t)sidx * (RP * 4);
              }
              uint64_t acc2[P];
              float acc1[P];
  #pragma unroll
              for (int pi = 0; pi < P; ++pi) {
                acc2[pi] = 0ull;
                acc1[pi] = 0.f;
              }
  #pragma unroll
              for (int a4 = 0; a4 < R / 4; ++a4) {
                float4 v[P];
  #pragma unroll
                for (int pi = 0; pi < P; ++pi) v[pi] = lds128(row[pi] + a4 * 16);
  #pragma unroll
                for (int pi = 0; pi < P; ++pi) {
                  ffma2(acc2[pi], g2[a4 * 4 + 0], v[pi].x);
                  ffma2(acc2[pi], g2[a4 * 4 + 1], v[pi].y);
                  ffma2(acc2[pi], g2[a4 * 4 + 2], v[pi].z);
                  ffma2(acc2[pi], g2[a4 * 4 + 3], v[pi].w);
                  if constexpr (C1) {
                    acc1[pi] = fmaf(v[pi].x, g1[a4 * 4 + 0], acc1[pi]);
                    acc1[pi] = fmaf(v[pi].y, g1[a4 * 4 + 1], acc1[pi]);
                    acc1[pi] = fmaf(v[pi].z, g1[a4 * 4 + 2], acc1[pi]);
                    acc1[pi] = fmaf(v[pi].w, g1[a4 * 4 + 3], acc1[pi]);
                  }
                }
              }
              __syncwarp();  // every lane of a group has read its sample's row
  #pragma unroll
              for (int pi = 0; pi < P; ++pi) {
                sts_b64(row[pi] + cp * 4, acc2[pi]);
                if constexpr (C1) sts32(row[pi] + cs * 4, acc1[pi]);
              }
              __syncwarp();
  p += n;
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

int pick_R(int rmax) {
  if (rmax <= 8) return 8;
  if (rmax <= 16) return 16;
  if (rmax <= 24) return 24;
  if (rmax <= 32) return 32;
  return 0;
}

int bucket_threads() {
  static int v = 0;
  if (v == 0) {
    const char* e = getenv("TNB_BUCKET_THREADS");
    v = (e && atoi(e) == 256) ? 256 : 512;
  }
  return v;
}

template <int R, typename IdxT, int NT>
int launch_nt(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err,
              int jcap, cudaStream_t st) {
  constexpr int RP = Geo<R>::RP;
  // 512/NT CTAs share an SM's 228 KB (1 KB reserved per CTA)
  const size_t budget = (size_t)(233472 / (512 / NT)) - 1024;
  int T = 65504;
  while (T > 32 && smem_bytes<IdxT>(T, RP, ch.n, jcap) > budget) T -= 32;
  const size_t smem = smem_bytes<IdxT>(T, RP, ch.n, jcap);
  if (smem > budget) return set_error(TNB_EINVAL, "bucketed: chain too long for smem");
  auto kern = entries_bucketed_kernel<R, IdxT, NT>;
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "bucketed smem attr");
  if (rc) return rc;
  const int64_t ntiles = (m + T - 1) / T;
  const int64_t slots = (int64_t)num_sms() * (512 / NT);
  const int grid = (int)(ntiles < slots ? ntiles : slots);
  kern<<<grid, NT, smem, st>>>(ch, idx, m, out, err, T, jcap);
  return check_launch("entries_bucketed");
}

template <int R, typename IdxT>
int launch_t(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err,
             int jcap, cudaStream_t st) {
  if (bucket_threads() == 512) return launch_nt<R, IdxT, 512>(ch, idx, m, out, err, jcap, st);
  return launch_nt<R, IdxT, 256>(ch, idx, m, out, err, jcap, st);
}

}  // namespace

bool bucketed_supported(const ChainDev& ch) {
  if (ch.batch != 1 || ch.n < 1 || ch.n > kMaxModes || pick_R(ch.rmax) == 0) return false;
  for (int k = 0; k < ch.n; ++k) {
    const ModeDev& md = ch.m[k];
    if (md.J <= 0 || md.J > 65535) return false;
    if (md.bstride != 0) return false;
    const bool sorted = k > 0 && k < ch.n - 1 && md.layout == TNB_LAYOUT_DENSE;
    if (sorted && md.J > kMaxJ) return false;
  }
  return true;
}

int launch_entries_bucketed(const ChainDev& ch, const int64_t* idx, int64_t m, float* out,
                            int32_t* err, cudaStream_t st) {
  int jmax = 1;
  bool small = true;
  for (int k = 0; k < ch.n; ++k) {
    if (ch.m[k].J > 256) small = false;
    if (k > 0 && k < ch.n - 1 && ch.m[k].layout == TNB_LAYOUT_DENSE && ch.m[k].J > jmax)
      jmax = ch.m[k].J;
  }
  const int jcap = jmax;
  switch (pick_R(ch.rmax)) {
    case 8:
      return small ? launch_t<8, uint8_t>(ch, idx, m, out, err, jcap, st)
                   : launch_t<8, uint16_t>(ch, idx, m, out, err, jcap, st);
    case 16:
      return small ? launch_t<16, uint8_t>(ch, idx, m, out, err, jcap, st)
                   : launch_t<16, uint16_t>(ch, idx, m, out, err, jcap, st);
    case 24:
      return small ? launch_t<24, uint8_t>(ch, idx, m, out, err, jcap, st)
                   : launch_t<24, uint16_t>(ch, idx, m, out, err, jcap, st);
    case 32:
      return small ? launch_t<32, uint8_t>(ch, idx, m, out, err, jcap, st)
                   : launch_t<32, uint16_t>(ch, idx, m, out, err, jcap, st);
  }
  return set_error(TNB_EINVAL, "bucketed: rank > 32");
}

}  // namespace tnb
