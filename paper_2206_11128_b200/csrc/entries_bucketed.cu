// K1 performance kernel: bucketed entry evaluation for unbatched chains with
// ranks <= 32 (BASELINE configs 2 and 5).
//
// Reference algorithm (core.py:432-444): per mode, argsort the samples by
// their index value so every group shares one core slice and the group's
// update is a real (n_j x r) @ (r x s) product.  A global re-sort per mode
// would cost 2 x M x r x 4 bytes of HBM traffic per mode, so
// here the grouping happens per tile, on chip, after the chain is shortened:
//
//   * mode merging (plan_merge): leading / trailing modes become prefix /
//     suffix tables and runs of interior CP modes diagonal product tables,
//     built per call and L2-resident; the kernels run that VIRTUAL chain;
//   * entries_prep_kernel (one CTA per tile): reads the tile's int64 index
//     rows, wraps and validates every ORIGINAL mode (lowest bad mode ->
//     *err, core.py:409-416), combines merged modes and writes the compact
//     uint8/uint16 [N][T] index block of the tile record -- HBM-bound;
//   * entries_sort_kernel (one warp per (tile, sorted mode)): counting sort
//     with a per-warp shared-memory histogram -> permutation + bucket starts;
//   * entries_compute_kernel (persistent, one 512-thread CTA per SM): streams
//     each tile record into shared memory with cp.async.bulk (the next tile's
//     rows are prefetched as soon as the current tile stops needing them);
//     the samples' r-vector states live in shared memory at FIXED slots, so
//     no state ever moves between modes.  First mode: a TMA bulk gather of
//     table rows.  Sorted modes: each warp takes an equal range of sorted
//     positions and, per bucket, loads the core slice once into registers
//     (K-split layout at r=32, lane groups at r<=24) and streams the bucket's
//     samples.  Diagonal runs: one vectorised pass, or folded into the last
//     mode's dot.  Last mode: lane groups per sample, several in flight.
// Each sample's arithmetic is a fixed FMA sequence, so results do not depend
// on the sort order or the tile a sample lands in.
#include <algorithm>

// state row padding in floats (sorted modes read rows in permuted order, so a
// pad buys little; 0 maximises the tile size)
#ifndef TNB_RPAD
#define TNB_RPAD 0
#endif

#include "common.cuh"

// state kernel: L2 prefetch of wide first / last mode rows
// state kernel: full-rank r = 32 sorted modes on mma.sync split-TF32 (state
// rows padded to 36 floats for conflict-light A-fragment loads)
// the per-tile counting sorts run inside the prep kernel (block-wide, on the
// compact indices it already holds in shared memory) instead of a separate
// one-warp-per-(tile, mode) sort kernel when every sorted mode has at least
// this many buckets (block-wide shared atomics contend on few buckets:
// measured faster at J = 128 (cfg5), slower at J = 32 (cfg2)); 0 = never
#ifndef TNB_SORT_IN_PREP
#define TNB_SORT_IN_PREP 64
#endif
#ifndef TNB_FAST_SPLIT
#define TNB_FAST_SPLIT 1
#endif
// state kernel: warp ranges balanced in tensor-core steps (write_splits)
#ifndef TNB_BALANCED
#define TNB_BALANCED 1
#endif
#ifndef TNB_STATE_MMA
#define TNB_STATE_MMA 1
#endif
// state kernel: the closing dot fused into the last sorted (MMA) mode
#ifndef TNB_FUSE_LAST
#define TNB_FUSE_LAST 1
#endif
// state kernel: the first mode's table rows read by the first sorted (MMA)
// mode directly (no gather pass)
#ifndef TNB_FUSE_FIRST
#define TNB_FUSE_FIRST 1
#endif
#ifndef TNB_LAST_U
#define TNB_LAST_U 4
#endif
#ifndef TNB_FFIRST_RING
#define TNB_FFIRST_RING 1
#endif
#ifndef TNB_FRING_G
#define TNB_FRING_G 16
#endif
#ifndef TNB_FRING_D
#define TNB_FRING_D 3
#endif
#ifndef TNB_STATE_PF
#define TNB_STATE_PF 3
#endif
// first-mode row rings (state and stream kernels): 1 = every group through
// L1 (.ca); 0 = .ca only for groups whose rows repeat (ring_cp16 / hot_rows)
#ifndef TNB_RING_CA
#define TNB_RING_CA 0
#endif
// state kernel, fused closing dot: L1 prefetch of this step's closing rows
// before its MMAs (measured: compute 2.36 vs 2.29 ms at cfg2)
#ifndef TNB_CLOSE_PF_EARLY
#define TNB_CLOSE_PF_EARLY 0
#endif
// state kernel, fused closing dot: L1 prefetch of the next step's closing
// rows (measured: compute 2.39 vs 2.28 ms at cfg2 -- the extra perm / index
// lookups cost more than the shorter closing-load latency saves)
#ifndef TNB_CLOSE_L1PF
#define TNB_CLOSE_L1PF 0
#endif
#ifndef TNB_STREAM_THREADS
#define TNB_STREAM_THREADS 384
#endif
#ifndef TNB_STREAM_T
#define TNB_STREAM_T 6144
#endif
#ifndef TNB_STREAM_MMA
#define TNB_STREAM_MMA 1
#endif
// first-mode row gathers: 0 = one cp.async.bulk (TMA) per row, 1 = 16-byte
// cp.async (LDGSTS) pieces, one commit group per ring chunk
#ifndef TNB_STREAM_LDGSTS
#define TNB_STREAM_LDGSTS 1
#endif
// L2 prefetch of the first-mode rows TNB_STREAM_PF chunks beyond the ring
// (same tile only): doubles the gathers in flight without shared memory
// tile records in flight (a warp may run one tile ahead of the slowest one
// before the producer's look-ahead stalls)
#ifndef TNB_STREAM_NREC
#define TNB_STREAM_NREC 2
#endif
// XOR-swizzled (unpadded) ring rows at R = 24
#ifndef TNB_STREAM_SWZ
#define TNB_STREAM_SWZ 1
#endif
// stream plans: sorted-mode index packed into the first mode's uint32
#ifndef TNB_STREAM_KPACK
#define TNB_STREAM_KPACK 1
#endif
#ifndef TNB_STREAM_PF
#define TNB_STREAM_PF 1
#endif

namespace tnb {
// full_tc.cu: the tcgen05 3xTF32 GEMM (large dense prefix table levels)
bool tc_gemm_supported(int64_t M, int64_t N, int K, int64_t lda, int64_t ldb, int64_t ldc);
int64_t tc_gemm_workspace(int64_t M);
int launch_tc_gemm(const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb, int64_t sB, float* C,
                   int64_t ldc, int64_t sC, int64_t M, int64_t N, int K, int64_t batch, void* ws, cudaStream_t st);
// full.cu: tiled SIMT GEMM (rank > 32 table levels)
int gemm_f32(const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb, int64_t sB, float* C,
             int64_t ldc, int64_t sC, int64_t M, int64_t N, int K, int64_t batch, cudaStream_t st);

namespace {

constexpr int kMaxJ = 1024;          // bucket count limit for sorted modes
#ifndef TNB_PREP_ILP2
#define TNB_PREP_ILP2 1
#endif
#ifndef TNB_PREP_THREADS
#define TNB_PREP_THREADS 512
#endif
constexpr int kPrepThreads = TNB_PREP_THREADS;
#ifndef TNB_STATE_CTAS
#define TNB_STATE_CTAS 1
#endif
constexpr int kStateCtas = TNB_STATE_CTAS;                // state-kernel CTAs per SM
constexpr int kComputeThreads = 512 / TNB_STATE_CTAS;     // 16 warps per SM



__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// ld.shared.v4 with a compile-time byte offset folded into the address
template <int OFF>
__device__ __forceinline__ float4 lds128o(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a), "n"(OFF));
  return v;
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
__device__ __forceinline__ ulonglong2 ldg_u2(const float* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
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

// split-TF32 on mma.sync m16n8k8: x = hi + lo, both rounded to tf32; the
// three products lo*hi + hi*lo + hi*hi keep fp32-level accuracy
// (rna on the bit pattern: cvt.rna.tf32.f32's value for every finite x in
// add + mask instead of add / NaN test / select / mask)
__device__ __forceinline__ uint32_t rna_tf32(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = rna_tf32(x);
  lo = rna_tf32(x - __uint_as_float(hi));
}
// the per-step A-fragment split: lo = x - rna(x) exact, passed unrounded (the
// tensor core truncates it; the dropped bits are below 2^-21 |x|) -- one
// instruction less than split_tf32
__device__ __forceinline__ void split_tf32_fast(float x, uint32_t& hi, uint32_t& lo) {
#if TNB_FAST_SPLIT
  hi = rna_tf32(x);
  lo = __float_as_uint(x - __uint_as_float(hi));
#else
  split_tf32(x, hi, lo);
#endif
}
// the A-fragment split of the per-entry kernels: hi = the fp32 bits as they
// are (the tensor core ignores the low 13 mantissa bits: truncation), lo =
// x - trunc(x) exact -- no conversion-pipe instruction per element
// (TNB_SPLIT_TRUNC=0: cvt.rna as above)
#ifndef TNB_SPLIT_TRUNC
#define TNB_SPLIT_TRUNC 1
#endif
__device__ __forceinline__ void split_tf32_step(float x, uint32_t& hi, uint32_t& lo) {
#if TNB_SPLIT_TRUNC
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
#else
  split_tf32_fast(x, hi, lo);
#endif
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
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
  static constexpr int RP = R + ((R == 32 && TNB_STATE_MMA) ? 4 : TNB_RPAD);  // state row stride (floats)
  static_assert(L * C == R && 32 % L == 0 && G * P == 8, "geometry");
};


// K-split pass group for R == 32: NP samples (one per pass) of one bucket.
// Lane (h, qq) holds rows 16h..16h+15 of the core slice, column pair
// (2qq, 2qq+1); the two row halves are summed with one 64-bit shuffle.
template <int NP, int RP>
__device__ __forceinline__ void ks_passes(const uint64_t (&g2)[16], const uint16_t* perm, int p,
                                          uint32_t s_state, int h, int qq) {
  uint32_t rowb[NP], rowh[NP];
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) {
    rowb[pi] = s_state + (uint32_t)perm[p + pi] * (RP * 4);
    rowh[pi] = rowb[pi] + h * 64;
  }
  uint64_t acc2[NP];
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) acc2[pi] = 0ull;
#pragma unroll
  for (int a4 = 0; a4 < 4; ++a4) {
    float4 v[NP];
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) {
      switch (a4) {  // immediate offsets: no per-load address arithmetic
        case 0: v[pi] = lds128o<0>(rowh[pi]); break;
        case 1: v[pi] = lds128o<16>(rowh[pi]); break;
        case 2: v[pi] = lds128o<32>(rowh[pi]); break;
        default: v[pi] = lds128o<48>(rowh[pi]); break;
      }
    }
    // consecutive FFMA2s hit different accumulators (no back-to-back RAW)
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 0], v[pi].x);
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 1], v[pi].y);
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 2], v[pi].z);
#pragma unroll
    for (int pi = 0; pi < NP; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 3], v[pi].w);
  }
  if constexpr (NP == 1) {
    acc2[0] = add2(acc2[0], __shfl_xor_sync(0xffffffffu, acc2[0], 16));
    __syncwarp();  // every lane has read its rows
    if (h == 0) sts_b64(rowb[0] + qq * 8, acc2[0]);
  } else {
    // sample pair (2i, 2i+1): half h finishes sample 2i+h, so each lane sends
    // the partial its partner finishes -- one 64-bit shuffle per pair
    uint64_t res[NP / 2];
#pragma unroll
    for (int i = 0; i < NP / 2; ++i) {
      const uint64_t keep = h ? acc2[2 * i + 1] : acc2[2 * i];
      const uint64_t send = h ? acc2[2 * i] : acc2[2 * i + 1];
      res[i] = add2(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
    __syncwarp();  // every lane has read its rows
#pragma unroll
    for (int i = 0; i < NP / 2; ++i) sts_b64((h ? rowb[2 * i + 1] : rowb[2 * i]) + qq * 8, res[i]);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Two kernels per call:
//   prep    (one CTA per tile): index validation/compaction and the counting
//           sort of every interior dense mode, written to a per-tile
//           workspace record [cidx | perm[slot] | starts[slot]];
//   compute (persistent): streams each tile's record into shared memory with
//           cp.async.bulk (the next tile's rows/slots are prefetched as soon
//           as the current tile stops needing them) and runs the modes; one
//           CTA barrier per mode, no sorting on the critical path.

struct BPlan {
  int T;           // samples per tile
  int nsort;       // interior dense modes (sorted)
  int jpad;        // bucket-start row length (>= max J + 1, multiple of 8)
  int idx_bytes;   // sizeof(IdxT)
  int64_t ntiles;
  int64_t tile_bytes;
  int64_t off_wide, off_perm, off_starts;
  // wide virtual modes: a prefix (mode 0) / suffix (mode N-1) table with more
  // than 65535 rows; their combined indices are uint32 rows [nw][T] stored
  // right after the compact [N][T] block (record and shared memory alike)
  int wide0, wideL, nw;
  // compact rows stored: virtual modes crow0 .. crow0 + ncrow - 1 (all N for
  // the state kernel; stream plans skip the first mode (always wide) and a
  // wide last mode)
  int crow0, ncrow;
  int psort;   // the prep kernel sorts (TNB_SORT_IN_PREP)
  int splits;  // balanced warp ranges are written after the bucket starts (state kernel)
  // stream plans: the sorted mode's index is packed above the first mode's
  // (uint32, bits kshift..) and its compact row dropped from the record
  int kpack, kshift;
  int8_t slot[kMaxModes];  // mode -> sorted slot or -1
  // mode merging: the kernels run a VIRTUAL chain whose first / last modes
  // may be prefix / suffix tables over several original modes; the prep
  // kernel reads the n0 original index columns, validates each against its
  // own extent oJ (error = lowest original mode) and combines the columns of
  // one virtual mode in C order (vmap: original mode -> virtual mode)
  int n0;
  int32_t oJ[kMaxModes];
  int8_t vmap[kMaxModes];
  int8_t smode[kMaxModes];  // sorted slot -> (virtual) mode
  int8_t lmaj[kMaxModes];   // sorted mode whose slices are in lane-major order
  int8_t mmal[kMaxModes];   // ... in the tensor-core fragment order (mma_slice_kernel)
  // device word set by detect_hot_kernel when the first-mode rows repeat
  // (slice queries): the compute kernels' rings then copy through L1
  const int32_t* hot = nullptr;
};

// Balanced warp ranges for the state kernel's sorted modes, written by ONE
// warp after the bucket starts gst[0..J] (gst[J] = tn): the tile's work is
// counted in 16-sample steps per bucket (the tensor-core step), and warp w of
// kSplitWarps starts at step floor(w S / kSplitWarps) -- a position inside
// its bucket, on a 16-sample boundary -- instead of at w tn / kSplitWarps
// (equal positions give a warp that straddles more buckets more steps, and
// the mode barrier waits for it).  gst[J + 1 + w] = start of warp w,
// gst[J + 1 + kSplitWarps] = tn.
constexpr int kSplitWarps = 16;
// `sm` holds the same starts in shared memory (entries 0..J-1).
__device__ void write_splits(uint16_t* gst, const int* sm, int J, int tn, int lane) {
  __syncwarp();
  const int per = (J + 31) >> 5;
  const int j0 = lane * per, j1 = min(j0 + per, J);
  auto start = [&](int j) { return j < J ? sm[j] : tn; };
  int my = 0;
  for (int j = j0; j < j1; ++j) my += (start(j + 1) - start(j) + 15) >> 4;
  int incl = my;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int S = __shfl_sync(0xffffffffu, incl, 31);
  const int excl = incl - my;
  __syncwarp();
  for (int w = 0; w < kSplitWarps; ++w) {
    const int t = (int)(((int64_t)w * S) / kSplitWarps);
    if (S == 0) {
      if (lane == 0) gst[J + 1 + w] = 0;
    } else if (t >= excl && t < incl) {
      int acc = excl;
      for (int j = j0; j < j1; ++j) {
        const int sj = (start(j + 1) - start(j) + 15) >> 4;
        if (t < acc + sj) {
          gst[J + 1 + w] = (uint16_t)(start(j) + 16 * (t - acc));
          break;
        }
        acc += sj;
      }
    }
  }
  if (lane == 0) gst[J + 1 + kSplitWarps] = (uint16_t)tn;
  __syncwarp();
}

// prep: one CTA per tile -- reads the tile's n0 int64 index columns
// (coalesced), validates and combines them, and writes the compact [N][T]
// index block of the tile record.
template <typename IdxT, bool PSORT, bool SPLITS>
__global__ void __launch_bounds__(kPrepThreads, PSORT ? 1024 / kPrepThreads : 1536 / kPrepThreads) entries_prep_kernel(const __grid_constant__ ChainDev ch,
                                                           const __grid_constant__ BPlan bp,
                                                           const int64_t* __restrict__ idx, int64_t m,
                                                           int32_t* __restrict__ err,
                                                           unsigned char* __restrict__ ws) {
  constexpr int NT = kPrepThreads;
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = ch.n, T = bp.T;
  IdxT* idxs = reinterpret_cast<IdxT*>(smem);                                         // [ncrow][T]
  uint32_t* widx = reinterpret_cast<uint32_t*>(smem + (size_t)bp.ncrow * T * sizeof(IdxT));  // [nw][T]
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t s0 = tile * T;
  const int tn = (int)((m - s0) < T ? (m - s0) : T);
  unsigned char* rec = ws + tile * bp.tile_bytes;

  // ---- indices: thread = sample row (n0 int64 values, 16-byte loads when
  //      the row stride allows), wrap/validate per original mode, combine
  //      merged modes, compact to [N][T]
  {
    const int N0 = bp.n0;
    const int64_t* src = idx + s0 * N0;
    const bool v2 = (N0 & 1) == 0 && (reinterpret_cast<uintptr_t>(idx) & 15) == 0;
#if TNB_PREP_ILP2
    // the sorting instance has registers to spare: rows of 8 indices (cfg5)
    // go two per thread, all eight 16-byte loads issued before either row is
    // combined
    if (PSORT && v2 && N0 == 8) {
      auto comb = [&](int s, const longlong2 (&r)[4]) {
        int vk = 0;
        uint32_t cur = 0;
        auto put = [&](int o, int64_t raw) {
          const int32_t J = bp.oJ[o];
          const uint32_t v = (uint32_t)norm_index(raw, J, o, err);
          const int tk = bp.vmap[o];
          if (tk != vk) {
            if (vk == 0 && bp.wide0) widx[s] = cur;
            else if (vk == N - 1 && bp.wideL) widx[(size_t)bp.wide0 * T + s] = cur;
            else idxs[(size_t)(vk - bp.crow0) * T + s] = (IdxT)cur;
            vk = tk;
            cur = 0;
          }
          cur = cur * (uint32_t)J + v;
        };
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          put(2 * q, r[q].x);
          put(2 * q + 1, r[q].y);
        }
        if (vk == 0 && bp.wide0) widx[s] = cur;
        else if (vk == N - 1 && bp.wideL) widx[(size_t)bp.wide0 * T + s] = cur;
        else idxs[(size_t)(vk - bp.crow0) * T + s] = (IdxT)cur;
      };
      for (int s = tid; s < tn; s += 2 * NT) {
        const int sb = s + NT;
        const bool hb = sb < tn;
        const longlong2* ra = reinterpret_cast<const longlong2*>(src + (int64_t)s * 8);
        const longlong2* rb = reinterpret_cast<const longlong2*>(src + (int64_t)(hb ? sb : s) * 8);
        longlong2 a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = __ldg(ra + q);
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = __ldg(rb + q);
        comb(s, a);
        if (hb) comb(sb, b);
      }
      for (int s = tn + tid; s < T; s += NT) {  // tail rows: index 0
        for (int k = 0; k < bp.ncrow; ++k) idxs[(size_t)k * T + s] = (IdxT)0;
        for (int w = 0; w < bp.nw; ++w) widx[(size_t)w * T + s] = 0u;
      }
    } else
#endif
    for (int s = tid; s < T; s += NT) {
      const int64_t* row = src + (int64_t)s * N0;
      if (s >= tn) {
        for (int k = 0; k < bp.ncrow; ++k) idxs[(size_t)k * T + s] = (IdxT)0;  // tail rows: index 0
        for (int w = 0; w < bp.nw; ++w) widx[(size_t)w * T + s] = 0u;
        continue;
      }
      auto store = [&](int v, uint32_t x) {
        if (v == 0 && bp.wide0) widx[s] = x;
        else if (v == N - 1 && bp.wideL) widx[(size_t)bp.wide0 * T + s] = x;
        else idxs[(size_t)(v - bp.crow0) * T + s] = (IdxT)x;
      };
      int vk = 0;
      uint32_t cur = 0;
      auto put = [&](int o, int64_t raw) {
        const int32_t J = bp.oJ[o];
        const uint32_t v = (uint32_t)norm_index(raw, J, o, err);
        const int tk = bp.vmap[o];
        if (tk != vk) {
          store(vk, cur);
          vk = tk;
          cur = 0;
        }
        cur = cur * (uint32_t)J + v;
      };
      if (v2) {
        for (int o = 0; o < N0; o += 2) {
          const longlong2 w = __ldg(reinterpret_cast<const longlong2*>(row + o));
          put(o, w.x);
          put(o + 1, w.y);
        }
      } else {
        for (int o = 0; o < N0; ++o) put(o, __ldg(row + o));
      }
      store(vk, cur);
    }
  }
  __syncthreads();
  const size_t cbytes = (size_t)bp.ncrow * T * sizeof(IdxT) + (size_t)bp.nw * T * 4;
  if (bp.kpack) {  // the sorted mode's index above the first mode's
    for (int s = tid; s < T; s += NT) widx[s] |= (uint32_t)idxs[s] << bp.kshift;
    __syncthreads();
  }
  {  // compact block (+ wide rows) -> record (16-byte stores), minus a packed row
    const size_t skip = bp.kpack ? (size_t)T * sizeof(IdxT) : 0;
    const int n16 = (int)((cbytes - skip) / 16);
    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(idxs) + skip);
    for (int i = tid; i < n16; i += NT) reinterpret_cast<uint4*>(rec)[i] = src[i];
  }
  // counting sort of each sorted slot: histogram (shared atomics), warp-0
  // scan into the bucket starts, scatter into a staged permutation, 16-byte
  // copy-out.  The order inside a bucket is not fixed, and need not be: a
  // sample's arithmetic does not depend on its position.
  const int JP = bp.jpad;
  int* hist = reinterpret_cast<int*>(smem + ((cbytes + 15) & ~(size_t)15));  // [jpad]
  uint16_t* pb = reinterpret_cast<uint16_t*>(hist + JP);                      // [T]
  const int lane = tid & 31;
  for (int sl = 0; sl < (PSORT ? bp.nsort : 0); ++sl) {
    const int k = bp.smode[sl];
    const int J = ch.m[k].J;
    const IdxT* col = idxs + (size_t)(k - bp.crow0) * T;
    for (int j = tid; j < JP; j += NT) hist[j] = 0;
    __syncthreads();
    for (int s = tid; s < tn; s += NT) atomicAdd(&hist[col[s]], 1);
    __syncthreads();
    if (tid < 32) {
      uint16_t* gst = reinterpret_cast<uint16_t*>(rec + bp.off_starts) + (size_t)sl * JP;
      const int per = (J + 31) >> 5;
      const int j0 = lane * per, j1 = min(j0 + per, J);
      int sum = 0;
      for (int j = j0; j < j1; ++j) sum += hist[j];
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - sum;
      for (int j = j0; j < j1; ++j) {
        const int c = hist[j];
        hist[j] = run;
        gst[j] = (uint16_t)run;
        run += c;
      }
      for (int j = J + lane; j < JP; j += 32) gst[j] = (uint16_t)tn;
      if constexpr (SPLITS) write_splits(gst, hist, J, tn, lane);
    }
    __syncthreads();
    for (int s = tid; s < tn; s += NT) pb[atomicAdd(&hist[col[s]], 1)] = (uint16_t)s;
    __syncthreads();
    uint16_t* pm = reinterpret_cast<uint16_t*>(rec + bp.off_perm) + (size_t)sl * T;
    for (int i = tid; i < T / 8; i += NT) reinterpret_cast<uint4*>(pm)[i] = reinterpret_cast<const uint4*>(pb)[i];
    __syncthreads();
  }
}

// sort: ONE WARP per (tile, sorted mode), independent of every other warp (no
// CTA barriers): counting sort of the tile's compact indices of that mode with
// a per-warp shared-memory histogram -- count (shared atomics), warp scan,
// scatter (shared atomics hand out the slots) -- writing the permutation and
// the bucket starts of the record.  The order inside a bucket is not fixed,
// and need not be: a sample's arithmetic does not depend on its position.
template <typename IdxT>
__global__ void __launch_bounds__(256) entries_sort_kernel(const __grid_constant__ ChainDev ch,
                                                           const __grid_constant__ BPlan bp, int64_t m,
                                                           unsigned char* __restrict__ ws) {
  extern __shared__ __align__(16) int hist_all[];  // per warp: [jpad] counts, [T] permutation
  const int NS = bp.nsort, T = bp.T, JP = bp.jpad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  const int64_t tile = gw / NS;
  if (tile >= bp.ntiles) return;
  const int sl = (int)(gw - tile * NS);
  const int64_t s0 = tile * T;
  const int tn = (int)((m - s0) < T ? (m - s0) : T);
  unsigned char* rec = ws + tile * bp.tile_bytes;
  const int k = bp.smode[sl];
  const int J = ch.m[k].J;
  const IdxT* col = reinterpret_cast<const IdxT*>(rec) + (size_t)(k - bp.crow0) * T;
  uint16_t* pm = reinterpret_cast<uint16_t*>(rec + bp.off_perm) + (size_t)sl * T;
  uint16_t* gst = reinterpret_cast<uint16_t*>(rec + bp.off_starts) + (size_t)sl * JP;
  int* h = hist_all + (size_t)warp * (JP + T / 2);
  uint16_t* pb = reinterpret_cast<uint16_t*>(h + JP);  // JP and T/2 are multiples of 4: 16-B aligned
  for (int j = lane; j < JP; j += 32) h[j] = 0;
  __syncwarp();
#pragma unroll 4
  for (int s = lane; s < tn; s += 32) atomicAdd(&h[col[s]], 1);
  __syncwarp();
  // exclusive scan: lane owns the contiguous bucket range [lane*per, ...)
  const int per = (J + 31) >> 5;
  const int j0 = lane * per, j1 = min(j0 + per, J);
  int sum = 0;
  for (int j = j0; j < j1; ++j) sum += h[j];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int run = incl - sum;
  for (int j = j0; j < j1; ++j) {
    const int c = h[j];
    h[j] = run;
    gst[j] = (uint16_t)run;
    run += c;
  }
  for (int j = J + lane; j < JP; j += 32) gst[j] = (uint16_t)tn;
  if (bp.splits) write_splits(gst, h, J, tn, lane);
#pragma unroll 4
  for (int s = lane; s < tn; s += 32) pb[atomicAdd(&h[col[s]], 1)] = (uint16_t)s;
  __syncwarp();
  // coalesced 16-byte copy-out of the permutation
  for (int i = lane; i < T / 8; i += 32) reinterpret_cast<uint4*>(pm)[i] = reinterpret_cast<const uint4*>(pb)[i];
}

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 16-byte ring copies: through L2 only (.cg, streaming) or through L1 too
// (.ca) when the group's rows repeat -- every sample of a slice query shares
// its first-mode row, and 2^24 copies of one L2 line serialise on its slice
// (cfg2 slice queries 14.0 -> 2.0 ms); random rows keep .cg (.ca for every
// group measured 3% slower on uniform indices)
__device__ __forceinline__ void ring_cp16(uint32_t dst, const void* src, bool hot) {
  if (hot)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// One warp per sampled tile: the first 32 samples' first-mode table rows;
// a majority equal to sample 0's sets *hot (the caller zeroes it).  A
// per-group vote inside the rings cost 2-8% on uniform indices; this is one
// tiny launch per call and a kernel-uniform flag.
template <typename IdxT>
__global__ void detect_hot_kernel(const __grid_constant__ BPlan bp, const unsigned char* __restrict__ ws, int64_t m,
                                  int32_t* __restrict__ hot) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (bp.ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t tile = (int64_t)blockIdx.x * stride;
  if (tile >= bp.ntiles) return;
  const int tn = (int)min((int64_t)bp.T, m - tile * bp.T);
  const int rows = tn < 32 ? tn : 32;
  const unsigned char* rec = ws + tile * bp.tile_bytes;
  uint32_t j = 0;
  if (lane < rows) {
    if (bp.crow0 > 0 || bp.wide0) {  // first mode in the uint32 row (stream records: sorted index packed above)
      const uint32_t kmask = bp.kpack ? (1u << bp.kshift) - 1u : ~0u;
      j = reinterpret_cast<const uint32_t*>(rec + bp.off_wide)[lane] & kmask;
    } else {
      j = (uint32_t)reinterpret_cast<const IdxT*>(rec)[lane];
    }
  }
  const uint32_t j0 = __shfl_sync(0xffffffffu, j, 0);
  const unsigned same = __ballot_sync(0xffffffffu, lane < rows && j == j0);
  if (lane == 0 && 2 * __popc(same) > rows) atomicOr(hot, 1);
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(s32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar))
      : "memory");
}

// FOLD: the chain ends in interior CP modes followed by the last mode; that
// run is folded into the last-mode dot product (separate instantiation so
// chains without it keep the leaner register allocation)
template <int R, typename IdxT, int NT, bool FOLD, bool HOT>
__global__ void __launch_bounds__(NT, kStateCtas)
    entries_compute_kernel(const __grid_constant__ ChainDev ch, const __grid_constant__ BPlan bp,
                           const unsigned char* __restrict__ ws, int64_t m, float* __restrict__ out) {
  if ((bp.hot != nullptr && __ldg(bp.hot) != 0) != HOT) return;  // see entries_stream_kernel
  using Gm = Geo<R>;
  constexpr int C = Gm::C, L = Gm::L, G = Gm::G, P = Gm::P, RP = Gm::RP;
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = ch.n, T = bp.T;
  float* state = reinterpret_cast<float*>(smem);                                   // [T+1][RP]
  IdxT* cidx = reinterpret_cast<IdxT*>(state + (size_t)(T + 1) * RP);              // [N][T]
  uint32_t* widx = reinterpret_cast<uint32_t*>(cidx + (size_t)N * T);              // [nw][T]
  uint16_t* permb = reinterpret_cast<uint16_t*>(widx + (size_t)bp.nw * T);         // [2][T]
  uint16_t* startb = permb + 2 * T;                                                // [2][jpad]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(startb + 2 * bp.jpad) + 15) & ~(uintptr_t)15);  // cbar, pbar[2], fbar
  uint64_t* cbar = bars;
  uint64_t* pbar = bars + 1;
  uint64_t* fbar = bars + 3;  // first-mode row gather

  const uint32_t s_state = s32(state);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = NT / 32;
  const int gi = lane / L;
  const int q = lane % L;
  const int64_t ntiles = bp.ntiles;
  const uint32_t row_bytes = (uint32_t)T * sizeof(IdxT);
  const uint32_t wrow_bytes = (uint32_t)T * 4;
  const uint32_t* widx0 = widx;                           // first mode (wide)
  const uint32_t* widxL = widx + (size_t)bp.wide0 * T;    // last mode (wide)
  const uint32_t slot_bytes = (uint32_t)T * 2 + (uint32_t)bp.jpad * 2;
  const int ns = bp.nsort;
  // ffirst: the first mode is a row table feeding a tensor-core sorted mode 1,
  // whose A fragments are then loaded straight from the table rows (no
  // first-mode gather into the state, no barrier after it)
  const bool ffirst = TNB_FUSE_FIRST && R == 32 && N >= 3 && bp.mmal[1] && ch.m[0].layout == TNB_LAYOUT_DENSE &&
                      ch.m[0].rl == 1 && ch.m[0].rr == R;

  // producer (tid 0): slot items in consumption order (tile-major, slot-minor)
  auto issue_slot = [&](int64_t item) {
    if (ns == 0) return;
    const int64_t ti = item / ns;
    const int sl = (int)(item - ti * ns);
    const int64_t tile = blockIdx.x + ti * gridDim.x;
    if (tile >= ntiles) return;
    const int b = (int)(item & 1);
    const unsigned char* rec = ws + tile * bp.tile_bytes;
    mb_expect(&pbar[b], slot_bytes);
    bulk(permb + b * T, rec + bp.off_perm + (size_t)sl * T * 2, (uint32_t)T * 2, &pbar[b]);
    bulk(startb + b * bp.jpad, rec + bp.off_starts + (size_t)sl * bp.jpad * 2, (uint32_t)bp.jpad * 2,
         &pbar[b]);
  };
  if (tid == 0) {
    mb_init(cbar, 1);
    mb_init(&pbar[0], 1);
    mb_init(&pbar[1], 1);
    mb_init(fbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < ntiles) {
      const unsigned char* rec = ws + (int64_t)blockIdx.x * bp.tile_bytes;
      mb_expect(cbar, row_bytes * N + wrow_bytes * bp.nw);
      for (int k = 0; k < N; ++k) bulk(cidx + (size_t)k * T, rec + (size_t)k * row_bytes, row_bytes, cbar);
      for (int w = 0; w < bp.nw; ++w) bulk(widx + (size_t)w * T, rec + bp.off_wide + (size_t)w * wrow_bytes, wrow_bytes, cbar);
      issue_slot(0);
      issue_slot(1);
    }
  }
  __syncthreads();

  uint32_t c_it = 0, f_it = 0;
  int64_t item = 0;  // slot items consumed
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t s0 = tile * T;
    const int tn = (int)((m - s0) < T ? (m - s0) : T);
    const int64_t ntile = tile + gridDim.x;
    mb_wait(cbar, c_it & 1);
    ++c_it;
    int fold = -1;  // first CP mode of a diagonal run folded into the last mode
    for (int k = 0; k < N; ++k) {
      if (k == 0 && ffirst) continue;  // the first sorted mode reads the first-mode rows itself
      const ModeDev& md = ch.m[k];
      const IdxT* col = cidx + (size_t)k * T;
      const int rl = md.rl, rr = md.rr;
      bool sorted = false;
      int k2 = k;  // last mode handled by this iteration (diagonal runs)
      if (k == 0) {
        if (N == 1) {  // [J][1][1]
          for (int s = tid; s < tn; s += NT) out[s0 + s] = __ldg(md.s + col[s]);
        } else if (rr == R) {
          // state row = G_0[j][0][:]: one bulk copy per sample, all of the
          // tile's rows in flight at once on the TMA engine (a prefix table
          // lives in L2: a register gather would be latency-bound)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
          if (tid == 0) mb_expect(fbar, (uint32_t)tn * R * 4);
          __syncthreads();
          for (int s = tid; s < tn; s += NT) {
            const int64_t j = bp.wide0 ? (int64_t)widx0[s] : (int64_t)col[s];
            bulk(state + s * RP, md.s + j * R, R * 4, fbar);
          }
          mb_wait(fbar, f_it & 1);
          ++f_it;
        } else {  // zero padded to R
          for (int e = tid; e < tn * R; e += NT) {
            const int s = e / R, c = e - (e / R) * R;
            const int64_t j = bp.wide0 ? (int64_t)widx0[s] : (int64_t)col[s];
            state[s * RP + c] = (c < rr) ? __ldg(md.s + j * rr + c) : 0.f;
          }
        }
      } else if (md.layout == TNB_LAYOUT_DIAG) {
        // a run of consecutive interior CP modes is one elementwise product:
        // v[c] *= D_k[j_k][c] * D_k+1[j_k+1][c] * ..., done in ONE pass over
        // the state (16-byte rows when the rank allows)
        while (k2 + 1 < N - 1 && ch.m[k2 + 1].layout == TNB_LAYOUT_DIAG) ++k2;
        if (FOLD && k2 == N - 2 && ch.m[N - 1].rl == R && ch.m[N - 1].rr == 1 && (R & 3) == 0) {
          fold = k;  // the last mode multiplies these rows in (no state pass)
        } else if ((rl & 3) == 0) {
          const int q4 = rl >> 2;
#pragma unroll 2
          for (int e = tid; e < tn * q4; e += NT) {
            const int s = e / q4, c4 = e - (e / q4) * q4;
            float4 f = *reinterpret_cast<const float4*>(state + s * RP + c4 * 4);
            for (int kk = k; kk <= k2; ++kk) {
              const ModeDev& mk = ch.m[kk];
              const float4 d = __ldg(reinterpret_cast<const float4*>(mk.s + (int64_t)cidx[(size_t)kk * T + s] * rl) + c4);
              f.x *= d.x;
              f.y *= d.y;
              f.z *= d.z;
              f.w *= d.w;
            }
            *reinterpret_cast<float4*>(state + s * RP + c4 * 4) = f;
          }
        } else {
          for (int e = tid; e < tn * rl; e += NT) {
            const int s = e / rl, c = e - (e / rl) * rl;
            float f = state[s * RP + c];
            for (int kk = k; kk <= k2; ++kk)
              f *= __ldg(ch.m[kk].s + (int64_t)cidx[(size_t)kk * T + s] * rl + c);
            state[s * RP + c] = f;
          }
        }
      } else if (k == N - 1) {  // rr == 1: out = state . G[j][:, 0]
        if (rl == R) {
          // groups of GS lanes per sample, lane c owns the 16-byte chunk c of
          // the random core row (one L1 line per group instead of one per
          // lane); folded CP rows multiply in before the dot; 2 samples per
          // group in flight
          constexpr int CH = R / 4;
          constexpr int GS = CH <= 2 ? 2 : (CH <= 4 ? 4 : 8);
          constexpr int SPW = 32 / GS;
          const int c = lane % GS, g = lane / GS;
          const int cc = c < CH ? c : 0;  // idle lanes (R = 24) re-read chunk 0
          const int kf = (FOLD && fold >= 0) ? fold : N - 1;
          const int nf = N - 1 - kf;  // folded CP modes
          // loop-invariant sources of the first MF folded modes (slot i >= nf
          // re-reads mode kf and is multiplied in as 1)
          constexpr int MF = 1;  // after diagonal merging a folded run is usually one mode
          const float* dps[MF];
          const IdxT* dcs[MF];
#pragma unroll
          for (int i = 0; i < MF; ++i) {
            const int kk = kf + (i < nf ? i : 0);
            dps[i] = FOLD ? ch.m[kk].s : md.s;
            dcs[i] = cidx + (size_t)kk * T;
          }
          constexpr int U = TNB_LAST_U;  // samples per lane group in flight (L2 / HBM latency)
          for (int base = warp * (U * SPW); base < tn; base += nwarps * U * SPW) {
            // every load of the U samples is issued before any use
            float4 gv[U], v[U], dv[U][MF];
            bool act[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int s = base + u * SPW + g;
              act[u] = s < tn && c < CH;
              const int sc = act[u] ? s : 0;
              const int64_t jl = bp.wideL ? (int64_t)widxL[sc] : (int64_t)col[sc];
              gv[u] = __ldg(reinterpret_cast<const float4*>(md.s + jl * R) + cc);
              if constexpr (FOLD) {
#pragma unroll
                for (int i = 0; i < MF; ++i)
                  dv[u][i] = __ldg(reinterpret_cast<const float4*>(dps[i] + (int64_t)dcs[i][sc] * R) + cc);
              }
              v[u] = lds128(s_state + (uint32_t)sc * (RP * 4) + cc * 16);
            }
            float part[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int s = act[u] ? base + u * SPW + g : 0;
              float4 w = gv[u];
              if constexpr (FOLD) {
#pragma unroll
                for (int i = 0; i < MF; ++i)
                  if (i < nf) {
                    w.x *= dv[u][i].x;
                    w.y *= dv[u][i].y;
                    w.z *= dv[u][i].z;
                    w.w *= dv[u][i].w;
                  }
                for (int kk = kf + MF; kk < N - 1; ++kk) {
                  const float4 d =
                      __ldg(reinterpret_cast<const float4*>(ch.m[kk].s + (int64_t)cidx[(size_t)kk * T + s] * R) + cc);
                  w.x *= d.x;
                  w.y *= d.y;
                  w.z *= d.z;
                  w.w *= d.w;
                }
              }
              float a = v[u].x * w.x;
              a = fmaf(v[u].y, w.y, a);
              a = fmaf(v[u].z, w.z, a);
              a = fmaf(v[u].w, w.w, a);
              part[u] = act[u] ? a : 0.f;
            }
#pragma unroll
            for (int o = GS / 2; o > 0; o >>= 1) {
#pragma unroll
              for (int u = 0; u < U; ++u) part[u] += __shfl_xor_sync(0xffffffffu, part[u], o);
            }
            if (c == 0) {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const int su = base + u * SPW + g;
                if (su < tn) out[s0 + su] = part[u];
              }
            }
          }
        } else {
          for (int s = tid; s < tn; s += NT) {
            const float* g = md.s + (bp.wideL ? (int64_t)widxL[s] : (int64_t)col[s]) * rl;
            const float* v = state + s * RP;
            float acc = 0.f;
#pragma unroll
            for (int a = 0; a < R; ++a)
              if (a < rl) acc = fmaf(v[a], __ldg(g + a), acc);
            out[s0 + s] = acc;
          }
        }
      } else {
        // ---- sorted mode: permutation + bucket starts from the prep kernel
        sorted = true;
#if TNB_STATE_PF
        // wide (HBM-resident) tables: L2 prefetch, while the last sorted mode
        // runs, of this tile's last-mode rows (bit 1) and of the NEXT tile's
        // first-mode rows (bit 2, indices from its record in global memory),
        // so neither gather waits on HBM latency
        if (k == N - 2) {
          if ((TNB_STATE_PF & 1) && bp.wideL) {
            const ModeDev& ml = ch.m[N - 1];
            for (int s = tid; s < tn; s += NT) prefetch_l2(ml.s + (int64_t)widxL[s] * ml.rl);
          }
          if ((TNB_STATE_PF & 2) && bp.wide0 && ntile < ntiles) {
            const int64_t ns0 = ntile * T;
            const int ntn = (int)((m - ns0) < T ? (m - ns0) : T);
            const uint32_t* nw = reinterpret_cast<const uint32_t*>(ws + ntile * bp.tile_bytes + bp.off_wide);
            // the index loads first (independent, all in flight), then the prefetches
            for (int base = tid; base < ntn; base += 4 * NT) {
              uint32_t jj[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) jj[u] = base + u * NT < ntn ? __ldg(nw + base + u * NT) : 0u;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (base + u * NT < ntn) prefetch_l2(ch.m[0].s + (int64_t)jj[u] * ch.m[0].rr);
            }
          }
        }
#endif
        const int b = (int)(item & 1);
        mb_wait(&pbar[b], (uint32_t)((item >> 1) & 1));
        const uint16_t* perm = permb + b * T;
        const uint16_t* st = startb + b * bp.jpad;
        const int lo = bp.splits ? (int)st[md.J + 1 + warp] : (int)(((int64_t)warp * tn) / nwarps);
        const int hi = bp.splits ? (int)st[md.J + 2 + warp] : (int)(((int64_t)(warp + 1) * tn) / nwarps);
        if constexpr (R == 32) {
        int p = lo;
#if TNB_STATE_MMA
        if (bp.mmal[k]) {
          // tensor cores: 16 samples of one bucket per step, rows g and g + 8
          // (sorted positions p + g, p + g + 8) of the m16n8k8 tiles; the
          // state rows are read as A fragments and overwritten in place by
          // the C fragments (v <- v G) after the whole step has read them.
          // fclose: this is the last sorted mode and the chain ends in a
          // dense R x 1 mode -- the closing dot runs on the C fragments (the
          // last-mode rows of the step's samples are loaded before its MMAs)
          // and the state is never written back: no separate last-mode pass.
          const int mg = lane >> 2, mt = lane & 3;
          const ModeDev& mlast = ch.m[N - 1];
          const bool fclose = TNB_FUSE_LAST && k == N - 2 && mlast.layout == TNB_LAYOUT_DENSE && mlast.rl == R &&
                              mlast.rr == 1;
          const IdxT* colL = cidx + (size_t)(N - 1) * T;
          if (fclose) k2 = N - 1;
          // fring: the first mode's table rows of this warp's positions are
          // copied with 16-byte cp.async (LDGSTS, one commit group per 16
          // positions, kFringD groups ahead) into the samples' own state rows,
          // which mode 1 then reads as A fragments and overwrites in place --
          // no CTA-wide gather barrier and no exposed load latency per step
          const bool fring = TNB_FFIRST_RING && ffirst && k == 1;
          constexpr int kFringG = TNB_FRING_G;  // positions per cp.async group (16 or 32)
          int g_issued = 0;
          auto issue_group = [&]() {
            const int base = lo + kFringG * g_issued;
            const int rows = min(kFringG, hi - base);
            if (rows > 0) {
              const uint32_t jr = lane < rows ? (bp.wide0 ? widx0[perm[base + lane]] : (uint32_t)cidx[perm[base + lane]])
                                              : 0u;
              const uint32_t sr = lane < rows ? (uint32_t)perm[base + lane] : 0u;
              constexpr bool hot = TNB_RING_CA || HOT;
#pragma unroll
              for (int it = 0; it < kFringG / 4; ++it) {  // kFringG rows x 8 pieces of 16 bytes
                const int i = lane + 32 * it;
                const int row = i >> 3, piece = i & 7;
                const uint32_t j = __shfl_sync(0xffffffffu, jr, row);
                const uint32_t srow = __shfl_sync(0xffffffffu, sr, row);
                if (row < rows)
                  ring_cp16(s_state + srow * (RP * 4) + piece * 16, ch.m[0].s + (int64_t)j * R + piece * 4, hot);
              }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            ++g_issued;
          };
          constexpr int kFringD = TNB_FRING_D;
          if (fring)
            for (int i = 0; i < kFringD; ++i) issue_group();
          while (p < hi) {
            const int key = col[perm[p]];
            const int bend = min((int)st[key + 1], hi);
            uint32_t bh[4][4][2], bl[4][4][2];
            {
              const uint4* gs = reinterpret_cast<const uint4*>(md.s + (int64_t)key * R * R * 2);
              uint32_t f[64];
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                const uint4 v = __ldg(gs + c * 32 + lane);
                f[4 * c] = v.x;
                f[4 * c + 1] = v.y;
                f[4 * c + 2] = v.z;
                f[4 * c + 3] = v.w;
              }
#pragma unroll
              for (int kt = 0; kt < 4; ++kt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    bh[kt][nt][e] = f[(kt * 4 + nt) * 2 + e];
                    bl[kt][nt][e] = f[32 + (kt * 4 + nt) * 2 + e];
                  }
            }
            while (p < bend) {
              const int n = min(16, bend - p);
              if (fring) {  // the groups holding positions p .. p + n - 1 have landed
                const int gneed = (p + n - 1 - lo) / kFringG;
                const int newer = g_issued - 1 - gneed;
                if (newer >= 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
                else if (newer == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
                else if (newer == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
                else asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncwarp();
              }
              const int sa = perm[p + min(mg, n - 1)], sb = perm[p + min(mg + 8, n - 1)];
              const uint32_t r0 = s_state + (uint32_t)sa * (RP * 4);
              const uint32_t r1 = s_state + (uint32_t)sb * (RP * 4);
#if TNB_CLOSE_L1PF
              if (fclose && mt == 0) {
                // the next step's closing rows (the warp's next 16 positions,
                // wherever their bucket): into L1 now, read after its MMAs
                const int pn = p + n;
                if (pn + mg < hi)
                  prefetch_l1(mlast.s + (int64_t)(bp.wideL ? widxL[perm[pn + mg]] : (uint32_t)colL[perm[pn + mg]]) * R);
                if (pn + mg + 8 < hi)
                  prefetch_l1(mlast.s +
                              (int64_t)(bp.wideL ? widxL[perm[pn + mg + 8]] : (uint32_t)colL[perm[pn + mg + 8]]) * R);
              }
#endif
              float2 da[4], db[4];  // closing rows, loaded after the MMAs (before them: spills)
#if TNB_CLOSE_PF_EARLY
              // this step's closing rows into L1 before the MMAs, read after them
              if (fclose && mt == 0) {
                prefetch_l1(mlast.s + (int64_t)(bp.wideL ? widxL[sa] : (uint32_t)colL[sa]) * R);
                prefetch_l1(mlast.s + (int64_t)(bp.wideL ? widxL[sb] : (uint32_t)colL[sb]) * R);
              }
#endif
              float acc[4][4];
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
              float av[4][4];  // A values: rows g, g + 8 x columns 8kt + t, 8kt + t + 4
              if (ffirst && k == 1 && !fring) {
                const float* pa = ch.m[0].s + (int64_t)(bp.wide0 ? widx0[sa] : (uint32_t)cidx[sa]) * R + mt;
                const float* pb = ch.m[0].s + (int64_t)(bp.wide0 ? widx0[sb] : (uint32_t)cidx[sb]) * R + mt;
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                  av[kt][0] = __ldg(pa + 8 * kt);
                  av[kt][1] = __ldg(pb + 8 * kt);
                  av[kt][2] = __ldg(pa + 8 * kt + 4);
                  av[kt][3] = __ldg(pb + 8 * kt + 4);
                }
              } else {
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                  av[kt][0] = lds32(r0 + kt * 32 + mt * 4);
                  av[kt][1] = lds32(r1 + kt * 32 + mt * 4);
                  av[kt][2] = lds32(r0 + kt * 32 + mt * 4 + 16);
                  av[kt][3] = lds32(r1 + kt * 32 + mt * 4 + 16);
                }
              }
#pragma unroll
              for (int kt = 0; kt < 4; ++kt) {
                uint32_t ah[4], al[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) split_tf32_step(av[kt][i], ah[i], al[i]);
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                  mma_tf32(acc[nt], al, bh[kt][nt][0], bh[kt][nt][1]);
                  mma_tf32(acc[nt], ah, bl[kt][nt][0], bl[kt][nt][1]);
                  mma_tf32(acc[nt], ah, bh[kt][nt][0], bh[kt][nt][1]);
                }
              }
              if (fclose) {
                const float* la = mlast.s + (int64_t)(bp.wideL ? widxL[sa] : (uint32_t)colL[sa]) * R + 2 * mt;
                const float* lb = mlast.s + (int64_t)(bp.wideL ? widxL[sb] : (uint32_t)colL[sb]) * R + 2 * mt;
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                  da[nt] = __ldg(reinterpret_cast<const float2*>(la + 8 * nt));
                  db[nt] = __ldg(reinterpret_cast<const float2*>(lb + 8 * nt));
                }
                float part0 = 0.f, part1 = 0.f;
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                  part0 = fmaf(acc[nt][0], da[nt].x, part0);
                  part0 = fmaf(acc[nt][1], da[nt].y, part0);
                  part1 = fmaf(acc[nt][2], db[nt].x, part1);
                  part1 = fmaf(acc[nt][3], db[nt].y, part1);
                }
                // reduce-scatter over the 4 lanes of a row: odd lanes finish row g + 8
                const bool odd = mt & 1;
                float keep = odd ? part1 : part0;
                keep += __shfl_xor_sync(0xffffffffu, odd ? part0 : part1, 1);
                keep += __shfl_xor_sync(0xffffffffu, keep, 2);
                if (mt < 2 && mg + 8 * mt < n) out[s0 + (mt ? sb : sa)] = keep;
              } else {
                __syncwarp();  // every row of the step has been read
                if (mg < n) {
#pragma unroll
                  for (int nt = 0; nt < 4; ++nt) sts_b64(r0 + nt * 32 + mt * 8, pack2(acc[nt][0], acc[nt][1]));
                }
                if (mg + 8 < n) {
#pragma unroll
                  for (int nt = 0; nt < 4; ++nt) sts_b64(r1 + nt * 32 + mt * 8, pack2(acc[nt][2], acc[nt][3]));
                }
                __syncwarp();
              }
              p += n;
              if (fring)  // groups wholly consumed -> the next ones
                while (g_issued < (p - lo) / kFringG + kFringD && lo + kFringG * g_issued < hi) issue_group();
            }
          }
          if (fring) asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
#endif
        while (p < hi) {
          const int key = col[perm[p]];
          const int bend = min((int)st[key + 1], hi);
          {
            // K-split geometry: lane (h, qq) owns rows 16h..16h+15 and the
            // column pair (2qq, 2qq+1); one sample per pass, the two row
            // halves are summed with one 64-bit shuffle.  Halves the core
            // registers (32) so 8 passes stay in flight.
            const int h = lane >> 4, qq = lane & 15;
            uint64_t g2[16];
            const float* gs = md.s + (int64_t)key * rl * rr;
            if (bp.lmaj[k]) {  // lane-major slice: 8 x 16-byte loads, chunk c = (g2[2c], g2[2c+1])
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const ulonglong2 v = ldg_u2(gs + (c * 32 + lane) * 4);
                g2[2 * c] = v.x;
                g2[2 * c + 1] = v.y;
              }
            } else if (rl == R && rr == R) {
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
          }
        }
        } else {
          // one bucket per warp at a time: all G groups take samples of it
          int p = lo;
          while (p < hi) {
            const int key = col[perm[p]];
            const int bend = min((int)st[key + 1], hi);
            // core slice -> registers (see Geo for the column ownership)
            constexpr int C1 = (C == 3) ? 1 : 0;
            uint64_t g2[R];
            float g1[C1 ? R : 1];
            const float* gs = md.s + (int64_t)key * rl * rr;
            const int cp = 2 * q, cs = 16 + q;
            if (bp.lmaj[k]) {  // lane-major slice: 16-byte loads (g2 pairs, then g1)
#pragma unroll
              for (int c = 0; c < R / 2; ++c) {
                const ulonglong2 v = ldg_u2(gs + (c * L + q) * 4);
                g2[2 * c] = v.x;
                g2[2 * c + 1] = v.y;
              }
              if constexpr (C1) {
#pragma unroll
                for (int c = 0; c < R / 4; ++c) {
                  const float4 v = __ldg(reinterpret_cast<const float4*>(gs + ((R / 2 + c) * L + q) * 4));
                  g1[4 * c] = v.x;
                  g1[4 * c + 1] = v.y;
                  g1[4 * c + 2] = v.z;
                  g1[4 * c + 3] = v.w;
                }
              }
            } else if (rl == R && rr == R) {  // full rank: unpredicated 8-byte loads
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
              for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 0], v[pi].x);
              #pragma unroll
              for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 1], v[pi].y);
              #pragma unroll
              for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 2], v[pi].z);
              #pragma unroll
              for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi], g2[a4 * 4 + 3], v[pi].w);
              if constexpr (C1) {
              #pragma unroll
                for (int pi = 0; pi < P; ++pi) {
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
      if (tid == 0) {
        // cidx rows k..k2 of this tile are dead: prefetch the next tile's rows
        if (ntile < ntiles) {
          const int kpost0 = ffirst ? 1 : 0;  // the first post-mode section of the tile
          if (k == kpost0) mb_expect(cbar, row_bytes * N + wrow_bytes * bp.nw);
          // rows of a folded diagonal run stay live until the last mode
          const int klo = (FOLD && k == N - 1 && fold >= 0) ? fold : (k == kpost0 ? 0 : k);
          if (!(FOLD && fold >= 0 && k >= fold && k < N - 1))
            for (int kk = klo; kk <= k2; ++kk)
              bulk(cidx + (size_t)kk * T, ws + ntile * bp.tile_bytes + (size_t)kk * row_bytes, row_bytes, cbar);
          const unsigned char* nrec = ws + ntile * bp.tile_bytes + bp.off_wide;
          if (k == kpost0 && bp.wide0) bulk(widx, nrec, wrow_bytes, cbar);
          if (k2 == N - 1 && bp.wideL) bulk(widx + (size_t)bp.wide0 * T, nrec + (size_t)bp.wide0 * wrow_bytes, wrow_bytes, cbar);
        }
        if (sorted) issue_slot(item + 2);  // this slot buffer is free again
      }
      if (sorted) ++item;
      k = k2;
    }
  }
}

// ---------------------------------------------------------------------------
// STREAM compute kernel: virtual chains with exactly ONE sorted mode, right
// after the first one:   first (row gather) . G (R x R, sorted) . D* . last
// (cfg5 after merging: P012 . G3 . D45 . S67).  There is no per-sample state
// array, so a tile is not bounded by shared memory (T = 4096: a bucket holds
// T / J samples, 32 at J = 128, against 16 in the state kernel).
//   * the CTA streams tile records (compact indices, permutation, bucket
//     starts) into a double buffer with one cp.async.bulk each;
//   * each warp owns a contiguous range of sorted positions and is its own
//     producer: its lanes gather the first-mode rows of the next samples, in
//     sorted order, into a per-warp ring of kSD chunks x kSC rows with
//     cp.async.bulk (the prefix table may be HBM-resident: the ring keeps
//     kSD*kSC rows in flight), running ahead into the next tile's range;
//   * per bucket the slice goes to registers once (Geo<R> column ownership)
//     and a lane group evaluates a whole sample: w = v G on its columns,
//     times the diagonal rows and the last row on those columns (direct L2
//     loads), reduced over the group -> out[s].
#ifndef TNB_STREAM_SC
#define TNB_STREAM_SC 32
#endif
#ifndef TNB_STREAM_SD
#define TNB_STREAM_SD 2
#endif
constexpr int kSC = TNB_STREAM_SC;  // rows per ring chunk (16 or 32)
constexpr int kSD = TNB_STREAM_SD;  // chunks per warp ring (power of two; ring row = sequence number % (kSC kSD))

__device__ __forceinline__ bool mb_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(s32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}

// ND: diagonal modes between the sorted and the last mode (0 or 1).  Stream
// plans store the first and last modes' indices as uint32 rows (wide0 and
// wideL are always set), the sorted and diagonal ones as IdxT.
// MMA: the per-bucket (n x R) @ (R x R) products run on the tensor cores
// (mma.sync m16n8k8, split TF32, 16 samples per warp step) with the slice's
// B fragments pre-split into hi / lo by the table build (mma_slice_kernel);
// otherwise FFMA2 lane groups (Geo<R>).
// HOT: the first-mode ring copies through L1 (repeated rows, see
// detect_hot_kernel).  Both instantiations are launched back to back; the one
// that does not match the device flag returns at once (~2 us), so each keeps
// the code generation of a compile-time copy instruction.
template <int R, typename IdxT, int NT, int ND, bool MMA, bool HOT>
__global__ void __launch_bounds__(NT, 1)
    entries_stream_kernel(const __grid_constant__ ChainDev ch, const __grid_constant__ BPlan bp,
                          const unsigned char* __restrict__ ws, int64_t m, float* __restrict__ out) {
  if ((bp.hot != nullptr && __ldg(bp.hot) != 0) != HOT) return;
  using Gm = Geo<R>;
  constexpr int C = Gm::C, L = Gm::L, G = Gm::G, P = Gm::P;
  constexpr int NW = NT / 32;
  constexpr int RING = kSC * kSD;
  constexpr int C1 = (C == 3) ? 1 : 0;
  // ring row stride (floats): R + 4 makes the A-fragment loads conflict-free;
  // at R = 24 an XOR swizzle of the 16-byte pieces does the same without the
  // padding (piece p of ring row q stored at p ^ ((q >> 2) & 1))
  constexpr bool SWZ = MMA && R == 24 && TNB_STREAM_SWZ;
  constexpr int RS = MMA ? (SWZ ? R : R + 4) : R;
  constexpr int KT = R / 8;            // MMA k- and n-tiles
  extern __shared__ __align__(128) unsigned char smem[];
  const int N = ch.n, T = bp.T;
  const int64_t TB = bp.tile_bytes;
  constexpr int NR = TNB_STREAM_NREC;
  unsigned char* recs = smem;                                                // [NR][tile_bytes]
  float* ring = reinterpret_cast<float*>(smem + NR * TB);                    // [NW][RING][RS]
  uint64_t* rbar = reinterpret_cast<uint64_t*>(ring + (size_t)NW * RING * RS);  // [2]
  uint64_t* gbar = rbar + NR;                                                // [NW][kSD]
  int* rdone = reinterpret_cast<int*>(gbar + NW * kSD);                      // [NR]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gi = lane / L, q = lane % L;
  const int cp = 2 * q, cs = 16 + q;
  const int64_t ntiles = bp.ntiles;
  const float* ftab = ch.m[0].s;
  const float* gtab = ch.m[1].s;
  const float* dtab = ch.m[ND ? 2 : 0].s;
  const float* ltab = ch.m[N - 1].s;
  const bool lmaj = bp.lmaj[1] != 0;
  uint64_t* wbar = gbar + warp * kSD;
  float* wring = ring + (size_t)warp * RING * RS;
  const uint32_t s_ring = s32(wring);

  auto tile_of = [&](int64_t ti) { return (int64_t)blockIdx.x + ti * gridDim.x; };
  // the warp's sorted-position range of tile iteration ti (empty past the end)
  auto range_of = [&](int64_t ti, int& lo, int& hi) {
    const int64_t tile = tile_of(ti);
    if (tile >= ntiles) {
      lo = hi = 0;
      return false;
    }
    const int64_t s0 = tile * T;
    const int tn = (int)((m - s0) < T ? (m - s0) : T);
    lo = (int)(((int64_t)warp * tn) / NW);
    hi = (int)(((int64_t)(warp + 1) * tn) / NW);
    return true;
  };
  auto load_rec = [&](int64_t ti) {  // tid 0
    const int64_t tile = tile_of(ti);
    if (tile >= ntiles) return;
    uint64_t* b = &rbar[ti % NR];
    mb_expect(b, (uint32_t)TB);
    bulk(recs + (ti % NR) * TB, ws + tile * TB, (uint32_t)TB, b);
  };
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) mb_init(&rbar[i], 1);
    for (int i = 0; i < NW * kSD; ++i) mb_init(&gbar[i], 1);
    for (int i = 0; i < NR; ++i) rdone[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < NR; ++i) load_rec(i);
  }
  __syncthreads();

  // Ring bookkeeping in per-warp SEQUENCE numbers: a tile's range occupies
  // [seq0, seq0 + hi - lo), seq0 a multiple of kSC, so a chunk (kSC
  // consecutive sequence numbers) never spans two tiles; ring row = seq & 63.
  int64_t pti = 0;  // producer: tile iteration being issued, its range, next chunk
  int plo, phi;
  bool pvalid = range_of(0, plo, phi);
  int pcc = 0;
  uint32_t c_issued = 0, c_waited = 0;
  int64_t cti = 0;  // consumer tile iteration
  auto try_issue = [&](bool block) -> bool {
    while (true) {
      if (!pvalid) return false;
      if (pcc * kSC < phi - plo) break;
      if (pti > cti) return false;  // never more than one tile ahead
      ++pti;
      pvalid = range_of(pti, plo, phi);
      pcc = 0;
    }
    const int b = (int)(pti % NR);
    if (pti > cti && !mb_test(&rbar[b], (uint32_t)((pti / NR) & 1))) {  // next tile's record
      if (!block) return false;
      mb_wait(&rbar[b], (uint32_t)((pti / NR) & 1));
    }
    const unsigned char* rec = recs + b * TB;
    const int n = min(kSC, phi - plo - pcc * kSC);
    const int slot = (int)(c_issued & (kSD - 1));
    __syncwarp();
#if TNB_STREAM_LDGSTS
    {
      // lane r < n looks up row r's table index once; the 16-byte pieces go
      // piece-major over the lanes (consecutive lanes, consecutive bytes of
      // a row) with the index broadcast by a shuffle
      const uint32_t jr = lane < n ? reinterpret_cast<const uint32_t*>(rec + bp.off_wide)[
                                         reinterpret_cast<const uint16_t*>(rec + bp.off_perm)[plo + pcc * kSC + lane]]
                                   : 0u;
      const uint32_t dst0 = s_ring + (uint32_t)(slot * kSC * RS * 4);
      const uint32_t kmask = bp.kpack ? (1u << bp.kshift) - 1u : ~0u;
      constexpr bool hot = TNB_RING_CA || HOT;
#pragma unroll
      for (int it = 0; it < (kSC * R / 4 + 31) / 32; ++it) {
        const int i = lane + 32 * it;
        const int row = i / (R / 4), piece = i - row * (R / 4);
        const uint32_t j = __shfl_sync(0xffffffffu, jr, row & 31) & kmask;
        if (row < n)
          ring_cp16(dst0 + (uint32_t)(row * RS * 4 + (SWZ ? piece ^ (((slot * kSC + row) >> 2) & 1) : piece) * 16),
                    ftab + (int64_t)j * R + piece * 4, hot);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
#else
    if (lane == 0) mb_expect(&wbar[slot], (uint32_t)(n * R * 4));
    __syncwarp();
    if (lane < n) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int s = reinterpret_cast<const uint16_t*>(rec + bp.off_perm)[plo + pcc * kSC + lane];
      const uint32_t j = reinterpret_cast<const uint32_t*>(rec + bp.off_wide)[s];
      bulk(wring + (slot * kSC + lane) * RS, ftab + (int64_t)j * R, R * 4, &wbar[slot]);
    }
#endif
#if TNB_STREAM_PF
    {
      const int pf = plo + (pcc + TNB_STREAM_PF) * kSC + (lane & (kSC - 1));
      if (pf < phi) {
        const int s = reinterpret_cast<const uint16_t*>(rec + bp.off_perm)[pf];
        const uint32_t j = reinterpret_cast<const uint32_t*>(rec + bp.off_wide)[s] & (bp.kpack ? (1u << bp.kshift) - 1u : ~0u);
        const float* a = ftab + (int64_t)j * R + (lane >= kSC ? R - 1 : 0);  // first and last line of the row
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        if (kSC == 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(a + R - 1));
      }
    }
#endif
    ++pcc;
    ++c_issued;
    return true;
  };

  uint32_t seq0 = 0, last_try = ~0u;
  for (;; ++cti) {
    const int64_t tile = tile_of(cti);
    if (tile >= ntiles) break;
    const int b = (int)(cti % NR);
    mb_wait(&rbar[b], (uint32_t)((cti / NR) & 1));
    const unsigned char* rec = recs + b * TB;
    // compact rows start at mode 1 (crow0 == 1): sorted mode 1, diagonal
    // mode 2, then the last mode unless it is wide (uint32 row after the
    // first mode's)
    const int rfirst = 1 + bp.kpack;  // first mode with a compact row in the record
    const IdxT* ckey = reinterpret_cast<const IdxT*>(rec);
    const uint32_t* cfirst = reinterpret_cast<const uint32_t*>(rec + bp.off_wide);
    const IdxT* cdiag = reinterpret_cast<const IdxT*>(rec) + (size_t)(2 - rfirst) * T;
    const IdxT* clastc = reinterpret_cast<const IdxT*>(rec) + (size_t)(N - 1 - rfirst) * T;
    const uint32_t* clastw = reinterpret_cast<const uint32_t*>(rec + bp.off_wide) + (size_t)T;
    const bool wl = bp.wideL != 0;
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(rec + bp.off_perm);
    const uint16_t* st = reinterpret_cast<const uint16_t*>(rec + bp.off_starts);
    float* otile = out + tile * T;
    int lo, hi;
    range_of(cti, lo, hi);
    const uint32_t sbase = seq0 - (uint32_t)lo;  // seq of position p = sbase + p
    // closing rows (last mode, diagonal mode) of positions q0 + w: raw loads
    // whose latency the next iteration's FMA loop covers
    float2 nlp[P], ndp[P];
    float nls[P], nds[P];
    auto load_close = [&](int q0) {
#pragma unroll
      for (int pi = 0; pi < P; ++pi) {
        const int pos = min(q0 + pi * G + gi, hi - 1);
        const int s = perm[pos];
        const float* lr = ltab + (int64_t)(wl ? clastw[s] : (uint32_t)clastc[s]) * R;
        nlp[pi] = __ldg(reinterpret_cast<const float2*>(lr + cp));
        nls[pi] = C1 ? __ldg(lr + cs) : 0.f;
        if constexpr (ND) {
          const float* dr = dtab + (int64_t)cdiag[s] * R;
          ndp[pi] = __ldg(reinterpret_cast<const float2*>(dr + cp));
          nds[pi] = C1 ? __ldg(dr + cs) : 0.f;
        }
      }
    };
    // MMA: the same for rows g, g + 8 of a 16-sample step, columns 8nt + 2t
    const int mg = lane >> 2, mt = lane & 3;
    float2 mlp[2][KT], mdp[2][KT];
    auto load_close_mma = [&](int q0) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int s = perm[min(q0 + mg + 8 * r, hi - 1)];
        const float* lr = ltab + (int64_t)(wl ? clastw[s] : (uint32_t)clastc[s]) * R + 2 * mt;
        const float* dr = dtab + (int64_t)cdiag[s] * R + 2 * mt;
#pragma unroll
        for (int nt = 0; nt < KT; ++nt) {
          mlp[r][nt] = __ldg(reinterpret_cast<const float2*>(lr + 8 * nt));
          if constexpr (ND) mdp[r][nt] = __ldg(reinterpret_cast<const float2*>(dr + 8 * nt));
        }
      }
    };
    if (lo < hi) {
      if constexpr (MMA) load_close_mma(lo);
      else load_close(lo);
    }
    while (c_issued < (seq0 / kSC) + kSD && try_issue(false)) {
    }
    int p = lo;
    while (p < hi) {
      const int key = bp.kpack ? (int)(cfirst[perm[p]] >> bp.kshift) : (int)ckey[perm[p]];
      const int bend = min((int)st[key + 1], hi);
      uint64_t g2[MMA ? 1 : R];
      float g1[(C1 && !MMA) ? R : 1];
      uint32_t bh[MMA ? KT : 1][MMA ? KT : 1][2], bl[MMA ? KT : 1][MMA ? KT : 1][2];
      const float* gs = gtab + (int64_t)key * R * R * (MMA ? 2 : 1);
      if constexpr (MMA) {
        // [chunk][lane][4]: hi fragments (kt, nt, 2) then lo fragments
        uint32_t f[4 * KT * KT];
#pragma unroll
        for (int c = 0; c < KT * KT; ++c) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(gs) + c * 32 + lane);
          f[4 * c] = v.x;
          f[4 * c + 1] = v.y;
          f[4 * c + 2] = v.z;
          f[4 * c + 3] = v.w;
        }
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int nt = 0; nt < KT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              bh[kt][nt][e] = f[(kt * KT + nt) * 2 + e];
              bl[kt][nt][e] = f[2 * KT * KT + (kt * KT + nt) * 2 + e];
            }
      } else if (lmaj) {
#pragma unroll
        for (int c = 0; c < R / 2; ++c) {
          const ulonglong2 v = ldg_u2(gs + (c * L + q) * 4);
          g2[2 * c] = v.x;
          g2[2 * c + 1] = v.y;
        }
        if constexpr (C1) {
#pragma unroll
          for (int c = 0; c < R / 4; ++c) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(gs + ((R / 2 + c) * L + q) * 4));
            g1[4 * c] = v.x;
            g1[4 * c + 1] = v.y;
            g1[4 * c + 2] = v.z;
            g1[4 * c + 3] = v.w;
          }
        }
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a) {
          g2[a] = ldg_b64(gs + a * R + cp);
          if constexpr (C1) g1[a] = __ldg(gs + a * R + cs);
        }
      }
      while (p < bend) {
        const int n = min(MMA ? 16 : P * G, bend - p);
        // ring chunks up to the one holding position p + n - 1
        const uint32_t cneed = (sbase + (uint32_t)(p + n - 1)) / kSC;
        while (c_waited <= cneed) {
          while (c_issued <= c_waited) try_issue(true);
#if TNB_STREAM_LDGSTS
          // chunk c_waited complete: at most c_issued - 1 - c_waited newer groups pending
          switch (min(c_issued - 1 - c_waited, (uint32_t)kSD - 1)) {
            case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
            case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
            case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
            default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
          }
          __syncwarp();
#else
          mb_wait(&wbar[c_waited & (kSD - 1)], (c_waited / kSD) & 1);
#endif
          ++c_waited;
        }
        if constexpr (MMA) {
          // rows g, g + 8 of the step = sorted positions p + g, p + g + 8
          // (clamped into the bucket: padding rows recompute a real sample)
          int sr[2];
          uint32_t vr[2], vb16[2];
          float2 dcl[2][KT];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int pos = p + min(mg + 8 * r, n - 1);
            sr[r] = perm[pos];
            const uint32_t q = (sbase + (uint32_t)pos) % RING;
            vr[r] = s_ring + q * (RS * 4) + mt * 4;
            vb16[r] = SWZ ? ((q >> 2) & 1) * 16 : 0;
#pragma unroll
            for (int nt = 0; nt < KT; ++nt) {
              dcl[r][nt] = mlp[r][nt];
              if constexpr (ND) {
                dcl[r][nt].x *= mdp[r][nt].x;
                dcl[r][nt].y *= mdp[r][nt].y;
              }
            }
          }
          if (p + n < hi) load_close_mma(p + n);
          float acc[KT][4];
#pragma unroll
          for (int nt = 0; nt < KT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            uint32_t ah[4], al[4];
            split_tf32_step(lds32(vr[0] + kt * 32 + vb16[0]), ah[0], al[0]);
            split_tf32_step(lds32(vr[1] + kt * 32 + vb16[1]), ah[1], al[1]);
            split_tf32_step(lds32(vr[0] + kt * 32 + 16 - vb16[0]), ah[2], al[2]);
            split_tf32_step(lds32(vr[1] + kt * 32 + 16 - vb16[1]), ah[3], al[3]);
#pragma unroll
            for (int nt = 0; nt < KT; ++nt) {
              mma_tf32(acc[nt], al, bh[kt][nt][0], bh[kt][nt][1]);
              mma_tf32(acc[nt], ah, bl[kt][nt][0], bl[kt][nt][1]);
              mma_tf32(acc[nt], ah, bh[kt][nt][0], bh[kt][nt][1]);
            }
          }
          float part0 = 0.f, part1 = 0.f;
#pragma unroll
          for (int nt = 0; nt < KT; ++nt) {
            part0 = fmaf(acc[nt][0], dcl[0][nt].x, part0);
            part0 = fmaf(acc[nt][1], dcl[0][nt].y, part0);
            part1 = fmaf(acc[nt][2], dcl[1][nt].x, part1);
            part1 = fmaf(acc[nt][3], dcl[1][nt].y, part1);
          }
          // reduce-scatter over the 4 lanes of a row: odd lanes finish row g + 8
          const bool odd = mt & 1;
          float keep = odd ? part1 : part0;
          keep += __shfl_xor_sync(0xffffffffu, odd ? part0 : part1, 1);
          keep += __shfl_xor_sync(0xffffffffu, keep, 2);
          if (mt < 2 && mg + 8 * mt < n) otile[mt ? sr[1] : sr[0]] = keep;
        } else {
        int sp[P];
        uint32_t vrow[P];
        float2 dp[P];
        float ds[P];
        // this iteration's closing rows (loaded one iteration ahead), then
        // the prefetch for positions p + n .. (the next iteration, whatever
        // its bucket)
#pragma unroll
        for (int pi = 0; pi < P; ++pi) {
          dp[pi] = nlp[pi];
          ds[pi] = nls[pi];
          if constexpr (ND) {
            dp[pi].x *= ndp[pi].x;
            dp[pi].y *= ndp[pi].y;
            if constexpr (C1) ds[pi] *= nds[pi];
          }
        }
        if (p + n < hi) load_close(p + n);
#pragma unroll
        for (int pi = 0; pi < P; ++pi) {
          const int w = pi * G + gi;
          const int pos = p + (w < n ? w : n - 1);
          sp[pi] = perm[pos];
          vrow[pi] = s_ring + ((sbase + (uint32_t)pos) % RING) * (R * 4);
        }
        // two accumulator sets per sample (even / odd rows): 2P independent
        // FFMA2 chains instead of P
        uint64_t acc2[P][2];
        float acc1[P][2];
#pragma unroll
        for (int pi = 0; pi < P; ++pi) {
          acc2[pi][0] = acc2[pi][1] = 0ull;
          acc1[pi][0] = acc1[pi][1] = 0.f;
        }
#pragma unroll
        for (int a4 = 0; a4 < R / 4; ++a4) {
          float4 v[P];
#pragma unroll
          for (int pi = 0; pi < P; ++pi) v[pi] = lds128(vrow[pi] + a4 * 16);
#pragma unroll
          for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi][0], g2[a4 * 4 + 0], v[pi].x);
#pragma unroll
          for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi][1], g2[a4 * 4 + 1], v[pi].y);
#pragma unroll
          for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi][0], g2[a4 * 4 + 2], v[pi].z);
#pragma unroll
          for (int pi = 0; pi < P; ++pi) ffma2(acc2[pi][1], g2[a4 * 4 + 3], v[pi].w);
          if constexpr (C1) {
#pragma unroll
            for (int pi = 0; pi < P; ++pi) {
              acc1[pi][0] = fmaf(v[pi].x, g1[a4 * 4 + 0], acc1[pi][0]);
              acc1[pi][1] = fmaf(v[pi].y, g1[a4 * 4 + 1], acc1[pi][1]);
              acc1[pi][0] = fmaf(v[pi].z, g1[a4 * 4 + 2], acc1[pi][0]);
              acc1[pi][1] = fmaf(v[pi].w, g1[a4 * 4 + 3], acc1[pi][1]);
            }
          }
        }
        float part[P];
#pragma unroll
        for (int pi = 0; pi < P; ++pi) {
          const uint64_t w2 = add2(acc2[pi][0], acc2[pi][1]);
          const float2 w = *reinterpret_cast<const float2*>(&w2);
          float a = w.x * dp[pi].x;
          a = fmaf(w.y, dp[pi].y, a);
          if constexpr (C1) a = fmaf(acc1[pi][0] + acc1[pi][1], ds[pi], a);
          part[pi] = a;
        }
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
#pragma unroll
          for (int pi = 0; pi < P; ++pi) part[pi] += __shfl_xor_sync(0xffffffffu, part[pi], o);
        }
        if (q == 0) {
#pragma unroll
          for (int pi = 0; pi < P; ++pi)
            if (pi * G + gi < n) otile[sp[pi]] = part[pi];
        }
        }
        p += n;
        // chunks wholly consumed -> refill the ring (this tile, then the
        // next); a failed look-ahead is retried only after the next chunk
        const uint32_t consumed = (sbase + (uint32_t)p) / kSC;
        if (consumed != last_try && c_issued < consumed + kSD) {
          last_try = consumed;
          while (c_issued < consumed + kSD && try_issue(false)) {
          }
        }
      }
    }
    seq0 += (uint32_t)((hi - lo + kSC - 1) / kSC * kSC);
    while (c_issued < seq0 / kSC + kSD && try_issue(false)) {
    }
    // the LAST warp done with record buffer b reloads it (no CTA barrier:
    // warps drift apart by up to a tile)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int old = atomicAdd(&rdone[b], 1);
      if (old == (int)((cti / NR) + 1) * NW - 1) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        load_rec(cti + NR);
      }
    }
  }
}

// large dense table levels on tcgen05
#include "table_tc5.cuh"

// ---- prefix / suffix tables for mode merging -------------------------------
// prefix step (rows in C order of the merged indices):
//   out[(p*J + j)*rr + c] = sum_a in[p*rl + a] * G(j, a, c)      (dense)
//                         = in[p*rl + c] * D(j, c)               (CP diagonal)
__global__ void table_prefix_step(ModeDev md, const float* __restrict__ in, int64_t P,
                                  float* __restrict__ out) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int64_t total = P * J * rr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t / ((int64_t)J * rr);
    const int64_t r = t - p * J * rr;
    const int j = (int)(r / rr), c = (int)(r - (int64_t)(r / rr) * rr);
    const float* x = in + p * rl;
    float acc;
    if (md.layout == TNB_LAYOUT_DIAG) {
      acc = x[c] * __ldg(md.s + (int64_t)j * rl + c);
    } else {
      acc = 0.f;
      const float* g = md.s + (int64_t)j * rl * rr + c;
      for (int a = 0; a < rl; ++a) acc = fmaf(x[a], __ldg(g + (int64_t)a * rr), acc);
    }
    out[t] = acc;
  }
}

// suffix step (row = j * n + x, the new mode's index slowest):
//   out[(j*n + x)*rl + a] = sum_c G(j, a, c) * in[x*rr + c]     (dense)
//                         = D(j, a) * in[x*rr + a]               (CP diagonal)
__global__ void __launch_bounds__(256) table_suffix_step(ModeDev md, const float* __restrict__ in,
                                                          int64_t n, float* __restrict__ out) {
  // block = (chunk of x, one j): the slice G(j) is staged transposed in
  // shared memory so lane a reads GT[c][a] (conflict-free) while in[x] rows
  // are broadcast; output rows are written coalesced
  __shared__ float gt[32 * 33];
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int j = blockIdx.y;
  if (md.layout != TNB_LAYOUT_DIAG)
    for (int e = threadIdx.x; e < rl * rr; e += blockDim.x) {
      const int a = e / rr, c = e - (e / rr) * rr;
      gt[c * 33 + a] = __ldg(md.s + (int64_t)j * rl * rr + e);
    }
  __syncthreads();
  const int per = blockDim.x / rl;  // x rows per pass
  const int xl = threadIdx.x / rl, a = threadIdx.x - xl * rl;
  if (xl >= per) return;
  for (int64_t x = blockIdx.x * (int64_t)per + xl; x < n; x += (int64_t)gridDim.x * per) {
    const float* y = in + x * rr;
    float acc;
    if (md.layout == TNB_LAYOUT_DIAG) {
      acc = __ldg(md.s + (int64_t)j * rl + a) * y[a];
    } else {
      acc = 0.f;
      for (int c = 0; c < rr; ++c) acc = fmaf(gt[c * 33 + a], y[c], acc);
    }
    out[((int64_t)j * n + x) * rl + a] = acc;
  }
  (void)J;
}

// suffix step for ranks above 32 (the staged kernel's 32 x 33 tile): slices
// read through L1 / L2 (two-table chains of rank 64 and up)
__global__ void __launch_bounds__(256) table_suffix_step_big(ModeDev md, const float* __restrict__ in, int64_t n,
                                                              float* __restrict__ out) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int64_t total = (int64_t)J * n * rl;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / rl;
    const int a = (int)(t - row * rl);
    const int j = (int)(row / n);
    const int64_t x = row - (int64_t)j * n;
    const float* y = in + x * rr;
    float acc;
    if (md.layout == TNB_LAYOUT_DIAG) {
      acc = __ldg(md.s + (int64_t)j * rl + a) * y[a];
    } else {
      acc = 0.f;
      const float* g = md.s + ((int64_t)j * rl + a) * rr;
      for (int c = 0; c < rr; ++c) acc = fmaf(__ldg(g + c), y[c], acc);
    }
    out[t] = acc;
  }
}

// Dense table steps as a tiled SIMT GEMM (the naive steps above re-read the
// input row per output element and ran the FMA pipe at < 10%).  Per z = j:
//   prefix: C_j[i][n] = sum_k A[i][k] G(j, k, n)  -> out[(i*J + j)*Nn + n]
//   suffix: C_j[i][n] = sum_k A[i][k] G(j, n, k)  -> out[(j*rows + i)*Nn + n]
// K, Nn <= 32 and Nn % 4 == 0.  CTA tile: 256 rows of A (transposed into
// shared memory once) x kTZ slices; thread = 8 rows x 4 columns, so a warp's
// 8 column quads of one row are one 128-byte store.
// dense table levels on tensor cores (split TF32) when K == Nn in {8..32}
#ifndef TNB_TABLE_TC
#define TNB_TABLE_TC 1
#endif
#ifndef TNB_TABLE_TZ
#define TNB_TABLE_TZ 4
#endif
constexpr int kTRows = 256, kTZ = TNB_TABLE_TZ;
template <bool SUFFIX>
__global__ void __launch_bounds__(256) table_gemm(ModeDev md, const float* __restrict__ A, int64_t rows,
                                                  float* __restrict__ out) {
  __shared__ __align__(16) float As[32][kTRows + 4];
  __shared__ __align__(16) float Bs[32][32];
  const int J = md.J;
  const int K = SUFFIX ? md.rr : md.rl, Nn = SUFFIX ? md.rl : md.rr;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  const int64_t i0 = (int64_t)blockIdx.x * kTRows;
  const int nr = (int)(rows - i0 < kTRows ? rows - i0 : kTRows);
  for (int e = tid; e < kTRows * K; e += 256) {
    const int r = e / K, k = e - r * K;
    As[k][r] = r < nr ? __ldg(A + i0 * K + e) : 0.f;
  }
  const bool colok = 4 * tx < Nn;
  for (int j = blockIdx.y * kTZ; j < min(J, (int)(blockIdx.y + 1) * kTZ); ++j) {
    __syncthreads();  // As ready / previous Bs consumed
    const float* g = md.s + (int64_t)j * md.rl * md.rr;
    for (int e = tid; e < md.rl * md.rr; e += 256) {
      const int a = e / md.rr, c = e - a * md.rr;
      if (SUFFIX) Bs[c][a] = __ldg(g + e);
      else Bs[a][c] = __ldg(g + e);
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
    if (colok) {
#pragma unroll 8
      for (int k = 0; k < K; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[k][4 * tx]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          acc[r][0] = fmaf(av[r], b.x, acc[r][0]);
          acc[r][1] = fmaf(av[r], b.y, acc[r][1]);
          acc[r][2] = fmaf(av[r], b.z, acc[r][2]);
          acc[r][3] = fmaf(av[r], b.w, acc[r][3]);
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int ri = ty * 8 + r;
        if (ri >= nr) break;
        const int64_t i = i0 + ri;
        float* dst = SUFFIX ? out + ((int64_t)j * rows + i) * Nn : out + (i * J + j) * Nn;
        *reinterpret_cast<float4*>(dst + 4 * tx) = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      }
    }
  }
}

// The same table steps on tensor cores (mma.sync m16n8k8, split TF32: hi =
// rna(x), lo = x - hi) for K, Nn in {8, 16, 24, 32}: CTA = 128 rows of A
// (staged in shared memory, row stride K + 4: conflict-free fragment loads)
// x 8 slices, warp w owns slice z0 + w (its B fragments stay in registers)
// and walks the 8 row tiles of 16.  Large levels (cfg2: 2^20-row tables)
// are write-bound instead of FFMA-bound.
constexpr int kTcRows = 128, kTcZ = 8;
// TNB_TABLE_STAGE: each 16-row tile of the CTA's 8 slices goes through
// shared memory and leaves as float4 runs (1 KB per prefix row, 2 KB per
// suffix slice) instead of 32-byte float2 pieces from the fragments
#ifndef TNB_TABLE_STAGE
#define TNB_TABLE_STAGE 0  /* measured: tables 0.187 vs 0.168 ms (serial, cfg2) */
#endif
template <int KT, int NTL, bool SUFFIX>
__global__ void __launch_bounds__(256) table_gemm_tc(ModeDev md, const float* __restrict__ A, int64_t rows,
                                                     float* __restrict__ out) {
  constexpr int K = 8 * KT, Nn = 8 * NTL, AS = K + 4;
  __shared__ __align__(16) float As[kTcRows * AS];
#if TNB_TABLE_STAGE
  __shared__ __align__(16) float Os[16 * kTcZ * Nn];  // [row][slice][Nn], 8-column blocks rotated by row
#endif
  const int J = md.J;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int z0 = blockIdx.y * kTcZ;
  const int j = z0 + warp;
  const bool jok = j < J;  // every warp stays for the staging barriers
  // B(k, n) = G(j, k, n) (prefix) or G(j, n, k) (suffix); fragment (kt, nt):
  // b0 = B(8kt + t, 8nt + g), b1 = B(8kt + t + 4, 8nt + g)
  const float* gj = md.s + (int64_t)(jok ? j : 0) * md.rl * md.rr;
  uint32_t bh[KT][NTL][2], bl[KT][NTL][2];
#pragma unroll
  for (int kt = 0; kt < KT; ++kt)
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = 8 * kt + t + 4 * e, n = 8 * nt + g;
        split_tf32(jok ? __ldg(gj + (SUFFIX ? n * K + k : k * Nn + n)) : 0.f, bh[kt][nt][e], bl[kt][nt][e]);
      }
  // the CTA's row chunks (the slice fragments above are loaded once)
  const bool a16 = (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  for (int64_t i0 = (int64_t)blockIdx.x * kTcRows; i0 < rows; i0 += (int64_t)gridDim.x * kTcRows) {
  const int nr = (int)(rows - i0 < kTcRows ? rows - i0 : kTcRows);
  __syncthreads();  // the previous chunk's fragment loads are done
  if (a16) {  // K % 4 == 0: 16-byte loads of the chunk's contiguous rows
    for (int e = tid; e < kTcRows * (K / 4); e += 256) {
      const int r = e / (K / 4), k4 = e - r * (K / 4);
      const float4 v = r < nr ? __ldg(reinterpret_cast<const float4*>(A + i0 * K) + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(As + r * AS + 4 * k4) = v;
    }
  } else {
    for (int e = tid; e < kTcRows * K; e += 256) {
      const int r = e / K, k = e - r * K;
      As[r * AS + k] = r < nr ? __ldg(A + i0 * K + e) : 0.f;
    }
  }
  __syncthreads();
  for (int mt = 0; mt < kTcRows / 16; ++mt) {
    if (mt * 16 >= nr || !jok) break;
    float acc[NTL][4];
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
    const float* a0 = As + (mt * 16 + g) * AS + t;
    const float* a1 = a0 + 8 * AS;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t ah[4], al[4];
      split_tf32_step(a0[8 * kt], ah[0], al[0]);
      split_tf32_step(a1[8 * kt], ah[1], al[1]);
      split_tf32_step(a0[8 * kt + 4], ah[2], al[2]);
      split_tf32_step(a1[8 * kt + 4], ah[3], al[3]);
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt) {
        mma_tf32(acc[nt], al, bh[kt][nt][0], bh[kt][nt][1]);
        mma_tf32(acc[nt], ah, bl[kt][nt][0], bl[kt][nt][1]);
        mma_tf32(acc[nt], ah, bh[kt][nt][0], bh[kt][nt][1]);
      }
    }
#if TNB_TABLE_STAGE
    __syncthreads();  // the previous tile's reads of Os are done
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = g + 8 * h;
      float* orow = Os + (r * kTcZ + warp) * Nn;
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt)
        *reinterpret_cast<float2*>(orow + 8 * ((nt + r) % NTL) + 2 * t) =
            make_float2(acc[nt][2 * h], acc[nt][2 * h + 1]);
    }
    __syncthreads();
    constexpr int F4 = Nn / 4;  // float4 per slice row
    for (int f = tid; f < 16 * kTcZ * F4; f += 256) {
      // prefix: row-major over (row, slice) -> 1 KB runs; suffix: slice-major -> 2 KB runs
      int r, w;
      if (SUFFIX) {
        w = f / (16 * F4);
        r = (f / F4) % 16;
      } else {
        r = f / (kTcZ * F4);
        w = (f / F4) % kTcZ;
      }
      const int c4 = (f % F4) * 4;
      if (mt * 16 + r >= nr || z0 + w >= J) continue;
      const float4 v = *reinterpret_cast<const float4*>(Os + (r * kTcZ + w) * Nn + 8 * ((c4 / 8 + r) % NTL) + c4 % 8);
      const int64_t i = i0 + mt * 16 + r;
      float* dst = SUFFIX ? out + ((int64_t)(z0 + w) * rows + i) * Nn : out + (i * J + z0 + w) * Nn;
      *reinterpret_cast<float4*>(dst + c4) = v;
    }
#else
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = mt * 16 + g + 8 * h;
      if (r >= nr) continue;
      const int64_t i = i0 + r;
      float* dst = SUFFIX ? out + ((int64_t)j * rows + i) * Nn : out + (i * J + j) * Nn;
#pragma unroll
      for (int nt = 0; nt < NTL; ++nt)
        *reinterpret_cast<float2*>(dst + 8 * nt + 2 * t) = make_float2(acc[nt][2 * h], acc[nt][2 * h + 1]);
    }
#endif
  }
  }
}

template <bool SUFFIX>
bool launch_table_tc(const ModeDev& md, const float* in, int64_t rows, float* out, cudaStream_t st) {
  const int K = SUFFIX ? md.rr : md.rl, Nn = SUFFIX ? md.rl : md.rr;
  if (!TNB_TABLE_TC || md.layout != TNB_LAYOUT_DENSE || K != Nn || (K & 7) || K < 8 || K > 32) return false;
  // ~4 CTAs per SM in all; a CTA walks its row chunks with the slice fragments loaded once
  const int64_t gy = ceil_div(md.J, kTcZ);
  const int64_t gx = std::min<int64_t>(ceil_div(rows, kTcRows), std::max<int64_t>(1, ((int64_t)num_sms() * 4) / gy));
  const dim3 grid((unsigned)gx, (unsigned)gy);
  switch (K) {
    case 8: table_gemm_tc<1, 1, SUFFIX><<<grid, 256, 0, st>>>(md, in, rows, out); break;
    case 16: table_gemm_tc<2, 2, SUFFIX><<<grid, 256, 0, st>>>(md, in, rows, out); break;
    case 24: table_gemm_tc<3, 3, SUFFIX><<<grid, 256, 0, st>>>(md, in, rows, out); break;
    default: table_gemm_tc<4, 4, SUFFIX><<<grid, 256, 0, st>>>(md, in, rows, out); break;
  }
  return true;
}

bool table_gemm_ok(const ModeDev& md, bool suffix) {
  const int K = suffix ? md.rr : md.rl, Nn = suffix ? md.rl : md.rr;
  return md.layout == TNB_LAYOUT_DENSE && K >= 1 && K <= 32 && Nn >= 4 && Nn <= 32 && (Nn & 3) == 0;
}

// Lane-major copy of a full-rank (R x R) sorted mode: the values one lane of
// the compute kernel holds are contiguous 16-byte chunks, chunk-major across
// lanes ([chunk][lane][4]) so a warp's load of chunk c is coalesced.
//   R == 32 (K-split, lane = 16h + qq): chunk c = G[16h+2c][2qq..], G[16h+2c+1][2qq..]
//   R <= 24 (Geo, lane q of L): float f < 2R -> G[f/2][2q + f%2],
//                                f >= 2R   -> G[f-2R][16+q]   (R == 24 only)
__global__ void lane_major_kernel(const float* __restrict__ src, float* __restrict__ dst, int J, int R) {
  const int L = R == 32 ? 32 : (R == 24 ? 8 : R / 2);
  const int per = R * R;
  const int64_t total = (int64_t)J * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / per;
    const int r = (int)(t - j * per);
    const int c = r / (L * 4), q = (r / 4) % L, e = r & 3;
    int a, col;
    if (R == 32) {
      a = 16 * (q >> 4) + 2 * c + (e >> 1);
      col = 2 * (q & 15) + (e & 1);
    } else {
      const int f = 4 * c + e;
      if (f < 2 * R) {
        a = f >> 1;
        col = 2 * q + (f & 1);
      } else {
        a = f - 2 * R;
        col = 16 + q;
      }
    }
    dst[t] = __ldg(src + j * per + a * R + col);
  }
}

// Tensor-core copy of the stream plan's sorted mode (R x R slices, R % 8 ==
// 0): per slice [chunk][lane][4] with the lane's m16n8k8 B fragments,
// b(kt, nt, e) = G[8kt + t + 4e][8nt + g] (g = lane / 4, t = lane % 4), first
// rounded to tf32 (hi) for every (kt, nt, e), then the tf32 remainders (lo).
__global__ void mma_slice_kernel(const float* __restrict__ src, float* __restrict__ dst, int J, int R) {
  const int KT = R / 8, nb = 2 * KT * KT;  // hi values per lane
  const int per = 32 * 2 * nb;             // floats per slice
  const int64_t total = (int64_t)J * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / per;
    const int r = (int)(i - j * per);
    const int c = r / 128, lane = (r / 4) % 32, f = 4 * c + (r & 3);
    const int lo = f >= nb, idx = f % nb;
    const int kt = idx / (2 * KT), nt = (idx / 2) % KT, e = idx & 1;
    const int g = lane >> 2, t = lane & 3;
    const float x = __ldg(src + j * R * R + (int64_t)(8 * kt + t + 4 * e) * R + 8 * nt + g);
    uint32_t h, l;
    split_tf32(x, h, l);
    dst[i] = __uint_as_float(lo ? l : h);
  }
}

int pick_R(int rmax);

int lane_major_env() {
  const char* e = getenv("TNB_LANE_MAJOR");
  return (e && e[0] == '0') ? 0 : 1;
}

// Mode merging: the original modes are partitioned into groups, each one
// VIRTUAL mode of the chain the kernels run:
//   prefix [0, a)      -> dense table P[(j_0..j_{a-1})][r_a]    (first mode)
//   suffix [n - b, n)  -> dense table S[(j_{n-b}..j_{n-1})][r]  (last mode)
//   runs of interior CP modes -> diagonal product table D[(j..)][R]
//   every other mode stays as it is.
// Table row indices are the C-order combinations of the original indices
// (the prep kernel combines them).  A group may hold at most min(m / 16,
// 65535) rows: uint16 compact indices, and building a table costs a small
// fraction of the per-entry work it removes (a gathered row replaces one
// dense r x r step or one diagonal gather per merged mode).
// TNB_ENTRIES_MERGE=0 disables merging.
enum GroupKind { kOrig = 0, kPrefix = 1, kSuffix = 2, kDiag = 3 };
struct MergePlan {
  int ng = 0;                    // virtual modes
  int lo[kMaxModes], hi[kMaxModes];
  int kind[kMaxModes];
  int64_t rows[kMaxModes];
  int64_t lvl[kMaxModes];        // byte offset of the level ending at original mode o
  int8_t lm[kMaxModes];          // virtual mode g gets a lane-major copy ...
  int64_t lm_off[kMaxModes];     // ... at this byte offset
  int R = 0;                     // register geometry of the virtual chain
  int64_t table_bytes = 0;       // 256-aligned
  int8_t mma[kMaxModes];         // the copy is the tensor-core fragment layout (hi / lo, 2x size)
  int64_t gemm_off = 0;          // scratch for GEMM-built table levels (transposed core + tcgen05 tiles)
  int64_t gemm_bytes = 0;        // ... its size (the last region of the tables)
  int a() const { return kind[0] == kPrefix ? hi[0] - lo[0] : 1; }
  int b() const { return kind[ng - 1] == kSuffix ? hi[ng - 1] - lo[ng - 1] : 1; }
};

int merge_env() {
  const char* e = getenv("TNB_ENTRIES_MERGE");
  return (e && e[0] == '0') ? 0 : 1;
}

int wide_env() {
  const char* e = getenv("TNB_MERGE_WIDE");
  return (e && e[0] == '0') ? 0 : 1;
}

bool gemm_level(const ModeDev& md) {
  return md.layout == TNB_LAYOUT_DENSE && (md.rl > 32 || md.rr > 32);
}

// A dense PREFIX level is one row-major GEMM, C (P x J*rr) = IN (P x rl) *
// Bt (rl x J*rr) with Bt[a][j][c] = G[j][a][c]: large ones can run on the
// tcgen05 3xTF32 GEMM of full() instead of the mma.sync table kernels.
// Off by default: on the high-priority side stream its one-CTA-per-SM
// persistent kernel takes whole SMs from the concurrent prep kernel (cfg2
// step 2.95 vs 2.80 ms: prep 0.55 vs 0.41 ms; TNB_TABLE_TCGEN05=1 enables it)
bool tc_prefix_level(const ModeDev& md, int64_t rows) {
  const char* e = getenv("TNB_TABLE_TCGEN05");
  const bool on = e && e[0] == '1';
  return on && md.layout == TNB_LAYOUT_DENSE && md.rl <= 64 &&
         tc_gemm_supported(rows, (int64_t)md.J * md.rr, md.rl, md.rl, (int64_t)md.J * md.rr, (int64_t)md.J * md.rr);
}

// G[j][a][c] -> prefix: Bt[a][j][c] (B of C = IN * Bt, rows p, columns (j, c));
//               suffix: GT[j][c][a] (per-j B of C_j = IN * G_j^T)
template <bool SUFFIX>
__global__ void core_transpose_kernel(ModeDev md, float* __restrict__ out) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int64_t total = (int64_t)J * rl * rr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / ((int64_t)rl * rr);
    const int r = (int)(t - j * rl * rr), a = r / rr, c = r - (r / rr) * rr;
    const float v = __ldg(md.s + t);
    if (SUFFIX) out[(j * rr + c) * rl + a] = v;
    else out[((int64_t)a * J + j) * rr + c] = v;
  }
}

int64_t env_rows(const char* name) {
  const char* e = getenv(name);
  return e ? atoll(e) : 0;
}

// wide_rows: row limit of the wide (HBM) prefix / suffix tables (0: m / 8)
void plan_merge(const ChainDev& ch, int64_t m, MergePlan* mp, int64_t wide_rows = 0) {
  const int N = ch.n;
  // uint16-indexed, L2-resident tables: up to min(m/16, 65535) rows.  A
  // prefix / suffix may grow further ("wide": uint32 indices, HBM-resident,
  // up to m/8 rows and 1.5 GB) but only by absorbing DENSE modes -- each
  // one removes a sorted r x r step per entry for one gathered row.
  const int64_t lim = (merge_env() && N >= 3) ? (m / 16 < 65535 ? m / 16 : 65535) : 0;
  const int64_t limw = (lim > 0 && wide_env()) ? std::min<int64_t>(wide_rows > 0 ? wide_rows : m / 8, (int64_t)1 << 30) : lim;
  const double max_table = 1.5e9;
  auto grow = [&](int64_t nr, const ModeDev& md, int width) {
    return nr <= lim || (nr <= limw && md.layout == TNB_LAYOUT_DENSE && (double)nr * width * 4 <= max_table);
  };
  int a = 1, b = 1;
  int64_t rows = ch.m[0].J, rs = ch.m[N - 1].J;
  // plan-exploration caps on the prefix / suffix table rows (0 = planner's choice)
  const int64_t pcap = env_rows("TNB_PREFIX_MAX_ROWS"), scap = env_rows("TNB_SUFFIX_MAX_ROWS");
  if (lim > 0) {
    while (a < N - 1 && grow(rows * ch.m[a].J, ch.m[a], ch.m[a].rr) && (!pcap || rows * ch.m[a].J <= pcap))
      rows *= ch.m[a++].J;
    while (N - 1 - b >= a && grow(rs * ch.m[N - 1 - b].J, ch.m[N - 1 - b], ch.m[N - 1 - b].rl) &&
           (!scap || rs * ch.m[N - 1 - b].J <= scap))
      rs *= ch.m[N - 1 - b++].J;
  }
  mp->table_bytes = 0;
  if (N == 1) {
    mp->ng = 1;
    mp->lo[0] = 0;
    mp->hi[0] = 1;
    mp->kind[0] = kOrig;
    mp->rows[0] = ch.m[0].J;
    mp->lm[0] = 0;
    mp->mma[0] = 0;
    return;
  }
  int g = 0;
  auto add = [&](int lo, int hi, int kind, int64_t r) {
    mp->lo[g] = lo;
    mp->hi[g] = hi;
    mp->kind[g] = kind;
    mp->rows[g] = r;
    ++g;
  };
  if (a > 1) add(0, a, kPrefix, rows);
  else add(0, 1, kOrig, ch.m[0].J);
  for (int o = a; o < N - b;) {
    int e = o + 1;
    int64_t r = ch.m[o].J;
    if (lim > 0 && ch.m[o].layout == TNB_LAYOUT_DIAG)
      while (e < N - b && ch.m[e].layout == TNB_LAYOUT_DIAG && r * ch.m[e].J <= lim) r *= ch.m[e++].J;
    add(o, e, e - o > 1 ? kDiag : kOrig, r);
    o = e;
  }
  if (b > 1) add(N - b, N, kSuffix, rs);
  else add(N - 1, N, kOrig, ch.m[N - 1].J);
  mp->ng = g;
  // table levels: prefix / diag levels end at original mode o (o > lo),
  // suffix levels start at o (o < hi - 1); the group's first level is a view
  int64_t off = 0;
  for (int v = 0; v < g; ++v) {
    const int lo = mp->lo[v], hi = mp->hi[v];
    if (mp->kind[v] == kPrefix || mp->kind[v] == kDiag) {
      int64_t r = ch.m[lo].J;
      for (int o = lo + 1; o < hi; ++o) {
        r *= ch.m[o].J;
        mp->lvl[o] = off;
        off += (r * ch.m[o].rr * 4 + 255) & ~(int64_t)255;
      }
    } else if (mp->kind[v] == kSuffix) {
      int64_t r = ch.m[hi - 1].J;
      for (int o = hi - 2; o >= lo; --o) {
        r *= ch.m[o].J;
        mp->lvl[o] = off;
        off += (r * ch.m[o].rl * 4 + 255) & ~(int64_t)255;
      }
    }
  }
  // lane-major copies of the full-rank sorted modes of the virtual chain
  int vr = 1;
  for (int v = 0; v < g; ++v) {
    const int lo = mp->lo[v], hi = mp->hi[v];
    const int rl = mp->kind[v] == kPrefix ? 1 : ch.m[lo].rl;
    const int rr = mp->kind[v] == kSuffix ? 1 : ch.m[hi - 1].rr;
    vr = max(vr, max(rl, rr));
  }
  mp->R = pick_R(vr);
  for (int v = 0; v < g; ++v) {
    const ModeDev& md = ch.m[mp->lo[v]];
    mp->lm[v] = (int8_t)(lane_major_env() && mp->R && v > 0 && v < g - 1 && mp->kind[v] == kOrig &&
                         md.layout == TNB_LAYOUT_DENSE && md.rl == mp->R && md.rr == mp->R);
    mp->mma[v] = (int8_t)(mp->lm[v] && mp->R == 32 && TNB_STATE_MMA);
    if (mp->lm[v]) {
      mp->lm_off[v] = off;
      off += ((int64_t)md.J * md.rl * md.rr * 4 * (mp->mma[v] ? 2 : 1) + 255) & ~(int64_t)255;
    }
  }
  // table levels of rank > 32 are built as GEMMs against a transposed copy
  // of the level's core (the staged / tensor-core table kernels stop at 32)
  int64_t scratch = 0;
  for (int v = 0; v < g; ++v) {
    if (mp->kind[v] != kPrefix && mp->kind[v] != kSuffix) continue;
    const int lo = mp->lo[v], hi = mp->hi[v];
    const int o0 = mp->kind[v] == kPrefix ? lo + 1 : lo, o1 = mp->kind[v] == kPrefix ? hi : hi - 1;
    int64_t rows = ch.m[lo].J;  // prefix: input rows of level o
    for (int o = o0; o < o1; ++o) {
      const int64_t bt = ((int64_t)ch.m[o].J * ch.m[o].rl * ch.m[o].rr * 4 + 255) & ~(int64_t)255;
      if (gemm_level(ch.m[o])) scratch = std::max<int64_t>(scratch, bt);
      if (mp->kind[v] == kPrefix && tc_prefix_level(ch.m[o], rows))
        scratch = std::max<int64_t>(scratch, bt + tc_gemm_workspace(rows));
      if (mp->kind[v] == kPrefix && t5_level_ok(ch.m[o], rows, false))
        scratch = std::max<int64_t>(scratch, t5_image_bytes(ch.m[o]));
      if (mp->kind[v] == kPrefix) rows *= ch.m[o].J;
    }
    if (mp->kind[v] == kSuffix) {  // suffix levels run from the last mode down: input rows = prod J of the modes above
      int64_t n = ch.m[hi - 1].J;
      for (int o = hi - 2; o >= lo; --o) {
        if (t5_level_ok(ch.m[o], n, true)) scratch = std::max<int64_t>(scratch, t5_image_bytes(ch.m[o]));
        n *= ch.m[o].J;
      }
    }
  }
  mp->gemm_off = off;
  // two halves: the prefix and the suffix chains may run concurrently (build_tables)
  mp->gemm_bytes = 2 * ((scratch + 255) & ~(int64_t)255);
  off += mp->gemm_bytes;
  mp->table_bytes = off;
}

// The virtual chain the kernels run; table pointers are filled when `base`
// is the workspace (nullptr for size queries).
void virtual_chain(const ChainDev& ch, const MergePlan& mp, unsigned char* base, ChainDev* v) {
  v->batch = 1;
  v->n = mp.ng;
  int rmax = 1;
  for (int g = 0; g < mp.ng; ++g) {
    const int lo = mp.lo[g], hi = mp.hi[g];
    ModeDev d = ch.m[lo];
    if (mp.kind[g] != kOrig) {
      const int64_t off = mp.kind[g] == kSuffix ? mp.lvl[lo] : mp.lvl[hi - 1];
      d.s = base ? reinterpret_cast<const float*>(base + off) : nullptr;
      d.bstride = 0;
      d.J = (int32_t)mp.rows[g];
      if (mp.kind[g] == kPrefix) {
        d.layout = TNB_LAYOUT_DENSE;
        d.rl = 1;
        d.rr = ch.m[hi - 1].rr;
      } else if (mp.kind[g] == kSuffix) {
        d.layout = TNB_LAYOUT_DENSE;
        d.rl = ch.m[lo].rl;
        d.rr = 1;
      }  // kDiag keeps layout DIAG and rl == rr == R
    }
    if (mp.lm[g]) d.s = base ? reinterpret_cast<const float*>(base + mp.lm_off[g]) : nullptr;
    v->m[g] = d;
    rmax = max(rmax, max(d.rl, d.rr));
  }
  v->rmax = rmax;
}

// st2 (with the events ea / eb): the suffix table's levels run there,
// concurrently with the prefix / diagonal ones on st -- the two chains are
// independent and their small first levels are launch-latency bound; st waits
// for st2 before build_tables returns.
int build_tables(const ChainDev& ch, const MergePlan& mp, unsigned char* base, cudaStream_t st,
                 cudaStream_t st2 = nullptr, cudaEvent_t ea = nullptr, cudaEvent_t eb = nullptr) {
  if (!mp.table_bytes) return TNB_OK;
  KTimer kt("entries_tables", st);
  bool forked = false;
  if (st2 && ea && eb && mp.ng > 1 && mp.kind[mp.ng - 1] == kSuffix && mp.kind[0] == kPrefix) {
    if (cudaEventRecord(ea, st) == cudaSuccess && cudaStreamWaitEvent(st2, ea, 0) == cudaSuccess) forked = true;
    else cudaGetLastError();
  }
  cudaStream_t sfx = forked ? st2 : st;
  struct Join {  // st waits for the suffix stream on every exit path
    bool on;
    cudaStream_t st, st2;
    cudaEvent_t eb;
    ~Join() {
      if (on) {
        if (cudaEventRecord(eb, st2) == cudaSuccess) cudaStreamWaitEvent(st, eb, 0);
        else cudaStreamSynchronize(st2);
      }
    }
  } join{forked, st, st2, eb};
  unsigned char* scratch2 = base + mp.gemm_off + mp.gemm_bytes / 2;  // the suffix chain's half
  const int grid_cap = num_sms() * 8;
  auto grid = [&](int64_t total) { return (int)std::min<int64_t>(ceil_div(total, 256), grid_cap); };
  for (int g = 0; g < mp.ng; ++g) {
    const int lo = mp.lo[g], hi = mp.hi[g];
    if (mp.kind[g] == kPrefix || mp.kind[g] == kDiag) {
      // [J_lo][r] view of the first mode (prefix: rl == 1; diag: the table)
      const float* in = ch.m[lo].s;
      int64_t rows = ch.m[lo].J;
      for (int o = lo + 1; o < hi; ++o) {
        float* out = reinterpret_cast<float*>(base + mp.lvl[o]);
        const int64_t total = rows * ch.m[o].J * ch.m[o].rr;
        if (total > 0 && mp.kind[g] == kPrefix && tc_prefix_level(ch.m[o], rows)) {
          const ModeDev& md = ch.m[o];
          float* bt = reinterpret_cast<float*>(base + mp.gemm_off);
          const int64_t btb = ((int64_t)md.J * md.rl * md.rr * 4 + 255) & ~(int64_t)255;
          core_transpose_kernel<false><<<grid((int64_t)md.J * md.rl * md.rr), 256, 0, st>>>(md, bt);
          int rc = launch_tc_gemm(in, md.rl, 0, bt, (int64_t)md.J * md.rr, 0, out, (int64_t)md.J * md.rr, 0, rows,
                                  (int64_t)md.J * md.rr, md.rl, 1, base + mp.gemm_off + btb, st);
          if (rc) return rc;
        } else if (total > 0 && gemm_level(ch.m[o])) {
          const ModeDev& md = ch.m[o];
          float* bt = reinterpret_cast<float*>(base + mp.gemm_off);
          core_transpose_kernel<false><<<grid((int64_t)md.J * md.rl * md.rr), 256, 0, st>>>(md, bt);
          int rc = gemm_f32(in, md.rl, 0, bt, (int64_t)md.J * md.rr, 0, out, (int64_t)md.J * md.rr, 0, rows,
                            (int64_t)md.J * md.rr, md.rl, 1, st);
          if (rc) return rc;
        } else if (total > 0 && mp.kind[g] == kPrefix && t5_level_ok(ch.m[o], rows, false) &&
                   (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
          int rc = launch_t5_level<false>(ch.m[o], in, rows, out, base + mp.gemm_off, st);
          if (rc) return rc;
        } else if (total > 0 && launch_table_tc<false>(ch.m[o], in, rows, out, st)) {
        } else if (total > 0 && table_gemm_ok(ch.m[o], false))
          table_gemm<false><<<dim3((unsigned)ceil_div(rows, kTRows), (unsigned)ceil_div(ch.m[o].J, kTZ)), 256, 0,
                              st>>>(ch.m[o], in, rows, out);
        else if (total > 0)
          table_prefix_step<<<grid(total), 256, 0, st>>>(ch.m[o], in, rows, out);
        int rc = check_launch("table_prefix_step");
        if (rc) return rc;
        in = out;
        rows *= ch.m[o].J;
      }
    } else if (mp.lm[g] && mp.mma[g]) {
      const ModeDev& md = ch.m[lo];
      mma_slice_kernel<<<grid((int64_t)md.J * md.rl * md.rr * 2), 256, 0, st>>>(
          md.s, reinterpret_cast<float*>(base + mp.lm_off[g]), md.J, md.rl);
    } else if (mp.lm[g]) {
      const ModeDev& md = ch.m[lo];
      lane_major_kernel<<<grid((int64_t)md.J * md.rl * md.rr), 256, 0, st>>>(
          md.s, reinterpret_cast<float*>(base + mp.lm_off[g]), md.J, md.rl);
      int rc = check_launch("lane_major");
      if (rc) return rc;
    } else if (mp.kind[g] == kSuffix) {
      const float* in = ch.m[hi - 1].s;  // [J][r][1] == [J][r]
      int64_t n = ch.m[hi - 1].J;
      for (int o = hi - 2; o >= lo; --o) {
        float* out = reinterpret_cast<float*>(base + mp.lvl[o]);
        const ModeDev& md = ch.m[o];
        if ((int64_t)md.J * n * md.rl > 0 && gemm_level(md)) {
          float* gt = reinterpret_cast<float*>(scratch2);
          core_transpose_kernel<true><<<grid((int64_t)md.J * md.rl * md.rr), 256, 0, sfx>>>(md, gt);
          int rc = gemm_f32(in, md.rr, 0, gt, md.rl, (int64_t)md.rr * md.rl, out, md.rl, n * md.rl, n, md.rl, md.rr,
                            md.J, sfx);
          if (rc) return rc;
        } else if ((int64_t)md.J * n * md.rl > 0 && t5_level_ok(md, n, true) && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
          int rc = launch_t5_level<true>(md, in, n, out, scratch2, sfx);
          if (rc) return rc;
        } else if ((int64_t)md.J * n * md.rl > 0 && launch_table_tc<true>(md, in, n, out, sfx)) {
        } else if ((int64_t)md.J * n * md.rl > 0 && table_gemm_ok(md, true)) {
          table_gemm<true><<<dim3((unsigned)ceil_div(n, kTRows), (unsigned)ceil_div(md.J, kTZ)), 256, 0, sfx>>>(
              md, in, n, out);
        } else if ((int64_t)md.J * n * md.rl > 0 && (md.rl > 32 || md.rr > 32)) {
          table_suffix_step_big<<<grid((int64_t)md.J * n * md.rl), 256, 0, sfx>>>(md, in, n, out);
        } else if ((int64_t)md.J * n * md.rl > 0) {
          const int per = 256 / md.rl;
          const int gx = (int)std::min<int64_t>(ceil_div(n, per), std::max<int64_t>(1, grid_cap / md.J));
          table_suffix_step<<<dim3(gx, md.J), 256, 0, sfx>>>(md, in, n, out);
        }
        int rc = check_launch("table_suffix_step");
        if (rc) return rc;
        in = out;
        n *= md.J;
      }
    }
  }
  return TNB_OK;
}

int table_launches(const MergePlan& mp) {
  int n = 0;
  for (int g = 0; g < mp.ng; ++g)
    n += mp.kind[g] != kOrig ? mp.hi[g] - mp.lo[g] - 1 : mp.lm[g];
  return n;
}

void set_vmap(const ChainDev& ch, const MergePlan& mp, BPlan* bp) {
  bp->n0 = ch.n;
  for (int g = 0; g < mp.ng; ++g) {
    bp->lmaj[g] = mp.lm[g];
    bp->mmal[g] = mp.mma[g];
  }
  for (int g = 0; g < mp.ng; ++g)
    for (int o = mp.lo[g]; o < mp.hi[g]; ++o) {
      bp->oJ[o] = ch.m[o].J;
      bp->vmap[o] = (int8_t)g;
    }
}

int pick_R(int rmax) {
  if (rmax <= 8) return 8;
  if (rmax <= 16) return 16;
  if (rmax <= 24) return 24;
  if (rmax <= 32) return 32;
  return 0;
}

size_t prep_smem_bytes(int N, int T, int idx_bytes, int nw, int psort, int jpad) {
  const size_t c = ((size_t)N * T * idx_bytes + (size_t)nw * T * 4 + 15) & ~(size_t)15;
  return c + (psort ? (size_t)jpad * 4 + (size_t)T * 2 : 0) + 256;
}

size_t compute_smem(int T, int RP, int N, int idx_bytes, int jpad, int nw) {
  size_t b = (size_t)(T + 1) * RP * 4 + (size_t)N * T * idx_bytes + (size_t)nw * T * 4 + (size_t)2 * T * 2 +
             (size_t)2 * jpad * 2;
  return ((b + 15) & ~(size_t)15) + 4 * 8;
}

// Shared by the workspace query and the launcher so both agree on T.
int make_bplan(const ChainDev& ch, int64_t m, BPlan* bp, int* R_out, int* nt_out, int t_force = 0,
               bool stream = false) {
  const int R = pick_R(ch.rmax);
  if (!R) return set_error(TNB_EINVAL, "bucketed: rank > 32");
  int jmax = 1, nsort = 0;
  bool small = true;
  const int N = ch.n;
  bp->wide0 = stream || ch.m[0].J > 65535;
  bp->wideL = N > 1 && ch.m[N - 1].J > 65535;
  bp->nw = bp->wide0 + bp->wideL;
  bp->crow0 = stream ? 1 : 0;
  bp->splits = !stream && TNB_BALANCED && kComputeThreads / 32 == kSplitWarps;
  bp->ncrow = stream ? N - 1 - bp->wideL : N;
  for (int k = 0; k < ch.n; ++k) {
    const bool wide = (k == 0 && bp->wide0) || (k == N - 1 && bp->wideL);
    if (!wide && ch.m[k].J > 256) small = false;
    const bool srt = k > 0 && k < ch.n - 1 && ch.m[k].layout == TNB_LAYOUT_DENSE;
    bp->slot[k] = srt ? (int8_t)nsort : (int8_t)-1;
    if (srt) {
      bp->smode[nsort] = (int8_t)k;
      ++nsort;
      jmax = ch.m[k].J > jmax ? ch.m[k].J : jmax;
    }
  }
  constexpr int NT = kComputeThreads;
  const int RP = R == 32 ? Geo<32>::RP : R + TNB_RPAD;
  const int idx_bytes = small ? 1 : 2;
  // starts, sentinel (+ the state kernel's warp splits)
  const int jpad = ((jmax + 1 + (stream ? 0 : 1 + kSplitWarps)) + 7) & ~7;
  const size_t budget = ((size_t)233472 - 1024 * kStateCtas) / kStateCtas;
  // the prep kernel holds every slot's permutation and per-warp counts at once
  int jmin = 1 << 30;
  for (int i = 0; i < nsort; ++i) jmin = std::min(jmin, (int)ch.m[bp->smode[i]].J);
  bp->psort = nsort > 0 && TNB_SORT_IN_PREP > 0 && jmin >= TNB_SORT_IN_PREP;
  auto prep_smem = [&](int t) { return prep_smem_bytes(bp->ncrow, t, idx_bytes, bp->nw, bp->psort, jpad); };
  auto comp_smem = [&](int t) { return compute_smem(t, RP, ch.n, idx_bytes, jpad, bp->nw); };
  int T = 65504;
  if (t_force > 0) {
    T = t_force;
    if (prep_smem(T) > 232448 - 1024) return set_error(TNB_EINVAL, "bucketed: chain too long for smem");
  } else {
    while (T > 32 && (comp_smem(T) > budget || prep_smem(T) > 232448 - 1024)) T -= 32;
    if (comp_smem(T) > budget || prep_smem(T) > 232448 - 1024)
      return set_error(TNB_EINVAL, "bucketed: chain too long for smem");
  }
  bp->T = T;
  bp->nsort = nsort;
  bp->jpad = jpad;
  bp->idx_bytes = idx_bytes;
  bp->ntiles = (m + T - 1) / T;
  // [N][T] compact rows, [nw][T] uint32 wide rows (contiguous: N*T*idx_bytes
  // is a multiple of 32), then the sorted slots
  {
    int ks = 0;
    while ((1LL << ks) < ch.m[0].J) ++ks;
    int kb = 0;
    while (nsort == 1 && (1LL << kb) < ch.m[bp->smode[0]].J) ++kb;
    bp->kshift = ks;
    bp->kpack = stream && TNB_STREAM_KPACK && bp->psort && nsort == 1 && bp->smode[0] == 1 && ks + kb <= 32;
  }
  bp->off_wide = (int64_t)(bp->ncrow - bp->kpack) * T * idx_bytes;
  const int64_t cidx_b = bp->off_wide + (int64_t)bp->nw * T * 4;
  bp->off_perm = cidx_b;
  bp->off_starts = cidx_b + (int64_t)nsort * T * 2;
  bp->tile_bytes = (bp->off_starts + (int64_t)nsort * jpad * 2 + 127) & ~(int64_t)127;
  *R_out = R;
  *nt_out = NT;
  return TNB_OK;
}

int stream_env() {
  const char* e = getenv("TNB_ENTRIES_STREAM");
  return (e && e[0] == '0') ? 0 : 1;
}

// first (rl 1, rr R) . G (R x R dense) . D (diagonal, R)* . last (rl R, rr 1)
bool stream_shape_ok(const ChainDev& v, int R) {
  if (!stream_env() || (R != 8 && R != 16 && R != 24) || v.n < 3 || v.n > 4) return false;
  const int N = v.n;
  const ModeDev &f = v.m[0], &g = v.m[1], &l = v.m[N - 1];
  if (f.layout != TNB_LAYOUT_DENSE || f.rl != 1 || f.rr != R) return false;
  if (g.layout != TNB_LAYOUT_DENSE || g.rl != R || g.rr != R || g.J > kMaxJ) return false;
  if (l.layout != TNB_LAYOUT_DENSE || l.rl != R || l.rr != 1) return false;
  for (int k = 2; k < N - 1; ++k)
    if (v.m[k].layout != TNB_LAYOUT_DIAG || v.m[k].rl != R) return false;
  return true;
}

constexpr int kStreamThreads = TNB_STREAM_THREADS;
constexpr bool kStreamMma = TNB_STREAM_MMA != 0;
size_t stream_smem(const BPlan& bp, int R) {
  const int rs = kStreamMma ? ((R == 24 && TNB_STREAM_SWZ) ? R : R + 4) : R;
  return TNB_STREAM_NREC * (size_t)bp.tile_bytes + (size_t)(kStreamThreads / 32) * kSD * kSC * rs * 4 + 128 +
         (size_t)(TNB_STREAM_NREC + (kStreamThreads / 32) * kSD) * 8 + 4 * TNB_STREAM_NREC + 16;
}

// Everything a call needs to know, shared by the workspace query, the plan
// report and the launcher so all three agree.
struct EPlan {
  MergePlan mp;
  ChainDev v;
  BPlan bp;
  int R = 0, nt = 0;
  bool stream = false;
};
int plan_entries(const ChainDev& ch, int64_t m, EPlan* P) {
  plan_merge(ch, m, &P->mp);
  virtual_chain(ch, P->mp, nullptr, &P->v);
  int rc = make_bplan(P->v, m, &P->bp, &P->R, &P->nt);
  if (rc) return rc;
  P->stream = false;
  if (P->bp.nsort == 1 && stream_shape_ok(P->v, P->R) && (!kStreamMma || P->mp.lm[1])) {
    // tiles of up to 4096 samples, at least two per SM when m allows
    int T = TNB_STREAM_T;
    while (T > 256 && (m + T - 1) / T < 2 * 148) T = std::max(256, (T >> 1) & ~31);
    BPlan bs;
    int R2, nt2;
    while (T >= 256) {  // the largest tile whose double-buffered record fits next to the rings
      if (make_bplan(P->v, m, &bs, &R2, &nt2, T, true) == TNB_OK &&
          stream_smem(bs, R2) <= (size_t)232448 - 1024) {
        P->bp = bs;
        P->stream = true;
        if (kStreamMma) {  // the sorted mode's copy doubles (hi / lo fragments); it is the last table
          const ModeDev& g1 = ch.m[P->mp.lo[1]];
          P->mp.mma[1] = 1;
          // the GEMM scratch moves behind the doubled copy
          P->mp.gemm_off = P->mp.lm_off[1] + (((int64_t)g1.J * g1.rl * g1.rr * 2 * 4 + 255) & ~(int64_t)255);
          P->mp.table_bytes = P->mp.gemm_off + P->mp.gemm_bytes;
        }
        break;
      }
      T = T > 1024 ? T - 512 : T >> 1;
    }
  }
  return TNB_OK;
}

template <int R, typename IdxT>
int launch_stream(const ChainDev& ch, const BPlan& bp, const unsigned char* ws, int64_t m, float* out,
                  cudaStream_t st) {
  const size_t smem = stream_smem(bp, R);
  auto k = ch.n == 4 ? entries_stream_kernel<R, IdxT, kStreamThreads, 1, kStreamMma, false>
                     : entries_stream_kernel<R, IdxT, kStreamThreads, 0, kStreamMma, false>;
  auto kh = ch.n == 4 ? entries_stream_kernel<R, IdxT, kStreamThreads, 1, kStreamMma, true>
                      : entries_stream_kernel<R, IdxT, kStreamThreads, 0, kStreamMma, true>;
  int rc = check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "stream smem attr");
  if (!rc && bp.hot)
    rc = check_cuda(cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "stream smem attr");
  if (rc) return rc;
  const int64_t slots = (int64_t)num_sms();
  const int grid = (int)(bp.ntiles < slots ? bp.ntiles : slots);
  {
    KTimer kt("entries_compute", st);
    k<<<grid, kStreamThreads, smem, st>>>(ch, bp, ws, m, out);
    if (bp.hot) kh<<<grid, kStreamThreads, smem, st>>>(ch, bp, ws, m, out);
  }
  return check_launch("entries_stream");
}

template <int R, typename IdxT, int NT, bool FOLD>
int launch_rt(const ChainDev& ch, const BPlan& bp, const int64_t* idx, int64_t m, float* out,
              int32_t* err, unsigned char* ws, bool stream, cudaStream_t st, cudaEvent_t tables_done,
              bool reuse_records) {
  int rc;
  if (reuse_records) goto compute;  // batched chains: the tile records of element 0 serve every element
  {
  // prep: one CTA per tile; sort: one warp per (tile, sorted mode)
  const size_t psmem = prep_smem_bytes(bp.ncrow, bp.T, (int)sizeof(IdxT), bp.nw, bp.psort, bp.jpad);
  auto pk = bp.psort ? (bp.splits ? entries_prep_kernel<IdxT, true, true> : entries_prep_kernel<IdxT, true, false>)
                     : entries_prep_kernel<IdxT, false, false>;
  rc = check_cuda(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem),
                  "prep smem attr");
  if (rc) return rc;
  {
    KTimer kt("entries_prep", st);
    pk<<<(unsigned)bp.ntiles, kPrepThreads, psmem, st>>>(ch, bp, idx, m, err, ws);
  }
  rc = check_launch("entries_prep");
  if (rc) return rc;
  if (bp.nsort > 0 && !bp.psort) {
    const int64_t warps = bp.ntiles * bp.nsort;
    const size_t per_warp = (size_t)bp.jpad * 4 + (size_t)bp.T * 2;
    int wpb = 8;
    while (wpb > 1 && wpb * per_warp > 96 * 1024) wpb >>= 1;
    rc = check_cuda(cudaFuncSetAttribute(entries_sort_kernel<IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(wpb * per_warp)),
                    "sort smem attr");
    if (rc) return rc;
    {
      KTimer kt("entries_sort", st);
      entries_sort_kernel<IdxT><<<(unsigned)ceil_div(warps, wpb), 32 * wpb, wpb * per_warp, st>>>(ch, bp, m, ws);
    }
    rc = check_launch("entries_sort");
    if (rc) return rc;
  }
  if (bp.hot) {
    const int64_t g = bp.ntiles < 256 ? bp.ntiles : 256;
    detect_hot_kernel<IdxT><<<(unsigned)g, 32, 0, st>>>(bp, ws, m, const_cast<int32_t*>(bp.hot));
    rc = check_launch("detect_hot");
    if (rc) return rc;
  }
  }
compute:
  if (tables_done) {  // the tables were built on the side stream, concurrently with prep / sort
    rc = check_cuda(cudaStreamWaitEvent(st, tables_done, 0), "join tables");
    if (rc) return rc;
  }
  if (stream) {
    if constexpr (R <= 24) return launch_stream<R, IdxT>(ch, bp, ws, m, out, st);
    return set_error(TNB_EINVAL, "stream kernel: rank > 24");
  }
  const size_t csmem = compute_smem(bp.T, Geo<R>::RP, ch.n, (int)sizeof(IdxT), bp.jpad, bp.nw);
  auto ck = entries_compute_kernel<R, IdxT, NT, FOLD, false>;
  auto ckh = entries_compute_kernel<R, IdxT, NT, FOLD, true>;
  rc = check_cuda(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem),
                  "compute smem attr");
  if (!rc && bp.hot)
    rc = check_cuda(cudaFuncSetAttribute(ckh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem),
                    "compute smem attr");
  if (rc) return rc;
  const int64_t slots = (int64_t)num_sms() * kStateCtas;
  const int grid = (int)(bp.ntiles < slots ? bp.ntiles : slots);
  {
    KTimer kt("entries_compute", st);
    ck<<<grid, NT, csmem, st>>>(ch, bp, ws, m, out);
    if (bp.hot) ckh<<<grid, NT, csmem, st>>>(ch, bp, ws, m, out);
  }
  return check_launch("entries_compute");
}

template <int R, typename IdxT>
int launch_ri(const ChainDev& ch, const BPlan& bp, int nt, const int64_t* idx, int64_t m, float* out,
              int32_t* err, unsigned char* ws, bool stream, cudaStream_t st, cudaEvent_t tables_done,
              bool reuse) {
  const int N = ch.n;
  const bool fold = !stream && (R & 3) == 0 && N >= 3 && ch.m[N - 2].layout == TNB_LAYOUT_DIAG &&
                    ch.m[N - 1].rl == R && ch.m[N - 1].rr == 1;
  (void)nt;
  if (fold)
    return launch_rt<R, IdxT, kComputeThreads, true>(ch, bp, idx, m, out, err, ws, stream, st, tables_done, reuse);
  return launch_rt<R, IdxT, kComputeThreads, false>(ch, bp, idx, m, out, err, ws, stream, st, tables_done, reuse);
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

int64_t bucketed_workspace(const ChainDev& ch, int64_t m) {
  if (m <= 0 || !bucketed_supported(ch)) return 0;
  EPlan P;
  if (plan_entries(ch, m, &P)) return 0;
  return P.mp.table_bytes + P.bp.ntiles * P.bp.tile_bytes + 256;
}

double chain_entry_flops(const ChainDev& ch);

void bucketed_info(const ChainDev& ch, int64_t m, tnb_entries_info* info) {
  EPlan P;
  plan_entries(ch, m, &P);
  const MergePlan& mp = P.mp;
  const ChainDev& v = P.v;
  info->compute_kernel = P.stream ? 1 : 0;
  info->tile = P.bp.T;
  info->tensor_flops = 0.0;
  for (int g = 0; g < v.n; ++g)
    if (mp.lm[g] && mp.mma[g]) info->tensor_flops += 3.0 * 2.0 * v.m[g].rl * v.m[g].rr * (double)m;
  info->n_virtual = v.n;
  info->prefix_modes = mp.a();
  info->suffix_modes = mp.b();
  info->prefix_rows = mp.a() > 1 ? mp.rows[0] : 0;
  info->suffix_rows = mp.b() > 1 ? mp.rows[mp.ng - 1] : 0;
  info->diag_tables = 0;
  info->table_launches = table_launches(mp);
  info->kernel_flops = chain_entry_flops(v) * (double)m;
  double tf = 0.0;
  for (int g = 0; g < mp.ng; ++g) {
    const int lo = mp.lo[g], hi = mp.hi[g];
    if (mp.kind[g] == kDiag) ++info->diag_tables;
    if (mp.kind[g] == kPrefix || mp.kind[g] == kDiag) {
      int64_t rows = ch.m[lo].J;
      for (int o = lo + 1; o < hi; ++o) {
        const ModeDev& md = ch.m[o];
        rows *= md.J;
        tf += (double)rows * md.rr * (md.layout == TNB_LAYOUT_DIAG ? 1.0 : 2.0 * md.rl);
      }
    } else if (mp.kind[g] == kSuffix) {
      int64_t rows = ch.m[hi - 1].J;
      for (int o = hi - 2; o >= lo; --o) {
        const ModeDev& md = ch.m[o];
        rows *= md.J;
        tf += (double)rows * md.rl * (md.layout == TNB_LAYOUT_DIAG ? 1.0 : 2.0 * md.rr);
      }
    }
  }
  info->table_flops = tf;
}

// One non-blocking side stream + fork / join events per (host thread,
// device), created on first use: the only state libtnb keeps besides the
// device-property cache (reentrant: each thread owns its own).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t join2 = nullptr;  // second join: batched global-sort calls build the next element's tables ahead
  cudaStream_t s2 = nullptr;    // the suffix table's levels, concurrent with the prefix's (build_tables)
  cudaEvent_t ea = nullptr, eb = nullptr;
};
SideStream* side_stream() {
  static thread_local SideStream ss[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  SideStream& x = ss[dev];
  if (!x.s) {
    // high priority (TNB_TABLE_PRIO, default on): the block scheduler hands
    // freed SMs to the short table kernels first, so the tables are ready
    // before the prep / sort that fills the GPU has finished
    int least = 0, greatest = 0;
    const char* pe = getenv("TNB_TABLE_PRIO");
    const bool prio = !(pe && pe[0] == '0');
    if (!prio || cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) greatest = 0;
    cudaGetLastError();
    if (cudaStreamCreateWithPriority(&x.s, cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join2, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithPriority(&x.s2, cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.ea, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.eb, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x = SideStream{};
      return nullptr;
    }
  }
  return &x;
}
int table_stream_env() {
  const char* e = getenv("TNB_TABLE_STREAM");
  return (e && e[0] == '0') ? 0 : 1;
}

int launch_entries_bucketed(const ChainDev& ch, const int64_t* idx, int64_t m, float* out,
                            int32_t* err, void* ws, int64_t ws_bytes, cudaStream_t st, bool reuse_records) {
  EPlan P;
  int rc = plan_entries(ch, m, &P);
  if (rc) return rc;
  const MergePlan& mp = P.mp;
  ChainDev& v = P.v;
  BPlan& bp = P.bp;
  const int R = P.R, nt = P.nt;
  const bool stream = P.stream;
  const int64_t need = mp.table_bytes + bp.ntiles * bp.tile_bytes + 256;  // + the hot-rows flag
  if (!ws || ws_bytes < need)
    return set_error(TNB_EWORKSPACE, "bucketed entries needs %lld workspace bytes, got %lld",
                     (long long)need, (long long)ws_bytes);
  unsigned char* base = static_cast<unsigned char*>(ws);
  cudaEvent_t tables = nullptr;
  if (mp.table_bytes) {
    // the tables depend only on the cores, prep / sort only on the indices:
    // build the tables on a side stream forked from st (after everything
    // already queued on st, e.g. the previous call still reading them) and
    // join it before the compute kernel
    SideStream* ss = table_stream_env() ? side_stream() : nullptr;
    if (ss) {
      rc = check_cuda(cudaEventRecord(ss->fork, st), "fork");
      if (!rc) rc = check_cuda(cudaStreamWaitEvent(ss->s, ss->fork, 0), "fork wait");
      if (rc) return rc;  // nothing was queued on the side stream
      const bool conc = reuse_records || 4 * (mp.rows[0] + mp.rows[mp.ng - 1]) >= m;  // tables on the critical path
      rc = build_tables(ch, mp, base, ss->s, conc ? ss->s2 : nullptr, ss->ea, ss->eb);
      const int rj = check_cuda(cudaEventRecord(ss->join, ss->s), "join");
      if (rc || rj) {
        // join on the error path too: the caller frees the workspace the
        // side stream may still be writing
        if (!rj) cudaStreamWaitEvent(st, ss->join, 0);
        else cudaStreamSynchronize(ss->s);
        return rc ? rc : rj;
      }
      tables = ss->join;
    } else {
      rc = build_tables(ch, mp, base, st);
      if (rc) return rc;
    }
    virtual_chain(ch, mp, base, &v);
  }
  set_vmap(ch, mp, &bp);
  ws = base + mp.table_bytes;
  const ChainDev& chv = v;
  unsigned char* w = static_cast<unsigned char*>(ws);
  {
    int32_t* hot = reinterpret_cast<int32_t*>(w + bp.ntiles * bp.tile_bytes);
    bp.hot = hot;
    if (!reuse_records) {  // batched elements reuse element 0's records and flag
      rc = check_cuda(cudaMemsetAsync(hot, 0, sizeof(int32_t), st), "hot flag");
      if (rc) {
        if (tables) cudaStreamWaitEvent(st, tables, 0);
        return rc;
      }
    }
  }
  const bool small = bp.idx_bytes == 1;
  switch (R) {
    case 8:
      rc = small ? launch_ri<8, uint8_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records)
                 : launch_ri<8, uint16_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records);
      break;
    case 16:
      rc = small ? launch_ri<16, uint8_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records)
                 : launch_ri<16, uint16_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records);
      break;
    case 24:
      rc = small ? launch_ri<24, uint8_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records)
                 : launch_ri<24, uint16_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records);
      break;
    default:
      rc = small ? launch_ri<32, uint8_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records)
                 : launch_ri<32, uint16_t>(chv, bp, nt, idx, m, out, err, w, stream, st, tables, reuse_records);
  }
  // a failed launch may return before its own join: the side stream's table
  // writes must still be ordered before anything the caller does with ws
  if (rc && tables) cudaStreamWaitEvent(st, tables, 0);
  return rc;
}


// ---------------------------------------------------------------------------
// Two-table chains.  When mode merging leaves a virtual chain of TWO modes
// -- a prefix table P[(j_0..j_{a-1})][R] and a suffix table
// S[(j_a..j_{n-1})][R] (either may be an original boundary mode) -- every
// entry is one dot product of two gathered rows, for ANY rank R (the state /
// stream kernels stop at R = 32; a rank-64 cfg3 chain of 4 modes lands here
// with 65536-row tables).  One fused kernel per call after the tables:
// thread = sample; it reads its int64 index row, wraps negatives, checks
// every ORIGINAL mode (lowest OOB mode -> err, core.py:409-416), combines the
// C-order row numbers and accumulates <P[p], S[q]> in 16-byte pieces.
struct TwoTab {
  const float* P;
  const float* S;
  int32_t n, a, R;
  int32_t J[kMaxModes];
  int64_t stride[kMaxModes];  // C-order weight of mode k inside its group
};

template <bool VEC>
__global__ void __launch_bounds__(256) two_table_kernel(const __grid_constant__ TwoTab tt, const int64_t* __restrict__ idx,
                                                        int64_t m, float* __restrict__ out, int32_t* __restrict__ err) {
  const int n = tt.n, R = tt.R;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = 0, q = 0;
    int bad = n;
    const int64_t* row = idx + s * n;
    for (int k = 0; k < n; ++k) {
      int64_t x = __ldcs(row + k);
      const int64_t J = tt.J[k];
      if (x < 0) x += J;
      if ((x < 0 || x >= J) && bad == n) bad = k;
      x = x < 0 ? 0 : (x >= J ? J - 1 : x);
      if (k < tt.a) p += x * tt.stride[k];
      else q += x * tt.stride[k];
    }
    if (bad < n) {
      atomicMin(err, bad);
      continue;
    }
    const float* pr = tt.P + p * R;
    const float* qr = tt.S + q * R;
    float acc0 = 0.f, acc1 = 0.f;
    if (VEC) {
      for (int c = 0; c < R; c += 4) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(pr + c));
        const float4 v = __ldg(reinterpret_cast<const float4*>(qr + c));
        acc0 = fmaf(u.x, v.x, acc0);
        acc1 = fmaf(u.y, v.y, acc1);
        acc0 = fmaf(u.z, v.z, acc0);
        acc1 = fmaf(u.w, v.w, acc1);
      }
    } else {
      for (int c = 0; c < R; ++c) acc0 = fmaf(__ldg(pr + c), __ldg(qr + c), acc0);
    }
    out[s] = acc0 + acc1;
  }
}

namespace {
bool two_table_plan(const ChainDev& ch, int64_t m, MergePlan* mp) {
  if (ch.batch != 1 || ch.n < 2 || ch.n > kMaxModes) return false;
  for (int k = 0; k < ch.n; ++k)
    if (ch.m[k].bstride != 0 || ch.m[k].J <= 0) return false;
  plan_merge(ch, m, mp);
  if (mp->ng != 2) return false;
  const int R = ch.m[mp->hi[0] - 1].rr;
  return R >= 1 && R <= 4096 && ch.m[mp->lo[1]].rl == R;
}
}  // namespace

bool two_table_ok(const ChainDev& ch, int64_t m) {
  MergePlan mp;
  return two_table_plan(ch, m, &mp);
}

int64_t two_table_workspace(const ChainDev& ch, int64_t m) {
  MergePlan mp;
  return two_table_plan(ch, m, &mp) ? mp.table_bytes : 0;
}

void two_table_info(const ChainDev& ch, int64_t m, tnb_entries_info* info) {
  MergePlan mp;
  two_table_plan(ch, m, &mp);
  ChainDev v;
  virtual_chain(ch, mp, nullptr, &v);
  info->n_virtual = 2;
  info->prefix_modes = mp.a();
  info->suffix_modes = mp.b();
  info->prefix_rows = mp.a() > 1 ? mp.rows[0] : 0;
  info->suffix_rows = mp.b() > 1 ? mp.rows[1] : 0;
  info->compute_kernel = 2;
  info->tile = 0;
  info->tensor_flops = 0.0;
  info->diag_tables = 0;
  info->table_launches = table_launches(mp);
  info->kernel_flops = 2.0 * v.m[0].rr * (double)m;
  double tf = 0.0;
  if (mp.kind[0] == kPrefix) {
    int64_t rows = ch.m[0].J;
    for (int o = 1; o < mp.hi[0]; ++o) {
      rows *= ch.m[o].J;
      tf += (double)rows * ch.m[o].rr * (ch.m[o].layout == TNB_LAYOUT_DIAG ? 1.0 : 2.0 * ch.m[o].rl);
    }
  }
  if (mp.kind[1] == kSuffix) {
    int64_t rows = ch.m[ch.n - 1].J;
    for (int o = ch.n - 2; o >= mp.lo[1]; --o) {
      rows *= ch.m[o].J;
      tf += (double)rows * ch.m[o].rl * (ch.m[o].layout == TNB_LAYOUT_DIAG ? 1.0 : 2.0 * ch.m[o].rr);
    }
  }
  info->table_flops = tf;
}

int launch_two_table(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                     int64_t ws_bytes, cudaStream_t st) {
  MergePlan mp;
  if (!two_table_plan(ch, m, &mp)) return set_error(TNB_EINVAL, "chain does not reduce to two tables");
  if (mp.table_bytes && (!ws || ws_bytes < mp.table_bytes))
    return set_error(TNB_EWORKSPACE, "two-table entries needs %lld workspace bytes, got %lld",
                     (long long)mp.table_bytes, (long long)ws_bytes);
  unsigned char* base = static_cast<unsigned char*>(ws);
  int rc = build_tables(ch, mp, base, st);
  if (rc) return rc;
  ChainDev v;
  virtual_chain(ch, mp, base, &v);
  TwoTab tt;
  tt.P = v.m[0].s;
  tt.S = v.m[1].s;
  tt.n = ch.n;
  tt.a = mp.hi[0];
  tt.R = v.m[0].rr;
  int64_t w = 1;
  for (int k = tt.a - 1; k >= 0; --k) {
    tt.stride[k] = w;
    w *= ch.m[k].J;
  }
  w = 1;
  for (int k = ch.n - 1; k >= tt.a; --k) {
    tt.stride[k] = w;
    w *= ch.m[k].J;
  }
  for (int k = 0; k < ch.n; ++k) tt.J[k] = ch.m[k].J;
  int64_t g = ceil_div(m, 256);
  if (g > (int64_t)num_sms() * 16) g = (int64_t)num_sms() * 16;
  const bool vec = (tt.R & 3) == 0 && (reinterpret_cast<uintptr_t>(tt.P) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(tt.S) & 15) == 0;
  {
    KTimer kt("entries_compute", st);
    if (vec)
      two_table_kernel<true><<<(unsigned)(g < 1 ? 1 : g), 256, 0, st>>>(tt, idx, m, out, err);
    else
      two_table_kernel<false><<<(unsigned)(g < 1 ? 1 : g), 256, 0, st>>>(tt, idx, m, out, err);
  }
  return check_launch("two_table");
}


// the global-sort tcgen05 path shares the planner and the table kernels above
#include "entries_gsort.cuh"

}  // namespace tnb
