// K2 tensor-core GEMM: the final contraction of full(), out = L @ R
// (reference: the last unfolding GEMM of full, core.py:345-351).
//
// fp32 accuracy from TF32 tensor cores via 3xTF32: x = hi + lo with
// hi = rna_tf32(x), lo = x - hi (exact), and C = Ahi*Bhi + Ahi*Blo + Alo*Bhi
// accumulated in fp32 in TMEM (the dropped lo*lo term is ~2^-22 relative).
//
// The kernel computes the TRANSPOSED product C^T = R^T L^T, so that
//   * the operand that stays put (a 384-column block of R, i.e. 384 rows of
//     R^T, split hi/lo; 256 with TNB_FULL_NB3=0) lives in TMEM as the MMA's A
//     operand -- loaded once per column block by a helper warpgroup
//     (tcgen05.st);
//   * the streamed operand (128-row tiles of L) is the MMA's B operand in
//     shared memory.  A tiny pre-pass writes L split into hi/lo AND already in
//     the UMMA canonical K-major SWIZZLE_128B image, so one cp.async.bulk of
//     64 KB lands a tile ready for tcgen05.mma (3-stage ring, one producer
//     lane, mbarrier full/empty);
//   * the accumulator tile has TMEM lane = output column n and TMEM column =
//     output row m, so after tcgen05.ld (thread = n) every st.global of a
//     warp writes 32 consecutive floats of one output row: whole 128-byte
//     lines, no transpose.
//   * an alternative epilogue (TNB_FULL_TMA_STORE=1) stages each warp's
//     32 x 32 sub-tile of the output in shared memory and writes it with one
//     TMA tensor store (cp.async.bulk.tensor.2d, 4 KB, double-buffered per
//     warp; TMA clips ragged tiles).  Measured slower (3.72 vs 3.45 ms): the
//     store stream of one CTA per SM caps near 5.9 TB/s either way
//     (tools/store_bench.cu), so the default stays st.global.
// Roles (384 threads, one persistent CTA per SM):
//   warp 0      MMA issuer (one lane) + TMEM allocator
//   warp 1      producer of L tiles (one lane)
//   warps 4-7   epilogue (TMEM -> registers -> HBM)
//   warps 8-11  resident-A loader (R^T block -> hi/lo -> TMEM)
// TMEM: 512 columns = acc | A(n-block 0) | A(n-block 1) | A(n-block 2)
// (TNB_FULL_NB3=0: acc0 | acc1 | A(n-block 0) | A(n-block 1)).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace tnb {
namespace {

constexpr int kThreads = 384;
constexpr int BMT = 128;       // L rows per tile (UMMA N)
constexpr int BNB = 128;       // R columns per n-block (UMMA M)
// TNB_FULL_NB3: 3 resident n-blocks (384 columns) and ONE accumulator,
// released as soon as the epilogue has it in registers: each L tile then
// serves 384 output columns instead of 256 (L2 reads of L: 2 -> 1.33 B per
// output element)
#ifndef TNB_FULL_NB3
#define TNB_FULL_NB3 1  /* measured: 3.66-3.73 vs 3.71-3.82 ms (NB 2, two accumulators) at cfg3 */
#endif
constexpr int NB = TNB_FULL_NB3 ? 3 : 2;  // resident n-blocks per column block
constexpr int kAccBufs = TNB_FULL_NB3 ? 1 : 2;
constexpr int KMAX = 64;       // max contraction length
constexpr int kTileBytes = 2 * 2 * BMT * 128;  // {hi,lo} x 2 K-blocks x 128 rows x 128 B = 64 KB
// TNB_FULL_BULK (with NB3): the epilogue stages 64-row halves of each tile
// in shared memory and writes them with 512-byte cp.async.bulk stores (one
// per output row segment) instead of 128-byte st.global per warp
#ifndef TNB_FULL_BULK
#define TNB_FULL_BULK 0  /* measured: 5.18 vs 3.66 ms at cfg3 */
#endif
constexpr int kStages = TNB_FULL_BULK ? 2 : 3;
static_assert(!TNB_FULL_BULK || TNB_FULL_NB3, "TNB_FULL_BULK needs TNB_FULL_NB3");
// epilogue: 1 = each warp transposes a 32 x 32 block through shared memory
// and writes 16-byte vectors (4 rows x 128 B per store instruction);
// 0 = one 128-byte row segment per st.global (thread = output column)
#ifndef TNB_FULL_V4
#define TNB_FULL_V4 0  /* measured: 3.80 vs 3.73 ms at cfg3 */
#endif
// TMA-store epilogue: per epilogue warp two 32 x 32 fp32 staging buffers
#ifndef TNB_FULL_TMA
#define TNB_FULL_TMA 1
#endif
// TNB_FULL_EPI8: 8 epilogue warps (the A-loader warps store the second half of
// each tile's rows between A loads).  Measured slower: 3.55-3.60 vs 3.37 ms
// at cfg3 (round 1 saw the same with another 8-warp split)
#ifndef TNB_FULL_EPI8
#define TNB_FULL_EPI8 0
#endif
static_assert(!(TNB_FULL_EPI8 && !TNB_FULL_NB3), "TNB_FULL_EPI8 needs TNB_FULL_NB3");
// TNB_FULL_ALT: two epilogue warpgroups (warps 4-7 and the A-loader warps
// 8-11) take ALTERNATE 128 x 128 sub-tiles: while one group is still storing
// its sub-tile, the other waits for the next MMA, drains the accumulator and
// starts storing, so the store stream has no gap at every tcgen05.ld.  Still
// one TMEM accumulator; acc_full / acc_empty [g] belong to group g.
#ifndef TNB_FULL_ALT
#define TNB_FULL_ALT 0
#endif
static_assert(!(TNB_FULL_ALT && (!TNB_FULL_NB3 || TNB_FULL_EPI8)), "TNB_FULL_ALT needs TNB_FULL_NB3 without EPI8");
constexpr int kTmaBox = 32;                                   // rows and columns per TMA store
constexpr int kTmaBufBytes = kTmaBox * kTmaBox * 4;           // 4 KB
constexpr int kTmaEpiBytes = TNB_FULL_TMA ? 4 * 2 * kTmaBufBytes : 0;
static_assert(!(TNB_FULL_TMA && (TNB_FULL_BULK || TNB_FULL_V4)), "one epilogue variant at a time");
constexpr int kEpiBytes = TNB_FULL_BULK ? 2 * 64 * 128 * 4 : TNB_FULL_V4 ? 4 * 32 * 32 * 4 : kTmaEpiBytes;
constexpr uint32_t kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L tiles are re-read once per column block: keep them in L2 (evict_last)
// while the output streams past them (st.global.cs = evict-first)
__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
#ifndef TNB_FULL_ST
#define TNB_FULL_ST 0  // 0: st.global.cs, 1: plain st.global, 2: st.global.L1::no_allocate
#endif
__device__ __forceinline__ void st_stream(float* p, uint32_t v) {
#if TNB_FULL_ST == 1
  asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#elif TNB_FULL_ST == 2
  asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// D[tmem] (+)= A[tmem] * B[smem desc]; kind::tf32, cta_group::1
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// K-major SWIZZLE_128B canonical descriptor: LBO=16B (unused), SBO=1024B
// (8-row groups), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

#define TMEM_ST32(taddr, v)                                                                    \
  asm volatile(                                                                                \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, " \
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "  \
      "%28, %29, %30, %31, %32};" ::"r"(taddr),                                                \
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),  \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),         \
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),      \
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),      \
      "r"(v[29]), "r"(v[30]), "r"(v[31]))

#define TMEM_LD32(taddr, v)                                                                    \
  asm volatile(                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "   \
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "  \
      "%28, %29, %30, %31}, [%32];"                                                            \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),             \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),          \
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),          \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),          \
        "=r"(v[31])                                                                            \
      : "r"(taddr))

// Pre-pass: L (M x K, row stride lda) -> per 128-row tile a 64 KB image
// [hi kb0 | hi kb1 | lo kb0 | lo kb1], each K-block 128 rows x 128 B with
// 16-byte chunks XOR-swizzled by (row % 8): the canonical K-major SW128 image.
__global__ void split_l_kernel(const float* __restrict__ L, int64_t lda, int64_t M, int K,
                               unsigned char* __restrict__ out) {
  const int64_t total = ((M + BMT - 1) / BMT) * BMT * (KMAX / 4);  // (row, k4) pairs
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / (KMAX / 4);
    const int k4 = (int)(t - row * (KMAX / 4));
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < M) {
      const float* src = L + row * lda + k4 * 4;
      if (k4 * 4 + 0 < K) x.x = __ldg(src + 0);
      if (k4 * 4 + 1 < K) x.y = __ldg(src + 1);
      if (k4 * 4 + 2 < K) x.z = __ldg(src + 2);
      if (k4 * 4 + 3 < K) x.w = __ldg(src + 3);
    }
    const int64_t tile = row / BMT;
    const int r = (int)(row - tile * BMT);
    const int kb = k4 >> 3, c = k4 & 7;
    const uint32_t off = (uint32_t)(kb * (BMT * 128) + (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) * 16));
    unsigned char* base = out + tile * kTileBytes;
    uint4 hi, lo;
    hi.x = f2tf32(x.x);
    hi.y = f2tf32(x.y);
    hi.z = f2tf32(x.z);
    hi.w = f2tf32(x.w);
    lo.x = __float_as_uint(x.x - __uint_as_float(hi.x));
    lo.y = __float_as_uint(x.y - __uint_as_float(hi.y));
    lo.z = __float_as_uint(x.z - __uint_as_float(hi.z));
    lo.w = __float_as_uint(x.w - __uint_as_float(hi.w));
    *reinterpret_cast<uint4*>(base + off) = hi;
    *reinterpret_cast<uint4*>(base + kTileBytes / 2 + off) = lo;
  }
}

struct alignas(64) TcArgs {
  CUtensorMap cmap;         // C as a 2-D [M][N] fp32 tensor, 32 x 32 boxes (TMA epilogue)
  int use_tma;              // 1: cmap is valid and the epilogue stores through it
  const unsigned char* Ls;  // split_l_kernel output
  const float* B;           // R: [K][ldb], N contiguous
  int64_t ldb;
  float* C;                 // [M][ldc]
  int64_t ldc;
  int64_t M, N;
  int K;
  int lockstep;             // tile order, see tile_at in the kernel
};

__global__ void __launch_bounds__(kThreads, 1) full_tc_gemm_kernel(const __grid_constant__ TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* sL = smem;  // [kStages][kTileBytes]
  float* sEpi = reinterpret_cast<float*>(smem + kStages * kTileBytes);  // [4 warps][32][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kTileBytes + kEpiBytes);
  uint64_t* full = bars + 0;        // [kStages] tx
  uint64_t* empty = bars + 3;       // [kStages] tcgen05.commit (kStages <= 3)
  uint64_t* acc_full = bars + 6;    // [2] tcgen05.commit
  uint64_t* acc_empty = bars + 8;   // [2] 128 epilogue threads
  uint64_t* mma_idle = bars + 10;   // tcgen05.commit before an A reload
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = args.M, N = args.N;
  const int K = args.K;
  const int nk = (K + 7) >> 3;
  const int64_t n_mt = (M + BMT - 1) / BMT, n_cb = (N + NB * BNB - 1) / (NB * BNB);
  // Tile order.  lockstep: CTA b owns column block b + G w for a whole pass
  // down the row tiles (w = 0 .. n_cb / G - 1, G = grid size), so at any time
  // every CTA writes the SAME 128-row band of C, each its own 1.5 KB of every
  // row -- the order DRAM likes (tools/store_bench.cu: 6.7 vs 5.5 TB/s for the
  // same stores) and every CTA reads the same L tile from L2 at the same
  // time.  The column blocks left over (n_cb mod G) are split evenly by
  // tiles, as everything is without lockstep.
  const int64_t G = gridDim.x, n_lock_cb = args.lockstep ? (n_cb / G) * G : 0;
  const int64_t lock_cnt = (n_lock_cb / G) * n_mt;
  const int64_t tail_tiles = (n_cb - n_lock_cb) * n_mt;
  const int64_t tail0 = n_lock_cb * n_mt + (tail_tiles * blockIdx.x) / G;
  const int64_t tail1 = n_lock_cb * n_mt + (tail_tiles * (blockIdx.x + 1)) / G;
  const int64_t t_cnt = lock_cnt + (tail1 - tail0);
  auto tile_at = [&](int64_t i) -> int64_t {  // i-th tile of this CTA as t = cb * n_mt + mt
    if (i < lock_cnt) {
      const int64_t w = i / n_mt;
      return (w * G + blockIdx.x) * n_mt + (i - w * n_mt);
    }
    return tail0 + (i - lock_cnt);
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full[0], 1);
    mbar_init(&acc_full[1], 1);
    mbar_init(&acc_empty[0], TNB_FULL_EPI8 ? 256 : 128);
    mbar_init(&acc_empty[1], TNB_FULL_EPI8 ? 256 : 128);
    mbar_init(mma_idle, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_acc0 = tmem, tm_a0 = tmem + kAccBufs * BMT;  // acc b at +b*128; A nb at +nb*128

  if (warp == 0) {
    // ================= MMA issuer =================
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BMT >> 3) << 17) |
                           ((uint32_t)(BNB >> 4) << 24);
    const uint32_t sL0 = smem_u32(sL);
    int64_t cur_cb = -1;
    uint32_t idle_phase = 0, it = 0, s_it = 0;
    for (int64_t ti = 0; ti < t_cnt; ++ti) {
      const int64_t t = tile_at(ti);
      const int64_t cb = t / n_mt;
      if (cb != cur_cb) {
        if (cur_cb >= 0) {  // MMAs reading the old A must be done
          if (lane == 0) tc_commit(mma_idle);
          __syncwarp();
          mbar_wait(mma_idle, idle_phase);
          idle_phase ^= 1;
        }
        named_sync(1, 160);  // -> A loader: go
        named_sync(2, 160);  // <- A loader: TMEM holds the new block
        tc_fence_after();
        cur_cb = cb;
      }
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      tc_fence_after();
      const uint32_t bhi = sL0 + s * kTileBytes, blo = bhi + kTileBytes / 2;
      for (int nb = 0; nb < NB; ++nb) {
#if TNB_FULL_ALT
        const int cbuf = 0;  // one accumulator; the barriers alternate with the epilogue groups
        if (s_it > 0) mbar_wait(&acc_empty[(s_it - 1) & 1], ((s_it - 1) >> 1) & 1);
#else
        const int cbuf = s_it % kAccBufs;
        mbar_wait(&acc_empty[cbuf], ((s_it / kAccBufs) & 1) ^ 1);
#endif
        tc_fence_after();
        if (lane == 0) {
          const uint32_t d = tm_acc0 + cbuf * BMT;
          const uint32_t ah = tm_a0 + nb * BNB, al = ah + KMAX;
          uint32_t acc = 0;
          for (int kk = 0; kk < nk; ++kk) {
            const uint32_t boff = (uint32_t)(kk >> 2) * (BMT * 128) + (uint32_t)(kk & 3) * 32;
            const uint64_t dh = sw128_desc(bhi + boff), dl = sw128_desc(blo + boff);
            mma_tf32_ts(d, ah + kk * 8, dh, idesc, acc);
            acc = 1;
            mma_tf32_ts(d, ah + kk * 8, dl, idesc, 1);
            mma_tf32_ts(d, al + kk * 8, dh, idesc, 1);
          }
          tc_commit(&acc_full[TNB_FULL_ALT ? (int)(s_it & 1) : cbuf]);
        }
        __syncwarp();
        ++s_it;
      }
      if (lane == 0) tc_commit(&empty[s]);  // the L stage is free once these MMAs finish
      __syncwarp();
      ++it;
    }
  } else if (warp == 1) {
    // ================= producer: L tiles -> smem ring =================
    if (lane == 0) {
      uint64_t keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      uint32_t it = 0;
      for (int64_t ti = 0; ti < t_cnt; ++ti) {
      const int64_t t = tile_at(ti);
        const int64_t mt = t % n_mt;
        const int s = it % kStages;
        mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], kTileBytes);
        bulk_g2s_keep(sL + s * kTileBytes, args.Ls + mt * kTileBytes, kTileBytes, &full[s], keep);
        ++it;
      }
    }
#if TNB_FULL_ALT
  } else if (warp >= 4) {
    // ===== two epilogue groups on alternate sub-tiles (TNB_FULL_ALT); group 1
    // (warps 8-11) also loads the resident A block when the column block changes
    const int q = warp & 3, g = (warp >> 2) - 1;
    const bool loader = warp >= 8;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t s_it = 0;
    int64_t cur_cb = -1;
    for (int64_t ti = 0; ti < t_cnt; ++ti) {
      const int64_t t = tile_at(ti);
      const int64_t cb = t / n_mt, mt = t - cb * n_mt;
      if (loader && cb != cur_cb) {
        cur_cb = cb;
        named_sync(1, 160);
        for (int nb = 0; nb < NB; ++nb) {
          const int64_t n = cb * NB * BNB + nb * BNB + q * 32 + lane;
          const bool nok = n < N;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t hi[32], lo[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int k = half * 32 + j;
              const float x = (nok && k < K) ? __ldg(args.B + (int64_t)k * args.ldb + n) : 0.f;
              hi[j] = f2tf32(x);
              lo[j] = __float_as_uint(x - __uint_as_float(hi[j]));
            }
            TMEM_ST32(tm_a0 + nb * BNB + lane_base + half * 32, hi);
            TMEM_ST32(tm_a0 + nb * BNB + lane_base + KMAX + half * 32, lo);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        named_sync(2, 160);
      }
      for (int nb = 0; nb < NB; ++nb, ++s_it) {
        if ((int)(s_it & 1) != g) continue;
        mbar_wait(&acc_full[g], (s_it >> 1) & 1);
        tc_fence_after();
        const int64_t col = cb * NB * BNB + nb * BNB + q * 32 + lane;
        uint32_t v[BMT];
#pragma unroll
        for (int ch = 0; ch < BMT / 32; ++ch) TMEM_LD32(tm_acc0 + lane_base + ch * 32, (v + ch * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&acc_empty[g]);
        const int64_t rows_left = M - mt * BMT;
        if (col < N) {
          float* p = args.C + (mt * BMT) * args.ldc + col;
          if (rows_left >= BMT) {
#pragma unroll
            for (int j = 0; j < BMT; ++j) {
              st_stream(p, v[j]);
              p += args.ldc;
            }
          } else {
#pragma unroll
            for (int j = 0; j < BMT; ++j) {
              if (j < rows_left) st_stream(p, v[j]);
              p += args.ldc;
            }
          }
        }
      }
    }
  }
#elif TNB_FULL_EPI8
  } else if (warp >= 4) {
    // ===== epilogue on 8 warps (TNB_FULL_EPI8): warps 4-7 store the tile's
    // first 64 rows, warps 8-11 its last 64 (TMEM lane quarter = warp % 4);
    // warps 8-11 also load the resident A block when the column block changes
    const int q = warp & 3, h = (warp >> 2) - 1;
    const bool loader = warp >= 8;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t s_it = 0;
    int64_t cur_cb = -1;
    for (int64_t ti = 0; ti < t_cnt; ++ti) {
      const int64_t t = tile_at(ti);
      const int64_t cb = t / n_mt, mt = t - cb * n_mt;
      if (loader && cb != cur_cb) {
        cur_cb = cb;
        named_sync(1, 160);
        for (int nb = 0; nb < NB; ++nb) {
          const int64_t n = cb * NB * BNB + nb * BNB + q * 32 + lane;
          const bool nok = n < N;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t hi[32], lo[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int k = half * 32 + j;
              const float x = (nok && k < K) ? __ldg(args.B + (int64_t)k * args.ldb + n) : 0.f;
              hi[j] = f2tf32(x);
              lo[j] = __float_as_uint(x - __uint_as_float(hi[j]));
            }
            TMEM_ST32(tm_a0 + nb * BNB + lane_base + half * 32, hi);
            TMEM_ST32(tm_a0 + nb * BNB + lane_base + KMAX + half * 32, lo);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        named_sync(2, 160);
      }
      for (int nb = 0; nb < NB; ++nb) {
        const int cbuf = s_it % kAccBufs;
        mbar_wait(&acc_full[cbuf], (s_it / kAccBufs) & 1);
        tc_fence_after();
        const int64_t col = cb * NB * BNB + nb * BNB + q * 32 + lane;
        uint32_t v[BMT / 2];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) TMEM_LD32(tm_acc0 + cbuf * BMT + lane_base + (2 * h + ch) * 32, (v + ch * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&acc_empty[cbuf]);
        ++s_it;
        const int64_t r0 = mt * BMT + 64 * h;
        const int64_t rows_left = M - r0;
        if (col < N) {
          float* p = args.C + r0 * args.ldc + col;
          if (rows_left >= 64) {
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              st_stream(p, v[j]);
              p += args.ldc;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              if (j < rows_left) st_stream(p, v[j]);
              p += args.ldc;
            }
          }
        }
      }
    }
  }
#else
  } else if (warp >= 4 && warp < 8) {
    // ================= epilogue: thread = output column =================
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t s_it = 0;
    uint32_t bulk_it = 0;
    uint32_t tma_it = 0;  // TMA stores this warp issued (staging buffer = tma_it & 1)
    (void)bulk_it;
    (void)tma_it;
    for (int64_t ti = 0; ti < t_cnt; ++ti) {
      const int64_t t = tile_at(ti);
      const int64_t cb = t / n_mt, mt = t - cb * n_mt;
      for (int nb = 0; nb < NB; ++nb) {
        const int cbuf = s_it % kAccBufs;
        mbar_wait(&acc_full[cbuf], (s_it / kAccBufs) & 1);
        tc_fence_after();
        const int64_t col = cb * NB * BNB + nb * BNB + q * 32 + lane;
#if TNB_FULL_NB3
        {
          // whole 128-row accumulator column into registers, release it, store
          const bool cok = col < N;
          const int64_t rows_left = M - mt * BMT;
          const int64_t ldc = args.ldc;
          float* p = args.C + (mt * BMT) * ldc + col;
          uint32_t v[BMT];
#pragma unroll
          for (int ch = 0; ch < BMT / 32; ++ch) TMEM_LD32(tm_acc0 + lane_base + ch * 32, (v + ch * 32));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          tc_fence_before();
          mbar_arrive(&acc_empty[cbuf]);
          ++s_it;
#if TNB_FULL_BULK
          {
            const int64_t c0 = cb * NB * BNB + nb * BNB;  // first column of this n-block
            const bool bulk_ok = rows_left >= BMT && c0 + BNB <= N && (ldc & 3) == 0 &&
                                 (reinterpret_cast<uintptr_t>(args.C) & 15) == 0;
            if (bulk_ok) {  // uniform over the 4 epilogue warps
              const int e = tid - 128;  // 0..127; 0..63 issue the row stores
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                float* sb = sEpi + (size_t)(bulk_it & 1) * (64 * 128);
                if (e < 64) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                named_sync(3, 128);
#pragma unroll
                for (int j = 0; j < 64; ++j) sb[j * 128 + q * 32 + lane] = __uint_as_float(v[h * 64 + j]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                named_sync(3, 128);
                if (e < 64) {
                  float* dst = args.C + (mt * BMT + h * 64 + e) * ldc + c0;
                  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(dst),
                               "r"(smem_u32(sb + e * 128))
                               : "memory");
                  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                ++bulk_it;
              }
              continue;
            }
          }
#endif
#if TNB_FULL_TMA
          if (args.use_tma) {
            // 4 chunks of 32 rows: stage the warp's 32 x 32 block, one TMA store
            // each; buffer reuse waits only for the store issued two chunks ago
            float* sb0 = sEpi + (size_t)q * 2 * (kTmaBufBytes / 4);
            const int c0 = (int)(cb * NB * BNB + nb * BNB + q * 32);
#pragma unroll
            for (int ch = 0; ch < BMT / kTmaBox; ++ch) {
              float* sb = sb0 + (size_t)(tma_it & 1) * (kTmaBufBytes / 4);
              if (lane == 0 && tma_it >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int j = 0; j < kTmaBox; ++j) sb[j * kTmaBox + lane] = __uint_as_float(v[ch * kTmaBox + j]);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                const int r0 = (int)(mt * BMT + ch * kTmaBox);
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                        reinterpret_cast<uint64_t>(&args.cmap)),
                    "r"(c0), "r"(r0), "r"(smem_u32(sb))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              }
              ++tma_it;
            }
            continue;
          }
#endif
          if (cok && rows_left >= BMT) {
#pragma unroll
            for (int j = 0; j < BMT; ++j) {
              st_stream(p, v[j]);
              p += ldc;
            }
          } else if (cok) {
#pragma unroll
            for (int j = 0; j < BMT; ++j) {
              if (j < rows_left) st_stream(p, v[j]);
              p += ldc;
            }
          }
          continue;
        }
#endif
        const bool cok = col < N;
        const int64_t rows_left = M - mt * BMT;
        const bool full_rows = rows_left >= BMT;
        const int64_t ldc = args.ldc;
        const bool v4ok = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(args.C) & 15) == 0;
        float* p = args.C + (mt * BMT) * ldc + col;  // row mt*128, advanced by ldc per row
        uint32_t va[32], vb[32];
        TMEM_LD32(tm_acc0 + cbuf * BMT + lane_base, va);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int ch = 0; ch < BMT / 32; ++ch) {
          uint32_t* cur = (ch & 1) ? vb : va;
          uint32_t* nxt = (ch & 1) ? va : vb;
          if (ch + 1 < BMT / 32) TMEM_LD32(tm_acc0 + cbuf * BMT + lane_base + (ch + 1) * 32, nxt);
          if (TNB_FULL_V4 && v4ok && full_rows && cb * NB * BNB + nb * BNB + q * 32 + 32 <= N) {
            // transpose the 32 rows x 32 columns through shared memory, then
            // 16-byte stores: lanes 8r..8r+7 write row r's 128 bytes
            float* tw = sEpi + q * 32 * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j) tw[j * 32 + lane] = __uint_as_float(cur[j]);
            __syncwarp();
            float* rowp = args.C + (mt * BMT + ch * 32 + (lane >> 3)) * ldc + (col - lane) + 4 * (lane & 7);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 v = *reinterpret_cast<const float4*>(tw + (4 * i + (lane >> 3)) * 32 + 4 * (lane & 7));
              __stcs(reinterpret_cast<float4*>(rowp + (int64_t)(4 * i) * ldc), v);
            }
            __syncwarp();
            p += 32 * ldc;
          } else if (cok && full_rows) {
            // one st.global per row: the warp's 32 lanes write 128 contiguous bytes
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              st_stream(p, cur[j]);
              p += ldc;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (cok && ch * 32 + j < rows_left) st_stream(p, cur[j]);
              p += ldc;
            }
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[cbuf]);
        ++s_it;
      }
    }
#if TNB_FULL_BULK
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
#if TNB_FULL_TMA
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
  } else if (warp >= 8) {
    // ================= resident A: R^T block -> hi/lo -> TMEM =================
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int64_t cur_cb = -1;
    for (int64_t ti = 0; ti < t_cnt; ++ti) {
      const int64_t t = tile_at(ti);
      const int64_t cb = t / n_mt;
      if (cb == cur_cb) continue;
      cur_cb = cb;
      named_sync(1, 160);
      for (int nb = 0; nb < NB; ++nb) {
        const int64_t n = cb * NB * BNB + nb * BNB + q * 32 + lane;
        const bool nok = n < N;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = half * 32 + j;
            const float x = (nok && k < K) ? __ldg(args.B + (int64_t)k * args.ldb + n) : 0.f;
            hi[j] = f2tf32(x);
            lo[j] = __float_as_uint(x - __uint_as_float(hi[j]));
          }
          TMEM_ST32(tm_a0 + nb * BNB + lane_base + half * 32, hi);
          TMEM_ST32(tm_a0 + nb * BNB + lane_base + KMAX + half * 32, lo);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      named_sync(2, 160);
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

constexpr size_t kSmemBytes = 1024 + (size_t)kStages * kTileBytes + kEpiBytes + 128;

bool tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TNB_FULL_NO_TC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

// TNB_FULL_TMA_STORE=1 selects the TMA-store epilogue.  Off by default:
// measured 3.72 vs 3.45 ms at cfg3 (profiles/r02_full_store_bench.txt: this
// one-CTA-per-SM store stream tops out at 5.6-5.9 TB/s whichever way the
// 128 x 128 tiles are written -- st.global.b32 / .v4, TMA 32x32 / 64x64 --
// and the staging round trip costs more than it saves)
bool tma_env() {
  const char* e = getenv("TNB_FULL_TMA_STORE");
  return e && e[0] == '1';
}

// C [M][N] (row stride ldc floats) as a 2-D tensor map with 32 x 32 boxes;
// false when TMA cannot describe it (the epilogue then uses st.global)
bool encode_c_map(CUtensorMap* map, float* C, int64_t M, int64_t N, int64_t ldc) {
  if (!TNB_FULL_TMA || !tma_env()) return false;
  if ((reinterpret_cast<uintptr_t>(C) & 15) || ((ldc * 4) & 15) || M >= (1LL << 31) || N >= (1LL << 31))
    return false;
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
  const cuuint64_t strides[1] = {(cuuint64_t)ldc * 4};
  const cuuint32_t box[2] = {kTmaBox, kTmaBox};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool tc_gemm_supported(int64_t M, int64_t N, int K, int64_t lda, int64_t ldb, int64_t ldc) {
  if (tc_disabled()) return false;
  (void)lda;
  (void)ldb;
  (void)ldc;
  return K >= 1 && K <= KMAX && M >= 1 && N >= BNB && M * N >= (1LL << 20);
}

int64_t tc_gemm_workspace(int64_t M) { return ((M + BMT - 1) / BMT) * (int64_t)kTileBytes; }

int launch_tc_gemm(const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb, int64_t sB,
                   float* C, int64_t ldc, int64_t sC, int64_t M, int64_t N, int K, int64_t batch,
                   void* ws, cudaStream_t st) {
  int rc = check_cuda(cudaFuncSetAttribute(full_tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kSmemBytes),
                      "tc smem attr");
  if (rc) return rc;
  const int64_t n_tiles = ((M + BMT - 1) / BMT) * ((N + NB * BNB - 1) / (NB * BNB));
  const int grid = (int)(n_tiles < num_sms() ? n_tiles : num_sms());
  unsigned char* Ls = static_cast<unsigned char*>(ws);
  for (int64_t e = 0; e < batch; ++e) {
    const int64_t pairs = ((M + BMT - 1) / BMT) * BMT * (KMAX / 4);
    int g = (int)ceil_div(pairs, 256);
    if (g > num_sms() * 16) g = num_sms() * 16;
    split_l_kernel<<<g, 256, 0, st>>>(A + e * sA, lda, M, K, Ls);
    rc = check_launch("split_l");
    if (rc) return rc;
    TcArgs a;
    a.use_tma = encode_c_map(&a.cmap, C + e * sC, M, N, ldc) ? 1 : 0;
    a.Ls = Ls;
    a.B = B + e * sB;
    a.ldb = ldb;
    a.C = C + e * sC;
    a.ldc = ldc;
    a.M = M;
    a.N = N;
    a.K = K;
    {
      const char* ev = getenv("TNB_FULL_LOCKSTEP");
      a.lockstep = !(ev && ev[0] == '0');
    }
    full_tc_gemm_kernel<<<grid, kThreads, kSmemBytes, st>>>(a);
    rc = check_launch("full_tc_gemm");
    if (rc) return rc;
  }
  return TNB_OK;
}

}  // namespace tnb
