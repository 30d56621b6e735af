// K2 tensor-core GEMM: the final contraction of full(), out = L @ R
// (reference: the last unfolding GEMM of full, core.py:345-351).
//
// fp32 accuracy from TF32 tensor cores via 3xTF32: x = hi + lo with
// hi = rna_tf32(x), lo = x - hi (exact), and C = Ahi*Bhi + Ahi*Blo + Alo*Bhi
// accumulated in fp32 in TMEM (the dropped lo*lo term is ~2^-22 relative).
//
// Design (one persistent CTA per SM, 512 threads, no cluster):
//   * B (= R^T block of BN=256 output columns, K <= 64) is RESIDENT in shared
//     memory in the UMMA canonical K-major SWIZZLE_128B layout, hi and lo
//     (128 KB); it is refilled only when the CTA's work moves to the next
//     column block (cb-major tile order).
//   * A (= 128 rows of L) never touches shared memory: loader warps (warps
//     4-11; thread = row, two warps per TMEM lane quadrant, one K half each)
//     read the rows from global/L2 one tile ahead, split them into hi/lo in
//     registers and tcgen05.st them into TMEM, where tcgen05.mma
//     takes its A operand (kind::tf32, A from TMEM, B from smem).  Two A
//     buffers of 128 columns (hi 64 | lo 64).
//   * MMA issuer (warp 0, one lane): per A tile, two 128x128 N-subtiles, each
//     24 MMAs (8 k-steps x 3 products) into one of two 128-column TMEM
//     accumulators; tcgen05.commit signals the epilogue and frees A.
//   * epilogue warps (12-15): tcgen05.ld 32 columns at a time (thread = row),
//     transposed through a per-warp smem tile so every st.global.cs.v4
//     writes whole 128-byte lines.  The output write (HBM) is the roof;
//     MMAs (~1.5k cycles per subtile) hide under it (~2.7k cycles at
//     ~24 B/clk/SM).
// TMEM: 512 columns = acc0 | acc1 | A0 | A1.
#include "common.cuh"

namespace tnb {
namespace {

constexpr int kThreads = 512;
constexpr int BM = 128;        // rows per A tile (UMMA M)
constexpr int BN = 256;        // resident B columns
constexpr int SUBN = 128;      // UMMA N
constexpr int KMAX = 64;       // max contraction length
constexpr int kBBytes = 2 * 2 * BN * 128;  // {hi,lo} x 2 K-blocks x 256 rows x 128 B
constexpr uint32_t kTmemCols = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(b))
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

// byte offset of B element (row n, k) inside one hi/lo half: K-block kb =
// k / 32 holds BN rows of 128 B; 16 B chunks XOR-swizzled with (row % 8).
__device__ __forceinline__ uint32_t b_offset(int n, int k) {
  const int kb = k >> 5, kk = k & 31;
  const int chunk = (kk >> 2) ^ (n & 7);
  return (uint32_t)(kb * (BN * 128) + (n >> 3) * 1024 + (n & 7) * 128 + chunk * 16 + (kk & 3) * 4);
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

#define TMEM_ST16(taddr, v)                                                                    \
  asm volatile(                                                                                \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, " \
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),                                          \
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),  \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),         \
      "r"(v[15]))

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

struct TcArgs {
  const float* A;  // [M][lda], K-major rows (left partial L)
  int64_t lda;
  const float* B;  // [K][ldb], N contiguous (right partial R)
  int64_t ldb;
  float* C;        // [M][ldc]
  int64_t ldc;
  int64_t M, N;
  int K;
};

__global__ void __launch_bounds__(kThreads, 1) full_tc_gemm_kernel(const __grid_constant__ TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-align the swizzled B region
  unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* sB = smem;  // hi: [0, kBBytes/2), lo: [kBBytes/2, kBBytes)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBBytes);
  uint64_t* a_full = bars + 0;     // [2] count 256 (loader threads)
  uint64_t* a_empty = bars + 2;    // [2] count 1 (tcgen05.commit)
  uint64_t* acc_full = bars + 4;   // [2] count 1 (tcgen05.commit)
  uint64_t* acc_empty = bars + 6;  // [2] count 128 (epilogue threads)
  uint64_t* mma_idle = bars + 8;   // count 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t M = args.M, N = args.N;
  const int K = args.K;
  const int nk = (K + 7) >> 3;  // k-steps of 8
  const int64_t n_rb = (M + BM - 1) / BM, n_cb = (N + BN - 1) / BN;
  const int64_t n_tiles = n_rb * n_cb;
  const int64_t t0 = (n_tiles * blockIdx.x) / gridDim.x;
  const int64_t t1 = (n_tiles * (blockIdx.x + 1)) / gridDim.x;

  if (tid == 0) {
    mbar_init(&a_full[0], 256);
    mbar_init(&a_full[1], 256);
    mbar_init(&a_empty[0], 1);
    mbar_init(&a_empty[1], 1);
    mbar_init(&acc_full[0], 1);
    mbar_init(&acc_full[1], 1);
    mbar_init(&acc_empty[0], 128);
    mbar_init(&acc_empty[1], 128);
    mbar_init(mma_idle, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_acc[2] = {tmem + 0, tmem + SUBN};
  const uint32_t tm_a[2] = {tmem + 2 * SUBN, tmem + 3 * SUBN};

  if (warp < 4) {
    // ================= WG0: B refills + MMA issue (warp 0) =================
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(SUBN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    const uint32_t sB_hi = smem_u32(sB), sB_lo = sB_hi + kBBytes / 2;
    int64_t cur_cb = -1;
    uint32_t idle_phase = 0;
    uint32_t a_it = 0, s_it = 0;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t cb = t / n_rb;
      if (cb != cur_cb) {
        if (warp == 0 && cur_cb >= 0) {  // all MMAs reading the old B must finish
          if (lane == 0) tc_commit(mma_idle);
          __syncwarp();
          mbar_wait(mma_idle, idle_phase);
          idle_phase ^= 1;
        }
        named_sync(1, 128);
        // B block: rows n = output columns cb*BN .. +BN, k < K; R is [K][ldb]
        // (n contiguous): 16-byte loads, 8 in flight per thread, each element
        // split into hi/lo and stored at its swizzled K-major position
        const int64_t n0 = cb * BN;
        const bool bvec = ((args.ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(args.B) & 15) == 0) &&
                          (n0 + BN <= N);
        for (int e0 = tid; e0 < (BN / 4) * KMAX; e0 += 128 * 8) {
          float4 xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * 128;
            const int k = e / (BN / 4), n4 = e - (e / (BN / 4)) * (BN / 4);
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < (BN / 4) * KMAX && k < K) {
              const float* src = args.B + (int64_t)k * args.ldb + n0 + n4 * 4;
              if (bvec) {
                x = __ldg(reinterpret_cast<const float4*>(src));
              } else {
                if (n0 + n4 * 4 + 0 < N) x.x = __ldg(src + 0);
                if (n0 + n4 * 4 + 1 < N) x.y = __ldg(src + 1);
                if (n0 + n4 * 4 + 2 < N) x.z = __ldg(src + 2);
                if (n0 + n4 * 4 + 3 < N) x.w = __ldg(src + 3);
              }
            }
            xv[u] = x;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * 128;
            if (e >= (BN / 4) * KMAX) continue;
            const int k = e / (BN / 4), n4 = e - (e / (BN / 4)) * (BN / 4);
            const float xs[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t hi = f2tf32(xs[j]);
              const uint32_t off = b_offset(n4 * 4 + j, k);
              *reinterpret_cast<uint32_t*>(sB + off) = hi;
              *reinterpret_cast<float*>(sB + kBBytes / 2 + off) = xs[j] - __uint_as_float(hi);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_sync(1, 128);
        cur_cb = cb;
      }
      if (warp == 0) {
        const int ab = a_it & 1;
        mbar_wait(&a_full[ab], (a_it >> 1) & 1);
        tc_fence_after();
        for (int sub = 0; sub < BN / SUBN; ++sub) {
          const int cbuf = s_it & 1;
          mbar_wait(&acc_empty[cbuf], ((s_it >> 1) & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t brow = (uint32_t)(sub * SUBN) * 128;  // 128 rows x 128 B
            uint32_t acc = 0;
            for (int kk = 0; kk < nk; ++kk) {
              const uint32_t boff = (uint32_t)(kk >> 2) * (BN * 128) + brow + (uint32_t)(kk & 3) * 32;
              const uint64_t dh = sw128_desc(sB_hi + boff), dl = sw128_desc(sB_lo + boff);
              const uint32_t ah = tm_a[ab] + kk * 8, al = tm_a[ab] + KMAX + kk * 8;
              mma_tf32_ts(tm_acc[cbuf], ah, dh, idesc, acc);
              acc = 1;
              mma_tf32_ts(tm_acc[cbuf], ah, dl, idesc, 1);
              mma_tf32_ts(tm_acc[cbuf], al, dh, idesc, 1);
            }
            tc_commit(&acc_full[cbuf]);
          }
          __syncwarp();
          ++s_it;
        }
        if (lane == 0) tc_commit(&a_empty[ab]);
        __syncwarp();
        ++a_it;
      }
    }
  } else if (warp < 12) {
    // ================= A loaders: thread = row, one K half per warp =========
    const int q = warp & 3;
    const int kh = (warp - 4) >> 2;  // columns kh*32 .. kh*32+31
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const bool vec = ((args.lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(args.A) & 15) == 0);
    auto load_row = [&](int64_t t, float4 (&x)[8]) {
      const int64_t rb = t - (t / n_rb) * n_rb;
      const int64_t row = rb * BM + r;
      const float* src = args.A + row * args.lda + kh * 32;
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const int k = kh * 32 + c4 * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < t1 && row < M) {
          if (vec && k + 3 < K) {
            v = __ldg(reinterpret_cast<const float4*>(src + c4 * 4));
          } else {
            if (k + 0 < K) v.x = __ldg(src + c4 * 4 + 0);
            if (k + 1 < K) v.y = __ldg(src + c4 * 4 + 1);
            if (k + 2 < K) v.z = __ldg(src + c4 * 4 + 2);
            if (k + 3 < K) v.w = __ldg(src + c4 * 4 + 3);
          }
        }
        x[c4] = v;
      }
    };
    float4 cur[8];
    load_row(t0, cur);
    uint32_t a_it = 0;
    for (int64_t t = t0; t < t1; ++t) {
      float4 nxt[8];
      load_row(t + 1, nxt);  // one tile ahead: the L2 latency overlaps this tile
      const int ab = a_it & 1;
      mbar_wait(&a_empty[ab], ((a_it >> 1) & 1) ^ 1);
      tc_fence_after();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // 16 columns at a time
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 v = cur[hh * 4 + c4];
          const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t h = f2tf32(xs[j]);
            hi[c4 * 4 + j] = h;
            lo[c4 * 4 + j] = __float_as_uint(xs[j] - __uint_as_float(h));
          }
        }
        const uint32_t col = kh * 32 + hh * 16;
        TMEM_ST16(tm_a[ab] + lane_base + col, hi);
        TMEM_ST16(tm_a[ab] + lane_base + KMAX + col, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&a_full[ab]);
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) cur[c4] = nxt[c4];
      ++a_it;
    }
  } else {
    // ================= WG2: epilogue =================
    // TMEM rows -> registers (thread = row) -> per-warp smem transpose ->
    // coalesced stores: each st.global.v4 writes 4 rows x 128 B full lines.
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const bool vec = ((args.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(args.C) & 15) == 0);
    float* tp = reinterpret_cast<float*>(smem + kBBytes + 1024) + q * (32 * 36);  // [32][36]
    const uint32_t tp_s = smem_u32(tp);
    uint32_t s_it = 0;
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t cb = t / n_rb, rb = t - cb * n_rb;
      const int64_t row0 = rb * BM + q * 32;  // this warp's 32 rows
      for (int sub = 0; sub < BN / SUBN; ++sub) {
        const int cbuf = s_it & 1;
        mbar_wait(&acc_full[cbuf], (s_it >> 1) & 1);
        tc_fence_after();
        const int64_t col0 = cb * BN + sub * SUBN;
        uint32_t va[32], vb[32];
        TMEM_LD32(tm_acc[cbuf] + lane_base, va);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int ch = 0; ch < SUBN / 32; ++ch) {
          uint32_t* cur = (ch & 1) ? vb : va;
          uint32_t* nxt = (ch & 1) ? va : vb;
          if (ch + 1 < SUBN / 32) TMEM_LD32(tm_acc[cbuf] + lane_base + (ch + 1) * 32, nxt);
          // my row (lane) -> smem row
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tp_s + (lane * 36 + j * 4) * 4),
                         "r"(cur[4 * j]), "r"(cur[4 * j + 1]), "r"(cur[4 * j + 2]), "r"(cur[4 * j + 3])
                         : "memory");
          __syncwarp();
          const int64_t c0 = col0 + ch * 32;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3), cq = (lane & 7) * 4;
            const int64_t grow = row0 + rr;
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(tp_s + (rr * 36 + cq) * 4));
            if (grow < M) {
              float* dst = args.C + grow * args.ldc + c0 + cq;
              if (vec && c0 + cq + 4 <= N) {
                asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y),
                             "f"(v.z), "f"(v.w)
                             : "memory");
              } else {
                const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (c0 + cq + u < N) dst[u] = vs[u];
              }
            }
          }
          __syncwarp();
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[cbuf]);
        ++s_it;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

constexpr size_t kSmemBytes = 1024 + kBBytes + 1024 + 4 * 32 * 36 * 4;

bool tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TNB_FULL_NO_TC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace

bool tc_gemm_supported(int64_t M, int64_t N, int K, int64_t lda, int64_t ldb, int64_t ldc) {
  if (tc_disabled()) return false;
  (void)lda;
  (void)ldb;
  (void)ldc;
  return K >= 1 && K <= KMAX && M >= BM && N >= SUBN && M * N >= (1LL << 20);
}

int launch_tc_gemm(const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb,
                   int64_t sB, float* C, int64_t ldc, int64_t sC, int64_t M, int64_t N, int K,
                   int64_t batch, cudaStream_t st) {
  int rc = check_cuda(cudaFuncSetAttribute(full_tc_gemm_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kSmemBytes),
                      "tc smem attr");
  if (rc) return rc;
  const int64_t n_tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = (int)(n_tiles < num_sms() ? n_tiles : num_sms());
  for (int64_t e = 0; e < batch; ++e) {
    TcArgs a;
    a.A = A + e * sA;
    a.lda = lda;
    a.B = B + e * sB;
    a.ldb = ldb;
    a.C = C + e * sC;
    a.ldc = ldc;
    a.M = M;
    a.N = N;
    a.K = K;
    full_tc_gemm_kernel<<<grid, kThreads, kSmemBytes, st>>>(a);
    rc = check_launch("full_tc_gemm");
    if (rc) return rc;
  }
  return TNB_OK;
}

}  // namespace tnb
