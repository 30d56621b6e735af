// K3 performance kernel: batched chain inner products / norms for TT chains
// of rank 16 (BASELINE config 4: 4096 pairs, N=16, I=64, r=16).
//
// Reference: chain_dot (core.py:362-384) propagates an r_a x r_b transfer
// matrix M mode by mode, M' = sum_j A_j^T M B_j, as numpy's einsum path
// "xaic,xab->bcix" then "bcix,xbid->xcd".  Here:
//   * one CTA per pair at a time (persistent, 4 CTAs per SM, 4 compute warps:
//     measured against 8 and 2 warps per pair, 1.45 vs 1.55 / 1.63 ms at cfg4)
//     plus a producer warp that streams the chunks (1.44 ms);
//   * core slices stream HBM -> shared memory with cp.async.bulk (TMA bulk
//     copies) in chunks of 8 slices (8 KB per operand), double buffered
//     behind an mbarrier full/empty pipeline -- each byte is read once;
//   * warp w takes slices j = w, w+4 of every chunk and, on tensor cores
//     (mma.sync m16n8k8 TF32 in split form, x = hi + lo, three MMAs per
//     product: lo*hi + hi*lo + hi*hi), computes
//       Y_j^T = B_j^T M^T   then   Mw += A_j^T Y_j
//     with the K slots of each 8-chunk permuted so that the accumulator
//     fragment of the first product IS the B-operand fragment of the second:
//     M and Y never leave registers; each slice's A_j^T Y_j starts from a
//     zero fragment and joins the warp's running partial with a rounded FADD
//     (long MMA accumulations drift: cfg4 relFro 2.5e-6 against float64);
//   * at the end of each core the per-warp partial M's are summed through
//     shared memory and reloaded (split once per mode) as fragments.
// The boundary cores (rank 1 outward) use FFMA2 (fma.rn.f32x2) special
// cases.  norm() streams only one operand (A == B) and splits each slice's
// fragments once for both products (the SAME instantiation).
// TNB_DOT_SIMT=1 selects the FFMA2 body (Y bounced through a per-warp smem
// tile; 6e-7 relFro, 2.40 vs 1.44 ms).
//
// Why not tcgen05: per pair the products are 16 x 16 x 16.  UMMA needs
// M >= 64 rows sharing ONE B operand; stacking 4-8 pairs' rows gives a
// block-diagonal product (3/4 - 7/8 of the MMA work wasted), and the second
// product M' = sum_j A_j^T Y_j is a 16 x 16 output with a 1024-long
// reduction -- no UMMA shape fits it.  HBM is the binding roof for dot
// (SURVEY 8(d)); the mma.sync path runs at 0.81 of it.
#include "common.cuh"

namespace tnb {
namespace {

// warps per pair (CTA) and slices per pipeline chunk; 16 warps per SM
#ifndef TNB_DOT_WARPS
#define TNB_DOT_WARPS 4
#endif
#ifndef TNB_DOT_CH
#define TNB_DOT_CH 8
#endif
constexpr int kWarps = TNB_DOT_WARPS;
// TNB_DOT_PRODUCER: one extra warp streams the chunks (thread 0 of the
// compute warps no longer blocks on the slowest warp to refill a stage)
#ifndef TNB_DOT_PRODUCER
#define TNB_DOT_PRODUCER 1
#endif
constexpr int kCompute = kWarps * 32;                           // compute threads
constexpr int kThreads = kCompute + (TNB_DOT_PRODUCER ? 32 : 0);
#ifndef TNB_DOT_CTAS
#define TNB_DOT_CTAS (16 / TNB_DOT_WARPS)
#endif
constexpr int kCtasPerSm = TNB_DOT_CTAS;
constexpr int R = 16;
constexpr int CH = TNB_DOT_CH;         // slices per chunk
static_assert(CH == 2 * kWarps, "the FFMA path takes two slices per warp and chunk");
#ifndef TNB_DOT_STAGES
#define TNB_DOT_STAGES 2
#endif
constexpr int kStages = TNB_DOT_STAGES;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// the producer lane's wait for a free stage: try_wait with a suspend-time
// hint, so the lane sleeps in the barrier unit instead of re-issuing the test
// every ~30 cycles beside the compute warps of its scheduler
#ifndef TNB_DOT_PSUSP
#define TNB_DOT_PSUSP 1
#endif
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* b, uint32_t parity) {
#if TNB_DOT_PSUSP
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity), "r"(20000u)
      : "memory");
#else
  mbar_wait(b, parity);
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void ffma2(uint64_t& acc, uint64_t a, float s) {
  asm("{\n\t.reg .b64 ss;\n\tmov.b64 ss, {%2, %2};\n\tfma.rn.f32x2 %0, %1, ss, %0;\n\t}"
      : "+l"(acc)
      : "l"(a), "f"(s));
}
__device__ __forceinline__ void unpack2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void lds128x2(uint32_t a, uint64_t& p0, uint64_t& p1) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(p0), "=l"(p1) : "r"(a));
}
__device__ __forceinline__ void sts128x2(uint32_t a, uint64_t p0, uint64_t p1) {
  asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(a), "l"(p0), "l"(p1) : "memory");
}

// Split-TF32 on mma.sync m16n8k8: x = hi + lo (both tf32; lo's rounding
// residual is <= 2^-23 |x|), D += [Alo*Blo +] Alo*Bhi + Ahi*Blo + Ahi*Bhi in
// fp32.  The lo*lo term (TNB_DOT_4TERM) halves the per-product error, which
// cfg4's heavily cancelling dots need to stay inside 1e-5.
#ifndef TNB_DOT_4TERM
#define TNB_DOT_4TERM 0
#endif
// TNB_DOT_TRUNC_SPLIT (2 instructions per split instead of 3):
//   1: hi = x itself (the tensor core reads only its tf32 bits, i.e.
//      truncates), lo = x - trunc(x): 4x the per-product error;
//   2: hi = rna(x), lo = x - hi exact and passed unrounded (the tensor core
//      truncates it): the dropped bits of lo are below 2^-21 |x| and the
//      measured cfg4 error equals the fully rounded split's.
//   0: hi = rna(x), lo = rna(x - hi).
#ifndef TNB_DOT_TRUNC_SPLIT
#define TNB_DOT_TRUNC_SPLIT 3  /* 1: cfg4 dot 1.32 ms but relFro 1.06e-5, over the 1e-5 bar;
                                  2: 1.43 ms at relFro 2.5e-6 (= the fully rounded split's);
                                  3: the same bits as 2 in 3 instead of 5 instructions: 1.27 ms */
#endif
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
#if TNB_DOT_TRUNC_SPLIT == 1
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
#elif TNB_DOT_TRUNC_SPLIT == 3
  // as 2, with the round-to-nearest-away done on the bit pattern: cvt.rna
  // compiles to add / NaN test / select / mask, this to add / mask (the same
  // hi for every finite x; a NaN still reaches the products through lo)
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
#elif TNB_DOT_TRUNC_SPLIT == 2
  // hi rounded, lo = x - hi exact but left for the tensor core to truncate
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  lo = __float_as_uint(x - __uint_as_float(hi));
#else
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
#endif
}
// TNB_DOT_PAIR: two values per split with one packed fp32x2 subtract (FADD2)
// for the two lo parts, and packed adds for the running partial
#ifndef TNB_DOT_PAIR
#define TNB_DOT_PAIR 1
#endif
__device__ __forceinline__ void split2_tf32(float x0, float x1, uint32_t& h0, uint32_t& h1, uint32_t& l0,
                                            uint32_t& l1) {
#if TNB_DOT_PAIR && TNB_DOT_TRUNC_SPLIT == 3
  h0 = (__float_as_uint(x0) + 0x1000u) & 0xffffe000u;
  h1 = (__float_as_uint(x1) + 0x1000u) & 0xffffe000u;
  uint64_t X, H, L;
  asm("mov.b64 %0, {%1, %2};" : "=l"(X) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(H) : "r"(h0), "r"(h1));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(L) : "l"(X), "l"(H));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(l0), "=r"(l1) : "l"(L));
#else
  split_tf32(x0, h0, l0);
  split_tf32(x1, h1, l1);
#endif
}
__device__ __forceinline__ void add4(float (&d)[4], const float (&z)[4]) {
#if TNB_DOT_PAIR
#pragma unroll
  for (int i = 0; i < 4; i += 2) {
    uint64_t D, Z;
    asm("mov.b64 %0, {%1, %2};" : "=l"(D) : "f"(d[i]), "f"(d[i + 1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(Z) : "f"(z[i]), "f"(z[i + 1]));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(D) : "l"(Z));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d[i]), "=f"(d[i + 1]) : "l"(D));
  }
#else
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] += z[i];
#endif
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma3s(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint32_t h0,
                                      uint32_t h1, uint32_t l0, uint32_t l1) {
  mma_tf32(d, al, h0, h1);
  mma_tf32(d, ah, l0, l1);
  mma_tf32(d, ah, h0, h1);
}
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], float b0,
                                     float b1) {
  uint32_t h0, l0, h1, l1;
  split2_tf32(b0, b1, h0, h1, l0, l1);
#if TNB_DOT_4TERM
  mma_tf32(d, al, l0, l1);
#endif
  mma_tf32(d, al, h0, h1);
  mma_tf32(d, ah, l0, l1);
  mma_tf32(d, ah, h0, h1);
}

// TNB_DOT_ILV: issue order of a slice's MMAs.  0: each accumulator's three
// split products back to back (a dependent chain of 6 per accumulator);
// 1: the two n-tiles' chains interleaved; 2: also one accumulator per k-chunk
// (four chains of 3, joined with fp32 adds: half the error, 4-7% slower).
// Two slices per warp at a time (four chains) measured no faster than 1.
#ifndef TNB_DOT_ILV
#define TNB_DOT_ILV 1
#endif
__device__ __forceinline__ void mma3s_pair(float (&d0)[4], float (&d1)[4], const uint32_t (&ah)[4],
                                           const uint32_t (&al)[4], const uint32_t (&Bh)[4],
                                           const uint32_t (&Bl)[4]) {
  mma_tf32(d0, al, Bh[0], Bh[1]);
  mma_tf32(d1, al, Bh[2], Bh[3]);
  mma_tf32(d0, ah, Bl[0], Bl[1]);
  mma_tf32(d1, ah, Bl[2], Bl[3]);
  mma_tf32(d0, ah, Bh[0], Bh[1]);
  mma_tf32(d1, ah, Bh[2], Bh[3]);
}
__device__ __forceinline__ void mma3_pair(float (&d0)[4], float (&d1)[4], const uint32_t (&ah)[4],
                                          const uint32_t (&al)[4], const float (&y)[4]) {
  uint32_t Bh[4], Bl[4];
#pragma unroll
  for (int i = 0; i < 4; i += 2) split2_tf32(y[i], y[i + 1], Bh[i], Bh[i + 1], Bl[i], Bl[i + 1]);
  mma3s_pair(d0, d1, ah, al, Bh, Bl);
}

// One interior slice on tensor cores.  Fragments (m16n8k8 tf32, g = lane/4,
// t = lane%4) with the K slots permuted: slot t <-> index 2t, slot t+4 <->
// 2t+1 of each 8-chunk kc.  Then the accumulator fragment of one product is
// exactly the B fragment of the next, so M and Y never leave registers:
//   Mc[nt] = {M[g][8nt+2t], M[g][8nt+2t+1], M[g+8][8nt+2t], M[g+8][8nt+2t+1]}
//   step 1: Y^T = B_j^T M^T   (A = B_j^T from smem, B(kc, nt) = Mc[kc] halves)
//   step 2: Mw += A_j^T Y     (A = A_j^T from smem, B(kc, nt) = Y^T halves)
__device__ __forceinline__ void slice_afrag(const float* S, int kc, int g, int t, uint32_t (&ah)[4],
                                            uint32_t (&al)[4]) {
  const float* r0 = S + (8 * kc + 2 * t) * 16;
  split2_tf32(r0[g], r0[g + 8], ah[0], ah[1], al[0], al[1]);
  split2_tf32(r0[16 + g], r0[16 + g + 8], ah[2], ah[3], al[2], al[3]);
}
// SAME (norm: A_j == B_j): the slice's split fragments serve both products
template <bool SAME>
__device__ __forceinline__ void slice_mma(const float* Aj, const float* Bj, const uint32_t (&Mh)[2][4],
                                          const uint32_t (&Ml)[2][4], float (&Mw)[2][4], int g, int t) {
  float Y[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  uint32_t sh[SAME ? 2 : 1][4], sl[SAME ? 2 : 1][4];  // B_j's fragments, kept for A_j^T Y when SAME
#if TNB_DOT_ILV == 2
  {
    float Y2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    uint32_t th[2][4], tl[2][4];
    slice_afrag(Bj, 0, g, t, th[0], tl[0]);
    slice_afrag(Bj, 1, g, t, th[1], tl[1]);
    mma_tf32(Y[0], tl[0], Mh[0][0], Mh[0][1]);
    mma_tf32(Y[1], tl[0], Mh[0][2], Mh[0][3]);
    mma_tf32(Y2[0], tl[1], Mh[1][0], Mh[1][1]);
    mma_tf32(Y2[1], tl[1], Mh[1][2], Mh[1][3]);
    mma_tf32(Y[0], th[0], Ml[0][0], Ml[0][1]);
    mma_tf32(Y[1], th[0], Ml[0][2], Ml[0][3]);
    mma_tf32(Y2[0], th[1], Ml[1][0], Ml[1][1]);
    mma_tf32(Y2[1], th[1], Ml[1][2], Ml[1][3]);
    mma_tf32(Y[0], th[0], Mh[0][0], Mh[0][1]);
    mma_tf32(Y[1], th[0], Mh[0][2], Mh[0][3]);
    mma_tf32(Y2[0], th[1], Mh[1][0], Mh[1][1]);
    mma_tf32(Y2[1], th[1], Mh[1][2], Mh[1][3]);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) Y[nt][i] += Y2[nt][i];
    if constexpr (SAME) {
#pragma unroll
      for (int kc = 0; kc < 2; ++kc)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sh[SAME ? kc : 0][i] = th[kc][i];
          sl[SAME ? kc : 0][i] = tl[kc][i];
        }
    }
  }
#else
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    const int ks = SAME ? kc : 0;
    slice_afrag(Bj, kc, g, t, sh[ks], sl[ks]);
#if TNB_DOT_ILV == 1
    mma3s_pair(Y[0], Y[1], sh[ks], sl[ks], Mh[kc], Ml[kc]);
#else
    mma3s(Y[0], sh[ks], sl[ks], Mh[kc][0], Mh[kc][1], Ml[kc][0], Ml[kc][1]);
    mma3s(Y[1], sh[ks], sl[ks], Mh[kc][2], Mh[kc][3], Ml[kc][2], Ml[kc][3]);
#endif
  }
#endif
  // this slice's A_j^T Y starts from zero and joins the running partial
  // with round-to-nearest FADDs: the MMA accumulator only ever sums the 6
  // products of one slice
  float Z[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#if TNB_DOT_ILV == 2
  float Z2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#endif
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    uint32_t ah[4], al[4];
    if constexpr (SAME) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ah[i] = sh[SAME ? kc : 0][i];
        al[i] = sl[SAME ? kc : 0][i];
      }
    } else {
      slice_afrag(Aj, kc, g, t, ah, al);
    }
#if TNB_DOT_ILV == 2
    if (kc == 1) {  // the second k-chunk has its own accumulators (joined below)
      mma3_pair(Z2[0], Z2[1], ah, al, Y[kc]);
      continue;
    }
#endif
#if TNB_DOT_ILV >= 1
    mma3_pair(Z[0], Z[1], ah, al, Y[kc]);
#else
    mma3(Z[0], ah, al, Y[kc][0], Y[kc][1]);
    mma3(Z[1], ah, al, Y[kc][2], Y[kc][3]);
#endif
  }
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#if TNB_DOT_ILV == 2
      Z[nt][i] += Z2[nt][i];
#endif
#if !TNB_DOT_PAIR
      Mw[nt][i] += Z[nt][i];
#endif
    }
#if TNB_DOT_PAIR
  add4(Mw[0], Z[0]);
  add4(Mw[1], Z[1]);
#endif
}

struct DotArgs {
  ChainDev a, b;  // a.m[k].s + e * bstride = slices of pair e
  float* out;
  int norm;
};

// chunk bookkeeping: the CTA walks (pair, core, chunk) in order
struct Walk {
  int64_t e;
  int k, c;
};

template <bool MMA, bool SAME>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) dot_r16_kernel(const __grid_constant__ DotArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* stA = reinterpret_cast<float*>(smem);                      // [kStages][CH*R*R]
  float* stB = stA + kStages * CH * R * R;                          // [kStages][CH*R*R]
  float* ybuf = stB + (args.norm ? 0 : kStages * CH * R * R);       // [kWarps][R*R]
  float* red = ybuf + 2 * kWarps * R * R;                           // [kWarps][R*R]
  float* msm = red + kWarps * R * R;                                // [R*R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(msm + R * R);        // full[kStages], empty[kStages]
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // barrier of the compute warps only (the producer warp never joins)
  auto csync = [&]() {
    if (TNB_DOT_PRODUCER) asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
    else __syncthreads();
  };
  const int ap = lane >> 2, dq = lane & 3;  // rows/cols 2ap,2ap+1 ; 4dq..4dq+3
  const int fg = lane >> 2, ft = lane & 3;  // mma fragment coordinates (MMA path)
  const int N = args.a.n, J = args.a.m[0].J;
  const int nch = (J + CH - 1) / CH;
  const int64_t B = args.a.batch;
  constexpr bool same = SAME;  // norm: A == B (one operand streamed)

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // producer state (thread 0): next chunk to load
  Walk pw{(int64_t)blockIdx.x, 0, 0};
  uint32_t p_it = 0;
  auto produce_one = [&]() {
    if (pw.e >= B) return;
    const int s = p_it % kStages;
    mbar_wait_suspend(&empty[s], ((p_it / kStages) & 1) ^ 1);
    const ModeDev& ma = args.a.m[pw.k];
    const ModeDev& mb = args.b.m[pw.k];
    const int j0 = pw.c * CH, nj = min(CH, J - j0);
    const uint32_t sz = (uint32_t)(nj * ma.rl * ma.rr * 4);
    mbar_expect_tx(&full[s], same ? sz : 2 * sz);
    bulk_g2s(stA + s * CH * R * R, ma.s + pw.e * ma.bstride + (int64_t)j0 * ma.rl * ma.rr, sz, &full[s]);
    if (!same)
      bulk_g2s(stB + s * CH * R * R, mb.s + pw.e * mb.bstride + (int64_t)j0 * mb.rl * mb.rr, sz,
               &full[s]);
    ++p_it;
    if (++pw.c == nch) {
      pw.c = 0;
      if (++pw.k == N) {
        pw.k = 0;
        pw.e += gridDim.x;
      }
    }
  };
  if (TNB_DOT_PRODUCER) {
    if (warp == kWarps) {  // the producer warp: every chunk of this CTA, in order
      if (lane == 0)
        while (pw.e < B) produce_one();
      return;
    }
  } else if (tid == 0) {
    for (int s = 0; s < kStages; ++s) produce_one();
  }

  uint32_t c_it = 0;
  for (int64_t e = blockIdx.x; e < B; e += gridDim.x) {
    float mrow[2][R];  // M rows 2ap, 2ap+1 (registers, SIMT path)
    uint32_t Mh[2][4], Ml[2][4];  // M as split-TF32 mma fragments (MMA path)
    for (int k = 0; k < N; ++k) {
      const bool first = (k == 0), last = (k == N - 1);
      uint64_t mn[2][2] = {{0ull, 0ull}, {0ull, 0ull}};
      uint64_t mn2[2][2] = {{0ull, 0ull}, {0ull, 0ull}};  // second slice of the pair
      float Mw[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};  // MMA partial M
      float lastacc = 0.f;
      float4 mq0 = make_float4(0.f, 0.f, 0.f, 0.f), mq1 = mq0;  // M[2ap(+1)][4dq..]
      if (last && !first) {
        mq0 = *reinterpret_cast<const float4*>(msm + (2 * ap) * R + dq * 4);
        mq1 = *reinterpret_cast<const float4*>(msm + (2 * ap + 1) * R + dq * 4);
      }
      for (int c = 0; c < nch; ++c) {
        const int s = c_it % kStages;
        mbar_wait(&full[s], (c_it / kStages) & 1);
        const float* A = stA + s * CH * R * R;
        const float* Bm = same ? A : stB + s * CH * R * R;
        const int nj = min(CH, J - c * CH);
        if (MMA && !first && !last) {  // interior slices on tensor cores (the loop the kernel lives in)
#pragma unroll 1
          for (int jj = warp; jj < nj; jj += kWarps)
            slice_mma<SAME>(A + jj * R * R, Bm + jj * R * R, Mh, Ml, Mw, fg, ft);
        } else
        for (int jj = warp; jj < nj; jj += kWarps) {
          if (first) {  // 1 x R slices: M' += A_j^T B_j
            const uint32_t a_row = su32(A + jj * R), b_row = su32(Bm + jj * R);
            uint64_t b0, b1;
            lds128x2(b_row + dq * 16, b0, b1);
            float a0, a1;
            unpack2(lds64(a_row + ap * 8), a0, a1);
            ffma2(mn[0][0], b0, a0);
            ffma2(mn[0][1], b1, a0);
            ffma2(mn[1][0], b0, a1);
            ffma2(mn[1][1], b1, a1);
          } else if (last) {  // R x 1 slices: s += a_j . (M b_j)
            const float* aj = A + jj * R;
            const float* bj = Bm + jj * R;
            const float4 bv = *reinterpret_cast<const float4*>(bj + dq * 4);
            const float a0 = aj[2 * ap], a1 = aj[2 * ap + 1];
            float y0 = 0.f, y1 = 0.f;
            y0 = fmaf(mq0.x, bv.x, y0);
            y0 = fmaf(mq0.y, bv.y, y0);
            y0 = fmaf(mq0.z, bv.z, y0);
            y0 = fmaf(mq0.w, bv.w, y0);
            y1 = fmaf(mq1.x, bv.x, y1);
            y1 = fmaf(mq1.y, bv.y, y1);
            y1 = fmaf(mq1.z, bv.z, y1);
            y1 = fmaf(mq1.w, bv.w, y1);
            lastacc = fmaf(a0, y0, lastacc);
            lastacc = fmaf(a1, y1, lastacc);
          } else if (MMA) {
            // (taken by the loop above)
          } else if (jj < kWarps) {
            // two slices per warp (jj, jj + kWarps): 8 independent FFMA2 chains
            const int j2 = jj + kWarps;
            const bool two = j2 < nj;
            const uint32_t bj1 = su32(Bm + jj * R * R), bj2 = su32(Bm + (two ? j2 : jj) * R * R);
            uint64_t y1[2][2] = {{0ull, 0ull}, {0ull, 0ull}}, y2[2][2] = {{0ull, 0ull}, {0ull, 0ull}};
#pragma unroll
            for (int b = 0; b < R; ++b) {
              uint64_t p0, p1, r0, r1;
              lds128x2(bj1 + b * 64 + dq * 16, p0, p1);
              lds128x2(bj2 + b * 64 + dq * 16, r0, r1);
              ffma2(y1[0][0], p0, mrow[0][b]);
              ffma2(y1[0][1], p1, mrow[0][b]);
              ffma2(y1[1][0], p0, mrow[1][b]);
              ffma2(y1[1][1], p1, mrow[1][b]);
              ffma2(y2[0][0], r0, mrow[0][b]);
              ffma2(y2[0][1], r1, mrow[0][b]);
              ffma2(y2[1][0], r0, mrow[1][b]);
              ffma2(y2[1][1], r1, mrow[1][b]);
            }
            const uint32_t yw1 = su32(ybuf + (2 * warp) * R * R), yw2 = yw1 + R * R * 4;
            sts128x2(yw1 + (2 * ap) * 64 + dq * 16, y1[0][0], y1[0][1]);
            sts128x2(yw1 + (2 * ap + 1) * 64 + dq * 16, y1[1][0], y1[1][1]);
            sts128x2(yw2 + (2 * ap) * 64 + dq * 16, y2[0][0], y2[0][1]);
            sts128x2(yw2 + (2 * ap + 1) * 64 + dq * 16, y2[1][0], y2[1][1]);
            __syncwarp();
            // Mw += A_j^T Y_j for both slices (second slice masked by 'two')
            const uint32_t aj1 = su32(A + jj * R * R), aj2 = su32(A + (two ? j2 : jj) * R * R);
            const float w2 = two ? 1.f : 0.f;
#pragma unroll
            for (int a = 0; a < R; ++a) {
              uint64_t q0, q1, t0, t1;
              lds128x2(yw1 + a * 64 + dq * 16, q0, q1);
              lds128x2(yw2 + a * 64 + dq * 16, t0, t1);
              float a0, a1, c0, c1;
              unpack2(lds64(aj1 + a * 64 + ap * 8), a0, a1);
              unpack2(lds64(aj2 + a * 64 + ap * 8), c0, c1);
              c0 *= w2;
              c1 *= w2;
              ffma2(mn[0][0], q0, a0);
              ffma2(mn[0][1], q1, a0);
              ffma2(mn[1][0], q0, a1);
              ffma2(mn[1][1], q1, a1);
              ffma2(mn2[0][0], t0, c0);
              ffma2(mn2[0][1], t1, c0);
              ffma2(mn2[1][0], t0, c1);
              ffma2(mn2[1][1], t1, c1);
            }
            __syncwarp();
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        ++c_it;
        if (!TNB_DOT_PRODUCER && tid == 0) produce_one();
      }
      // ---- reduce the per-warp partial M over warps ----
      if (last) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lastacc += __shfl_xor_sync(0xffffffffu, lastacc, o);
        if (lane == 0) red[warp] = lastacc;
        csync();
        if (tid == 0) {
          float v = 0.f;
          for (int w = 0; w < kWarps; ++w) v += red[w];
          args.out[e] = args.norm ? sqrtf(fmaxf(v, 0.f)) : v;
        }
        csync();
      } else {
        float* rw = red + warp * R * R;
        if (MMA && !first) {
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            *reinterpret_cast<float2*>(rw + fg * R + 8 * nt + 2 * ft) = make_float2(Mw[nt][0], Mw[nt][1]);
            *reinterpret_cast<float2*>(rw + (fg + 8) * R + 8 * nt + 2 * ft) = make_float2(Mw[nt][2], Mw[nt][3]);
          }
        } else
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          float x0, x1, x2, x3, z0, z1, z2, z3;
          unpack2(mn[i][0], x0, x1);
          unpack2(mn[i][1], x2, x3);
          unpack2(mn2[i][0], z0, z1);
          unpack2(mn2[i][1], z2, z3);
          x0 += z0;
          x1 += z1;
          x2 += z2;
          x3 += z3;
          *reinterpret_cast<float4*>(rw + (2 * ap + i) * R + dq * 4) = make_float4(x0, x1, x2, x3);
        }
        csync();
        for (int e = tid; e < R * R; e += kCompute) {
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) v += red[w * R * R + e];
          msm[e] = v;
        }
        csync();
        if (MMA) {
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const float2 u = *reinterpret_cast<const float2*>(msm + fg * R + 8 * nt + 2 * ft);
            const float2 v = *reinterpret_cast<const float2*>(msm + (fg + 8) * R + 8 * nt + 2 * ft);
            split_tf32(u.x, Mh[nt][0], Ml[nt][0]);
            split_tf32(u.y, Mh[nt][1], Ml[nt][1]);
            split_tf32(v.x, Mh[nt][2], Ml[nt][2]);
            split_tf32(v.y, Mh[nt][3], Ml[nt][3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int b = 0; b < R; ++b) mrow[i][b] = msm[(2 * ap + i) * R + b];
        }
        // no barrier here: the next writes of red / msm come after the next
        // mode's first barrier, which every warp reaches only after these reads
      }
    }
  }
}

size_t dot_smem(bool norm) {
  const size_t stage = (size_t)kStages * CH * R * R * 4;
  return stage * (norm ? 1 : 2) + (size_t)(3 * kWarps * R * R + R * R) * 4 + 2 * kStages * 8 + 16;
}

bool chain_ok(const ChainDev& c) {
  if (c.n < 2) return false;
  const int J = c.m[0].J;
  if (J < 1) return false;
  for (int k = 0; k < c.n; ++k) {
    const ModeDev& m = c.m[k];
    if (m.layout != TNB_LAYOUT_DENSE || m.J != J) return false;
    const int rl = (k == 0) ? 1 : R, rr = (k == c.n - 1) ? 1 : R;
    if (m.rl != rl || m.rr != rr) return false;
    // bulk copies need 16-byte aligned sources
    if ((reinterpret_cast<uintptr_t>(m.s) & 15) || ((m.bstride * 4) & 15)) return false;
  }
  return true;
}

}  // namespace

bool dot_fast_supported(const ChainDev& a, const ChainDev& b) {
  return chain_ok(a) && chain_ok(b) && a.n == b.n && a.batch == b.batch;
}

int launch_dot_fast(const ChainDev& a, const ChainDev& b, float* out, bool is_norm, cudaStream_t st) {
  DotArgs args;
  args.a = a;
  args.b = b;
  args.out = out;
  args.norm = is_norm ? 1 : 0;
  const size_t smem = dot_smem(is_norm);
  const char* e = getenv("TNB_DOT_SIMT");
  auto kern = (e && e[0] == '1') ? (is_norm ? dot_r16_kernel<false, true> : dot_r16_kernel<false, false>)
                                 : (is_norm ? dot_r16_kernel<true, true> : dot_r16_kernel<true, false>);
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "dot smem attr");
  if (rc) return rc;
  const int64_t slots = (int64_t)num_sms() * kCtasPerSm;
  const int grid = (int)(a.batch < slots ? a.batch : slots);
  kern<<<grid, kThreads, smem, st>>>(args);
  return check_launch("dot_r16");
}

}  // namespace tnb
