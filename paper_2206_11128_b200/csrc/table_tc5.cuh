// Dense table levels on tcgen05 (round 2): the large levels of the prefix /
// suffix tables that mode merging builds per call (entries_bucketed.cu,
// plan_merge / build_tables; reference: the core-by-core products of
// core.py:432-444 hoisted out of the per-sample loop).
//
//   prefix level:  out[(p*J + j)*Nn + c] = sum_a in[p*K + a] G(j, a, c)    (K = rl, Nn = rr)
//   suffix level:  out[(j*rows + x)*Nn + a] = sum_c G(j, a, c) in[x*K + c]  (K = rr, Nn = rl)
//
// Both are, per slice j, D_j (rows x Nn) = IN (rows x K) . B_j with B_j = G_j
// (prefix) or G_j^T (suffix), K, Nn <= 32.  One CTA takes 128 rows of IN as
// the A operand (SW128 K-major tile, hi = the fp32 bits the tensor core
// truncates itself, lo = x - trunc(x)) and walks the slices in groups of 8:
// the group's B operands are 8 consecutive 32-row images (N = 256 per MMA),
// prepared once per level by t5_image_kernel (tf32 hi and lo), so a group
// costs 3 MMAs per k-step.  Accumulators: 2 x 256 TMEM columns.  The
// epilogue warps read each slice's 128 x 32 block from TMEM (thread = row),
// turn it through shared memory and write whole 128-byte lines.
// The mma.sync kernel (table_gemm_tc) stays for small levels and odd shapes.
#pragma once

namespace {

#ifndef TNB_TABLE_T5
#define TNB_TABLE_T5 1
#endif
constexpr int kT5Threads = 256;  // warp 0 MMA, warp 1 image loader, warps 4-7 A loader + epilogue
constexpr int kT5Grp = 8;        // slices per MMA group
constexpr int kT5Tile = 128 * 128;                      // operand tile: 128 rows x 128 B
constexpr int kT5Slot = 2 * kT5Grp * 4096;              // hi + lo images of a group: 64 KB
constexpr int kT5Stage = 4 * 2 * 4096;                  // per epilogue warp two 32-row x 128-byte staging blocks
constexpr int kT5Smem = 2 * kT5Tile + 2 * kT5Slot + kT5Stage + 128 + 1024;

bool t5_env() {
  const char* e = getenv("TNB_TABLE_T5");
  return TNB_TABLE_T5 && !(e && e[0] == '0');
}

// levels worth a tcgen05 launch: dense, both ranks multiples of 4 up to 32, at least 4096 input rows
bool t5_level_ok(const ModeDev& md, int64_t rows, bool suffix) {
  const int K = suffix ? md.rr : md.rl, Nn = suffix ? md.rl : md.rr;
  return t5_env() && md.layout == TNB_LAYOUT_DENSE && K >= 4 && K <= 32 && (K & 3) == 0 && Nn >= 4 && Nn <= 32 &&
         (Nn & 3) == 0 && rows >= 4096 && md.J >= 1;
}

int64_t t5_image_bytes(const ModeDev& md) { return (int64_t)md.J * 8192; }

// B_j[n][k]: prefix G(j, k, n), suffix G(j, n, k); image row n = 128 bytes, 16-byte piece c at c ^ (n & 7);
// all hi images first (J x 4 KB), then all lo images
template <bool SUFFIX>
__global__ void t5_image_kernel(ModeDev md, unsigned char* __restrict__ img) {
  const int J = md.J, rl = md.rl, rr = md.rr;
  const int K = SUFFIX ? rr : rl, Nn = SUFFIX ? rl : rr;
  const int64_t total = (int64_t)J * 256;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t >> 8;
    const int n = (int)(t >> 3) & 31, c = (int)t & 7;
    uint4 hi, lo;
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 4 * c + i;
      float x = 0.f;
      if (n < Nn && k < K) x = __ldg(md.s + (SUFFIX ? ((j * rl + n) * rr + k) : ((j * rl + k) * rr + n)));
      split_tf32(x, h[i], l[i]);
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
    unsigned char* dst = img + j * 4096 + n * 128 + ((c ^ (n & 7)) << 4);
    *reinterpret_cast<uint4*>(dst) = hi;
    *reinterpret_cast<uint4*>(dst + (int64_t)J * 4096) = lo;
  }
}

__device__ __forceinline__ void t5_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = s32(b);
  uint32_t done;
  int spins = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(1000000u)
        : "memory");
    if (done) return;
    if (++spins > 30000) __trap();  // a protocol bug, not a slow tile
  }
}
__device__ __forceinline__ void t5_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void t5_commit(uint64_t* b) {  // whole warp, one elected lane
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(s32(b))
      : "memory");
}
__device__ __forceinline__ void t5_mma(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
#define T5_TMEM_LD32(taddr, v)                                                                 \
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

template <bool SUFFIX>
__global__ void __launch_bounds__(kT5Threads, 1) t5_level_kernel(ModeDev md, const float* __restrict__ in, int64_t rows,
                                                                float* __restrict__ out,
                                                                const unsigned char* __restrict__ img) {
  extern __shared__ __align__(1024) unsigned char t5_raw[];
  unsigned char* smem = t5_raw + ((1024 - (s32(t5_raw) & 1023)) & 1023);
  unsigned char* sAhi = smem;
  unsigned char* sAlo = smem + kT5Tile;
  unsigned char* sB = smem + 2 * kT5Tile;              // [2 slots][hi 32 KB | lo 32 KB]
  unsigned char* sStage = sB + 2 * kT5Slot;            // [4 warps][2][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + kT5Stage);
  uint64_t* a_ready = bars;        // 128 loader threads
  uint64_t* b_full = bars + 1;     // [2] tx
  uint64_t* b_empty = bars + 3;    // [2] tcgen05.commit
  uint64_t* acc_full = bars + 5;   // [2] tcgen05.commit
  uint64_t* acc_empty = bars + 7;  // [2] 128 epilogue threads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = md.J;
  const int K = SUFFIX ? md.rr : md.rl, Nn = SUFFIX ? md.rl : md.rr;
  const int nk = (K + 7) >> 3;
  const int ng = (J + kT5Grp - 1) / kT5Grp;
  const int64_t i0 = (int64_t)blockIdx.x * 128;

  if (tid == 0) {
    mb_init(a_ready, 128);
    for (int s = 0; s < 2; ++s) {
      mb_init(&b_full[s], 1);
      mb_init(&b_empty[s], 1);
      mb_init(&acc_full[s], 1);
      mb_init(&acc_empty[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = s32(smem);

  if (warp == 0) {
    // ================= MMA issuer =================
    const uint64_t dc = ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
    const uint32_t ah = sbase >> 4, al = (sbase + kT5Tile) >> 4;
    t5_wait(a_ready, 0);
    for (int g = 0; g < ng; ++g) {
      const int slot = g & 1;
      const int cnt = min(kT5Grp, J - g * kT5Grp);
      t5_wait(&b_full[slot], (g >> 1) & 1);
      t5_wait(&acc_empty[slot], ((g >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((32 * cnt) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t bh = (sbase + 2 * kT5Tile + slot * kT5Slot) >> 4, bl = bh + ((kT5Grp * 4096) >> 4);
      const uint32_t d = tmem + slot * 256;
      for (int kk = 0; kk < nk; ++kk) {
        const uint64_t dah = dc | (uint64_t)(ah + 2 * kk), dal = dc | (uint64_t)(al + 2 * kk);
        const uint64_t dbh = dc | (uint64_t)(bh + 2 * kk), dbl = dc | (uint64_t)(bl + 2 * kk);
        t5_mma(d, dal, dbh, idesc, kk > 0);
        t5_mma(d, dah, dbl, idesc, 1);
        t5_mma(d, dah, dbh, idesc, 1);
      }
      t5_commit(&acc_full[slot]);
      t5_commit(&b_empty[slot]);
    }
  } else if (warp == 1) {
    // ================= slice images -> shared memory =================
    if (lane == 0) {
      for (int g = 0; g < ng; ++g) {
        const int slot = g & 1;
        const int cnt = min(kT5Grp, J - g * kT5Grp);
        t5_wait(&b_empty[slot], ((g >> 1) & 1) ^ 1);
        mb_expect(&b_full[slot], (uint32_t)cnt * 8192u);
        unsigned char* dst = sB + slot * kT5Slot;
        bulk(dst, img + (int64_t)g * kT5Grp * 4096, (uint32_t)cnt * 4096u, &b_full[slot]);
        bulk(dst + kT5Grp * 4096, img + (int64_t)J * 4096 + (int64_t)g * kT5Grp * 4096, (uint32_t)cnt * 4096u,
             &b_full[slot]);
      }
    }
  } else if (warp >= 4) {
    // ================= A tile, then the epilogue: thread = row =================
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t swz = (uint32_t)(row & 7);
    const bool rok = i0 + row < rows;
    {
      const float* src = in + (i0 + row) * K;
      const uint32_t a = sbase + (uint32_t)row * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rok && 4 * c < K) x = __ldg(reinterpret_cast<const float4*>(src) + c);
        const uint32_t off = ((uint32_t)c ^ swz) << 4;
        const uint32_t l0 = __float_as_uint(x.x - __uint_as_float(__float_as_uint(x.x) & 0xffffe000u));
        const uint32_t l1 = __float_as_uint(x.y - __uint_as_float(__float_as_uint(x.y) & 0xffffe000u));
        const uint32_t l2 = __float_as_uint(x.z - __uint_as_float(__float_as_uint(x.z) & 0xffffe000u));
        const uint32_t l3 = __float_as_uint(x.w - __uint_as_float(__float_as_uint(x.w) & 0xffffe000u));
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a + off), "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w) : "memory");
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + kT5Tile + off), "r"(l0), "r"(l1), "r"(l2), "r"(l3)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      t5_arrive(a_ready);
    }
    const uint32_t stg = s32(sStage) + (uint32_t)q * 8192;
    const int n4 = Nn >> 2;
    const int c = lane & 7, rsub = lane >> 3;
    uint32_t nst = 0;  // staging blocks used so far (alternating)
    for (int g = 0; g < ng; ++g) {
      const int slot = g & 1;
      const int cnt = min(kT5Grp, J - g * kT5Grp);
      t5_wait(&acc_full[slot], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int s = 0; s < cnt; ++s, ++nst) {
        uint32_t v[32];
        T5_TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + slot * 256 + s * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // the warp's 32 rows x Nn floats of slice j through shared memory: whole lines per store
        const uint32_t sb = stg + (nst & 1) * 4096;
        __syncwarp();  // the block's previous readers are done
#pragma unroll
        for (int p = 0; p < 8; ++p)
          if (p < n4)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sb + (uint32_t)lane * 128 + (((uint32_t)p ^ (uint32_t)(lane & 7)) << 4)),
                         "r"(v[4 * p]), "r"(v[4 * p + 1]), "r"(v[4 * p + 2]), "r"(v[4 * p + 3])
                         : "memory");
        __syncwarp();
        const int64_t j = (int64_t)g * kT5Grp + s;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 4 * i + rsub;           // row of the warp's block
          const int64_t gi = i0 + q * 32 + r;   // table row
          if (c < n4 && gi < rows) {
            const float4 x = lds128(sb + (uint32_t)r * 128 + (((uint32_t)c ^ (uint32_t)(r & 7)) << 4));
            float* dst = SUFFIX ? out + (j * rows + gi) * Nn : out + (gi * J + j) * Nn;
            *reinterpret_cast<float4*>(dst + 4 * c) = x;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      t5_arrive(&acc_empty[slot]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
  }
}

// one level on tcgen05; `img` = scratch for the level's slice images (t5_image_bytes)
template <bool SUFFIX>
int launch_t5_level(const ModeDev& md, const float* in, int64_t rows, float* out, unsigned char* img, cudaStream_t st) {
  int rc = check_cuda(cudaFuncSetAttribute(t5_level_kernel<SUFFIX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT5Smem),
                      "t5 smem attr");
  if (rc) return rc;
  const int gi = (int)std::min<int64_t>(ceil_div((int64_t)md.J * 256, 256), (int64_t)num_sms() * 4);
  t5_image_kernel<SUFFIX><<<gi, 256, 0, st>>>(md, img);
  t5_level_kernel<SUFFIX><<<(unsigned)ceil_div(rows, 128), kT5Threads, kT5Smem, st>>>(md, in, rows, out, img);
  return check_launch("t5 table level");
}

}  // namespace
