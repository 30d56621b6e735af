// K1, global-sort path (TNB_ALGO_GSORT): entry evaluation on tcgen05.
//
// Reference algorithm (core.py:432-444): per mode, argsort the samples by
// their index so every group shares one core slice and the group's update is
// a real GEMM.  The bucketed kernels (entries_bucketed.cu) group per tile,
// on chip, which leaves ~45 samples per bucket: too few rows for a tcgen05
// tile, so they run mma.sync.  This path sorts ONCE, globally, by the index
// of a MERGED interior mode, so that every bucket is thousands of samples
// that share one B operand and the per-entry work is ONE r x r product:
//
//   * mode merging (plan_merge) shortens the chain to
//       first . [dense interior modes] . [diag table] . last
//     and plan_gsort merges the dense interior modes into one table of
//     K = prod J slices M[key] = G_a[j_a] ... G_b[j_b] (r0 x r1), each stored
//     as the UMMA K-major SWIZZLE_128B image of its transpose, split into
//     tf32 hi / lo (gs_mid_image_kernel).  cfg2: P0123 . G45 (1024 slices) .
//     S6789;  cfg5: P012 . G3 (128 slices) . D45 . S67;
//   * gs_prep_kernel: reads the int64 index rows once, wraps and validates
//     every ORIGINAL mode (lowest bad mode -> *err, core.py:409-416), and
//     writes one 16-byte record per sample {key, first row, last row, diag
//     row} plus the global histogram of the keys;
//   * gs_scan_kernel: bucket starts, and the start of every bucket in
//     128-sample tiles (the compute kernel's work list, balanced by tiles
//     whatever the skew); gs_tilemap_kernel: per tile {first sorted position,
//     bucket, rows};
//   * gs_scatter_kernel: counting-sort scatter of the records by key (the
//     order inside a bucket is not fixed, and need not be: a sample's
//     arithmetic does not depend on its position);
//   * entries_gsort_kernel (persistent, one 896-thread CTA per SM), per tile
//     of 128 sorted samples of one bucket:
//       16 producer warps gather the samples' first-table rows into the A
//                        operand tile (K-major SW128 layout) and their
//                        closing rows (last / diag tables) into shared memory
//                        with 16-byte cp.async, several tiles ahead (records
//                        through a per-warp cp.async ring; L2 policies:
//                        big tables stream, results stay; repeated rows go
//                        through L1);
//       4 splitter warps  lo = x - trunc_tf32(x) into a second tile (the MMA
//                        reads the gathered tile itself as hi: the tensor
//                        core ignores the low 13 mantissa bits);
//       one MMA warp     D[128 x 64] = A [Bhi | Blo], D[:, :32] += Alo Bhi
//                        (tcgen05.mma.kind::tf32, accumulators in TMEM, issued
//                        by one elected lane);
//       4 epilogue warps tcgen05.ld the D row of their sample, add the halves,
//                        dot it with the closing rows, write out[orig].
// The kernel runs at the rate the SM can keep random row gathers in flight
// (DESIGN 3 K1 2c, tools/gather_bench.cu); the MMAs take 13% of the tensor pipe.
// Results are bitwise reproducible and independent of the input order.
#pragma once

#define TMEM_LD16_GS(taddr, v)                                                                   \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, " \
      "%12, %13, %14, %15}, [%16];"                                                              \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),      \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), \
        "=r"(v[14]), "=r"(v[15])                                                                 \
      : "r"(taddr))

namespace {

constexpr int kGsSmemK = 8192;           // up to here the histograms live in shared memory
constexpr int kGsMaxK = 65536;           // buckets (above kGsSmemK: warp-aggregated global atomics)
constexpr int kGsTile = 128;             // samples per tile (UMMA M)
constexpr int kGsRow = 128;              // bytes per operand row (one SW128 atom row)
constexpr int kGsTileBytes = kGsTile * kGsRow;  // 16 KB
constexpr int kGsImgBytes = 2 * 32 * kGsRow;    // hi + lo image of one slice: 8 KB
constexpr int kGsNA = 4;                 // TMEM accumulators (64 columns each: A Bhi | A Blo)
constexpr int kGsNB = 2;                 // slice images in flight
// warps: 0 MMA, 1 image loader, 2-3 idle, 4-7 epilogue, 8-11 splitters, 12-27 producers
// (a warp holds at most ~8 LDGSTS in flight -- tools/gather_bench.cu -- so the
// gather rate and a tile's gather latency are set by the number of producer warps)
#ifndef TNB_GS_PW
#define TNB_GS_PW 16
#endif
// splitter: 1 = the MMA reads the gathered tile itself (hi = truncation by the
// tensor core), only lo is written; 0 = hi rounded to nearest, stored in place
#ifndef TNB_GS_TRUNC_HI
#define TNB_GS_TRUNC_HI 1
#endif
constexpr int kGsPW = TNB_GS_PW;         // producer warps (128 / kGsPW rows of every tile each)
constexpr int kGsRW = kGsTile / kGsPW;   // rows per producer warp
constexpr int kGsPasses = kGsRW / 4;     // 4 rows per copy instruction
static_assert(kGsRW * kGsPW == kGsTile && kGsPasses * 4 == kGsRW && kGsRW <= 32, "producer geometry");
constexpr int kGsThreads = (12 + kGsPW) * 32;
constexpr int kGsPrepThreads = 512;
constexpr int kGsScatThreads = 512, kGsScatPer = 8;  // 1024 x 4 and 256 x 8 measured equal / slower

struct GPlan {
  MergePlan mp;
  int gdiag = -1;          // virtual group of the diagonal table, or -1
  int omid_lo = 0, omid_hi = 0;  // original modes merged into the sorted mode
  int r0 = 0, r1 = 0;      // its slices are r0 x r1
  int64_t K = 0;           // sort buckets: Kmid slices x nsub row ranges of the first table
  int64_t Kmid = 0;        // slices of the merged sorted mode
  int nsub = 1;            // row ranges of the first table in the sort key (L2 locality)
  int64_t sub_rows = 0;    // rows per range (0: none)
  int chunk_shift = 0;     // > 0: the sample index >> chunk_shift leads the sort key (result windows, below)
  int64_t tinfo_off = 0;   // per-tile {first sorted position, bucket, rows}
  int64_t lvl_off[kMaxModes];  // mid level ending at original mode o (o > omid_lo)
  int64_t img_off = 0, hist_off = 0, bstart_off = 0, tbase_off = 0, cursor_off = 0;
  int64_t recu_off = 0, recs_off = 0, total_bytes = 0;
};

struct GsPrep {
  int32_t n0;
  uint32_t K;
  uint32_t Kmid, sub_rows;  // key = (first row / sub_rows) * Kmid + merged index (sub_rows 0: no row ranges)
  uint32_t chunk_shift;     // or key = (sample >> chunk_shift) * Kmid + merged index (0: none)
  int32_t oJ[kMaxModes];
  // C-order weight of mode o inside its group, in the group's field (first /
  // sorted / diag / last) and zero in the other three: no branches per mode
  uint32_t w0[kMaxModes], w1[kMaxModes], w2[kMaxModes], w3[kMaxModes];
};

// TNB_ENTRIES_GSORT: 0 = AUTO never picks this path, 2 = AUTO picks it for
// every chain it supports, default = when it merges at least two interior modes
int gsort_env() {
  const char* e = getenv("TNB_ENTRIES_GSORT");
  return (e && e[0] == '0') ? 0 : ((e && e[0] == '2') ? 2 : 1);
}

bool plan_gsort_with(const ChainDev& ch, int64_t m, GPlan* G, int64_t wide_rows);
// The merge the bucketed kernels use (wide tables of up to m / 8 rows), or --
// when that leaves too many interior modes for one sort (K > m / 512) -- the
// same with tables of up to m / 2, then m rows: a table row costs as much as
// one sorted step of one sample, and every absorbed mode removes that step
// from all m samples (cfg2 chain: P0123 . G45 . S6789 instead of six modes on
// the state kernel -- 0.38 against 1.0 ms at 2^22 tuples, 0.18 against 0.30 ms
// at 2^20).
// (batched: the chain is one element of a batched chain; same plan.)
bool plan_gsort(const ChainDev& ch, int64_t m, GPlan* G, bool batched = false) {
  if (plan_gsort_with(ch, m, G, 0) && G->K * 512 <= m) return true;
  // (small ranks stay with the first plan: 40^9, r = 8 at 2^22 tuples ran 0.41 against 0.39 ms)
  if (plan_gsort_with(ch, m, G, m / 2) && G->K * 512 <= m && G->r0 * G->r1 >= 256) return true;
  if (plan_gsort_with(ch, m, G, m) && G->K * 512 <= m && G->r0 * G->r1 >= 256) return true;
  return plan_gsort_with(ch, m, G, 0);
}

bool plan_gsort_with(const ChainDev& ch, int64_t m, GPlan* G, int64_t wide_rows) {
  const int N = ch.n;
  if (ch.batch != 1 || N < 3 || N > kMaxModes || m < 1 || m >= ((int64_t)1 << 31)) return false;
  for (int k = 0; k < N; ++k)
    if (ch.m[k].bstride != 0 || ch.m[k].J <= 0) return false;
  MergePlan& mp = G->mp;
  plan_merge(ch, m, &mp, wide_rows);
  if (mp.ng < 3) return false;
  // first: a [rows][r0] table
  const ModeDev& f = ch.m[mp.hi[0] - 1];
  if (mp.kind[0] == kOrig && (ch.m[0].layout != TNB_LAYOUT_DENSE || ch.m[0].rl != 1)) return false;
  if (mp.kind[0] != kOrig && mp.kind[0] != kPrefix) return false;
  const int r0 = f.rr;
  // the dense interior modes right after it
  int g = 1;
  int64_t K = 1;
  while (g < mp.ng - 1 && mp.kind[g] == kOrig && ch.m[mp.lo[g]].layout == TNB_LAYOUT_DENSE) {
    K *= ch.m[mp.lo[g]].J;
    if (K > kGsMaxK) return false;
    ++g;
  }
  if (g == 1) return false;
  G->omid_lo = mp.lo[1];
  G->omid_hi = mp.hi[g - 1];
  if (ch.m[G->omid_lo].rl != r0) return false;
  const int r1 = ch.m[G->omid_hi - 1].rr;
  for (int o = G->omid_lo; o < G->omid_hi; ++o)
    if (ch.m[o].rl > 32 || ch.m[o].rr > 32) return false;
  // at most one diagonal table
  G->gdiag = -1;
  if (g < mp.ng - 1) {
    const ModeDev& d = ch.m[mp.lo[g]];
    if (d.layout != TNB_LAYOUT_DIAG || d.rl != r1) return false;
    G->gdiag = g;
    ++g;
  }
  if (g != mp.ng - 1) return false;
  // last: a [rows][r1] table
  if (mp.kind[g] != kOrig && mp.kind[g] != kSuffix) return false;
  const ModeDev& l = ch.m[mp.lo[g]];
  if (mp.kind[g] == kOrig && (l.layout != TNB_LAYOUT_DENSE || l.rr != 1)) return false;
  if (l.rl != r1) return false;
  if (r0 < 4 || r0 > 32 || (r0 & 3) || r1 < 4 || r1 > 32 || (r1 & 3)) return false;
  G->r0 = r0;
  G->r1 = r1;
  G->Kmid = K;
  // A first table too large for L2 is gathered one row range at a time: the
  // range index leads the sort key and the compute kernel's CTAs sweep the
  // sorted tiles together (interleaved), so at any time the gathers fall into
  // one range (<= 16 MB, L2-resident: every row is fetched from HBM once per
  // call instead of once per sample).  Limits: shared-memory histograms
  // (kGsSmemK buckets) and buckets of >= 512 samples on average.
  G->nsub = 1;
  G->sub_rows = 0;
  {
    const int64_t rowsP = mp.rows[0];
    const int64_t bytesP = rowsP * r0 * 4;
    const char* e = getenv("TNB_GS_SUBRANGES");
    const int want = e ? atoi(e) : 1;  // measured: no gain at cfg2 (the kernel is issue-bound, not DRAM-bound) and a slower 8192-bucket scatter
    int ns = 1;
    while (bytesP / ns > ((int64_t)16 << 20) && ns * 2 <= want && K * ns * 2 <= kGsSmemK && K * ns * 2 * 512 <= m) ns *= 2;
    if (ns > 1) {
      G->nsub = ns;
      G->sub_rows = (rowsP + ns - 1) / ns;
    }
  }
  // A result too large for L2 is written one window of samples at a time: the
  // compute kernel stores every value at its sample's position (4 scattered
  // bytes), which the memory system retires at ~16 G stores/s once the result
  // no longer fits in L2 (2^26 samples: 4.2 ms of stores alone).  With the
  // sample index's high bits leading the sort key, the CTAs (interleaved)
  // sweep one 2^23-sample window at a time and its 32 MB of results fill
  // whole lines in L2 before they are written back (cfg2 chain, 2^26 tuples:
  // 7.7 -> 6.2 ms; 2^25: 3.76 -> 2.90 ms, 3.22 with 2^22-sample windows and
  // their 8192 buckets).
  G->chunk_shift = 0;
  {
    const char* e = getenv("TNB_GS_CHUNK_LOG2");  // 0: off; n: 2^n-sample windows whatever the result size (tests)
    int sh = e ? atoi(e) : 23;
    if (G->nsub == 1 && sh > 0 && sh < 31 && (e || m * 4 > ((int64_t)64 << 20))) {
      auto nchunk = [&](int b) { return (m + ((int64_t)1 << b) - 1) >> b; };
      // windows of up to 64 MB when the bucket count would outgrow the shared-memory histograms
      while (!e && sh < 24 && K * nchunk(sh) > kGsSmemK) ++sh;
      const int64_t nc = nchunk(sh);
      if (nc > 1 && K * nc <= kGsSmemK && K * nc * 512 <= m) {
        G->chunk_shift = sh;
        G->nsub = (int)nc;  // the windows take the row ranges' place in the key
      }
    }
  }
  K *= G->nsub;
  G->K = K;
  // the bucketed kernels' slice copies are not needed here
  for (int v = 0; v < mp.ng; ++v) mp.lm[v] = mp.mma[v] = 0;
  int64_t off = mp.table_bytes;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += (bytes + 1023) & ~(int64_t)1023;
    return o;
  };
  int64_t rows = (int64_t)ch.m[G->omid_lo].J * r0;
  for (int o = G->omid_lo + 1; o < G->omid_hi; ++o) {
    rows *= ch.m[o].J;
    G->lvl_off[o] = take(rows * ch.m[o].rr * 4);
  }
  G->img_off = take(G->Kmid * kGsImgBytes);
  G->hist_off = take(K * 4 + 16);  // + 3 hot-row counters (gs_detect_hot_kernel)
  G->bstart_off = take((K + 1) * 4);
  G->tbase_off = take((K + 1) * 4);
  G->cursor_off = take(K * 4);
  G->tinfo_off = take(((m + kGsTile - 1) / kGsTile + K + 1) * 8);
  G->recu_off = take(m * 16);
  G->recs_off = take(m * 16);
  G->total_bytes = off;
  return true;
}

// ---------------------------------------------------------------------------
// slice images: M (levels layout [j_lo][a][j_rest][c]) -> per key the K-major
// SW128 image of M[key]^T (row n, 16-byte piece c at (c ^ (n & 7))), tf32 hi
// then lo, zero padded to 32 x 32
__global__ void gs_mid_image_kernel(const float* __restrict__ M, int64_t K, int64_t Jrest, int r0, int r1,
                                    unsigned char* __restrict__ img) {
  const int64_t total = K * 256;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t >> 8;
    const int n = (int)(t >> 3) & 31, c = (int)t & 7;
    const int64_t jlo = k / Jrest, jr = k - jlo * Jrest;
    float x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int a = 4 * c + i;
      x[i] = (n < r1 && a < r0) ? __ldg(M + ((jlo * r0 + a) * Jrest + jr) * r1 + n) : 0.f;
    }
    uint4 hi, lo;
    uint32_t h, l;
    split_tf32(x[0], h, l); hi.x = h; lo.x = l;
    split_tf32(x[1], h, l); hi.y = h; lo.y = l;
    split_tf32(x[2], h, l); hi.z = h; lo.z = l;
    split_tf32(x[3], h, l); hi.w = h; lo.w = l;
    unsigned char* dst = img + k * kGsImgBytes + n * kGsRow + ((c ^ (n & 7)) << 4);
    *reinterpret_cast<uint4*>(dst) = hi;
    *reinterpret_cast<uint4*>(dst + kGsImgBytes / 2) = lo;
  }
}

// one prefix-style level: out[(p*J + j)*rr + c] = sum_a in[p*rl + a] G(j, a, c)
int gs_prefix_level(const ModeDev& md, const float* in, int64_t rows, float* out, cudaStream_t st) {
  const int64_t total = rows * md.J * md.rr;
  if (total <= 0) return TNB_OK;
  if (launch_table_tc<false>(md, in, rows, out, st)) {
  } else if (table_gemm_ok(md, false)) {
    table_gemm<false><<<dim3((unsigned)ceil_div(rows, kTRows), (unsigned)ceil_div(md.J, kTZ)), 256, 0, st>>>(md, in, rows,
                                                                                                         out);
  } else {
    const int g = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8);
    table_prefix_step<<<g, 256, 0, st>>>(md, in, rows, out);
  }
  return check_launch("gsort mid level");
}

int gs_build_mid(const ChainDev& ch, const GPlan& G, unsigned char* base, cudaStream_t st) {
  KTimer kt("entries_mid", st);
  const ModeDev& m0 = ch.m[G.omid_lo];
  const float* in = m0.s;
  int64_t rows = (int64_t)m0.J * G.r0, jrest = 1;
  for (int o = G.omid_lo + 1; o < G.omid_hi; ++o) {
    float* out = reinterpret_cast<float*>(base + G.lvl_off[o]);
    int rc = gs_prefix_level(ch.m[o], in, rows, out, st);
    if (rc) return rc;
    in = out;
    rows *= ch.m[o].J;
    jrest *= ch.m[o].J;
  }
  // one image per slice of the merged mode (the kernel maps bucket -> bucket % Kmid)
  const int g = (int)std::min<int64_t>(ceil_div(G.Kmid * 256, 256), (int64_t)num_sms() * 8);
  gs_mid_image_kernel<<<g, 256, 0, st>>>(in, G.Kmid, jrest, G.r0, G.r1, base + G.img_off);
  return check_launch("gsort mid image");
}

// ---------------------------------------------------------------------------
// prep: thread = sample row; record {key, first row, last row, diag row}.
// STAGE: each warp copies the 32 rows of its pass into shared memory with
// coalesced 16-byte loads (all in flight at once) and every lane then reads
// its own row back (row stride 8 N0 bytes: conflict-free for N0 = 8, 10);
// otherwise each thread loads its row straight from global memory.
constexpr int kGsStageN0 = 16;  // rows of up to 16 indices are staged
template <bool SH, bool STAGE>
__global__ void __launch_bounds__(kGsPrepThreads) gs_prep_kernel(const __grid_constant__ GsPrep gp,
                                                                 const int64_t* __restrict__ idx, int64_t m,
                                                                 int32_t* __restrict__ err, uint4* __restrict__ recu,
                                                                 uint32_t* __restrict__ hist) {
  extern __shared__ __align__(16) uint32_t gs_sh[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, N0 = gp.n0;
  const uint32_t K = gp.K;
  if (SH) {
    for (uint32_t j = tid; j < K; j += kGsPrepThreads) gs_sh[j] = 0;
    __syncthreads();
  }
  uint32_t f0, f1, f2, f3;
  int badm;
  // wrap and check one index on 32-bit halves: valid raw values have a high
  // word of 0 (then lo < J) or -1 (then lo + J wraps below J); core.py:409-416
  auto put = [&](int o, int64_t raw) {
    const uint32_t J = (uint32_t)gp.oJ[o];
    const uint32_t lo = (uint32_t)raw;
    const int32_t hi = (int32_t)(raw >> 32);
    uint32_t v = lo + ((uint32_t)hi & J);
    const bool bad = v >= J || (uint32_t)(hi + 1) > 1u;
    badm = (bad && o < badm) ? o : badm;
    v = bad ? 0u : v;
    f0 += v * gp.w0[o];
    f1 += v * gp.w1[o];
    f2 += v * gp.w2[o];
    f3 += v * gp.w3[o];
  };
  auto emit = [&](int64_t s) {
    if (badm < N0) atomicMin(err, badm);
    if (gp.sub_rows) f1 += (f0 / gp.sub_rows) * gp.Kmid;
    if (gp.chunk_shift) f1 += (uint32_t)(s >> gp.chunk_shift) * gp.Kmid;
    recu[s] = make_uint4(f1, f0, f3, f2);
    if (SH) {
      atomicAdd(&gs_sh[f1], 1u);
    } else {  // many buckets: one global atomic per distinct key of the warp
      const unsigned mk = __match_any_sync(__activemask(), f1);
      if (lane == __ffs(mk) - 1) atomicAdd(&hist[f1], (uint32_t)__popc(mk));
    }
  };
  if (STAGE) {
    const int h = N0 >> 1;  // 16-byte pieces per row
    uint4* stage = reinterpret_cast<uint4*>(gs_sh + (SH ? ((K + 3) & ~3u) : 0)) + (size_t)warp * 32 * h;
    constexpr int W = kGsPrepThreads / 32;
    for (int64_t base = ((int64_t)blockIdx.x * W + warp) * 32; base < m; base += (int64_t)gridDim.x * W * 32) {
      const int rows = (int)min((int64_t)32, m - base);
      const int np = rows * h;
      const uint4* src = reinterpret_cast<const uint4*>(idx + base * N0);
      uint4 buf[kGsStageN0 / 2];
#pragma unroll
      for (int i = 0; i < kGsStageN0 / 2; ++i)
        if (i < h && lane + 32 * i < np) buf[i] = __ldcs(src + lane + 32 * i);
#pragma unroll
      for (int i = 0; i < kGsStageN0 / 2; ++i)
        if (i < h && lane + 32 * i < np) {
          const int pi = lane + 32 * i;  // rows of 4 pieces (64 B) are XOR-swizzled against bank conflicts
          stage[h == 4 ? (pi ^ ((pi >> 3) & 3)) : pi] = buf[i];
        }
      __syncwarp();
      if (lane < rows) {
        f0 = f1 = f2 = f3 = 0;
        badm = N0;
        const longlong2* row = reinterpret_cast<const longlong2*>(stage + lane * h);
        for (int o = 0; o < h; ++o) {
          const longlong2 w = row[h == 4 ? (o ^ ((lane >> 1) & 3)) : o];
          put(2 * o, w.x);
          put(2 * o + 1, w.y);
        }
        emit(base + lane);
      }
      __syncwarp();
    }
  } else {
    for (int64_t s = blockIdx.x * (int64_t)kGsPrepThreads + tid; s < m; s += (int64_t)gridDim.x * kGsPrepThreads) {
      const int64_t* row = idx + s * N0;
      f0 = f1 = f2 = f3 = 0;
      badm = N0;
      for (int o = 0; o < N0; ++o) put(o, __ldg(row + o));
      emit(s);
    }
  }
  if (SH) {
    __syncthreads();
    for (uint32_t j = tid; j < K; j += kGsPrepThreads) {
      const uint32_t c = gs_sh[j];
      if (c) atomicAdd(&hist[j], c);
    }
  }
}

// scan (one CTA): bucket starts, tile starts, scatter cursors
__global__ void __launch_bounds__(1024) gs_scan_kernel(const uint32_t* __restrict__ hist, uint32_t K,
                                                       uint32_t* __restrict__ bstart, uint32_t* __restrict__ tbase,
                                                       uint32_t* __restrict__ cursor) {
  __shared__ uint32_t wc[32], wt[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (K + 1023) / 1024;
  const uint32_t j0 = min(K, tid * per), j1 = min(K, j0 + per);
  uint32_t c = 0, t = 0;
  for (uint32_t j = j0; j < j1; ++j) {
    const uint32_t h = hist[j];
    c += h;
    t += (h + kGsTile - 1) / kGsTile;
  }
  uint32_t ic = c, it = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yc = __shfl_up_sync(0xffffffffu, ic, o), yt = __shfl_up_sync(0xffffffffu, it, o);
    if (lane >= o) {
      ic += yc;
      it += yt;
    }
  }
  if (lane == 31) {
    wc[warp] = ic;
    wt[warp] = it;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t xc = wc[lane], xt = wt[lane];
    uint32_t sc = xc, stt = xt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yc = __shfl_up_sync(0xffffffffu, sc, o), yt = __shfl_up_sync(0xffffffffu, stt, o);
      if (lane >= o) {
        sc += yc;
        stt += yt;
      }
    }
    wc[lane] = sc - xc;
    wt[lane] = stt - xt;
    if (lane == 31) {
      bstart[K] = sc;
      tbase[K] = stt;
    }
  }
  __syncthreads();
  uint32_t rc = wc[warp] + ic - c, rt = wt[warp] + it - t;
  for (uint32_t j = j0; j < j1; ++j) {
    const uint32_t h = hist[j];
    bstart[j] = rc;
    cursor[j] = rc;
    tbase[j] = rt;
    rc += h;
    rt += (h + kGsTile - 1) / kGsTile;
  }
}

// tile map: for every 128-sample tile of the sorted order its first position,
// its bucket and its number of rows (the last tile of a bucket is ragged) --
// one 8-byte load per tile and role in the compute kernel
__global__ void __launch_bounds__(256) gs_tilemap_kernel(const uint32_t* __restrict__ bstart,
                                                        const uint32_t* __restrict__ tbase, uint32_t K,
                                                        uint2* __restrict__ tinfo) {
  const uint32_t Nt = __ldg(tbase + K);
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < Nt; t += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = K - 1;  // first b with tbase[b + 1] > t
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(tbase + mid + 1) > t) hi = mid;
      else lo = mid + 1;
    }
    const uint32_t p0 = __ldg(bstart + lo) + (t - __ldg(tbase + lo)) * kGsTile;
    const uint32_t left = __ldg(bstart + lo + 1) - p0;
    tinfo[t] = make_uint2(p0, (lo << 8) | ((left < (uint32_t)kGsTile ? left : (uint32_t)kGsTile) - 1));
  }
}

// scatter: each CTA takes 4096 records, counts its keys in shared memory
// (the count a sample draws is its rank inside the CTA's share of the bucket),
// reserves the CTA's range of every bucket with one atomicAdd, sorts the
// records by key in shared memory and writes {orig, first row, last row, diag
// row} runs to the sorted positions (a bucket's share is contiguous)
__global__ void __launch_bounds__(kGsScatThreads, 2) gs_scatter_kernel(const uint4* __restrict__ recu, int64_t m, uint32_t K,
                                                                     uint32_t* __restrict__ cursor,
                                                                     uint4* __restrict__ recs) {
  extern __shared__ __align__(16) uint32_t gs_sh[];
  constexpr int TS = kGsScatThreads * kGsScatPer;
  uint4* stg = reinterpret_cast<uint4*>(gs_sh);               // [TS] records in key order
  uint16_t* skey = reinterpret_cast<uint16_t*>(stg + TS);     // [TS] their keys
  uint32_t* cnt = reinterpret_cast<uint32_t*>(skey + TS);     // [K] counts, then local starts
  uint32_t* bas = cnt + K;                                    // [K] global start of the CTA's share
  __shared__ uint32_t wsum[kGsScatThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (K + kGsScatThreads - 1) / kGsScatThreads;
  for (int64_t tile = blockIdx.x; tile * TS < m; tile += gridDim.x) {
    const int n = (int)min((int64_t)TS, m - tile * TS);
    for (uint32_t j = tid; j < K; j += kGsScatThreads) cnt[j] = 0;
    __syncthreads();
    uint4 r[kGsScatPer];
    uint32_t rk[kGsScatPer];
#pragma unroll
    for (int i = 0; i < kGsScatPer; ++i) {
      const int l = i * kGsScatThreads + tid;
      if (l < n) r[i] = __ldcs(recu + tile * TS + l);
    }
#pragma unroll
    for (int i = 0; i < kGsScatPer; ++i) {
      const int l = i * kGsScatThreads + tid;
      if (l < n) rk[i] = atomicAdd(&cnt[r[i].x], 1u);
    }
    __syncthreads();
    // reserve, and turn the counts into local starts (block exclusive scan)
    const uint32_t j0 = min(K, tid * per), j1 = min(K, j0 + per);
    uint32_t sum = 0;
    for (uint32_t j = j0; j < j1; ++j) {
      const uint32_t c = cnt[j];
      if (c) bas[j] = atomicAdd(&cursor[j], c);
      sum += c;
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = lane < kGsScatThreads / 32 ? wsum[lane] : 0;
      uint32_t sc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, sc, o);
        if (lane >= o) sc += y;
      }
      if (lane < kGsScatThreads / 32) wsum[lane] = sc - x;
    }
    __syncthreads();
    uint32_t run = wsum[warp] + inc - sum;
    for (uint32_t j = j0; j < j1; ++j) {
      const uint32_t c = cnt[j];
      cnt[j] = run;
      run += c;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kGsScatPer; ++i) {
      const int l = i * kGsScatThreads + tid;
      if (l < n) {
        const uint32_t slot = cnt[r[i].x] + rk[i];
        stg[slot] = make_uint4((uint32_t)(tile * TS + l), r[i].y, r[i].z, r[i].w);
        skey[slot] = (uint16_t)r[i].x;
      }
    }
    __syncthreads();
    for (int l = tid; l < n; l += kGsScatThreads) {
      const uint32_t k = skey[l];
      recs[bas[k] + ((uint32_t)l - cnt[k])] = stg[l];
    }
    __syncthreads();
  }
}

// scatter with many buckets: thread = record, the warp's records of one key
// reserve their slots with one global atomicAdd
__global__ void __launch_bounds__(256) gs_scatter_big_kernel(const uint4* __restrict__ recu, int64_t m,
                                                             uint32_t* __restrict__ cursor, uint4* __restrict__ recs) {
  const int lane = threadIdx.x & 31;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = __ldcs(recu + s);
    const unsigned mk = __match_any_sync(__activemask(), r.x);
    const int leader = __ffs(mk) - 1;
    uint32_t b = 0;
    if (lane == leader) b = atomicAdd(&cursor[r.x], (uint32_t)__popc(mk));
    b = __shfl_sync(mk, b, leader);
    recs[b + __popc(mk & ((1u << lane) - 1u))] = make_uint4((uint32_t)s, r.y, r.z, r.w);
  }
}

// Repeated table rows (slice queries: every sample shares its leading or
// trailing indices): all SMs would gather ONE L2 line, and 2^24 copies of it
// serialise on its slice (cfg2 compute 0.84 -> 3.7 ms).  Each of kGsHotBlocks
// warps looks at 32 consecutive records: a majority equal to the first one,
// per table, counts a vote; the compute kernel copies a table's rows through
// L1 (cp.async.ca) when most warps voted.
constexpr int kGsHotBlocks = 64;
__global__ void gs_detect_hot_kernel(const uint4* __restrict__ recu, int64_t m, uint32_t* __restrict__ hot) {
  const int lane = threadIdx.x & 31;
  const int64_t base = (m / kGsHotBlocks) * blockIdx.x;
  const int64_t s = base + lane;
  uint4 r = make_uint4(0, 0, 0, 0);
  const bool ok = s < m;
  if (ok) r = __ldg(recu + s);
  const uint32_t y0 = __shfl_sync(0xffffffffu, r.y, 0), z0 = __shfl_sync(0xffffffffu, r.z, 0),
                 w0 = __shfl_sync(0xffffffffu, r.w, 0);
  const int n = __popc(__ballot_sync(0xffffffffu, ok));
  const int ny = __popc(__ballot_sync(0xffffffffu, ok && r.y == y0));
  const int nz = __popc(__ballot_sync(0xffffffffu, ok && r.z == z0));
  const int nw = __popc(__ballot_sync(0xffffffffu, ok && r.w == w0));
  if (lane == 0 && n >= 8) {
    if (2 * ny > n) atomicAdd(hot + 0, 1u);
    if (2 * nz > n) atomicAdd(hot + 1, 1u);
    if (2 * nw > n) atomicAdd(hot + 2, 1u);
  }
}

// ---------------------------------------------------------------------------
// compute kernel
struct GsArgs {
  const float* P;             // [rows][r0]
  const float* S;             // [rows][r1]
  const float* D;             // [rows][r1] or null
  const unsigned char* img;   // [K][8 KB]
  const uint4* recs;          // sorted records
  const uint2* tinfo;         // [tiles] {first sorted position, bucket << 8 | rows - 1}
  const uint32_t* tbase;      // [K + 1] (tbase[K] = number of tiles)
  uint32_t K, Kmid, m;
  int32_t interleave;         // CTAs take runs of kGsRun tiles round-robin instead of one contiguous range
  int32_t r0, r1;
  int32_t pfP, pfS, pfD;      // tables too large for L2: their rows are streamed (evict_first)
  int32_t keep_out;           // the result fits in L2: keep its lines there (evict_last)
  const uint32_t* hot;        // [3] gs_detect_hot_kernel votes: first / last / diag rows repeat
  float* out;
#ifdef TNB_GS_TRACE
  unsigned long long* trace;  // [block][4 roles][6 phases] clock64 cycles
#endif
};

// try_wait with a suspend-time hint: the waiting warp sleeps in hardware
// until the phase completes instead of re-issuing the poll every ~20 cycles
// (16 polling warps otherwise take most of the SM's issue slots from the few
// working ones: the roles ran 2-3x slower)
__device__ __forceinline__ void gs_wait(uint64_t* b, uint32_t parity) {
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
    if (++spins > 30000) __trap();  // ~30 s without progress: a protocol bug, not a slow tile
  }
}
// producers waiting for a free stage are not on the critical path: they
// sleep between polls instead of taking issue slots from the working warps
__device__ __forceinline__ void gs_wait_relaxed(uint64_t* b, uint32_t parity) {
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
    __nanosleep(128);
    if (++spins > 100000000) __trap();
  }
}
__device__ __forceinline__ void gs_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void gs_cp_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void gs_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void gs_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// rows of a table too large for L2 are streamed (evict_first): they would
// otherwise push out the result lines, whose scattered 4-byte writes only
// merge into whole sectors while they stay in L2
__device__ __forceinline__ void gs_cp16_stream(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void gs_cp16_l1(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// mode 0: through L2 only; 1: streamed (evict_first); 2: through L1 (repeated rows)
__device__ __forceinline__ void gs_cp16_mode(uint32_t dst, const void* src, int mode, uint64_t pol) {
  if (mode == 2) gs_cp16_l1(dst, src);
  else if (mode == 1) gs_cp16_stream(dst, src, pol);
  else gs_cp16(dst, src);
}
__device__ __forceinline__ uint64_t gs_desc(uint32_t saddr) {  // K-major SWIZZLE_128B, SBO 1024
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// issued by the whole (converged) warp: one elected lane executes the MMA
__device__ __forceinline__ void gs_mma(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void gs_commit_elect(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "elect.sync _|q, 0xffffffff;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(s32(b))
      : "memory");
}

// TNB_GS_TRACE builds: every role's lane 0 accumulates the clock64 cycles it
// spends in each phase of its loop and writes the sums at the end
// (trace[block][role][phase]); tools/gs_trace.py prints the averages
#ifdef TNB_GS_TRACE
#define GS_TRACE_INIT() \
  long long gs_acc_[6] = {0, 0, 0, 0, 0, 0}; \
  long long gs_last_ = clock64()
#define GS_TRACE(role, it, ev)              \
  do {                                      \
    const long long now_ = clock64();       \
    gs_acc_[ev] += now_ - gs_last_;         \
    gs_last_ = now_;                        \
  } while (0)
#define GS_STAMP(it, ev)                                                                 \
  do {                                                                                   \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (it) >= 256 && (it) < 288)         \
      ga.trace[8192 + ((it) - 256) * 16 + (ev)] = (unsigned long long)clock64();         \
  } while (0)
#define GS_TRACE_END(role)                                                               \
  do {                                                                                   \
    if ((threadIdx.x & 31) == 0)                                                         \
      for (int e_ = 0; e_ < 6; ++e_) ga.trace[(blockIdx.x * 4 + (role)) * 6 + e_] = (unsigned long long)gs_acc_[e_]; \
  } while (0)
#else
#define GS_TRACE_INIT() \
  do {                  \
  } while (0)
#define GS_TRACE(role, it, ev) \
  do {                         \
  } while (0)
#define GS_TRACE_END(role) \
  do {                     \
  } while (0)
#define GS_STAMP(it, ev) \
  do {                   \
  } while (0)
#endif

// The CTA's tile sequence.  Contiguous: tiles [Nt b / G, Nt (b + 1) / G).
// Interleaved (row ranges in the sort key): runs of kGsRun consecutive tiles
// dealt round-robin, so all CTAs work in the same part of the sorted order.
constexpr uint32_t kGsRun = 4;
struct GsSeq {
  uint32_t first, cnt, G, inter;
  __device__ void init(uint32_t Nt, uint32_t bid, uint32_t grid, int interleave) {
    G = grid;
    inter = (uint32_t)interleave;
    if (!inter) {
      first = (uint32_t)(((uint64_t)Nt * bid) / grid);
      cnt = (uint32_t)(((uint64_t)Nt * (bid + 1)) / grid) - first;
    } else {
      first = bid;
      const uint32_t NR = (Nt + kGsRun - 1) / kGsRun;  // runs
      const uint32_t nr = bid < NR ? (NR - bid + grid - 1) / grid : 0;
      cnt = nr * kGsRun;
      if (nr && (NR - 1) % grid == bid) cnt -= NR * kGsRun - Nt;  // the last run is short
    }
  }
  __device__ __forceinline__ uint32_t tile(uint32_t i) const {
    return inter ? ((i / kGsRun) * G + first) * kGsRun + (i % kGsRun) : first + i;
  }
};

// CSB: bytes between the closing rows (last / diag tables) of a stage: 128
// (pieces XOR-swizzled like the operand tile) or 96 (compact rows of up to 24
// floats: a fourth stage fits next to a diagonal table)
template <bool DIAG, int CSB>
struct GsSmem {
  static constexpr int kClose = kGsTile * CSB;                               // one closing table's rows
  static constexpr int kOrigOff = kGsTileBytes + (DIAG ? 2 : 1) * kClose;    // A | S | (D) | orig[128]
  static constexpr int kStage = (kOrigOff + 512 + 1023) & ~1023;
  static constexpr int NS = DIAG ? (CSB == 96 ? 4 : 3) : 5;                  // gather stages
  static constexpr int kAlo = NS * kStage;                                   // 2 x 16 KB
  static constexpr int kB = kAlo + 2 * kGsTileBytes;                         // kGsNB x 8 KB
  static constexpr int RR = 4;                                               // record ring depth (tiles)
  static constexpr int kRec = kB + kGsNB * kGsImgBytes;                      // kGsPW warps x RR x kGsRW records x 16 B
  static constexpr int kBars = kRec + kGsPW * RR * kGsRW * 16;
  static constexpr int kNBars = 3 * NS + 2 + 2 * kGsNA + 2 * kGsNB;
  static constexpr int kBytes = kBars + kNBars * 8 + 16;
  static_assert(kBytes + 1024 <= 232448, "shared memory");
};

template <bool DIAG, int CSB>
__global__ void __launch_bounds__(kGsThreads, 1) entries_gsort_kernel(const __grid_constant__ GsArgs ga) {
  using L = GsSmem<DIAG, CSB>;
  constexpr int NS = L::NS;
  extern __shared__ __align__(1024) unsigned char gs_raw[];
  unsigned char* smem = gs_raw + ((1024 - (s32(gs_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBars);
  uint64_t* full_raw = bars;                  // [NS] every producer thread: one cp.async arrival + one plain (orig stores)
  uint64_t* a_ready = bars + NS;              // [NS] 128 splitter threads
  uint64_t* empty = bars + 2 * NS;            // [NS] 128 epilogue threads
  uint64_t* alo_empty = bars + 3 * NS;        // [2] tcgen05.commit
  uint64_t* acc_full = alo_empty + 2;         // [NA] tcgen05.commit
  uint64_t* acc_empty = acc_full + kGsNA;     // [NA] 128 epilogue threads
  uint64_t* b_full = acc_empty + kGsNA;       // [NB] tx
  uint64_t* b_empty = b_full + kGsNB;         // [NB] tcgen05.commit
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_empty + kGsNB);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  GsSeq seq;
  seq.init(__ldg(ga.tbase + ga.K), blockIdx.x, gridDim.x, ga.interleave);
  const uint32_t ntile = seq.cnt;
  const int r0 = ga.r0, r1 = ga.r1;

  // operand pad columns (r0 up to a multiple of 8 floats) must read as zero
  for (int i = tid; i < L::kB / 16; i += kGsThreads) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mb_init(&full_raw[s], 2 * 32 * kGsPW);
      mb_init(&a_ready[s], 128);
      mb_init(&empty[s], 128);
    }
    mb_init(&alo_empty[0], 1);
    mb_init(&alo_empty[1], 1);
    for (int a = 0; a < kGsNA; ++a) {
      mb_init(&acc_full[a], 1);
      mb_init(&acc_empty[a], 128);
    }
    for (int b = 0; b < kGsNB; ++b) {
      mb_init(&b_full[b], 1);
      mb_init(&b_empty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "r"((uint32_t)(kGsNA * 64)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = s32(smem);

  if (ntile > 0) {
    if (warp == 0) {
      // ================= MMA issuer =================
      const uint32_t idesc32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) |
                               ((uint32_t)(kGsTile >> 4) << 24);
      const uint32_t idesc64 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) |
                               ((uint32_t)(kGsTile >> 4) << 24);
      const int nk = (r0 + 7) >> 3;
      uint32_t nb = 0, slot = 0, prev_b = 0xffffffffu;  // bucket changes so far: the slice-image ring position
      uint32_t nxt = __ldg(&ga.tinfo[seq.tile(0)].y);
      GS_TRACE_INIT();
      for (uint32_t it = 0; it < ntile; ++it) {
        const uint32_t b = nxt >> 8;
        if (it + 1 < ntile) nxt = __ldg(&ga.tinfo[seq.tile(it + 1)].y);
        if (b != prev_b) {
          if (prev_b != 0xffffffffu) {
            gs_commit_elect(&b_empty[slot]);  // the previous bucket's MMAs are all issued
            ++nb;
          }
          prev_b = b;
          slot = nb % kGsNB;
          gs_wait(&b_full[slot], (nb / kGsNB) & 1);
        }
        const uint32_t s = it % NS, a = it % kGsNA;
        gs_wait(&a_ready[s], (it / NS) & 1);
        GS_TRACE(0, it, 0);
        GS_STAMP(it, 6);
        gs_wait(&acc_empty[a], ((it / kGsNA) & 1) ^ 1);
        GS_TRACE(0, it, 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        {
          // K-major SWIZZLE_128B descriptors: constant bits | (address >> 4); a
          // k-step advances 32 bytes inside the 128-byte swizzle row.  Per
          // k-step: Ahi x [Bhi | Blo] (N = 64: the image's hi and lo rows are
          // contiguous) and Alo x Bhi (N = 32) -- the epilogue adds the halves
          const uint64_t dc = ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
          const uint32_t ah = (sbase + s * L::kStage) >> 4, al = (sbase + L::kAlo + (it & 1) * kGsTileBytes) >> 4;
          const uint32_t bh = (sbase + L::kB + slot * kGsImgBytes) >> 4;
          const uint32_t d = tmem + a * 64;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (kk < nk) {
              const uint64_t dah = dc | (uint64_t)(ah + 2 * kk), dal = dc | (uint64_t)(al + 2 * kk);
              const uint64_t dbh = dc | (uint64_t)(bh + 2 * kk);
              gs_mma(d, dah, dbh, idesc64, kk > 0);
              gs_mma(d, dal, dbh, idesc32, 1);
            }
          }
          gs_commit_elect(&acc_full[a]);
          gs_commit_elect(&alo_empty[it & 1]);
        }
        GS_TRACE(0, it, 2);
        GS_STAMP(it, 7);
        __syncwarp();
      }
      GS_TRACE_END(0);
    } else if (warp == 1) {
      // ================= slice images -> ring =================
      if (lane == 0) {
        uint32_t nb = 0, prev_b = 0xffffffffu;
        uint32_t nxt = __ldg(&ga.tinfo[seq.tile(0)].y);
        for (uint32_t it = 0; it < ntile; ++it) {
          const uint32_t b = nxt >> 8;
          if (it + 1 < ntile) nxt = __ldg(&ga.tinfo[seq.tile(it + 1)].y);
          if (b != prev_b) {
            if (prev_b != 0xffffffffu) ++nb;
            prev_b = b;
            const uint32_t slot = nb % kGsNB;
            gs_wait(&b_empty[slot], ((nb / kGsNB) & 1) ^ 1);
            mb_expect(&b_full[slot], kGsImgBytes);
            bulk(smem + L::kB + slot * kGsImgBytes, ga.img + (size_t)(b % ga.Kmid) * kGsImgBytes, kGsImgBytes,
                 &b_full[slot]);
          }
        }
      }
    } else if (warp >= 4 && warp < 8) {
      // ================= epilogue: thread = sample row =================
      const int q = warp & 3, row = q * 32 + lane;
      const uint32_t swz = (uint32_t)(row & 7);
      const int n4 = r1 >> 2;
      uint32_t it = 0;
      // the results land at random positions: their lines are kept in L2
      // (evict_last) when the whole result fits, so the 4-byte writes merge
      uint64_t keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      GS_TRACE_INIT();
      for (; it < ntile; ++it) {
        const uint32_t s = it % NS, a = it % kGsNA;
        gs_wait(&full_raw[s], (it / NS) & 1);
        GS_TRACE(1, it, 0);
        const uint32_t st = sbase + s * L::kStage;
        uint32_t orig;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(orig) : "r"(st + (uint32_t)L::kOrigOff + 4u * (uint32_t)row) : "memory");
        const uint32_t srow = st + kGsTileBytes + (uint32_t)row * CSB;
        gs_wait(&acc_full[a], (it / kGsNA) & 1);
        GS_TRACE(1, it, 1);
        if (q == 0) GS_STAMP(it, 8);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // D = (A Bhi + Alo Bhi)[0:32] + (A Blo)[32:64]: 16 columns of each half at a time
        const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + a * 64;
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (4 * h < n4) {
            uint32_t vh[16], vl[16];
            TMEM_LD16_GS(tacc + 16 * h, vh);
            TMEM_LD16_GS(tacc + 32 + 16 * h, vl);
            float wv[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (4 * h + c < n4) {
                const uint32_t off = (CSB == 128 ? ((uint32_t)(4 * h + c) ^ swz) : (uint32_t)(4 * h + c)) << 4;
                float4 x = lds128(srow + off);
                if (DIAG) {
                  const float4 y = lds128(srow + L::kClose + off);
                  x.x *= y.x;
                  x.y *= y.y;
                  x.z *= y.z;
                  x.w *= y.w;
                }
                wv[4 * c] = x.x;
                wv[4 * c + 1] = x.y;
                wv[4 * c + 2] = x.z;
                wv[4 * c + 3] = x.w;
              }
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
              if (16 * h + c < r1) {
                acc0 = fmaf(__uint_as_float(vh[c]) + __uint_as_float(vl[c]), wv[c], acc0);
                acc1 = fmaf(__uint_as_float(vh[c + 1]) + __uint_as_float(vl[c + 1]), wv[c + 1], acc1);
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        gs_arrive(&acc_empty[a]);
        if (orig != 0xffffffffu) {
          if (ga.keep_out)
            asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ga.out + orig), "f"(acc0 + acc1), "l"(keep) : "memory");
          else
            ga.out[orig] = acc0 + acc1;
        }
        gs_arrive(&empty[s]);
        GS_TRACE(1, it, 2);
        if (q == 0) GS_STAMP(it, 9);
      }
      if (q == 0) GS_TRACE_END(1);
    } else if (warp >= 12) {
      // ================= producers: gathers (kGsPW warps x 8 rows of every tile) =================
      // lanes 8g..8g+7 copy the 16-byte pieces of one row (one 128-byte line
      // per lane group and table); the warp's 8 rows take 2 passes.
      const int pw = warp - 12;
      const int c = lane & 7, rsub = lane >> 3;
      const bool okA = c < (r0 >> 2), okS = c < (r1 >> 2);
      const unsigned char* Pc = reinterpret_cast<const unsigned char*>(ga.P) + 16 * c;
      const unsigned char* Sc = reinterpret_cast<const unsigned char*>(ga.S) + 16 * c;
      const unsigned char* Dc = reinterpret_cast<const unsigned char*>(ga.D) + 16 * c;
      const uint32_t rbA = (uint32_t)r0 * 4, rbS = (uint32_t)r1 * 4;
      uint32_t offA[kGsPasses], offS[kGsPasses];
#pragma unroll
      for (int i = 0; i < kGsPasses; ++i) {
        const uint32_t r = (uint32_t)(pw * kGsRW + 4 * i + rsub);
        offA[i] = r * kGsRow + (((uint32_t)c ^ (r & 7)) << 4);
        offS[i] = kGsTileBytes + r * CSB + ((CSB == 128 ? ((uint32_t)c ^ (r & 7)) : (uint32_t)c) << 4);
      }
      uint64_t stream_pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream_pol));
      const int modeP = 2 * __ldg(ga.hot + 0) > kGsHotBlocks ? 2 : (ga.pfP && !ga.interleave ? 1 : 0);
      const int modeS = 2 * __ldg(ga.hot + 1) > kGsHotBlocks ? 2 : (ga.pfS ? 1 : 0);
      const int modeD = DIAG && 2 * __ldg(ga.hot + 2) > kGsHotBlocks ? 2 : (ga.pfD ? 1 : 0);
      uint64_t normal_pol;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(normal_pol));
      const bool anyhot = modeP == 2 || modeS == 2 || modeD == 2;
      const uint64_t polP = modeP == 1 ? stream_pol : normal_pol, polS = modeS == 1 ? stream_pol : normal_pol,
                     polD = modeD == 1 ? stream_pol : normal_pol;
      const int row = pw * kGsRW + (lane % kGsRW);  // lanes 0 .. kGsRW-1 hold the warp's records
      // record ring in shared memory (per warp: RR tiles x 8 records), filled
      // with cp.async RR tiles ahead: one commit group per tile, so
      // wait_group RR-1 at the top of a tile means its record has landed
      // (register prefetches of several tiles share a scoreboard: waiting for
      // the oldest load also waited for the newest).  The tile map entry of
      // the tile after the one being requested is loaded one step ahead.
      constexpr int RR = L::RR;
      const uint32_t ring = sbase + L::kRec + (uint32_t)pw * (RR * kGsRW * 16) + (uint32_t)(lane % kGsRW) * 16;
      uint2 tnext = __ldg(ga.tinfo + seq.tile(0));
      uint32_t jreq = 0;  // next tile (sequence index) whose records are requested
      auto issue_rec = [&](uint32_t slot) {
        const uint2 ti = tnext;
        ++jreq;
        if (jreq < ntile) tnext = __ldg(ga.tinfo + seq.tile(jreq));
        if (lane < kGsRW) {
          const uint32_t dst = ring + slot * (kGsRW * 16);
          if (row <= (int)(ti.y & 0xff)) {
            gs_cp16_stream(dst, ga.recs + ti.x + row, stream_pol);
          } else {
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %2, %2};" ::"r"(dst), "r"(0xffffffffu), "r"(0u) : "memory");
          }
        }
      };
#pragma unroll 1
      for (int j = 0; j < RR; ++j) {
        if ((uint32_t)j < ntile) issue_rec((uint32_t)j);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      GS_TRACE_INIT();
      for (uint32_t it = 0; it < ntile; ++it) {
        asm volatile("cp.async.wait_group %0;" ::"n"(RR - 1) : "memory");
        const uint32_t slot = it % RR;
        uint4 rec = make_uint4(0xffffffffu, 0, 0, 0);
        if (lane < kGsRW) {
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(rec.x), "=r"(rec.y), "=r"(rec.z), "=r"(rec.w)
                       : "r"(ring + slot * (kGsRW * 16))
                       : "memory");
        }
        GS_TRACE(2, it, 5);
        if (pw == 0) GS_STAMP(it, 0);
        if (jreq < ntile) issue_rec(slot);
        GS_TRACE(2, it, 3);
        const uint32_t s = it % NS;
        gs_wait_relaxed(&empty[s], ((it / NS) & 1) ^ 1);
        GS_TRACE(2, it, 1);
        if (pw == 0) GS_STAMP(it, 1);
        const uint32_t sa = sbase + s * L::kStage;
        if (lane < kGsRW) {
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(sa + (uint32_t)L::kOrigOff + 4u * (uint32_t)row), "r"(rec.x)
                       : "memory");
        }
        if (!anyhot) {  // the usual case: one copy instruction per piece, the L2 policy in a register
#pragma unroll
          for (int i = 0; i < kGsPasses; ++i) {
            const int src = 4 * i + rsub;
            const uint32_t og = __shfl_sync(0xffffffffu, rec.x, src);
            const uint32_t pr = __shfl_sync(0xffffffffu, rec.y, src);
            const uint32_t sr = __shfl_sync(0xffffffffu, rec.z, src);
            uint32_t dr = 0;
            if (DIAG) dr = __shfl_sync(0xffffffffu, rec.w, src);
            if (og != 0xffffffffu) {
              if (okA) gs_cp16_stream(sa + offA[i], Pc + (uint64_t)pr * rbA, polP);
              if (okS) {
                gs_cp16_stream(sa + offS[i], Sc + (uint64_t)sr * rbS, polS);
                if (DIAG) gs_cp16_stream(sa + offS[i] + L::kClose, Dc + (uint64_t)dr * rbS, polD);
              }
            }
          }
        } else {  // some table's rows repeat: those go through L1
#pragma unroll
          for (int i = 0; i < kGsPasses; ++i) {
            const int src = 4 * i + rsub;
            const uint32_t og = __shfl_sync(0xffffffffu, rec.x, src);
            const uint32_t pr = __shfl_sync(0xffffffffu, rec.y, src);
            const uint32_t sr = __shfl_sync(0xffffffffu, rec.z, src);
            uint32_t dr = 0;
            if (DIAG) dr = __shfl_sync(0xffffffffu, rec.w, src);
            if (og != 0xffffffffu) {
              if (okA) gs_cp16_mode(sa + offA[i], Pc + (uint64_t)pr * rbA, modeP, stream_pol);
              if (okS) {
                gs_cp16_mode(sa + offS[i], Sc + (uint64_t)sr * rbS, modeS, stream_pol);
                if (DIAG) gs_cp16_mode(sa + offS[i] + L::kClose, Dc + (uint64_t)dr * rbS, modeD, stream_pol);
              }
            }
          }
        }
        gs_cp_arrive(&full_raw[s]);
        gs_arrive(&full_raw[s]);
        asm volatile("cp.async.commit_group;" ::: "memory");
        GS_TRACE(2, it, 2);
        if (pw == 0) GS_STAMP(it, 2);
      }
      if (pw == 0) GS_TRACE_END(2);
    } else if (warp >= 8 && warp < 12) {
      // ================= splitters: x -> tf32 hi (in place), lo =================
      const int row = (warp - 8) * 32 + lane;
      const uint32_t swz = (uint32_t)(row & 7);
      const int nph = ((r0 + 7) >> 3) * 2;  // pieces (r0 padded to 8 floats)
      const int c0 = 0;
      const uint32_t rowoff = (uint32_t)row * kGsRow;
      uint32_t it = 0;
      GS_TRACE_INIT();
      for (; it < ntile; ++it) {
        const uint32_t s = it % NS;
        gs_wait(&full_raw[s], (it / NS) & 1);
        GS_TRACE(3, it, 0);
        if (warp == 8) GS_STAMP(it, 3);
        gs_wait(&alo_empty[it & 1], ((it >> 1) & 1) ^ 1);
        GS_TRACE(3, it, 1);
        const uint32_t A = sbase + s * L::kStage + rowoff;
        const uint32_t Alo = sbase + L::kAlo + (it & 1) * kGsTileBytes + rowoff;
        float4 x[8];  // all loads first: the in-place stores alias them
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < nph) x[c] = lds128(A + (((uint32_t)(c0 + c) ^ swz) << 4));
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < nph) {
            const uint32_t off = ((uint32_t)(c0 + c) ^ swz) << 4;
#if TNB_GS_TRUNC_HI
            // The MMA reads the gathered tile as it is: the tensor core ignores
            // the low 13 mantissa bits, i.e. hi = x truncated to tf32.  Only
            // lo = x - hi (exact) is written -- no in-place store of hi.
            const uint32_t l0 = __float_as_uint(x[c].x - __uint_as_float(__float_as_uint(x[c].x) & 0xffffe000u));
            const uint32_t l1 = __float_as_uint(x[c].y - __uint_as_float(__float_as_uint(x[c].y) & 0xffffe000u));
            const uint32_t l2 = __float_as_uint(x[c].z - __uint_as_float(__float_as_uint(x[c].z) & 0xffffe000u));
            const uint32_t l3 = __float_as_uint(x[c].w - __uint_as_float(__float_as_uint(x[c].w) & 0xffffe000u));
#else
            // hi = x rounded to tf32 (nearest, ties away: add half an ulp of the
            // 10-bit mantissa to the magnitude and truncate -- what cvt.rna does,
            // on the full-rate integer pipe instead of the conversion pipe);
            // lo = x - hi exact, truncated to tf32 by the tensor core
            uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
            h0 = (__float_as_uint(x[c].x) + 0x1000u) & 0xffffe000u;
            h1 = (__float_as_uint(x[c].y) + 0x1000u) & 0xffffe000u;
            h2 = (__float_as_uint(x[c].z) + 0x1000u) & 0xffffe000u;
            h3 = (__float_as_uint(x[c].w) + 0x1000u) & 0xffffe000u;
            l0 = __float_as_uint(x[c].x - __uint_as_float(h0));
            l1 = __float_as_uint(x[c].y - __uint_as_float(h1));
            l2 = __float_as_uint(x[c].z - __uint_as_float(h2));
            l3 = __float_as_uint(x[c].w - __uint_as_float(h3));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(A + off), "r"(h0), "r"(h1), "r"(h2), "r"(h3)
                         : "memory");
#endif
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(Alo + off), "r"(l0), "r"(l1), "r"(l2), "r"(l3)
                         : "memory");
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        gs_arrive(&a_ready[s]);
        GS_TRACE(3, it, 2);
        if (warp == 8) GS_STAMP(it, 5);
      }
      if (warp == 8) GS_TRACE_END(3);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(kGsNA * 64)));
  }
}

void gs_fill_prep(const ChainDev& ch, const GPlan& G, GsPrep* gp) {
  const MergePlan& mp = G.mp;
  gp->n0 = ch.n;
  gp->K = (uint32_t)G.K;
  gp->Kmid = (uint32_t)G.Kmid;
  gp->sub_rows = (uint32_t)G.sub_rows;
  gp->chunk_shift = (uint32_t)G.chunk_shift;
  for (int g = 0; g < mp.ng; ++g) {
    const int f = g == 0 ? 0 : (g == mp.ng - 1 ? 3 : (g == G.gdiag ? 2 : 1));
    // the sorted field runs over ALL merged interior groups (one original mode each)
    uint32_t w = 1;
    if (f == 1)
      for (int o = mp.hi[g]; o < G.omid_hi; ++o) w *= (uint32_t)ch.m[o].J;
    for (int o = mp.hi[g] - 1; o >= mp.lo[g]; --o) {
      gp->oJ[o] = ch.m[o].J;
      gp->w0[o] = gp->w1[o] = gp->w2[o] = gp->w3[o] = 0;
      (f == 0 ? gp->w0 : f == 1 ? gp->w1 : f == 2 ? gp->w2 : gp->w3)[o] = w;
      w *= (uint32_t)ch.m[o].J;
    }
  }
}

}  // namespace

bool gsort_ok(const ChainDev& ch, int64_t m, bool batched) {
  static thread_local GPlan G;
  if (!plan_gsort(ch, m, &G, batched)) return false;
  // 16-byte row pieces: original boundary modes must be 16-byte aligned
  if (G.mp.kind[0] == kOrig && (reinterpret_cast<uintptr_t>(ch.m[0].s) & 15)) return false;
  if (G.mp.kind[G.mp.ng - 1] == kOrig && (reinterpret_cast<uintptr_t>(ch.m[ch.n - 1].s) & 15)) return false;
  if (G.gdiag >= 0 && G.mp.kind[G.gdiag] == kOrig && (reinterpret_cast<uintptr_t>(ch.m[G.mp.lo[G.gdiag]].s) & 15))
    return false;
  return true;
}

// AUTO: large calls whose buckets average at least 512 samples (4 tiles) and
// whose sorted mode is a product of at least two interior modes -- the global
// sort then removes a whole r x r step per entry -- or is a single interior
// mode that the bucketed path would run on the state kernel (48^7, r = 32 at
// 2^22 tuples: 0.34 against 0.47 ms; r = 20: against 1.08 ms).  A single
// interior mode that fits the stream kernel stays there: its per-tile sort is
// cheaper than the global one (cfg5: 4.6 against 5.5 ms at 2^26 tuples).
bool gsort_auto(const ChainDev& ch, int64_t m, bool batched) {
  const int env = gsort_env();
  if (!env || m < (1 << 18) || !gsort_ok(ch, m, batched)) return false;
  static thread_local GPlan G;
  plan_gsort(ch, m, &G, batched);
  if (G.K * 512 > m) return false;
  if (env == 2 || G.omid_hi - G.omid_lo >= 2) return true;
  static thread_local EPlan P;
  return bucketed_supported(ch) && plan_entries(ch, m, &P) == TNB_OK && !P.stream;
}

int64_t gsort_workspace(const ChainDev& ch, int64_t m, bool batched) {
  static thread_local GPlan G;
  return plan_gsort(ch, m, &G, batched) ? G.total_bytes : 0;
}

void gsort_info(const ChainDev& ch, int64_t m, tnb_entries_info* info, bool batched) {
  static thread_local GPlan G;
  if (!plan_gsort(ch, m, &G, batched)) return;
  const MergePlan& mp = G.mp;
  info->compute_kernel = 3;
  info->tile = kGsTile;
  info->n_virtual = 3 + (G.gdiag >= 0 ? 1 : 0);
  info->prefix_modes = mp.a();
  info->suffix_modes = mp.b();
  info->prefix_rows = mp.a() > 1 ? mp.rows[0] : 0;
  info->suffix_rows = mp.b() > 1 ? mp.rows[mp.ng - 1] : 0;
  info->diag_tables = 0;
  info->table_launches = table_launches(mp) + (G.omid_hi - G.omid_lo);
  // per entry: one r0 x r1 product (3 tf32 MMAs), the diagonal scale, the closing dot
  info->tensor_flops = 3.0 * 2.0 * G.r0 * G.r1 * (double)m;
  info->kernel_flops = (2.0 * G.r0 * G.r1 + (G.gdiag >= 0 ? G.r1 : 0) + 2.0 * G.r1) * (double)m;
  double tf = 0.0;
  for (int g = 0; g < mp.ng; ++g) {
    const int lo = mp.lo[g], hi = mp.hi[g];
    if (mp.kind[g] == kDiag) ++info->diag_tables;
    if (mp.kind[g] == kPrefix || mp.kind[g] == kDiag) {
      int64_t rows = ch.m[lo].J;
      for (int o = lo + 1; o < hi; ++o) {
        rows *= ch.m[o].J;
        tf += (double)rows * ch.m[o].rr * (ch.m[o].layout == TNB_LAYOUT_DIAG ? 1.0 : 2.0 * ch.m[o].rl);
      }
    } else if (mp.kind[g] == kSuffix) {
      int64_t rows = ch.m[hi - 1].J;
      for (int o = hi - 2; o >= lo; --o) {
        rows *= ch.m[o].J;
        tf += (double)rows * ch.m[o].rl * (ch.m[o].layout == TNB_LAYOUT_DIAG ? 1.0 : 2.0 * ch.m[o].rr);
      }
    }
  }
  int64_t rows = (int64_t)ch.m[G.omid_lo].J * G.r0;
  for (int o = G.omid_lo + 1; o < G.omid_hi; ++o) {
    rows *= ch.m[o].J;
    tf += (double)rows * ch.m[o].rr * 2.0 * ch.m[o].rl;
  }
  info->table_flops = tf;
}

// Bytes of the core-dependent head of the workspace: tables, levels of the
// merged mode and its slice images.  Batched calls keep two of them and
// build element b + 1's while element b's compute kernel runs.
int64_t gsort_table_bytes(const ChainDev& ch, int64_t m, bool batched) {
  static thread_local GPlan G;
  return plan_gsort(ch, m, &G, batched) ? G.hist_off : 0;
}

// Phase 1 of a call: tables (first / last / diag) and the slice images of the
// chain `ch` into table_ws.  They depend only on the cores: side stream
// (forked from st: after everything queued there), concurrent with whatever
// st runs next; *done = the event the compute kernel has to wait for (null
// when they were built on st itself).  slot picks one of the two join events.
int gsort_tables(const ChainDev& ch, int64_t m, bool batched, void* table_ws, cudaStream_t st, int slot,
                 cudaEvent_t* done) {
  static thread_local GPlan G;
  if (!plan_gsort(ch, m, &G, batched))
    return set_error(TNB_EINVAL, "the global-sort algorithm does not support this chain");
  unsigned char* tb = static_cast<unsigned char*>(table_ws);
  *done = nullptr;
  int rc;
  SideStream* ss = table_stream_env() ? side_stream() : nullptr;
  if (ss) {
    cudaEvent_t join = slot ? ss->join2 : ss->join;
    rc = check_cuda(cudaEventRecord(ss->fork, st), "fork");
    if (!rc) rc = check_cuda(cudaStreamWaitEvent(ss->s, ss->fork, 0), "fork wait");
    if (rc) return rc;
    // prefix and suffix chains side by side when the tables are on the critical path (batched elements
    // after the first have no index passes to hide behind; else when the tables are large against m:
    // next to the index passes of a 2^24-tuple call the second stream only takes bandwidth from them)
    const bool conc = batched || 4 * (G.mp.rows[0] + G.mp.rows[G.mp.ng - 1]) >= m;
    rc = build_tables(ch, G.mp, tb, ss->s, conc ? ss->s2 : nullptr, ss->ea, ss->eb);
    if (!rc) rc = gs_build_mid(ch, G, tb, ss->s);
    const int rj = check_cuda(cudaEventRecord(join, ss->s), "join");
    if (rc || rj) {
      // join on the error path too: the caller frees the workspace the side stream may still be writing
      if (!rj) cudaStreamWaitEvent(st, join, 0);
      else cudaStreamSynchronize(ss->s);
      return rc ? rc : rj;
    }
    *done = join;
    return TNB_OK;
  }
  rc = build_tables(ch, G.mp, tb, st);
  if (!rc) rc = gs_build_mid(ch, G, tb, st);
  return rc;
}

// Phase 2: the index passes (unless the records of a previous element of the
// batch are reused) and the compute kernel, which waits for `tables`.
// batched / reuse_records: the chain is one element of a batched chain; every
// element shares the index matrix, so the sorted records, the tile map and the
// hot-row votes of element 0 serve the others.
int gsort_compute(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                  int64_t ws_bytes, void* table_ws, cudaStream_t st, bool batched, bool reuse_records,
                  cudaEvent_t tables) {
  static thread_local GPlan G;
  auto fail0 = [&](int code) {
    if (tables) cudaStreamWaitEvent(st, tables, 0);
    return code;
  };
  if (!plan_gsort(ch, m, &G, batched))
    return fail0(set_error(TNB_EINVAL, "the global-sort algorithm does not support this chain"));
  if (!ws || ws_bytes < G.total_bytes)
    return fail0(set_error(TNB_EWORKSPACE, "global-sort entries needs %lld workspace bytes, got %lld",
                           (long long)G.total_bytes, (long long)ws_bytes));
  unsigned char* base = static_cast<unsigned char*>(ws);
  unsigned char* tb = static_cast<unsigned char*>(table_ws);
  const MergePlan& mp = G.mp;
  int rc;
  auto fail = [&](int code) {
    if (tables) cudaStreamWaitEvent(st, tables, 0);
    return code;
  };
  static thread_local ChainDev v;
  virtual_chain(ch, mp, tb, &v);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + G.hist_off);
  uint32_t* bstart = reinterpret_cast<uint32_t*>(base + G.bstart_off);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(base + G.tbase_off);
  uint32_t* cursor = reinterpret_cast<uint32_t*>(base + G.cursor_off);
  uint2* tinfo = reinterpret_cast<uint2*>(base + G.tinfo_off);
  uint4* recu = reinterpret_cast<uint4*>(base + G.recu_off);
  uint4* recs = reinterpret_cast<uint4*>(base + G.recs_off);
  const uint32_t K = (uint32_t)G.K;
  if (!reuse_records) {
    rc = check_cuda(cudaMemsetAsync(hist, 0, (size_t)K * 4 + 16, st), "gsort hist");
    if (rc) return fail(rc);
    {
      static thread_local GsPrep gp;
      gs_fill_prep(ch, G, &gp);
      const bool sh = K <= (uint32_t)kGsSmemK;
      const bool stage = (ch.n & 1) == 0 && ch.n <= kGsStageN0 && (reinterpret_cast<uintptr_t>(idx) & 15) == 0;
      const size_t sm = (sh ? (size_t)((K + 3) & ~3u) * 4 : 0) + (stage ? (size_t)kGsPrepThreads * (ch.n / 2) * 16 : 0);
      auto pk = sh ? (stage ? gs_prep_kernel<true, true> : gs_prep_kernel<true, false>)
                   : (stage ? gs_prep_kernel<false, true> : gs_prep_kernel<false, false>);
      if (sm > 48 * 1024) {
        rc = check_cuda(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "gsort prep smem");
        if (rc) return fail(rc);
      }
      const int per_sm = sm > 56 * 1024 ? 2 : 4;
      const int64_t g = std::min<int64_t>(ceil_div(m, kGsPrepThreads), (int64_t)num_sms() * per_sm);
      KTimer kt("entries_prep", st);
      pk<<<(unsigned)g, kGsPrepThreads, sm, st>>>(gp, idx, m, err, recu, hist);
    }
    rc = check_launch("gsort prep");
    if (rc) return fail(rc);
    gs_detect_hot_kernel<<<kGsHotBlocks, 32, 0, st>>>(recu, m, hist + K);
    rc = check_launch("gsort detect hot");
    if (rc) return fail(rc);
    {
      KTimer kt("entries_sort", st);
      gs_scan_kernel<<<1, 1024, 0, st>>>(hist, K, bstart, tbase, cursor);
      gs_tilemap_kernel<<<(unsigned)std::min<int64_t>(ceil_div(ceil_div(m, kGsTile) + K, 256), (int64_t)num_sms() * 8), 256, 0,
                          st>>>(bstart, tbase, K, tinfo);
      const size_t sm = (size_t)kGsScatThreads * kGsScatPer * 18 + (size_t)K * 8;
      if (K > (uint32_t)kGsSmemK) {
        const int64_t g = std::min<int64_t>(ceil_div(m, 256), (int64_t)num_sms() * 16);
        gs_scatter_big_kernel<<<(unsigned)g, 256, 0, st>>>(recu, m, cursor, recs);
      } else {
        if (sm > 48 * 1024)
          rc = check_cuda(cudaFuncSetAttribute(gs_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                          "gsort scatter smem");
        if (!rc) {
          const int64_t g =
              std::min<int64_t>(ceil_div(m, (int64_t)kGsScatThreads * kGsScatPer), (int64_t)num_sms() * 8);
          gs_scatter_kernel<<<(unsigned)g, kGsScatThreads, sm, st>>>(recu, m, K, cursor, recs);
        }
      }
    }
    if (rc) return fail(rc);
    rc = check_launch("gsort sort");
    if (rc) return fail(rc);
  }
  if (tables) {
    rc = check_cuda(cudaStreamWaitEvent(st, tables, 0), "join tables");
    if (rc) return rc;
  }
  GsArgs ga;
  ga.P = v.m[0].s;
  ga.S = v.m[mp.ng - 1].s;
  ga.D = G.gdiag >= 0 ? v.m[G.gdiag].s : nullptr;
  ga.img = tb + G.img_off;
  ga.recs = recs;
  ga.tinfo = tinfo;
  ga.tbase = tbase;
  ga.K = K;
  ga.Kmid = (uint32_t)G.Kmid;
  ga.interleave = G.nsub > 1;
  ga.hot = hist + K;
  ga.m = (uint32_t)m;
  {  // L2 policies: big tables stream, a result that fits stays
    const int64_t big = (int64_t)16 << 20;
    const int gl = mp.ng - 1;
    ga.pfP = (int64_t)v.m[0].J * G.r0 * 4 > big;
    ga.pfS = (int64_t)v.m[gl].J * G.r1 * 4 > big;
    ga.pfD = G.gdiag >= 0 && (int64_t)v.m[G.gdiag].J * G.r1 * 4 > big;
    ga.keep_out = m * 4 <= ((int64_t)64 << 20);
  }
  ga.r0 = G.r0;
  ga.r1 = G.r1;
  ga.out = out;
  const bool diag = G.gdiag >= 0;
  const bool compact = diag && G.r1 <= 24;  // 96-byte closing rows: a fourth stage
  const size_t smem = 1024 + (compact ? GsSmem<true, 96>::kBytes
                                      : (diag ? GsSmem<true, 128>::kBytes : GsSmem<false, 128>::kBytes));
  auto kfn = compact ? entries_gsort_kernel<true, 96>
                     : (diag ? entries_gsort_kernel<true, 128> : entries_gsort_kernel<false, 128>);
  rc = check_cuda(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "gsort smem attr");
  if (rc) return rc;
  const int64_t tiles_max = ceil_div(m, kGsTile) + (int64_t)K;
  const int grid = (int)std::min<int64_t>(tiles_max, num_sms());
#ifdef TNB_GS_TRACE
  static unsigned long long* tr = nullptr;
  if (!tr) cudaMalloc(&tr, 16384 * 8);
  cudaMemsetAsync(tr, 0, 16384 * 8, st);
  ga.trace = tr;
#endif
  {
    KTimer kt("entries_compute", st);
    kfn<<<grid, kGsThreads, smem, st>>>(ga);
  }
#ifdef TNB_GS_TRACE
  if (const char* tp = getenv("TNB_GS_TRACE_FILE")) {
    static unsigned long long host[16384];
    cudaStreamSynchronize(st);
    cudaMemcpy(host, tr, sizeof(host), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(tp, "wb")) {
      fwrite(host, 1, sizeof(host), f);
      fclose(f);
    }
  }
#endif
  return check_launch("entries_gsort");
}

int launch_entries_gsort(const ChainDev& ch, const int64_t* idx, int64_t m, float* out, int32_t* err, void* ws,
                         int64_t ws_bytes, cudaStream_t st) {
  if (!ws || ws_bytes < gsort_workspace(ch, m, false))
    return set_error(TNB_EWORKSPACE, "global-sort entries needs %lld workspace bytes, got %lld",
                     (long long)gsort_workspace(ch, m, false), (long long)ws_bytes);
  cudaEvent_t tables = nullptr;
  const int rc = gsort_tables(ch, m, false, ws, st, 0, &tables);
  if (rc) return rc;
  return gsort_compute(ch, idx, m, out, err, ws, ws_bytes, ws, st, false, false, tables);
}
