// Random-row gather microbenchmark (B200): how fast can one SM pull random
// 128-byte table rows into shared memory / registers?  Informs the entries
// kernels' gather design (csrc/entries_gsort.cuh).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bench tools/gather_bench.cu
//   ./gather_bench [log2_rows=20] [samples_log2=24]
// Modes: 0 = 16-byte cp.async (LDGSTS), 8 lanes per row, per-warp ring with wait_group
//        1 = LDG.128 into registers, 8 lanes per row, UNROLL rows in flight per lane group
//        2 = cp.async.bulk (TMA) 128 B per row, one mbarrier per batch of 32 rows per warp
//        3 = TMA tile::gather4 (UTMALDG.2D.GATHER4): 4 rows per instruction, SWIZZLE_128B tensor map;
//            checked against the table (row r holds the value r in every column)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));            \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: each warp processes batches of 32 rows (8 LDGSTS instructions), DEPTH batches in flight
template <int DEPTH>
__global__ void __launch_bounds__(256) k_ldgsts(const float* __restrict__ tab, const uint32_t* __restrict__ idx, int64_t m,
                                                float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = sm + (size_t)warp * DEPTH * 4096;
  const int64_t nb = m / 32;  // batches
  const int64_t gw = blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  float acc = 0.f;
  auto issue = [&](int64_t b, int slot) {
    const uint32_t r = __ldg(idx + b * 32 + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int src = 4 * i + (lane >> 3);
      const uint32_t row = __shfl_sync(0xffffffffu, r, src);
      const uint32_t dst = s32(ring + slot * 4096 + src * 128 + (lane & 7) * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(tab + (size_t)row * 32 + 4 * (lane & 7)) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t b = gw;
  for (int d = 0; d < DEPTH; ++d) {
    if (b + (int64_t)d * nw < nb) issue(b + (int64_t)d * nw, d);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int slot = 0;
  for (; b < nb; b += nw) {
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");
    __syncwarp();
    acc += *reinterpret_cast<const float*>(ring + slot * 4096 + lane * 128 + (lane & 7) * 4);
    __syncwarp();
    const int64_t nxt = b + (int64_t)DEPTH * nw;
    if (nxt < nb) issue(nxt, slot);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    slot = slot + 1 == DEPTH ? 0 : slot + 1;
  }
  if (acc == 12345.f) out[0] = acc;
}

// mode 1: LDG.128, 8 lanes per row, 4 rows per instruction, UNROLL instructions in flight
template <int UNROLL>
__global__ void __launch_bounds__(256) k_ldg(const float* __restrict__ tab, const uint32_t* __restrict__ idx, int64_t m,
                                             float* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nb = m / 32;
  const int64_t gw = blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  float acc = 0.f;
  for (int64_t b = gw; b < nb; b += nw) {
    const uint32_t r = __ldg(idx + b * 32 + lane);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int src = 4 * i + (lane >> 3);
      const uint32_t row = __shfl_sync(0xffffffffu, r, src);
      v[i] = __ldcg(reinterpret_cast<const float4*>(tab + (size_t)row * 32 + 4 * (lane & 7)));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].w;
  }
  if (acc == 12345.f) out[0] = acc;
  (void)UNROLL;
}

// mode 2: TMA bulk row copies: lane l copies row l of the batch (128 B), one mbarrier per slot
template <int DEPTH>
__global__ void __launch_bounds__(256) k_bulk(const float* __restrict__ tab, const uint32_t* __restrict__ idx, int64_t m,
                                              float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = sm + (size_t)warp * DEPTH * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)8 * DEPTH * 4096) + warp * DEPTH;
  if (lane == 0)
    for (int d = 0; d < DEPTH; ++d) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bars + d)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t nb = m / 32;
  const int64_t gw = blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  float acc = 0.f;
  auto issue = [&](int64_t b, int slot) {
    const uint32_t row = __ldg(idx + b * 32 + lane);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bars + slot)), "r"(4096u) : "memory");
    __syncwarp();
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(ring + slot * 4096 + lane * 128)),
                 "l"(tab + (size_t)row * 32), "r"(128u), "r"(s32(bars + slot))
                 : "memory");
  };
  int64_t b = gw;
  for (int d = 0; d < DEPTH; ++d)
    if (b + (int64_t)d * nw < nb) issue(b + (int64_t)d * nw, d);
  int slot = 0;
  uint32_t ph = 0;
  for (; b < nb; b += nw) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(s32(bars + slot)),
        "r"(ph)
        : "memory");
    acc += *reinterpret_cast<const float*>(ring + slot * 4096 + lane * 128 + (lane & 7) * 4);
    __syncwarp();
    const int64_t nxt = b + (int64_t)DEPTH * nw;
    if (nxt < nb) issue(nxt, slot);
    if (++slot == DEPTH) {
      slot = 0;
      ph ^= 1;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

// mode 3: TMA gather4: lanes 0..7 of a warp issue one gather4 each per batch of 32 rows
template <int DEPTH>
__global__ void __launch_bounds__(256) k_gather4(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ idx,
                                                 int64_t m, float* __restrict__ out, unsigned long long* __restrict__ bad) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024 - (s32(sm_raw) & 1023)) & 1023);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = sm + (size_t)warp * DEPTH * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)8 * DEPTH * 4096) + warp * DEPTH;
  if (lane == 0)
    for (int d = 0; d < DEPTH; ++d) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bars + d)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t nb = m / 32;
  const int64_t gw = blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
  float acc = 0.f;
  unsigned long long nbad = 0;
  auto issue = [&](int64_t b, int slot) {
    const uint32_t row = __ldg(idx + b * 32 + lane);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bars + slot)), "r"(4096u) : "memory");
    const int r0 = __shfl_sync(0xffffffffu, (int)row, (4 * lane) & 31), r1 = __shfl_sync(0xffffffffu, (int)row, (4 * lane + 1) & 31),
              r2 = __shfl_sync(0xffffffffu, (int)row, (4 * lane + 2) & 31), r3 = __shfl_sync(0xffffffffu, (int)row, (4 * lane + 3) & 31);
    __syncwarp();
    if (lane < 8)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
          "%6}], [%7];" ::"r"(s32(ring + slot * 4096 + lane * 512)),
          "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(s32(bars + slot))
          : "memory");
  };
  int64_t b = gw;
  for (int d = 0; d < DEPTH; ++d)
    if (b + (int64_t)d * nw < nb) issue(b + (int64_t)d * nw, d);
  int slot = 0;
  uint32_t ph = 0;
  for (; b < nb; b += nw) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(s32(bars + slot)),
        "r"(ph)
        : "memory");
    // row `lane` of the batch, column 4 * (lane & 7): SWIZZLE_128B puts 16-byte piece c at c ^ (row & 7)
    const float v = *reinterpret_cast<const float*>(ring + slot * 4096 + lane * 128 + ((0 ^ (lane & 7)) << 4));
    const float w = *reinterpret_cast<const float*>(ring + slot * 4096 + lane * 128 + ((3 ^ (lane & 7)) << 4) + 4);
    const uint32_t want = __ldg(idx + b * 32 + lane);
    if (v != (float)(want & 0xffff) || w != (float)(want & 0xffff) + 13.f) ++nbad;
    acc += v;
    __syncwarp();
    const int64_t nxt = b + (int64_t)DEPTH * nw;
    if (nxt < nb) issue(nxt, slot);
    if (++slot == DEPTH) {
      slot = 0;
      ph ^= 1;
    }
  }
  if (nbad) atomicAdd(bad, nbad);
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int lr = argc > 1 ? atoi(argv[1]) : 20, lm = argc > 2 ? atoi(argv[2]) : 24;
  const int64_t rows = (int64_t)1 << lr, m = (int64_t)1 << lm;
  float *tab, *out;
  uint32_t* idx;
  CK(cudaMalloc(&tab, rows * 128));
  {  // row r: column c holds (r & 0xffff) + c (exact in fp32)
    std::vector<float> ht((size_t)rows * 32);
    for (int64_t r = 0; r < rows; ++r)
      for (int c = 0; c < 32; ++c) ht[(size_t)r * 32 + c] = (float)(r & 0xffff) + (float)c;
    CK(cudaMemcpy(tab, ht.data(), (size_t)rows * 128, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&out, 4));
  CK(cudaMalloc(&idx, m * 4));
  std::vector<uint32_t> h(m);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < m; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    h[i] = (uint32_t)(s % (uint64_t)rows);
  }
  CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-34s rows 2^%d: %7.3f ms  %7.1f GB/s  (%5.1f GB/s per SM)\n", name, lr, ms, m * 128.0 / ms / 1e6,
           m * 128.0 / ms / 1e6 / 148);
  };
#define LDGSTS(D, CTAS)                                                                                          \
  {                                                                                                              \
    CK(cudaFuncSetAttribute(k_ldgsts<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * D * 4096));            \
    run("ldgsts depth " #D " x " #CTAS " CTA/SM", [&] { k_ldgsts<D><<<148 * CTAS, 256, 8 * D * 4096>>>(tab, idx, m, out); }); \
  }
  LDGSTS(1, 1)
  LDGSTS(2, 1)
  LDGSTS(4, 1)
  LDGSTS(6, 1)
  LDGSTS(2, 2)
  LDGSTS(3, 2)
  LDGSTS(1, 4)
  LDGSTS(1, 6)
  run("ldg.128 x 2 CTA/SM", [&] { k_ldg<8><<<148 * 2, 256>>>(tab, idx, m, out); });
  run("ldg.128 x 4 CTA/SM", [&] { k_ldg<8><<<148 * 4, 256>>>(tab, idx, m, out); });
  run("ldg.128 x 8 CTA/SM", [&] { k_ldg<8><<<148 * 8, 256>>>(tab, idx, m, out); });
#define BULK(D, CTAS)                                                                                             \
  {                                                                                                               \
    CK(cudaFuncSetAttribute(k_bulk<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * D * 4096 + 8 * D * 8));   \
    run("bulk depth " #D " x " #CTAS " CTA/SM", [&] { k_bulk<D><<<148 * CTAS, 256, 8 * D * 4096 + 8 * D * 8>>>(tab, idx, m, out); }); \
  }
  BULK(1, 1)
  BULK(2, 1)
  BULK(4, 1)
  BULK(6, 1)
  BULK(3, 2)
  {  // mode 3: TMA gather4 through a SWIZZLE_128B tensor map, box height 1 and 4
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    unsigned long long* bad;
    CK(cudaMalloc(&bad, 8));
    for (int bh : {1}) {  // box height 4 is rejected at run time (illegal instruction)
      CUtensorMap tm;
      const cuuint64_t dims[2] = {32, (cuuint64_t)rows};
      const cuuint64_t strides[1] = {128};
      const cuuint32_t box[2] = {32, (cuuint32_t)bh};
      const cuuint32_t estr[2] = {1, 1};
      const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("tensor map box height %d: encode rc %d\n", bh, (int)r);
      if (r != CUDA_SUCCESS) continue;
#define G4(D, CTAS)                                                                                              \
  {                                                                                                              \
    const int smb = 8 * D * 4096 + 8 * D * 8 + 1024;                                                             \
    CK(cudaFuncSetAttribute(k_gather4<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));                    \
    CK(cudaMemset(bad, 0, 8));                                                                                   \
    run("gather4 depth " #D " x " #CTAS " CTA/SM", [&] { k_gather4<D><<<148 * CTAS, 256, smb>>>(tm, idx, m, out, bad); }); \
    unsigned long long hb = 0;                                                                                   \
    CK(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));                                                         \
    printf("    mismatching rows: %llu of %lld\n", hb, (long long)(6 * m));                                      \
  }
      G4(2, 1)
      G4(4, 1)
      G4(4, 2)
      G4(2, 4)
    }
  }
  return 0;
}
