// Store-stream microbenchmark for the full() epilogue design (no MMA):
// 148 persistent CTAs write a 65536 x 65536 fp32 C (17.18 GB) in 128 x 128
// tiles, tile order as in full_tc_gemm_kernel (down the rows of a column
// block), with
//   mode 0: W warps, thread = column, 128 st.global.cs.b32 per tile per warp
//           group of 4 (the current epilogue when W = 4)
//   mode 1: W warps, TMA 2-D tensor stores of 32 x 32 boxes staged in smem
//   mode 2: W warps, thread = 4 columns: st.global.cs.v4 (512 B per warp row)
//   mode 3: W warps, TMA stores of 64 x 64 boxes (16 KB)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/store_bench tools/store_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

constexpr int64_t NN = 65536;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Args {
  CUtensorMap m32, m64;
  float* C;
};

template <int MODE, int W>
__global__ void __launch_bounds__(W * 32, 1) store_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_mt = NN / 128, n_cb = NN / 128;
  const int64_t nt = n_mt * n_cb;
  const int64_t t0 = nt * blockIdx.x / gridDim.x, t1 = nt * (blockIdx.x + 1) / gridDim.x;
  uint32_t it = 0;
  // MODE 4 / 5: the b32 stores of mode 0 with the CTAs in lockstep on one 128-row
  // band: 4 = tiles in row-major order, grid-strided (adjacent CTAs write
  // adjacent column tiles); 5 = CTA b keeps column tile b + 148 w for a whole
  // pass down the rows (what a resident-operand GEMM needs), all CTAs at the
  // same row band
  const int64_t t_lo = MODE >= 4 ? 0 : t0, t_hi = MODE == 6 ? 2 * 3 * n_mt : MODE >= 4 ? (nt + gridDim.x - 1) / gridDim.x : t1;
  for (int64_t tt = t_lo; tt < t_hi; ++tt) {
    int64_t t = tt, cb, mt;
    if (MODE == 4) {
      t = tt * gridDim.x + blockIdx.x;
      if (t >= nt) break;
      mt = t / n_cb;
      cb = t - mt * n_cb;
    } else if (MODE == 5) {
      const int64_t w = tt / n_mt;
      mt = tt - w * n_mt;
      cb = w * gridDim.x + blockIdx.x;
      if (cb >= n_cb) break;
    } else if (MODE == 6) {
      // the GEMM's order: CTA b owns 384 columns (3 column tiles) of wave w; per
      // row tile it writes the three 128 x 128 sub-tiles one after the other
      const int64_t per = 3 * n_mt, w = tt / per, r = tt - w * per;
      mt = r / 3;
      cb = (w * gridDim.x + blockIdx.x) * 3 + (r - mt * 3);
      if (cb >= n_cb) {
        if (r - mt * 3 == 0 && (w * gridDim.x + blockIdx.x) * 3 >= n_cb) break;
        continue;
      }
    } else {
      cb = t / n_mt;
      mt = t - cb * n_mt;
    }
    const float base = (float)(t + lane);
#define V(j) (base + (float)(j))
    if (MODE == 0 || MODE >= 4) {
      // W warps split the 128 columns x 128 rows: warp w: column group w % 4, rows half
      constexpr int RG = W / 4;  // row groups
      const int cg = warp & 3, rg = warp >> 2;
      float* p = a.C + (mt * 128 + rg * (128 / RG)) * NN + cb * 128 + cg * 32 + lane;
#pragma unroll
      for (int j = 0; j < 128 / RG; ++j) {
        asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "f"(V(j)) : "memory");
        p += NN;
      }
    } else if (MODE == 2) {
      // thread = 4 consecutive columns; a warp writes 512 B of one row; W warps split rows
      float* p = a.C + (mt * 128 + warp) * NN + cb * 128 + lane * 4;
      for (int j = warp; j < 128; j += W) {
        __stcs(reinterpret_cast<float4*>(p), make_float4(V(j), V(j + 1), V(j + 2), V(j + 3)));
        p += (int64_t)W * NN;
      }
    } else if (MODE == 1) {
      // warp w: column group w % 4 (32 cols), row groups of 32 split over W/4
      const int cg = warp & 3, rg = warp >> 2;
      float* sb0 = sm + warp * 2 * 1024;
      for (int ch = rg; ch < 4; ch += W / 4) {
        float* sb = sb0 + (it & 1) * 1024;
        if (lane == 0 && it >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) sb[j * 32 + lane] = V(ch * 32 + j);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                           reinterpret_cast<uint64_t>(&a.m32)),
                       "r"((int)(cb * 128 + cg * 32)), "r"((int)(mt * 128 + ch * 32)), "r"(smem_u32(sb))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++it;
      }
    } else {
      // MODE 3: 64 x 64 boxes, 4 per tile; warp w takes box w % 4 (W >= 4), rows staged by the warp
      if (warp < 4) {
        const int bx = warp & 1, by = warp >> 1;
        float* sb = sm + warp * 2 * 4096 + (it & 1) * 4096;
        if (lane == 0 && it >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll 8
        for (int j = 0; j < 64; ++j) {
          sb[j * 64 + lane] = V(j);
          sb[j * 64 + 32 + lane] = V(j + 1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                           reinterpret_cast<uint64_t>(&a.m64)),
                       "r"((int)(cb * 128 + bx * 64)), "r"((int)(mt * 128 + by * 64)), "r"(smem_u32(sb))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++it;
      }
    }
  }
  if (MODE == 1 || MODE == 3)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// tile shape sweep: TR rows x TC cols per tile, st.global.cs.v4 by W warps
// (each warp instruction: 512 contiguous bytes of one row); RIGHT: a CTA's
// consecutive tiles go along the row (else down the column block)
template <int TR, int TC, int W, bool RIGHT>
__global__ void __launch_bounds__(W * 32, 1) shape_kernel(float* C) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_mt = NN / TR, n_ct = NN / TC;
  const int64_t nt = n_mt * n_ct;
  const int64_t t0 = nt * blockIdx.x / gridDim.x, t1 = nt * (blockIdx.x + 1) / gridDim.x;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t ct = RIGHT ? t % n_ct : t / n_mt, mt = RIGHT ? t / n_ct : t - (t / n_mt) * n_mt;
    const float base = (float)(t + lane);
    constexpr int SEG = TC / 128;  // 512-byte segments per row
    for (int e = warp; e < TR * SEG; e += W) {
      const int r = e / SEG, sg = e % SEG;
      float* p = C + (mt * TR + r) * NN + ct * TC + sg * 128 + lane * 4;
      __stcs(reinterpret_cast<float4*>(p), make_float4(base, base + 1.f, base + 2.f, base + (float)e));
    }
  }
}

template <int TR, int TC, int W, bool RIGHT>
float run_shape(float* C) {
  auto k = shape_kernel<TR, TC, W, RIGHT>;
  for (int i = 0; i < 2; ++i) k<<<148, W * 32>>>(C);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) k<<<148, W * 32>>>(C);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

template <int MODE, int W>
float run(Args& a, int smem) {
  auto k = store_kernel<MODE, W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 2; ++i) k<<<148, W * 32, smem>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k<<<148, W * 32, smem>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / reps;
}

int main() {
  Args a;
  size_t bytes = (size_t)NN * NN * 4;
  if (cudaMalloc(&a.C, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cuuint64_t dims[2] = {(cuuint64_t)NN, (cuuint64_t)NN}, str[1] = {(cuuint64_t)NN * 4};
  cuuint32_t b32[2] = {32, 32}, b64[2] = {64, 64}, es[2] = {1, 1};
  enc(&a.m32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a.C, dims, str, b32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&a.m64, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a.C, dims, str, b64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto rep = [&](const char* name, float ms) {
    printf("%-34s %8.3f ms %8.1f GB/s\n", name, ms, bytes / (ms * 1e-3) / 1e9);
  };
  rep("st.b32 4 warps (current)", run<0, 4>(a, 0));
  rep("st.b32 4 warps lockstep row-major", run<4, 4>(a, 0));
  rep("st.b32 4 warps lockstep col-block", run<5, 4>(a, 0));
  rep("st.b32 4 warps lockstep 384-col block", run<6, 4>(a, 0));
  rep("st.b32 8 warps lockstep row-major", run<4, 8>(a, 0));
  rep("st.b32 8 warps", run<0, 8>(a, 0));
  rep("st.b32 16 warps", run<0, 16>(a, 0));
  rep("st.v4 4 warps", run<2, 4>(a, 0));
  rep("st.v4 8 warps", run<2, 8>(a, 0));
  rep("st.v4 16 warps", run<2, 16>(a, 0));
  rep("tma 32x32 4 warps", run<1, 4>(a, 4 * 2 * 4096));
  rep("tma 32x32 8 warps", run<1, 8>(a, 8 * 2 * 4096));
  rep("tma 32x32 16 warps", run<1, 16>(a, 16 * 2 * 4096));
  rep("tma 64x64 4 warps", run<3, 4>(a, 4 * 2 * 16384));
  rep("v4 128x128 down 8w", run_shape<128, 128, 8, false>(a.C));
  rep("v4 128x128 right 8w", run_shape<128, 128, 8, true>(a.C));
  rep("v4 128x384 down 8w", run_shape<128, 384, 8, false>(a.C));
  rep("v4 64x256 down 8w", run_shape<64, 256, 8, false>(a.C));
  rep("v4 32x512 down 8w", run_shape<32, 512, 8, false>(a.C));
  rep("v4 16x1024 down 8w", run_shape<16, 1024, 8, false>(a.C));
  rep("v4 8x2048 down 8w", run_shape<8, 2048, 8, false>(a.C));
  rep("v4 128x128 right 16w", run_shape<128, 128, 16, true>(a.C));
  rep("v4 32x512 right 8w", run_shape<32, 512, 8, true>(a.C));
  rep("v4 1x65536 (rows) 8w", run_shape<1, 65536, 8, false>(a.C));
  rep("v4 1x65536 (rows) 32w", run_shape<1, 65536, 32, false>(a.C));
  cudaFree(a.C);
  return 0;
}
