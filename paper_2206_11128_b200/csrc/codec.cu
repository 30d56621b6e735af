// Device side of the index transport codec (host side: host_codec.cpp):
// widens an int8 / int16 index matrix that crossed PCIe back to the int64
// matrix the entries kernels read (core.py:394-416 semantics unchanged: the
// values are the caller's raw indices, wrapped and bounds-checked by prep).
// HBM-bound: 1 (2) B read + 8 B written per index.
#include "common.cuh"

namespace tnb {
namespace {

// each thread widens 16 consecutive values: one 16-byte (int8) or two
// 16-byte (int16) loads, eight 16-byte stores
template <typename N>
__global__ void __launch_bounds__(256) widen_kernel(const N* __restrict__ in, int64_t count,
                                                    int64_t* __restrict__ out) {
  const int64_t groups = count / 16;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    N v[16];
    const uint4* src = reinterpret_cast<const uint4*>(in + g * 16);
#pragma unroll
    for (int q = 0; q < (int)sizeof(N); ++q) reinterpret_cast<uint4*>(v)[q] = __ldcs(src + q);
    longlong2* dst = reinterpret_cast<longlong2*>(out + g * 16);
#pragma unroll
    for (int q = 0; q < 8; ++q) __stcs(dst + q, make_longlong2((long long)v[2 * q], (long long)v[2 * q + 1]));
  }
  // ragged tail (count % 16 values)
  const int64_t t = groups * 16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && t < count) out[t] = (int64_t)in[t];
}

}  // namespace

int launch_widen(const void* in, int width, int64_t count, int64_t* out, cudaStream_t st) {
  if (count == 0) return TNB_OK;
  if (!in || !out || (width != 1 && width != 2)) return set_error(TNB_EINVAL, "widen: bad arguments");
  if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return set_error(TNB_EINVAL, "widen: buffers must be 16-byte aligned");
  const int64_t groups = count / 16;
  int64_t grid = (groups + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  grid = grid < 1 ? 1 : (grid > cap ? cap : grid);
  if (width == 1)
    widen_kernel<int8_t><<<(unsigned)grid, 256, 0, st>>>(static_cast<const int8_t*>(in), count, out);
  else
    widen_kernel<int16_t><<<(unsigned)grid, 256, 0, st>>>(static_cast<const int16_t*>(in), count, out);
  return check_launch("widen");
}

}  // namespace tnb

extern "C" int tnb_widen_indices(const void* in, int32_t width, int64_t count, int64_t* out, void* stream) {
  return tnb::launch_widen(in, width, count, out, static_cast<cudaStream_t>(stream));
}
