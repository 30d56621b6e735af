// Device side of the index transport codec (host side: host_codec.cpp):
// widens an int8 / int16 index matrix that crossed PCIe back to the int64
// matrix the entries kernels read (core.py:394-416 semantics unchanged: the
// values are the caller's raw indices, wrapped and bounds-checked by prep).
// HBM-bound: 1 (2) B read + 8 B written per index.
#include "common.cuh"

namespace tnb {
namespace {

// each thread widens 2 consecutive values per step: a 2 (4)-byte load and
// one 16-byte store, so a warp's stores cover 512 contiguous bytes (the
// 16-values-per-thread variant wrote 128-byte runs at a 128-byte lane
// stride and ran at 1.1 TB/s)
template <typename N>
__global__ void __launch_bounds__(256) widen_kernel(const N* __restrict__ in, int64_t count,
                                                    int64_t* __restrict__ out) {
  const int64_t pairs = count / 2;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < pairs;
       g += (int64_t)gridDim.x * blockDim.x) {
    N v[2];
    if constexpr (sizeof(N) == 1)
      *reinterpret_cast<uint16_t*>(v) = __ldcs(reinterpret_cast<const unsigned short*>(in) + g);
    else
      *reinterpret_cast<uint32_t*>(v) = __ldcs(reinterpret_cast<const unsigned int*>(in) + g);
    __stcs(reinterpret_cast<longlong2*>(out) + g, make_longlong2((long long)v[0], (long long)v[1]));
  }
  if (count & 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0) out[count - 1] = (int64_t)in[count - 1];
  }
}

}  // namespace

int launch_widen(const void* in, int width, int64_t count, int64_t* out, cudaStream_t st) {
  if (count == 0) return TNB_OK;
  if (!in || !out || (width != 1 && width != 2)) return set_error(TNB_EINVAL, "widen: bad arguments");
  if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return set_error(TNB_EINVAL, "widen: buffers must be 16-byte aligned");
  const int64_t pairs = count / 2;
  int64_t grid = (pairs + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
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
