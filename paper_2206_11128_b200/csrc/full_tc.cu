// tcgen05 3xTF32 GEMM for the final full() contraction (placeholder).
#include "common.cuh"

namespace tnb {
bool tc_gemm_supported(int64_t, int64_t, int, int64_t, int64_t, int64_t) { return false; }
int launch_tc_gemm(const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*, int64_t,
                   int64_t, int64_t, int64_t, int, int64_t, cudaStream_t) {
  return set_error(TNB_EINVAL, "tensor-core gemm not built");
}
}  // namespace tnb
