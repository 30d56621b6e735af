// K1 performance kernel (placeholder until the bucketed kernel lands).
#include "common.cuh"

namespace tnb {
bool bucketed_supported(const ChainDev&) { return false; }
int launch_entries_bucketed(const ChainDev&, const int64_t*, int64_t, float*, int32_t*,
                            cudaStream_t) {
  return set_error(TNB_EINVAL, "bucketed entries not built");
}
}  // namespace tnb
