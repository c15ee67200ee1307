// k_mlp_tc.cu -- K2b: the bf16 tcgen05 fused MLP (placeholder until the kernel lands).
#include "gcdf_internal.h"

namespace gcdf {
bool tc_compiled() { return false; }
cudaError_t launch_mlp_tc(int, const WeightsBF16 &, const QueryArgs &, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace gcdf
