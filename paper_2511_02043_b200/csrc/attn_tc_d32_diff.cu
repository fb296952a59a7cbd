// attn_tc_d32_diff.cu -- instantiates the tcgen05 attention kernel family (attn_tc.cuh) for D = 32,
// differential attention true (one translation unit per (D, DIFF) so the build compiles in parallel).
#include "attn_tc.cuh"

namespace fl {
cudaError_t launch_attn_tc_32_1(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream) {
  return launch_mod<32, true>(p, maps, stream);
}
cudaError_t debug_timing_32_1(unsigned long long* out, int reset) { return debug_timing_tu<0>(out, reset); }
}  // namespace fl
