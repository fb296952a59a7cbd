// attn_tc_d64_diff.cu -- instantiates the tcgen05 attention kernel family (attn_tc.cuh) for D = 64,
// differential attention true (one translation unit per (D, DIFF) so the build compiles in parallel).
#include "attn_tc.cuh"

namespace fl {
cudaError_t launch_attn_tc_64_1(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream) {
  return launch_mod<64, true>(p, maps, stream);
}
cudaError_t debug_timing_64_1(unsigned long long* out, int reset) { return debug_timing_tu<0>(out, reset); }
}  // namespace fl
