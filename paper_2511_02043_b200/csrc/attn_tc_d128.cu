// attn_tc_d128.cu -- instantiates the tcgen05 attention kernel family (attn_tc.cuh) for D = 128,
// differential attention false (one translation unit per (D, DIFF) so the build compiles in parallel).
#include "attn_tc.cuh"

namespace fl {
cudaError_t launch_attn_tc_128_0(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream) {
  return launch_mod<128, false>(p, maps, stream);
}
cudaError_t debug_timing_128_0(unsigned long long* out, int reset) { return debug_timing_tu<0>(out, reset); }
}  // namespace fl
