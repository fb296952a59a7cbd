// attn_tc.cu -- dispatch of the bf16 tcgen05 attention family (attn_tc.cuh) by head dim and
// differential attention; the instantiations live in attn_tc_d{128,64,32}[_diff].cu.
#include <cuda_runtime.h>

#include "params.h"

namespace fl {
#define FL_DECL(D, F) cudaError_t launch_attn_tc_##D##_##F(const AttnParams&, const TmaMaps&, cudaStream_t);
FL_DECL(128, 0) FL_DECL(128, 1) FL_DECL(64, 0) FL_DECL(64, 1) FL_DECL(32, 0) FL_DECL(32, 1)
#undef FL_DECL

cudaError_t launch_attn_tc(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream) {
  const bool diff = p.maps == 2;
  switch (p.Dqk) {
    case 128: return diff ? launch_attn_tc_128_1(p, maps, stream) : launch_attn_tc_128_0(p, maps, stream);
    case 64: return diff ? launch_attn_tc_64_1(p, maps, stream) : launch_attn_tc_64_0(p, maps, stream);
    case 32: return diff ? launch_attn_tc_32_1(p, maps, stream) : launch_attn_tc_32_0(p, maps, stream);
    default: return cudaErrorInvalidValue;
  }
}

int tc_chunk_elems(int D) { return D >= 64 ? 64 : 32; }
}  // namespace fl
