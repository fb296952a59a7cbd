// attn_tc.cu -- dispatch of the bf16 tcgen05 attention family (attn_tc.cuh) by head dim and
// differential attention; the instantiations live in attn_tc_d{128,64,32}[_diff].cu.
#include <cuda_runtime.h>

#include "attn_tc.cuh"
#include "params.h"

namespace fl {
#define FL_DECL(D, F)                                                                     \
  cudaError_t launch_attn_tc_##D##_##F(const AttnParams&, const TmaMaps&, cudaStream_t); \
  cudaError_t debug_timing_##D##_##F(unsigned long long*, int);
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

// fl_debug_schedule: the persistent kernel's work units and tile classes for p (interval masks, bf16
// path), written by sched_dump_kernel with the unit decomposition launch_one uses.
cudaError_t launch_sched_dump(const AttnParams& p, int32_t* out, int64_t out_words, int64_t* n_records,
                              int32_t* max_tiles, cudaStream_t stream) {
  const bool diff = p.maps == 2;
  const bool pair = small_head_pair(p);
  AttnParams pp = p;
  pp.unit_order = pair && bias_resident(p) ? 1 : 0;   // the order launch_one gives the kernel
  const int rows_per_unit = (diff || pair) ? 128 : 256;
  const long long units =
      (long long)p.B * (pair ? (p.G + 1) / 2 : p.G) * p.Hq * ((p.Sq + rows_per_unit - 1) / rows_per_unit);
  const int mt = (p.Sk + 127) / 128;
  *n_records = units * 2;
  *max_tiles = mt;
  if (!out) return cudaSuccess;                        // size query
  if (out_words < units * 2 * (8 + mt)) return cudaErrorInvalidValue;
  const int blocks = (int)((units * 2 + 127) / 128);
  if (diff) sched_dump_kernel<true, false><<<blocks, 128, 0, stream>>>(pp, (int)units, mt, out);
  else if (pair) sched_dump_kernel<false, true><<<blocks, 128, 0, stream>>>(pp, (int)units, mt, out);
  else sched_dump_kernel<false, false><<<blocks, 128, 0, stream>>>(pp, (int)units, mt, out);
  return cudaGetLastError();
}

// fl_debug_timing: the FL_TIMING counters summed over the instantiating translation units
cudaError_t debug_timing(unsigned long long* out, int reset) {
  cudaError_t (*fns[])(unsigned long long*, int) = {debug_timing_128_0, debug_timing_128_1, debug_timing_64_0,
                                                    debug_timing_64_1, debug_timing_32_0, debug_timing_32_1};
  for (int i = 0; i < 48; ++i) out[i] = 0;
  for (auto f : fns) {
    unsigned long long t[48];
    cudaError_t e = f(t, reset);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < 48; ++i) out[i] += t[i];
  }
  return cudaSuccess;
}
}  // namespace fl
