// masks.cuh -- every non-blocklist mask of fl_attn.h is a per-row key INTERVAL
// [lo, hi): causal [0, q_abs+1), sliding window [q_abs-w, q_abs+1) (Listing 2
// P:L296, G4), PrefixLM [0, max(P, q_abs+1)) (G5), document [off[j], off[j+1])
// (G6, optionally cut at q_abs+1), none [0, S_k).  That turns FlexAttention's
// inspected block_mask into O(1) arithmetic per tile:
// a KV tile is skipped, full (no per-element test) or partial (two compares).
#pragma once
#include "params.h"

namespace fl {

struct Interval {
  int32_t lo, hi;  // admissible keys [lo, hi); empty when hi <= lo
};

__host__ __device__ inline Interval row_interval(const AttnParams& p, int32_t b, int32_t q) {
  const int32_t q_abs = q + p.q_off;
  int32_t lo = 0, hi = p.Sk;
  switch (p.mask) {
    case MASK_CAUSAL:
    case MASK_BLOCKLIST:
      hi = q_abs + 1 < hi ? q_abs + 1 : hi;
      break;
    case MASK_SLIDING:
      hi = q_abs + 1 < hi ? q_abs + 1 : hi;
      lo = q_abs - p.window > 0 ? q_abs - p.window : 0;
      break;
    case MASK_PREFIX: {
      int32_t e = p.prefix > q_abs + 1 ? p.prefix : q_abs + 1;
      hi = e < hi ? e : hi;
      break;
    }
    case MASK_DOCUMENT: {
      const int32_t* off = p.doc_offsets + (int64_t)b * p.doc_stride_b;
      lo = 0;
      hi = 0;
      if (q_abs >= 0 && q_abs < p.Sk) {
        for (int32_t j = 0; j < p.n_docs; ++j) {
          int32_t a = off[j], e = off[j + 1];
          if (q_abs >= a && q_abs < e) {
            lo = a;
            hi = e;
          }
        }
        if (p.doc_causal && q_abs + 1 < hi) hi = q_abs + 1;
      }
      break;
    }
    default:
      break;
  }
  if (hi < lo) hi = lo;
  return {lo, hi};
}

// A 128-key tile starting at k0 needs no per-element mask for a row with interval iv iff it lies
// inside the interval and inside [0, S_k).  The kernel (attn_tc.cuh) and the schedule dump
// (fl_debug_schedule) classify tiles with this one predicate.
__host__ __device__ inline bool tile_inside(const Interval& iv, int32_t k0, int32_t Sk) {
  return k0 >= iv.lo && k0 + 128 <= iv.hi && k0 + 128 <= Sk;
}

// Union of the row intervals of rows [q_first, q_last] (all intervals are monotone in q).
__host__ __device__ inline Interval rows_union(const AttnParams& p, int32_t b, int32_t q_first, int32_t q_last) {
  Interval a = row_interval(p, b, q_first), z = row_interval(p, b, q_last);
  bool ea = a.hi <= a.lo, ez = z.hi <= z.lo;
  if (ea && ez) return {0, 0};
  if (ea) return z;
  if (ez) return a;
  return {a.lo < z.lo ? a.lo : z.lo, a.hi > z.hi ? a.hi : z.hi};
}

}  // namespace fl
