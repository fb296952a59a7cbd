// attn_simt.cu -- the exact-fp32 path (BASELINE config 1, tolerance 1e-5):
// fused tiled online-softmax attention on the FFMA pipe with warp-shuffle row
// max / sum, for EVERY variant of fl_attn.h.  No tensor cores: tcgen05 has no
// fp32-input kind (tf32 rounds to 10 mantissa bits, ~1e-3), so an fp32 kernel
// that must hold 1e-5 runs on CUDA cores.  It is also the semantic reference
// for the bf16 tcgen05 family: same inputs, tighter tolerance.
//
// Layout: one CTA = 16 query rows of one (b, g, h) (4 warps x 4 rows).  K/V
// tiles of 32 keys are staged in shared memory (rows padded by one float so a
// warp's 32 lanes -- one key each -- hit 32 banks).  Per row and tile: lane j
// scores key j, warp max/sum by shuffles, online update (Alg.2 P:L162-175,
// rescale exp(m_old - m_new) P:L685-697), and lane d accumulates O[d].
#include <cuda_runtime.h>
#include <math.h>

#include "masks.cuh"
#include "params.h"

namespace fl {

// RPW rows per warp, 4 warps: 16-row CTAs for big problems (K/V tiles shared by 16 rows); 4-row CTAs
// when the problem has too few 16-row tiles to fill the SMs (C1: 128 rows -> 32 CTAs instead of 8)
constexpr int SIMT_MAX_ROWS = 16;
constexpr int SIMT_KT = 32;
constexpr int SIMT_THREADS = 128;

__device__ __forceinline__ float ld_in(const void* base, int64_t off, int32_t dtype) {
  if (dtype == 1) return static_cast<const float*>(base)[off];
  unsigned short u = static_cast<const unsigned short*>(base)[off];
  return __uint_as_float(static_cast<uint32_t>(u) << 16);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int RPW>
__global__ void __launch_bounds__(SIMT_THREADS) attn_simt_kernel(const __grid_constant__ AttnParams p) {
  constexpr int SIMT_ROWS = 4 * RPW;
  extern __shared__ float sm[];
  const int Dq = p.Dqk, Dv = p.Dv;
  float* Ks = sm;                              // [KT][Dq+1]
  float* Vs = Ks + SIMT_KT * (Dq + 1);         // [KT][Dv+1]
  float* Qs = Vs + SIMT_KT * (Dv + 1);         // [ROWS][Dq]
  uint32_t* blkbits = reinterpret_cast<uint32_t*>(Qs + SIMT_ROWS * Dq);  // blocklist bitmap

  const int nrb = (p.Sq + SIMT_ROWS - 1) / SIMT_ROWS;
  const int64_t bgh = blockIdx.x / nrb;
  const int rb = blockIdx.x % nrb;
  const int h = static_cast<int>(bgh % p.Hq);
  const int g = static_cast<int>((bgh / p.Hq) % p.G);
  const int b = static_cast<int>(bgh / ((int64_t)p.Hq * p.G));
  const int hkv = h / p.grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_first = rb * SIMT_ROWS;
  const int q_last = min(p.Sq, q_first + SIMT_ROWS) - 1;

  Interval blk = rows_union(p, b, q_first, q_last);
  const bool blocklist = p.mask == MASK_BLOCKLIST;
  const int nkb = blocklist ? (p.Sk + p.blk_k - 1) / p.blk_k : 0;
  if (blocklist) {
    const int qb = q_first / p.blk_q;
    for (int w = threadIdx.x; w < (nkb + 31) / 32; w += blockDim.x) blkbits[w] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t base = bgh * p.n_qblk + qb;
      const int cnt = p.blk_cnt[base];
      for (int i = 0; i < cnt && i < p.max_sel; ++i) {
        int j = p.blk_idx[base * p.max_sel + i];
        if (j >= 0 && j < nkb) blkbits[j >> 5] |= 1u << (j & 31);
      }
    }
  }

  float slope = 0.f;
  if (p.mod == MOD_ALIBI) slope = p.alibi ? p.alibi[h] : exp2f(-8.f * (float)(h + 1) / (float)p.Hq);
  const float lam = p.maps == 2 ? diff_lambda(p, h) : 0.f;

  float res[RPW][4];                           // final output accumulators (rows x d-chunks)
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) res[r][c] = 0.f;
  float lse_out[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) lse_out[r] = 0.f;

  for (int map = 0; map < p.maps; ++map) {
    const int qh = h + map * p.Hq, kh = hkv + map * p.Hkv;
    // stage this CTA's Q rows
    __syncthreads();
    for (int i = threadIdx.x; i < SIMT_ROWS * Dq; i += blockDim.x) {
      int r = i / Dq, d = i % Dq, q = q_first + r;
      Qs[i] = q < p.Sq ? ld_in(p.q, b * p.qs.b + g * p.qs.g + qh * p.qs.h + q * p.qs.s + d, p.in_dtype) : 0.f;
    }
    float m[RPW], l[RPW], acc[RPW][4];
    int klo[RPW], khi[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      m[r] = -INFINITY;
      l[r] = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
      Interval iv = row_interval(p, b, q_first + warp * RPW + r);
      klo[r] = iv.lo;
      khi[r] = iv.hi;
    }
    const int t_lo = blk.lo / SIMT_KT, t_hi = (blk.hi + SIMT_KT - 1) / SIMT_KT;
    for (int t = t_lo; t < t_hi; ++t) {
      const int k0 = t * SIMT_KT;
      if (blocklist && !((blkbits[(k0 / p.blk_k) >> 5] >> ((k0 / p.blk_k) & 31)) & 1u)) continue;
      __syncthreads();
      for (int i = threadIdx.x; i < SIMT_KT * Dq; i += blockDim.x) {
        int j = i / Dq, d = i % Dq, k = k0 + j;
        Ks[j * (Dq + 1) + d] =
            k < p.Sk ? ld_in(p.k, b * p.ks.b + g * p.ks.g + kh * p.ks.h + (int64_t)k * p.ks.s + d, p.in_dtype) : 0.f;
      }
      for (int i = threadIdx.x; i < SIMT_KT * Dv; i += blockDim.x) {
        int j = i / Dv, d = i % Dv, k = k0 + j;
        Vs[j * (Dv + 1) + d] =
            k < p.Sk ? ld_in(p.v, b * p.vs.b + g * p.vs.g + hkv * p.vs.h + (int64_t)k * p.vs.s + d, p.in_dtype)
                     : 0.f;
      }
      __syncthreads();
      const int k = k0 + lane;
      bool key_ok = k < p.Sk;
      if (key_ok && p.keybits) {
        const uint32_t* kb = p.keybits + ((int64_t)b * p.G + g) * p.keybits_words;
        key_ok = (kb[k >> 5] >> (k & 31)) & 1u;
      }
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int qrow = warp * RPW + r, q = q_first + qrow;
        if (q >= p.Sq) continue;                       // warp-uniform
        const float* qv = Qs + qrow * Dq;
        const float* kv = Ks + lane * (Dq + 1);
        float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;   // four chains: latency, not the FMA pipe, bounds a row
        int d = 0;
        for (; d + 4 <= Dq; d += 4) {
          d0 = fmaf(qv[d], kv[d], d0);
          d1 = fmaf(qv[d + 1], kv[d + 1], d1);
          d2 = fmaf(qv[d + 2], kv[d + 2], d2);
          d3 = fmaf(qv[d + 3], kv[d + 3], d3);
        }
        for (; d < Dq; ++d) d0 = fmaf(qv[d], kv[d], d0);
        const float dot = (d0 + d1) + (d2 + d3);
        float s = dot * p.scale;                       // Listing 1: scores *= 1/sqrt(d)
        if (p.mod == MOD_ALIBI) s += slope * (float)(k - (q + p.q_off));
        if (p.bias)
          s += ld_in(p.bias, b * p.bs.b + g * p.bs.g + h * p.bs.h + (int64_t)q * p.bs.s + (int64_t)k * p.bs.d,
                     p.bias_dtype);
        if (p.mod == MOD_SOFTCAP) s = p.softcap * tanhf(s / p.softcap);
        bool keep = key_ok && k >= klo[r] && k < khi[r];
        if (blocklist) keep = keep && ((blkbits[(k / p.blk_k) >> 5] >> ((k / p.blk_k) & 31)) & 1u);
        s = keep ? s : -INFINITY;
        const float m_new = fmaxf(m[r], warp_max(s));
        if (m_new == -INFINITY) continue;               // nothing kept yet (warp-uniform)
        const float corr = expf(m[r] - m_new);          // 0 when m = -inf
        const float pk = keep ? expf(s - m_new) : 0.f;
        l[r] = l[r] * corr + warp_sum(pk);
        m[r] = m_new;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] *= corr;
        for (int j = 0; j < SIMT_KT; ++j) {
          const float pj = __shfl_sync(0xffffffffu, pk, j);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int d = lane + 32 * c;
            if (d < Dv) acc[r][c] = fmaf(pj, Vs[j * (Dv + 1) + d], acc[r][c]);
          }
        }
      }
    }
    const float coef = map == 0 ? 1.f : -lam;          // Listing 4: attn0 - lambda * attn1
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const float inv = l[r] > 0.f ? 1.f / l[r] : 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) res[r][c] += coef * acc[r][c] * inv;
      lse_out[r] = l[r] > 0.f ? m[r] + logf(l[r]) : -INFINITY;
    }
  }

  // DIFF-Transformer epilogue (NEXT-2): per-head RMSNorm of A_0 - lambda A_1 over D_v, times (1 - lambda_init)
  float norm_k[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) norm_k[r] = 1.f;
  if (p.maps == 2 && p.diff_norm) {
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      float ss = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (lane + 32 * c < Dv) ss = fmaf(res[r][c], res[r][c], ss);
      ss = warp_sum(ss);
      norm_k[r] = (1.f - p.lambda_init) / sqrtf(ss / (float)Dv + p.diff_norm_eps);
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int q = q_first + warp * RPW + r;
    if (q >= p.Sq) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int d = lane + 32 * c;
      if (d >= Dv) continue;
      float o = res[r][c];
      if (p.maps == 2 && p.diff_norm) o *= norm_k[r] * (p.diff_norm_w ? p.diff_norm_w[d] : 1.f);
      if (p.gate_mode != GATE_NONE) {
        float gv = ld_in(p.gate, b * p.gs.b + g * p.gs.g + h * p.gs.h + (int64_t)q * p.gs.s + d, p.gate_dtype);
        o *= p.gate_mode == GATE_SIGMOID ? 1.f / (1.f + expf(-gv)) : gv;
      }
      static_cast<float*>(p.o)[b * p.os.b + g * p.os.g + h * p.os.h + (int64_t)q * p.os.s + d] = o;
    }
    if (p.lse && lane == 0)
      p.lse[b * p.lses.b + g * p.lses.g + h * p.lses.h + (int64_t)q * p.lses.s] = lse_out[r];
  }
}

size_t simt_smem_bytes(const AttnParams& p) {
  const int nkb = p.mask == MASK_BLOCKLIST ? (p.Sk + p.blk_k - 1) / p.blk_k : 0;
  return sizeof(float) * (SIMT_KT * (p.Dqk + 1) + SIMT_KT * (p.Dv + 1) + SIMT_MAX_ROWS * p.Dqk) +
         sizeof(uint32_t) * ((nkb + 31) / 32 + 1);
}

cudaError_t launch_attn_simt(const AttnParams& p, cudaStream_t stream) {
  const long long bgh = (long long)p.B * p.G * p.Hq;
  const bool small = bgh * ((p.Sq + SIMT_MAX_ROWS - 1) / SIMT_MAX_ROWS) < 2 * 148;
  const int rows = small ? 4 : SIMT_MAX_ROWS;
  const long long grid = bgh * ((p.Sq + rows - 1) / rows);
  const size_t smem = simt_smem_bytes(p);
  auto kern = small ? attn_simt_kernel<1> : attn_simt_kernel<4>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<(unsigned)grid, SIMT_THREADS, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace fl
