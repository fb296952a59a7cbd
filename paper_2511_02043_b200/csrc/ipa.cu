// ipa.cu -- AlphaFold's Invariant Point Attention core (named by the paper among the
// variants FlexAttention cannot express, P:L47 / P:L443, "12 heads and head dimension 16" P:L891; the formula
// is reading G23 = AF2 Suppl. Alg.22 lines 7-10):
//   logit_ij = w_L ( c^-1/2 q_i.k_j + b_ij - (gamma_h w_C / 2) sum_p |T_i q_ip - T_j k_jp|^2 )
// The point term is a squared distance of GLOBAL points, |x_i|^2 + |y_j|^2 - 2 x_i.y_j: the cross term is a
// dot product over 3 Pq dimensions and |y_j|^2 a per-key term, |x_i|^2 cancels in the softmax.  So the
// logits are ONE tensor-core contraction over augmented operands of 64 columns (ipa_prep_kernel):
//   Q'_i = [ w_L c^-1/2 q_i | a x_hi | a x_hi | a x_lo | 1 | 1 | 0 ],   a = w_L gamma_h w_C (x = T_i q_ip)
//   K'_j = [ k_j            | y_hi   | y_lo   | y_hi   | u_hi | u_lo | 0 ],   u = -a/2 |y_j|^2
// (hi/lo = a bf16 value and its bf16 remainder: global coordinates of tens of A would lose the small
// distances in a single bf16 term), and the fused attention kernel (fl_attn_fwd, scale 1, additive bias
// w_L b) computes softmax and the scalar output o = sum_j a_ij v_j on the tensor cores and returns the LSE.
// ipa_finish_kernel then recomputes a_ij = exp(Q'_i.K'_j + w_L b_ij - LSE_i) per row i (fp32) for the two
// outputs whose "values" are not shared across rows or need more than bf16: the pair output
// sum_j a_ij z_ij and the point output T_i^-1 sum_j a_ij T_j v_jp, accumulated in fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "params.h"
#include "ptx.cuh"

namespace fl {


constexpr int kIpaD = 64;

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// one warp per (n, h): every lane transforms the (n, h) points (a few FMAs), then writes columns lane and
// lane + 32 of Q'_n, K'_n (coalesced 64-byte rows) and lanes < 3 Pv the global value points
__global__ void ipa_prep_kernel(const IpaParams p) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= p.N * p.H) return;
  const int n = w / p.H, h = w % p.H;
  const float wL = sqrtf(1.f / 3.f), wC = p.Pq > 0 ? sqrtf(2.f / (9.f * (float)p.Pq)) : 0.f;
  const float a = wL * p.gamma[h] * wC;
  const float* R = p.R + n * 9;
  const float* t = p.t + n * 3;
  float y2 = 0.f;
  for (int m = 0; m < 3 * p.Pq; ++m) {             // |y|^2 over every query/key point coordinate
    const int pp = m / 3, e = m % 3;
    float y = t[e];
    for (int f = 0; f < 3; ++f) y += R[e * 3 + f] * __bfloat162float(p.kp[((int64_t)w * p.Pq + pp) * 3 + f]);
    y2 += y * y;
  }
  const int P3 = 3 * p.Pq, o1 = p.c, o2 = p.c + P3, o3 = p.c + 2 * P3, o4 = p.c + 3 * P3;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int d = lane + 32 * half;
    float qv = 0.f, kv = 0.f;
    if (d < p.c) {
      qv = wL * rsqrtf((float)p.c) * __bfloat162float(p.q[(int64_t)w * p.c + d]);
      kv = __bfloat162float(p.k[(int64_t)w * p.c + d]);
    } else if (d < o4) {
      const int seg = (d - o1) / P3, m = (d - o1) % P3, pp = m / 3, e = m % 3;
      float x = t[e], y = t[e];
      for (int f = 0; f < 3; ++f) {
        x += R[e * 3 + f] * __bfloat162float(p.qp[((int64_t)w * p.Pq + pp) * 3 + f]);
        y += R[e * 3 + f] * __bfloat162float(p.kp[((int64_t)w * p.Pq + pp) * 3 + f]);
      }
      __nv_bfloat16 xh, xl, yh, yl;
      split_bf16(a * x, xh, xl);
      split_bf16(y, yh, yl);
      // seg 0: a x_hi . y_hi, seg 1: a x_hi . y_lo, seg 2: a x_lo . y_hi
      qv = __bfloat162float(seg == 2 ? xl : xh);
      kv = __bfloat162float(seg == 1 ? yl : yh);
    } else if (d < o4 + 2) {                       // 1 . (-a/2 |y|^2) as hi + lo
      __nv_bfloat16 uh, ul;
      split_bf16(-0.5f * a * y2, uh, ul);
      qv = 1.f;
      kv = __bfloat162float(d == o4 ? uh : ul);
    }
    p.qa[(int64_t)w * kIpaD + d] = __float2bfloat16_rn(qv);   // exact: the values are already bf16
    p.ka[(int64_t)w * kIpaD + d] = __float2bfloat16_rn(kv);
  }
  if (lane < 3 * p.Pv) {                           // global value point coordinate T_n v_np
    const int pp = lane / 3, e = lane % 3;
    float g = t[e];
    for (int f = 0; f < 3; ++f) g += R[e * 3 + f] * __bfloat162float(p.vp[((int64_t)w * p.Pv + pp) * 3 + f]);
    p.gv[((int64_t)w * p.Pv + pp) * 3 + e] = g;
  }
}

// w_L b: the additive bias the attention kernel takes (natural-log units, scale 1)
__global__ void ipa_bias_kernel(const IpaParams p) {
  const int64_t n = (int64_t)p.H * p.N * p.N;
  const float wL = sqrtf(1.f / 3.f);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p.bias_s[i] = __float2bfloat16_rn(wL * __bfloat162float(p.bias[i]));
}

// One CTA per (row i, head h), 128 threads (many small CTAs: the per-row loops are latency-bound, so the
// kernel relies on occupancy): a_ij (recomputed from Q', K', w_L b and the forward's LSE, fp32), then
// opair_i^h = sum_j a_ij z_ij (thread = feature) and the point output op_ip^h = R_i^T (sum_j a_ij g_jp^h - t_i)
// (24 sums split over 5 j-partitions of the threads, reduced in shared memory).
constexpr int kIpaThreads = 128;
constexpr int kIpaParts = kIpaThreads / 24;        // 5 j-partitions for the (<= 24) point sums
__global__ void __launch_bounds__(kIpaThreads) ipa_finish_kernel(const IpaParams p, const float* __restrict__ lse,
                                                                 __nv_bfloat16* __restrict__ opair,
                                                                 float* __restrict__ op) {
  extern __shared__ float ipa_smem[];
  float* a = ipa_smem;                             // [N]
  float* qs = a + p.N;                             // [64]
  float* gs = qs + kIpaD;                          // [kIpaParts][24]
  const int i = blockIdx.x / p.H, h = blockIdx.x % p.H, tid = threadIdx.x;
  if (tid < kIpaD) qs[tid] = __bfloat162float(p.qa[((int64_t)i * p.H + h) * kIpaD + tid]);
  __syncthreads();
  const float l = lse[(int64_t)h * p.N + i];      // lse [1, H, N] (natural log, G19)
  // ---- a_ij
  for (int j = tid; j < p.N; j += kIpaThreads) {
    const uint4* kr = reinterpret_cast<const uint4*>(p.ka + ((int64_t)j * p.H + h) * kIpaD);
    uint4 u[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) u[d] = __ldg(kr + d);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      const uint32_t w[4] = {u[d].x, u[d].y, u[d].z, u[d].w};
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        s0 = fmaf(qs[d * 8 + 2 * x], bf16_lo(w[x]), s0);
        s1 = fmaf(qs[d * 8 + 2 * x + 1], bf16_hi(w[x]), s1);
      }
    }
    const float s = s0 + s1 + __bfloat162float(p.bias_s[((int64_t)h * p.N + i) * p.N + j]);
    a[j] = __expf(s - l);
  }
  __syncthreads();
  // ---- pair output: thread -> 8 consecutive features (one 16-byte load of z per j) and a j-partition
  // (8 partitions), reduced over the partitions in shared memory
  const __nv_bfloat16* zi = p.z + (int64_t)i * p.N * p.cz;
  float* red = ipa_smem + ((p.N + kIpaD + kIpaParts * 24 + 3) & ~3);   // [8][128], 16-byte aligned
  for (int fb = 0; fb < p.cz; fb += 128) {
    const int f8 = fb + (tid % 16) * 8, part = tid / 16;
    float acc[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) acc[x] = 0.f;
    if (f8 < p.cz) {
#pragma unroll 4
      for (int j = part; j < p.N; j += 8) {
        const uint4 zv = __ldg(reinterpret_cast<const uint4*>(zi + (int64_t)j * p.cz + f8));
        const uint32_t w[4] = {zv.x, zv.y, zv.z, zv.w};
        const float aj = a[j];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          acc[2 * x] = fmaf(aj, bf16_lo(w[x]), acc[2 * x]);
          acc[2 * x + 1] = fmaf(aj, bf16_hi(w[x]), acc[2 * x + 1]);
        }
      }
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) red[part * 128 + (tid % 16) * 8 + x] = acc[x];
    __syncthreads();
    if (fb + tid < p.cz) {
      float v = 0.f;
#pragma unroll
      for (int q8 = 0; q8 < 8; ++q8) v += red[q8 * 128 + tid];
      opair[((int64_t)i * p.H + h) * p.cz + fb + tid] = __float2bfloat16_rn(v);
    }
    __syncthreads();
  }
  // ---- point output: thread -> (float4 of the <= 24 sums, j-partition), reduced in shared memory
  const int PV3 = p.Pv * 3;
  const int64_t jstride = (int64_t)p.H * PV3;
  constexpr int kPtParts = kIpaThreads / 6;        // 21
  if (tid < 6 * kPtParts) {
    const int f4 = tid % 6, part = tid / 6;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (f4 * 4 < PV3) {
      const float* gj = p.gv + (int64_t)h * PV3 + f4 * 4;
#pragma unroll 4
      for (int j = part; j < p.N; j += kPtParts) {
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(gj + (int64_t)j * jstride));
        const float aj = a[j];
        acc.x = fmaf(aj, g4.x, acc.x);
        acc.y = fmaf(aj, g4.y, acc.y);
        acc.z = fmaf(aj, g4.z, acc.z);
        acc.w = fmaf(aj, g4.w, acc.w);
      }
    }
    reinterpret_cast<float4*>(red)[part * 6 + f4] = acc;
  }
  __syncthreads();
  if (tid < PV3) {
    float v = 0.f;
    for (int part = 0; part < kPtParts; ++part) v += red[part * 24 + tid];
    gs[tid] = v;
  }
  __syncthreads();
  if (tid < p.Pv) {
    const float* g = gs + tid * 3;
    const float* R = p.R + i * 9;
    const float* t = p.t + i * 3;
    for (int x = 0; x < 3; ++x)
      op[(((int64_t)i * p.H + h) * p.Pv + tid) * 3 + x] =
          R[0 * 3 + x] * (g[0] - t[0]) + R[1 * 3 + x] * (g[1] - t[1]) + R[2 * 3 + x] * (g[2] - t[2]);
  }
}

cudaError_t launch_ipa_prep(const IpaParams& p, cudaStream_t s) {
  ipa_prep_kernel<<<(p.N * p.H + 7) / 8, 256, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ipa_bias_kernel<<<4 * 148, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ipa_finish(const IpaParams& p, const float* lse, void* opair, float* op, cudaStream_t s) {
  const int smem = (((p.N + kIpaD + kIpaParts * 24 + 3) & ~3) + 8 * 128) * 4;
  cudaError_t e = cudaFuncSetAttribute(ipa_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  ipa_finish_kernel<<<p.N * p.H, kIpaThreads, smem, s>>>(p, lse, static_cast<__nv_bfloat16*>(opair), op);
  return cudaGetLastError();
}

}  // namespace fl
