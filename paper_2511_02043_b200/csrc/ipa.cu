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
  const int P3 = 3 * p.Pq, o1 = p.c, o4 = p.c + 3 * P3;   // column blocks: [o1, o1 + 3 P3) points, o4, o4 + 1 norms
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

// a_ij^h = exp(Q'_i.K'_j + w_L b_ij - LSE_i) for a block of kProbRows query rows of one head, fp32 into
// A [H, N, N] (for the pair output): thread = key j (its K' row of 64 bf16 in registers), the block's Q'
// rows and LSEs in shared memory -- each K' row is read once per row block instead of once per row.  The
// point output of the block's rows is summed here as well, over key chunks of kJC staged in shared memory
// (the chunk's a_ij and global value points g_jp^h): thread (row, float4 of the <= 24 coordinates) --
// op_ip^h = R_i^T (sum_j a_ij g_jp^h - t_i).
constexpr int kProbRows = 16;
constexpr int kProbThreads = 128;
constexpr int kJC = 256;                           // keys per chunk
size_t ipa_probs_smem() { return (size_t)(kProbRows * kJC + kJC * 24 + kProbRows * 24) * 4; }
__global__ void __launch_bounds__(kProbThreads) ipa_probs_kernel(const IpaParams p, const float* __restrict__ lse,
                                                                 float* __restrict__ A, float* __restrict__ op) {
  __shared__ __align__(16) float qs[kProbRows][kIpaD];
  __shared__ float ls[kProbRows];
  extern __shared__ __align__(16) float pr_smem[];
  float* as = pr_smem;                             // [kProbRows][kJC]
  float* gs = as + kProbRows * kJC;                // [kJC][24]
  float* gsum = gs + kJC * 24;                     // [kProbRows][24]
  const int h = blockIdx.y, i0 = blockIdx.x * kProbRows, tid = threadIdx.x;
  const int nr = min(kProbRows, p.N - i0);
  const int PV3 = p.Pv * 3;
  {                                                 // the rows' Q' (8 bf16 per thread and load, batched)
    constexpr int kB = (kProbRows * kIpaD / 8 + kProbThreads - 1) / kProbThreads;
    uint4 tmp[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int e = tid + k * kProbThreads, r = e / (kIpaD / 8), d8 = e % (kIpaD / 8);
      tmp[k] = make_uint4(0u, 0u, 0u, 0u);
      if (r < nr) tmp[k] = __ldg(reinterpret_cast<const uint4*>(p.qa + ((int64_t)(i0 + r) * p.H + h) * kIpaD) + d8);
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int e = tid + k * kProbThreads, r = e / (kIpaD / 8), d8 = e % (kIpaD / 8);
      if (r < kProbRows) {
        const uint32_t w[4] = {tmp[k].x, tmp[k].y, tmp[k].z, tmp[k].w};
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          qs[r][d8 * 8 + 2 * x] = bf16_lo(w[x]);
          qs[r][d8 * 8 + 2 * x + 1] = bf16_hi(w[x]);
        }
      }
    }
  }
  if (tid < kProbRows) ls[tid] = tid < nr ? lse[(int64_t)h * p.N + i0 + tid] : 0.f;   // lse [1, H, N] (G19)
  const int pr_r = tid / 6, pr_f4 = tid % 6;       // point sums: threads < 96
  const bool pt_on = tid < kProbRows * 6 && pr_r < nr && pr_f4 * 4 < PV3;
  float4 pacc = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  for (int j0 = 0; j0 < p.N; j0 += kJC) {
    const int cnt = min(kJC, p.N - j0);
    {                                               // the chunk's g_jp^h (<= 6 float4 per key), loads batched
      constexpr int kB = kJC * 6 / kProbThreads;    // 12
      const int nq = PV3 / 4, n4 = cnt * nq;
      float4 tmp[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int e = tid + k * kProbThreads;
        if (e < n4)
          tmp[k] = __ldg(reinterpret_cast<const float4*>(p.gv + ((int64_t)(j0 + e / nq) * p.H + h) * PV3) + e % nq);
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int e = tid + k * kProbThreads;
        if (e < n4) *reinterpret_cast<float4*>(gs + (e / nq) * 24 + (e % nq) * 4) = tmp[k];
      }
    }
    for (int jj = tid; jj < cnt; jj += kProbThreads) {
      const int j = j0 + jj;
      const uint4* kr = reinterpret_cast<const uint4*>(p.ka + ((int64_t)j * p.H + h) * kIpaD);
      uint4 u[8];
#pragma unroll
      for (int d = 0; d < 8; ++d) u[d] = __ldg(kr + d);
      float bv[kProbRows];                          // the rows' biases, all in flight at once
#pragma unroll
      for (int r = 0; r < kProbRows; ++r)
        bv[r] = r < nr ? __bfloat162float(p.bias_s[((int64_t)h * p.N + i0 + r) * p.N + j]) : 0.f;
#pragma unroll
      for (int r = 0; r < kProbRows; ++r) {
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const uint32_t w[4] = {u[d].x, u[d].y, u[d].z, u[d].w};
          const float4 qa = *reinterpret_cast<const float4*>(&qs[r][d * 8]);
          const float4 qb = *reinterpret_cast<const float4*>(&qs[r][d * 8 + 4]);
          s0 = fmaf(qa.x, bf16_lo(w[0]), s0);
          s1 = fmaf(qa.y, bf16_hi(w[0]), s1);
          s0 = fmaf(qa.z, bf16_lo(w[1]), s0);
          s1 = fmaf(qa.w, bf16_hi(w[1]), s1);
          s0 = fmaf(qb.x, bf16_lo(w[2]), s0);
          s1 = fmaf(qb.y, bf16_hi(w[2]), s1);
          s0 = fmaf(qb.z, bf16_lo(w[3]), s0);
          s1 = fmaf(qb.w, bf16_hi(w[3]), s1);
        }
        const float av = r < nr ? __expf(s0 + s1 + bv[r] - ls[r]) : 0.f;
        as[r * kJC + jj] = av;
        if (r < nr) A[((int64_t)h * p.N + i0 + r) * p.N + j] = av;
      }
    }
    __syncthreads();
    if (pt_on) {
      const float* ar = as + pr_r * kJC;
#pragma unroll 4
      for (int jj = 0; jj < cnt; ++jj) {
        const float aj = ar[jj];
        const float4 g4 = *reinterpret_cast<const float4*>(gs + jj * 24 + pr_f4 * 4);
        pacc.x = fmaf(aj, g4.x, pacc.x);
        pacc.y = fmaf(aj, g4.y, pacc.y);
        pacc.z = fmaf(aj, g4.z, pacc.z);
        pacc.w = fmaf(aj, g4.w, pacc.w);
      }
    }
    __syncthreads();
  }
  if (PV3 == 0) return;
  if (pt_on) *reinterpret_cast<float4*>(gsum + pr_r * 24 + pr_f4 * 4) = pacc;
  __syncthreads();
  for (int e = tid; e < nr * p.Pv; e += kProbThreads) {
    const int r = e / p.Pv, pp = e % p.Pv, i = i0 + r;
    const float* g = gsum + r * 24 + pp * 3;
    const float* R = p.R + i * 9;
    const float* t = p.t + i * 3;
    for (int x = 0; x < 3; ++x)
      op[(((int64_t)i * p.H + h) * p.Pv + pp) * 3 + x] =
          R[0 * 3 + x] * (g[0] - t[0]) + R[1 * 3 + x] * (g[1] - t[1]) + R[2 * 3 + x] * (g[2] - t[2]);
  }
}

// One CTA per (row i, group of kOutHG heads): z_i (the row's N x c_z pair features) is streamed once for
// the group's heads, opair_i^h = sum_j a_ij^h z_ij (thread = 8 consecutive features x one of 16
// j-partitions).  The group's a_i^h [kOutHG][N] is staged in shared memory.
constexpr int kOutThreads = 256;
constexpr int kOutHG = 6;                          // heads per pass over z_i (6 x 8 accumulators)
__global__ void __launch_bounds__(kOutThreads) ipa_out_kernel(const IpaParams p, const float* __restrict__ A,
                                                              __nv_bfloat16* __restrict__ opair) {
  extern __shared__ __align__(16) float ipa_smem[];
  float* a = ipa_smem;                             // [kOutHG][N]
  float* red = a + (((int64_t)kOutHG * p.N + 3) & ~3);   // [8 warps][kOutHG][128] / point partials
  const int i = blockIdx.x, hg = blockIdx.y * kOutHG, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ng = min(kOutHG, p.H - hg);
  for (int e0 = 0; e0 < ng * p.N; e0 += 8 * kOutThreads) {   // 8 loads in flight per thread
    float tmp[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = e0 + tid + k * kOutThreads;
      if (e < ng * p.N) tmp[k] = __ldg(A + ((int64_t)(hg + e / p.N) * p.N + i) * p.N + e % p.N);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = e0 + tid + k * kOutThreads;
      if (e < ng * p.N) a[e] = tmp[k];
    }
  }
  __syncthreads();
  // ---- pair output
  const __nv_bfloat16* zi = p.z + (int64_t)i * p.N * p.cz;
  const int fl8 = (tid & 15) * 8, part = tid >> 4;   // 16 j-partitions; lanes l, l ^ 16 hold parts 2w, 2w + 1
  for (int fb = 0; fb < p.cz; fb += 128) {
    const int f8 = fb + fl8;
    {
      const int h0 = 0, nh = ng;                   // local head index; global head = hg + local
      float acc[kOutHG][8];
#pragma unroll
      for (int hh = 0; hh < kOutHG; ++hh)
#pragma unroll
        for (int x = 0; x < 8; ++x) acc[hh][x] = 0.f;
      if (f8 < p.cz) {
#pragma unroll 6
        for (int j = part; j < p.N; j += 16) {
          const uint4 zv = __ldg(reinterpret_cast<const uint4*>(zi + (int64_t)j * p.cz + f8));
          const uint32_t w[4] = {zv.x, zv.y, zv.z, zv.w};
#pragma unroll
          for (int hh = 0; hh < kOutHG; ++hh) {
            const float aj = hh < nh ? a[(h0 + hh) * p.N + j] : 0.f;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              acc[hh][2 * x] = fmaf(aj, bf16_lo(w[x]), acc[hh][2 * x]);
              acc[hh][2 * x + 1] = fmaf(aj, bf16_hi(w[x]), acc[hh][2 * x + 1]);
            }
          }
        }
      }
#pragma unroll
      for (int hh = 0; hh < kOutHG; ++hh)
#pragma unroll
        for (int x = 0; x < 8; ++x) acc[hh][x] += __shfl_xor_sync(0xffffffffu, acc[hh][x], 16);
      if (lane < 16)
#pragma unroll
        for (int hh = 0; hh < kOutHG; ++hh)
#pragma unroll
          for (int x = 0; x < 8; ++x) red[(warp * kOutHG + hh) * 128 + fl8 + x] = acc[hh][x];
      __syncthreads();
      for (int e = tid; e < nh * 128; e += kOutThreads) {
        const int hh = e / 128, f = e % 128;
        if (fb + f < p.cz) {
          float v = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < kOutThreads / 32; ++w2) v += red[(w2 * kOutHG + hh) * 128 + f];
          opair[((int64_t)i * p.H + hg + h0 + hh) * p.cz + fb + f] = __float2bfloat16_rn(v);
        }
      }
      __syncthreads();
    }
  }
}

cudaError_t launch_ipa_prep(const IpaParams& p, cudaStream_t s) {
  ipa_prep_kernel<<<(p.N * p.H + 7) / 8, 256, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ipa_bias_kernel<<<4 * 148, 256, 0, s>>>(p);
  return cudaGetLastError();
}

size_t ipa_out_smem(const IpaParams& p) {
  return ((((size_t)kOutHG * p.N + 3) & ~size_t(3)) + (size_t)(kOutThreads / 32) * kOutHG * 128) * 4;
}

cudaError_t launch_ipa_finish(const IpaParams& p, const float* lse, float* A, void* opair, float* op, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(ipa_probs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ipa_probs_smem());
  if (e != cudaSuccess) return e;
  ipa_probs_kernel<<<dim3((p.N + kProbRows - 1) / kProbRows, p.H), kProbThreads, ipa_probs_smem(), s>>>(p, lse, A, op);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = ipa_out_smem(p);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(ipa_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ipa_out_kernel<<<dim3(p.N, (p.H + kOutHG - 1) / kOutHG), kOutThreads, smem, s>>>(
      p, A, static_cast<__nv_bfloat16*>(opair));
  return cudaGetLastError();
}

}  // namespace fl
