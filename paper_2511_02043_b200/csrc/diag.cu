// diag.cu -- bring-up diagnostic (fl_diag_umma_gemm): one 128 x N x K bf16 GEMM
// through exactly the TMA / swizzle / UMMA-descriptor / TMEM conventions the
// attention kernels use, so a descriptor bug shows up as a wrong GEMM against
// torch.matmul instead of as a subtly wrong attention output.
//   C[128, N] (f32) = A[128, K] . B^T      B given [N, K] (K-major, like K tiles)
//                                   or B  given [K, N] (MN-major, like V tiles)
//   a_from_tmem: A is first written to TMEM by the threads (like P) -> TS MMA.
#include <cuda_runtime.h>

#include "params.h"
#include "ptx.cuh"

namespace fl {

template <int N, int K, bool BMN, bool ATMEM>
__global__ void __launch_bounds__(128, 1)
    diag_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                     const unsigned short* a_glob, float* c) {
  constexpr int CHK = K >= 64 ? 64 : 32, SWK = CHK * 2;            // A / K-major B chunking along K
  constexpr int CHN = N >= 64 ? 64 : 32, SWN = CHN * 2;            // MN-major B chunking along N
  constexpr uint32_t LK = SWK == 128 ? kLayoutSW128 : kLayoutSW64;
  constexpr uint32_t LN = SWN == 128 ? kLayoutSW128 : kLayoutSW64;
  constexpr int A_BYTES = 128 * K * 2, B_BYTES = N * K * 2;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SW128 atoms); offset arithmetic on smem_raw keeps the shared address space visible
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + A_BYTES + B_BYTES);
  uint64_t* done = bar + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  constexpr uint32_t COL_A = 128;   // A (bf16 pairs) at columns [128, 128 + K/2)

  if (ATMEM) {  // each thread writes its row of A into TMEM, packed like P
    const int r = threadIdx.x;
    uint32_t pk[64];
#pragma unroll
    for (int t = 0; t < K / 2; ++t)
      pk[t] = (uint32_t)a_glob[r * K + 2 * t] | ((uint32_t)a_glob[r * K + 2 * t + 1] << 16);
#pragma unroll
    for (int t = 0; t < K / 2; t += 16) tmem_st16(tmem + lane_base + COL_A + t, &pk[t]);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, (ATMEM ? 0 : A_BYTES) + B_BYTES);
    if (!ATMEM)
      for (int cc = 0; cc < K / CHK; ++cc) tma_load_5d(sA + cc * 128 * SWK, &ta, bar, cc * CHK, 0, 0, 0, 0);
    if (BMN)
      for (int cc = 0; cc < N / CHN; ++cc) tma_load_5d(sB + cc * K * SWN, &tb, bar, cc * CHN, 0, 0, 0, 0);
    else
      for (int cc = 0; cc < K / CHK; ++cc) tma_load_5d(sB + cc * N * SWK, &tb, bar, cc * CHK, 0, 0, 0, 0);
    mbar_wait(bar, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(128, N, BMN ? 1 : 0);
#pragma unroll
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint32_t koff = (kk * 16 / CHK) * 0 + (kk * 16 % CHK) * 2;
      uint64_t bdesc;
      if (BMN)
        bdesc = smem_desc(smem_u32(sB) + kk * 16 * SWN, K * SWN, 8 * SWN, LN);
      else
        bdesc = smem_desc(smem_u32(sB) + (kk * 16 / CHK) * N * SWK + koff, 16, 8 * SWK, LK);
      if (ATMEM) {
        umma_ts(tmem, tmem + COL_A + kk * 8, bdesc, idesc, kk > 0);
      } else {
        const uint64_t adesc = smem_desc(smem_u32(sA) + (kk * 16 / CHK) * 128 * SWK + koff, 16, 8 * SWK, LK);
        umma_ss(tmem, adesc, bdesc, idesc, kk > 0);
      }
    }
    umma_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int cc = 0; cc < N; cc += 32) {
    tmem_ld32(tmem + lane_base + cc, v);
    tmem_wait_ld();
    for (int t = 0; t < 32; ++t) c[threadIdx.x * N + cc + t] = __uint_as_float(v[t]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

template <int N, int K, bool BMN, bool ATMEM>
static cudaError_t diag_launch(const CUtensorMap& ta, const CUtensorMap& tb, const void* a, float* c,
                               cudaStream_t s) {
  const int smem = 128 * K * 2 + N * K * 2 + 64 + 1024;
  auto kern = diag_gemm_kernel<N, K, BMN, ATMEM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<1, 128, smem, s>>>(ta, tb, static_cast<const unsigned short*>(a), c);
  return cudaGetLastError();
}

template <int N, int K>
static cudaError_t diag_nk(const CUtensorMap& ta, const CUtensorMap& tb, const void* a, float* c, bool bmn,
                           bool atmem, cudaStream_t s) {
  if (bmn) return atmem ? diag_launch<N, K, true, true>(ta, tb, a, c, s) : diag_launch<N, K, true, false>(ta, tb, a, c, s);
  return atmem ? diag_launch<N, K, false, true>(ta, tb, a, c, s) : diag_launch<N, K, false, false>(ta, tb, a, c, s);
}

template <int N>
static cudaError_t diag_n(int k, const CUtensorMap& ta, const CUtensorMap& tb, const void* a, float* c, bool bmn,
                          bool atmem, cudaStream_t s) {
  switch (k) {
    case 32: return diag_nk<N, 32>(ta, tb, a, c, bmn, atmem, s);
    case 64: return diag_nk<N, 64>(ta, tb, a, c, bmn, atmem, s);
    case 128: return diag_nk<N, 128>(ta, tb, a, c, bmn, atmem, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_diag_gemm(int n, int k, const CUtensorMap& ta, const CUtensorMap& tb, const void* a, float* c,
                             bool bmn, bool atmem, cudaStream_t s) {
  switch (n) {
    case 32: return diag_n<32>(k, ta, tb, a, c, bmn, atmem, s);
    case 64: return diag_n<64>(k, ta, tb, a, c, bmn, atmem, s);
    case 128: return diag_n<128>(k, ta, tb, a, c, bmn, atmem, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace fl

// ------------------------------------------------------------------ pipe-rate microbenchmark
// fl_diag_pipe_rate: the measured MUFU / FMA throughput that bench.py uses as the roofline denominator of
// the MUFU-bound kernels (ex2.approx.f32, ex2.approx.ftz.bf16x2, tanh.approx.f32, FFMA2).
// One CTA per SM, 512 threads (4 warps per SM sub-partition), 8 independent dependency chains per
// thread so the pipe, not its latency, is the limit.  x <- ex2(-x) / tanh(x) stay bounded.
namespace fl {
template <int OP>
__global__ void __launch_bounds__(512, 1) pipe_rate_kernel(float* sink, int iters) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = 0.01f * (float)(threadIdx.x + j);
  uint32_t h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = pack_bf16(x[j], -x[j]);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) {
        asm volatile("{.reg .f32 t;\n\tneg.f32 t, %1;\n\tex2.approx.ftz.f32 %0, t;}" : "=f"(x[j]) : "f"(x[j]));
      } else if (OP == 1) {
        asm volatile("{.reg .b32 t;\n\txor.b32 t, %1, 0x80008000;\n\tex2.approx.ftz.bf16x2 %0, t;}"
                     : "=r"(h[j]) : "r"(h[j]));
      } else if (OP == 2) {
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x[j]));
      } else if ((j & 1) == 0) {                  // 4 independent packed pairs (x[j], x[j+1])
        ffma2(x[j], x[j + 1], x[j], x[j + 1], 0.999f, 0.998f, 1e-3f, 2e-3f);
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += x[j] + bf16_lo(h[j]);
  if (acc == 123.456f) sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

cudaError_t launch_pipe_rate(int op, int iters, int n_sms, float* sink, cudaStream_t s) {
  switch (op) {
    case 0: pipe_rate_kernel<0><<<n_sms, 512, 0, s>>>(sink, iters); break;
    case 1: pipe_rate_kernel<1><<<n_sms, 512, 0, s>>>(sink, iters); break;
    case 2: pipe_rate_kernel<2><<<n_sms, 512, 0, s>>>(sink, iters); break;
    case 3: pipe_rate_kernel<3><<<n_sms, 512, 0, s>>>(sink, iters); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
}  // namespace fl
