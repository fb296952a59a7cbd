// linear.cu -- the memory passes on either side of the attention kernel (Flashlight's
// claim to fuse "complex element-wise prologues"): a tcgen05 GEMM  y = [LN(x)] W^T + bias  whose
// prologue is a row LayerNorm of its A operand and whose epilogue adds the bias and writes any output
// strides.  Used for the Evoformer row-attention block (AF2 Alg.7, the paper's second workload P:L865):
// line 1 + 2 + 4 (m <- LN(m); q, k, v, g = Linear(m), one GEMM with N = 4 H c), line 3 (pair bias
// b = Linear(LN(z)), written head-major [H, i, j] by the strided epilogue) and line 7 (output Linear).
//
// One CTA per 128-row x N_t output tile (N_t <= 256), 160 threads:
//   warps 0-3 (thread = row = TMEM lane): LayerNorm of the landed X tile in place in shared memory (fp32
//     stats, two passes over the row, bf16 write-back in the same 128-B swizzled layout the MMA reads),
//     then the epilogue (tcgen05.ld of the accumulator, + bias, bf16, strided store);
//   warp 4: TMEM allocation; lane 0 issues the TMA loads (X: K/64 slabs of 128 rows x 64, W: K/64 slabs
//     of N_t rows x 64, 128-B swizzle) and the K/16 tcgen05.mma (M = 128, N = N_t) into TMEM.
// K <= 256 (the whole row is one tile, so the row statistics need no second kernel).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "params.h"
#include "ptx.cuh"

namespace fl {

constexpr int kLinThreads = 160;

__global__ void __launch_bounds__(kLinThreads, 1)
    linear_ln_kernel(const __grid_constant__ LinParams p, const __grid_constant__ CUtensorMap tx,
                     const __grid_constant__ CUtensorMap tw) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nkc = p.K / 64;                            // 64-column slabs
  uint8_t* sX = smem;                                  // [nkc][128 rows x 128 B]
  const int nrow_boxes = (p.NT + 127) / 128;           // W boxes are 128 rows (rows past N: TMA zero fill)
  const int wslab = nrow_boxes * 128 * 128;            // one 64-column slab of W
  uint8_t* sW = smem + nkc * 128 * 128;                // [nkc][nrow_boxes * 128 rows x 128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + nkc * wslab);
  uint64_t* x_full = bars;
  uint64_t* w_full = bars + 1;
  uint64_t* ln_done = bars + 2;
  uint64_t* acc_full = bars + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * p.NT;
  const bool ln = p.ln_g != nullptr;

  if (threadIdx.x == 0) {
    mbar_init(x_full, 1);
    mbar_init(w_full, 1);
    mbar_init(ln_done, 128);
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      tma_prefetch_desc(&tx);
      tma_prefetch_desc(&tw);
      mbar_arrive_expect_tx(x_full, nkc * 128 * 128);
      for (int c = 0; c < nkc; ++c) tma_load_5d(sX + c * 128 * 128, &tx, x_full, c * 64, m0, 0, 0, 0);
      mbar_arrive_expect_tx(w_full, nkc * wslab);
      for (int c = 0; c < nkc; ++c)
        for (int rb = 0; rb < nrow_boxes; ++rb)
          tma_load_5d(sW + c * wslab + rb * 128 * 128, &tw, w_full, c * 64, n0 + rb * 128, 0, 0, 0);
      // MMA: A = X (K-major, 128 rows), B = W (K-major, NT rows), D = TMEM [128 x NT] f32
      mbar_wait(ln ? ln_done : x_full, 0);
      mbar_wait(w_full, 0);
      tc_fence_after();
      const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)p.NT, 0);
      const uint32_t xa = smem_u32(sX), wa = smem_u32(sW);
      for (int kk = 0; kk < p.K / 16; ++kk) {
        const uint32_t cx = (kk >> 2) * 128 * 128 + (kk & 3) * 32;
        const uint32_t cw = (kk >> 2) * wslab + (kk & 3) * 32;
        umma_ss(tmem, smem_desc(xa + cx, 16, 1024, kLayoutSW128), smem_desc(wa + cw, 16, 1024, kLayoutSW128), idesc,
                kk > 0);
      }
      umma_commit(acc_full);
    }
  } else {
    const int r = threadIdx.x;                         // row within the tile == TMEM lane
    if (ln) {
      // LayerNorm of row r in place: 16-B piece pc of slab c sits at (pc ^ (r & 7)) * 16 (128-B swizzle)
      mbar_wait(x_full, 0);
      float s1 = 0.f;
      for (int c = 0; c < nkc; ++c)
#pragma unroll
        for (int pc = 0; pc < 8; ++pc) {
          const uint4 u = *reinterpret_cast<const uint4*>(sX + c * 16384 + r * 128 + ((pc ^ (r & 7)) << 4));
          const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) s1 += bf16_lo(ww[t]) + bf16_hi(ww[t]);
        }
      const float mean = s1 / (float)p.K;
      float s2 = 0.f;
      for (int c = 0; c < nkc; ++c)
#pragma unroll
        for (int pc = 0; pc < 8; ++pc) {
          const uint4 u = *reinterpret_cast<const uint4*>(sX + c * 16384 + r * 128 + ((pc ^ (r & 7)) << 4));
          const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float d0 = bf16_lo(ww[t]) - mean, d1 = bf16_hi(ww[t]) - mean;
            s2 = fmaf(d0, d0, fmaf(d1, d1, s2));
          }
        }
      const float rstd = rsqrtf(s2 / (float)p.K + p.eps);
      for (int c = 0; c < nkc; ++c)
#pragma unroll
        for (int pc = 0; pc < 8; ++pc) {
          uint4* a = reinterpret_cast<uint4*>(sX + c * 16384 + r * 128 + ((pc ^ (r & 7)) << 4));
          const uint4 u = *a;
          const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
          uint32_t o[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int k = c * 64 + pc * 8 + 2 * t;
            const float y0 = fmaf((bf16_lo(ww[t]) - mean) * rstd, __ldg(p.ln_g + k), p.ln_b ? __ldg(p.ln_b + k) : 0.f);
            const float y1 =
                fmaf((bf16_hi(ww[t]) - mean) * rstd, __ldg(p.ln_g + k + 1), p.ln_b ? __ldg(p.ln_b + k + 1) : 0.f);
            o[t] = pack_bf16(y0, y1);
          }
          *a = make_uint4(o[0], o[1], o[2], o[3]);
        }
      fence_proxy_async_smem();                        // generic stores -> the tensor core's reads
      mbar_arrive(ln_done);
    }
    // ---- epilogue: row m0 + r, columns [n0, n0 + NT)
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int m = m0 + r;
    const bool row_ok = m < p.M;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    __nv_bfloat16* yr = static_cast<__nv_bfloat16*>(p.y) + (int64_t)(row_ok ? m : 0) * p.ys_m;
    const bool vec = p.ys_n == 1 && (reinterpret_cast<uintptr_t>(p.y) % 16 == 0) && (p.ys_m % 8 == 0);
    for (int c = 0; c < p.NT; c += 32) {
      uint32_t acc[32];
      tmem_ld32(tmem + lane_base + c, acc);           // every lane loads (.sync.aligned)
      tmem_wait_ld();
      float f[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int n = n0 + c + t;
        f[t] = __uint_as_float(acc[t]) + ((p.bias && n < p.N) ? __ldg(p.bias + n) : 0.f);
      }
      if (!row_ok) continue;
      if (vec && c + 32 <= p.NT && n0 + c + 32 <= p.N) {
        uint4* yp = reinterpret_cast<uint4*>(yr + n0 + c);
#pragma unroll
        for (int t8 = 0; t8 < 4; ++t8)
          yp[t8] = make_uint4(pack_bf16(f[8 * t8], f[8 * t8 + 1]), pack_bf16(f[8 * t8 + 2], f[8 * t8 + 3]),
                              pack_bf16(f[8 * t8 + 4], f[8 * t8 + 5]), pack_bf16(f[8 * t8 + 6], f[8 * t8 + 7]));
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (c + t < p.NT && n0 + c + t < p.N) yr[(int64_t)(n0 + c + t) * p.ys_n] = __float2bfloat16_rn(f[t]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 4) tmem_dealloc<256>(tmem);
}

int linear_smem_bytes(int K, int NT) { return (K / 64) * 128 * 128 + (K / 64) * ((NT + 127) / 128) * 128 * 128 + 64 + 1024; }

cudaError_t launch_linear(const LinParams& p, const CUtensorMap& tx, const CUtensorMap& tw, cudaStream_t stream) {
  const int smem = linear_smem_bytes(p.K, p.NT);
  cudaError_t e = cudaFuncSetAttribute(linear_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((p.M + 127) / 128), (unsigned)((p.N + p.NT - 1) / p.NT));
  linear_ln_kernel<<<grid, kLinThreads, smem, stream>>>(p, tx, tw);
  return cudaGetLastError();
}

}  // namespace fl
