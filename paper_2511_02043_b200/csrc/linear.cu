// linear.cu -- the memory passes on either side of the attention kernel (Flashlight's
// claim to fuse "complex element-wise prologues"): a tcgen05 GEMM  y = [LN(x)] W^T + bias  whose
// prologue is a row LayerNorm of its A operand and whose epilogue adds the bias and writes any output
// strides.  Used for the Evoformer row-attention block (AF2 Alg.7, the paper's second workload P:L865):
// line 1 + 2 + 4 (m <- LN(m); q, k, v, g = Linear(m), one GEMM with N = 4 H c), line 3 (pair bias
// b = Linear(LN(z)), written head-major [H, i, j] by the strided epilogue) and line 7 (output Linear).
//
// One CTA per 128-row block of x (X read from HBM and normalised ONCE), looping over the output column
// tiles of N_t <= 128 (W tiles streamed through a double buffer from L2, two TMEM accumulators so the
// epilogue of tile n overlaps the MMAs of tile n + 1), 192 threads:
//   warps 0-3 (thread = row = TMEM lane): LayerNorm of the landed X tile in place in shared memory (fp32
//     stats, two passes over the row, bf16 write-back in the same 128-B swizzled layout the MMA reads),
//     then per column tile the epilogue (tcgen05.ld of the accumulator, + bias, bf16, strided store);
//   warp 4 (lane 0): TMA loads (X: K/64 slabs of 128 rows x 64; W: K/64 slabs of 128 rows x 64 per column
//     tile, 128-B swizzle), TMEM allocation;
//   warp 5 (lane 0): K/16 tcgen05.mma (M = 128, N = N_t) per column tile into accumulator nt & 1.
// K <= 256 (the whole row is one tile, so the row statistics need no second kernel).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "params.h"
#include "ptx.cuh"

namespace fl {

constexpr int kLinThreads = 320;     // warps 0-3: rows [0, 128), 4: TMA, 5: MMA, 6-9: rows [128, 256)
constexpr int kLinNT = 64;           // output columns per tile (TMEM accumulator width)

// One CTA per 256 rows of x (two 128-row halves: every W tile brought into shared memory serves both, so
// W -- re-read from L2 by every CTA -- moves half as often as with 128-row CTAs), 64-column output tiles,
// W double-buffered, two TMEM accumulators per half (the epilogue of tile n overlaps the MMAs of n + 1).
__global__ void __launch_bounds__(kLinThreads, 1)
    linear_ln_kernel(const __grid_constant__ LinParams p, const __grid_constant__ CUtensorMap tx,
                     const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap ty, int y_tma) {
  (void)ty;
  (void)y_tma;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nkc = p.K / 64;                            // 64-column slabs
  constexpr int kXSlab = 128 * 128;                    // 128 X rows x 128 B
  constexpr int kWSlab = kLinNT * 128;                 // 64 W rows (rows past N: TMA zero fill) x 128 B
  uint8_t* sX = smem;                                  // [2 halves][nkc][kXSlab]
  uint8_t* sW = smem + 2 * nkc * kXSlab;               // [2][nkc][kWSlab]
  float* sBias = reinterpret_cast<float*>(sW + 2 * nkc * kWSlab);   // [2][64]: the bias of tile nt (parity nt & 1)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBias + 2 * kLinNT);
  uint64_t* x_full = bars;
  uint64_t* ln_done = bars + 1;
  uint64_t* w_full = bars + 2;                         // [2]
  uint64_t* w_empty = bars + 4;                        // [2]
  uint64_t* acc_full = bars + 6;                       // [2]
  uint64_t* acc_empty = bars + 8;                      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 256;
  const int n_nt = (p.N + p.NT - 1) / p.NT;
  const bool ln = p.ln_g != nullptr;

  if (threadIdx.x == 0) {
    mbar_init(x_full, 1);
    mbar_init(ln_done, 256);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 256);
    }
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<4 * kLinNT>(tmem_slot);    // accumulator (half h, buffer b) at (2 h + b) * 64
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {                                   // ---- TMA producer
      tma_prefetch_desc(&tx);
      tma_prefetch_desc(&tw);
      mbar_arrive_expect_tx(x_full, 2 * nkc * kXSlab);
      for (int hf = 0; hf < 2; ++hf)                   // rows past M: TMA zero fill
        for (int c = 0; c < nkc; ++c)
          tma_load_5d(sX + (hf * nkc + c) * kXSlab, &tx, x_full, c * 64, m0 + 128 * hf, 0, 0, 0);
      for (int nt = 0; nt < n_nt; ++nt) {
        const int b = nt & 1;
        if (nt >= 2) mbar_wait(&w_empty[b], ((nt >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&w_full[b], nkc * kWSlab);
        for (int c = 0; c < nkc; ++c)
          tma_load_5d(sW + (b * nkc + c) * kWSlab, &tw, &w_full[b], c * 64, nt * p.NT, 0, 0, 0);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {                                   // ---- MMA issuer: A = X half, B = W tile (both K-major)
      mbar_wait(ln ? ln_done : x_full, 0);
      tc_fence_after();
      const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)p.NT, 0);
      const uint32_t xa = smem_u32(sX), wa = smem_u32(sW);
      for (int nt = 0; nt < n_nt; ++nt) {
        const int b = nt & 1;
        mbar_wait(&w_full[b], (nt >> 1) & 1);
        if (nt >= 2) mbar_wait(&acc_empty[b], ((nt >> 1) - 1) & 1);
        tc_fence_after();
        for (int hf = 0; hf < 2; ++hf)
          for (int kk = 0; kk < p.K / 16; ++kk) {
            const uint32_t cx = (hf * nkc + (kk >> 2)) * kXSlab + (kk & 3) * 32;
            const uint32_t cw = (b * nkc + (kk >> 2)) * kWSlab + (kk & 3) * 32;
            umma_ss(tmem + (2 * hf + b) * kLinNT, smem_desc(xa + cx, 16, 1024, kLayoutSW128),
                    smem_desc(wa + cw, 16, 1024, kLayoutSW128), idesc, kk > 0);
          }
        umma_commit(&w_empty[b]);
        umma_commit(&acc_full[b]);
      }
    }
  } else {
    const int hf = warp >= 6 ? 1 : 0;                  // row half
    const int r = 32 * (warp & 3) + lane;              // row within the half == TMEM lane
    uint8_t* sXh = sX + hf * nkc * kXSlab;
    if (ln) {
      // LayerNorm of row r in place: 16-B piece pc of slab c sits at (pc ^ (r & 7)) * 16 (128-B swizzle)
      mbar_wait(x_full, 0);
      float s1 = 0.f;
      for (int c = 0; c < nkc; ++c)
#pragma unroll
        for (int pc = 0; pc < 8; ++pc) {
          const uint4 u = *reinterpret_cast<const uint4*>(sXh + c * kXSlab + r * 128 + ((pc ^ (r & 7)) << 4));
          const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) s1 += bf16_lo(ww[t]) + bf16_hi(ww[t]);
        }
      const float mean = s1 / (float)p.K;
      float s2 = 0.f;
      for (int c = 0; c < nkc; ++c)
#pragma unroll
        for (int pc = 0; pc < 8; ++pc) {
          const uint4 u = *reinterpret_cast<const uint4*>(sXh + c * kXSlab + r * 128 + ((pc ^ (r & 7)) << 4));
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
          uint4* a = reinterpret_cast<uint4*>(sXh + c * kXSlab + r * 128 + ((pc ^ (r & 7)) << 4));
          const uint4 u = *a;
          const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
          uint32_t o[4];
          const int k8 = c * 64 + pc * 8;              // gamma / beta of these 8 columns: 4 vector loads
          const float4 g0 = __ldg(reinterpret_cast<const float4*>(p.ln_g + k8));
          const float4 g1 = __ldg(reinterpret_cast<const float4*>(p.ln_g + k8 + 4));
          const float4 b0 = p.ln_b ? __ldg(reinterpret_cast<const float4*>(p.ln_b + k8)) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 b1 = p.ln_b ? __ldg(reinterpret_cast<const float4*>(p.ln_b + k8 + 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float y0 = fmaf((bf16_lo(ww[t]) - mean) * rstd, gg[2 * t], bb[2 * t]);
            const float y1 = fmaf((bf16_hi(ww[t]) - mean) * rstd, gg[2 * t + 1], bb[2 * t + 1]);
            o[t] = pack_bf16(y0, y1);
          }
          *a = make_uint4(o[0], o[1], o[2], o[3]);
        }
      fence_proxy_async_smem();                        // generic stores -> the tensor core's reads
      mbar_arrive(ln_done);
    }
    // ---- epilogue per column tile: row m0 + 128 hf + r, columns [n0, n0 + NT)
    const int m = m0 + 128 * hf + r;
    const bool row_ok = m < p.M;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    __nv_bfloat16* yr = static_cast<__nv_bfloat16*>(p.y) + (int64_t)(row_ok ? m : 0) * p.ys_m;
    const bool vec = p.ys_n == 1 && (reinterpret_cast<uintptr_t>(p.y) % 16 == 0) && (p.ys_m % 8 == 0);
    // the tile's bias in shared memory: thread r < 64 of the first half fetches column r of tile nt + 1 while
    // tile nt is processed (a per-chunk global load stalled the epilogue on its latency: 19 % of the samples)
    const bool bias_thread = hf == 0 && r < p.NT;
    auto bias_of = [&](int nt2) {
      const int n = nt2 * p.NT + r;
      return (bias_thread && p.bias && n < p.N) ? __ldg(p.bias + n) : 0.f;
    };
    if (hf == 0 && r < kLinNT) sBias[r] = bias_of(0);
    float bias_next = n_nt > 1 ? bias_of(1) : 0.f;
    named_bar_sync(2, 256);
    for (int nt = 0; nt < n_nt; ++nt) {
      const int b = nt & 1, n0 = nt * p.NT;
      const float* sb = sBias + b * kLinNT;
      mbar_wait(&acc_full[b], (nt >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < p.NT; c += 32) {
        uint32_t acc[32];
        tmem_ld32(tmem + lane_base + (2 * hf + b) * kLinNT + c, acc);   // every lane loads (.sync.aligned)
        tmem_wait_ld();
        float f[32];
#pragma unroll
        for (int t4 = 0; t4 < 8; ++t4) {
          const float4 bb = *reinterpret_cast<const float4*>(sb + c + 4 * t4);   // broadcast
          f[4 * t4] = __uint_as_float(acc[4 * t4]) + bb.x;
          f[4 * t4 + 1] = __uint_as_float(acc[4 * t4 + 1]) + bb.y;
          f[4 * t4 + 2] = __uint_as_float(acc[4 * t4 + 2]) + bb.z;
          f[4 * t4 + 3] = __uint_as_float(acc[4 * t4 + 3]) + bb.w;
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
      tc_fence_before();
      mbar_arrive(&acc_empty[b]);                      // the accumulator may take tile nt + 2
      if (nt + 1 < n_nt) {                             // publish tile nt + 1's bias, fetch tile nt + 2's
        if (hf == 0 && r < kLinNT) sBias[((nt + 1) & 1) * kLinNT + r] = bias_next;
        bias_next = nt + 2 < n_nt ? bias_of(nt + 2) : 0.f;
        named_bar_sync(2, 256);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 4) tmem_dealloc<4 * kLinNT>(tmem);
}

int linear_smem_bytes(int K) { return 2 * (K / 64) * 128 * 128 + 2 * (K / 64) * kLinNT * 128 + 2 * kLinNT * 4 + 128 + 1024; }
int linear_nt_max() { return kLinNT; }
int linear_rows_per_cta() { return 256; }

cudaError_t launch_linear(const LinParams& p, const CUtensorMap& tx, const CUtensorMap& tw, const CUtensorMap& ty,
                          int y_tma, cudaStream_t stream) {
  const int smem = linear_smem_bytes(p.K);
  cudaError_t e = cudaFuncSetAttribute(linear_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  linear_ln_kernel<<<(unsigned)((p.M + 255) / 256), kLinThreads, smem, stream>>>(p, tx, tw, ty, y_tma);
  return cudaGetLastError();
}

}  // namespace fl
