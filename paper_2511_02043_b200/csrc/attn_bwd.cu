// attn_bwd.cu -- bf16 backward of the fused attention forward on the 5th-generation tensor cores
// (the training half of the same attention program, which Flashlight hands to
// AOTAutograd as a forward and a backward graph, §2.4).  Given Q, K, V, O, dO and the forward's
// natural-log LSE (G19), with s = score_mod(scale QK^T) and P = exp(s - LSE) (no online softmax: the LSE
// is known):
//     Dvec_q = <dO_q, O_q>                                  (bwd_dvec_kernel)
//     dV_k   = sum_q P_qk dO_q
//     dS_qk  = P_qk (<dO_q, V_k> - Dvec_q) * (softcap: 1 - (s_qk / cap)^2)
//     dK_k   = scale sum_q dS_qk Q_q,   dQ_q = scale sum_k dS_qk K_k
// Two tcgen05 kernels, each a 128-row tile of TMEM lanes with TMA-fed operands (the forward's tensor
// maps, 128-B swizzle) and one softmax-like warpgroup (thread = TMEM lane):
//  * bwd_dkdv_kernel: CTA = one 128-key tile of one (b, kv head); walks the query tiles (of every query
//    head of its GQA group) whose mask interval meets the tile:  S^T = K Q^T and dP^T = V dO^T (SS),
//    P^T and dS^T (bf16) written back to TMEM, dV += P^T dO and dK += dS^T Q (TS, P / dS from TMEM).
//  * bwd_dq_kernel: CTA = one 128-query tile of one (b, head); walks its KV tiles: S = Q K^T,
//    dP = dO V^T, dS to TMEM, dQ += dS K.
// TMEM columns (dkdv): S^T [0,128) with P^T (bf16) at [64,128) and dS^T at [0,64); dP^T [128,256);
// dV [256, 256+D); dK [256+D, 256+2D).  (dq): S [0,128) with dS at [64,128); dP [128,256); dQ [256,256+D).
// No atomics: every output element has one writer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "masks.cuh"
#include "params.h"
#include "ptx.cuh"

namespace fl {

constexpr float kBwdLog2e = 1.4426950408889634f;
// two compute warpgroups (warps 0-7; each takes 64 of a tile's 128 columns), TMA warp 8, MMA warp 9
constexpr int kBwdThreads = 320;

// ---------------------------------------------------------------- Dvec = rowsum(dO * O)
// one warp per output row, 16-byte loads; dvec [B, G, Hq, Sq] f32 contiguous
__global__ void __launch_bounds__(256) bwd_dvec_kernel(const AttnParams p, const __nv_bfloat16* __restrict__ dout,
                                                      Strided5 dos, float* __restrict__ dvec) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t n_rows = (int64_t)p.B * p.G * p.Hq * p.Sq;
  if (row >= n_rows) return;
  const int q = (int)(row % p.Sq);
  const int64_t bgh = row / p.Sq;
  const int h = (int)(bgh % p.Hq), g = (int)((bgh / p.Hq) % p.G), b = (int)(bgh / ((int64_t)p.Hq * p.G));
  const __nv_bfloat16* o = static_cast<const __nv_bfloat16*>(p.o) + b * p.os.b + g * p.os.g + h * p.os.h + q * p.os.s;
  const __nv_bfloat16* d = dout + b * dos.b + g * dos.g + h * dos.h + q * dos.s;
  float acc = 0.f;
  for (int c = lane * 8; c < p.Dv; c += 256) {
    const uint4 uo = *reinterpret_cast<const uint4*>(o + c), ud = *reinterpret_cast<const uint4*>(d + c);
    const uint32_t wo[4] = {uo.x, uo.y, uo.z, uo.w}, wd[4] = {ud.x, ud.y, ud.z, ud.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      acc = fmaf(bf16_lo(wo[t]), bf16_lo(wd[t]), acc);
      acc = fmaf(bf16_hi(wo[t]), bf16_hi(wd[t]), acc);
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) dvec[row] = acc;
}

// ---------------------------------------------------------------- sigmoid gate (reading G9, AF2 Alg.7 line 6)
// out = s(g) * A:  dA = dO * s(g) (written as the dO the tcgen05 kernels read, contiguous [B,G,Hq,Sq,Dv]),
// dg = dO * out * (1 - s(g))  (= dO * A * s (1 - s), no division by s), Dvec = rowsum(dA * A) = rowsum(dO * out).
// One warp per output row, 8 elements per lane and step.
// Mul gate (O = G * A): dA = dO * G, dg = dO * A with A the ungated output the host recomputed into `aun`
// (contiguous [rows, Dv]; no division by G), Dvec = rowsum(dO * out) as above.
template <bool MUL>
__global__ void __launch_bounds__(256) bwd_gate_kernel(const AttnParams p, const __nv_bfloat16* __restrict__ dout,
                                                      Strided5 dos, __nv_bfloat16* __restrict__ da,
                                                      __nv_bfloat16* __restrict__ dgate, Strided5 dgs,
                                                      float* __restrict__ dvec, const __nv_bfloat16* __restrict__ aun) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t n_rows = (int64_t)p.B * p.G * p.Hq * p.Sq;
  if (row >= n_rows) return;
  const int q = (int)(row % p.Sq);
  const int64_t bgh = row / p.Sq;
  const int h = (int)(bgh % p.Hq), g = (int)((bgh / p.Hq) % p.G), b = (int)(bgh / ((int64_t)p.Hq * p.G));
  const __nv_bfloat16* o = static_cast<const __nv_bfloat16*>(p.o) + b * p.os.b + g * p.os.g + h * p.os.h + q * p.os.s;
  const __nv_bfloat16* d = dout + b * dos.b + g * dos.g + h * dos.h + q * dos.s;
  const __nv_bfloat16* gl = static_cast<const __nv_bfloat16*>(p.gate) + b * p.gs.b + g * p.gs.g + h * p.gs.h + q * p.gs.s;
  __nv_bfloat16* dar = da + row * p.Dv;
  __nv_bfloat16* dgr = dgate ? dgate + b * dgs.b + g * dgs.g + h * dgs.h + q * dgs.s : nullptr;
  float acc = 0.f;
  for (int c = lane * 8; c < p.Dv; c += 256) {
    const uint4 uo = *reinterpret_cast<const uint4*>(o + c), ud = *reinterpret_cast<const uint4*>(d + c),
                ug = *reinterpret_cast<const uint4*>(gl + c);
    const uint32_t wo[4] = {uo.x, uo.y, uo.z, uo.w}, wd[4] = {ud.x, ud.y, ud.z, ud.w}, wg[4] = {ug.x, ug.y, ug.z, ug.w};
    uint32_t pa[4], pg[4];
    if constexpr (MUL) {
      const uint4 ua = *reinterpret_cast<const uint4*>(aun + row * p.Dv + c);
      const uint32_t wa[4] = {ua.x, ua.y, ua.z, ua.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float d0 = bf16_lo(wd[t]), d1 = bf16_hi(wd[t]);
        acc = fmaf(bf16_lo(wo[t]), d0, fmaf(bf16_hi(wo[t]), d1, acc));
        pa[t] = pack_bf16(d0 * bf16_lo(wg[t]), d1 * bf16_hi(wg[t]));
        pg[t] = pack_bf16(d0 * bf16_lo(wa[t]), d1 * bf16_hi(wa[t]));
      }
      *reinterpret_cast<uint4*>(dar + c) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
      if (dgr) *reinterpret_cast<uint4*>(dgr + c) = make_uint4(pg[0], pg[1], pg[2], pg[3]);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float o0 = bf16_lo(wo[t]), o1 = bf16_hi(wo[t]), d0 = bf16_lo(wd[t]), d1 = bf16_hi(wd[t]);
        const float s0 = 1.f / (1.f + __expf(-bf16_lo(wg[t]))), s1 = 1.f / (1.f + __expf(-bf16_hi(wg[t])));
        acc = fmaf(o0, d0, fmaf(o1, d1, acc));
        pa[t] = pack_bf16(d0 * s0, d1 * s1);
        pg[t] = pack_bf16(d0 * o0 * (1.f - s0), d1 * o1 * (1.f - s1));
      }
      *reinterpret_cast<uint4*>(dar + c) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
      if (dgr && p.grad_accum) {                        // second diff map: add to the first map's dgate
        const uint4 u = *reinterpret_cast<const uint4*>(dgr + c);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float o0 = bf16_lo(wo[t]), o1 = bf16_hi(wo[t]), d0 = bf16_lo(wd[t]), d1 = bf16_hi(wd[t]);
          const float s0 = 1.f / (1.f + __expf(-bf16_lo(wg[t]))), s1 = 1.f / (1.f + __expf(-bf16_hi(wg[t])));
          pg[t] = pack_bf16(fmaf(d0 * o0, 1.f - s0, bf16_lo(w[t])), fmaf(d1 * o1, 1.f - s1, bf16_hi(w[t])));
        }
        *reinterpret_cast<uint4*>(dgr + c) = make_uint4(pg[0], pg[1], pg[2], pg[3]);
      } else if (dgr) {
        *reinterpret_cast<uint4*>(dgr + c) = make_uint4(pg[0], pg[1], pg[2], pg[3]);
      }
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) dvec[row] = acc;
}

// Differential attention (Listing 4; reading G8), O = A_0 - lambda_h A_1: the backward runs the
// single-map kernels once per map (host.cu) with the map-1 seed dO_1 = -lambda_h dO; this kernel writes that
// seed (contiguous, [rows, Dv]) and dL/dlambda_h = -sum_{b,g,q,d} dO * o_1, o_1 the recomputed map-1 output
// (gated when the forward is: o_1 = gate' A_1).  One warp per row; the block's 8 rows share one head when
// they lie in one (b, g, h) (S_q % 8 == 0), then one atomic per block.
__global__ void __launch_bounds__(256) diff_bwd_seed_kernel(const AttnParams p, const __nv_bfloat16* __restrict__ dout,
                                                           Strided5 dos, const __nv_bfloat16* __restrict__ o1,
                                                           __nv_bfloat16* __restrict__ do1, float* __restrict__ dlambda) {
  __shared__ float part[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + warp;
  const int64_t n_rows = (int64_t)p.B * p.G * p.Hq * p.Sq;
  float acc = 0.f;
  int h = 0;
  if (row < n_rows) {
    const int q = (int)(row % p.Sq);
    const int64_t bgh = row / p.Sq;
    h = (int)(bgh % p.Hq);
    const int g = (int)((bgh / p.Hq) % p.G), b = (int)(bgh / ((int64_t)p.Hq * p.G));
    const float c = -diff_lambda(p, h);
    const __nv_bfloat16* d = dout + b * dos.b + g * dos.g + h * dos.h + q * dos.s;
    const __nv_bfloat16* o = o1 + row * p.Dv;
    __nv_bfloat16* out = do1 + row * p.Dv;
    for (int col = lane * 8; col < p.Dv; col += 256) {
      const uint4 ud = *reinterpret_cast<const uint4*>(d + col), uo = *reinterpret_cast<const uint4*>(o + col);
      const uint32_t wd[4] = {ud.x, ud.y, ud.z, ud.w}, wo[4] = {uo.x, uo.y, uo.z, uo.w};
      uint32_t pd[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float d0 = bf16_lo(wd[t]), d1 = bf16_hi(wd[t]);
        acc = fmaf(d0, bf16_lo(wo[t]), fmaf(d1, bf16_hi(wo[t]), acc));
        pd[t] = pack_bf16(c * d0, c * d1);
      }
      *reinterpret_cast<uint4*>(out + col) = make_uint4(pd[0], pd[1], pd[2], pd[3]);
    }
  }
  if (!dlambda) return;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  const int64_t r0 = (int64_t)blockIdx.x * 8, r1 = r0 + 7;
  const bool one_head = r1 < n_rows && r0 / p.Sq == r1 / p.Sq;
  if (!one_head) {
    if (lane == 0 && row < n_rows) atomicAdd(dlambda + h, -acc);
    return;
  }
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w];
    atomicAdd(dlambda + h, -t);
  }
}

// Zero a strided [B, G, H, S, D] bf16 view (contiguous last dim): the gradients the kernels never visit
// when the problem has no queries (dK, dV) or no keys (dQ, dgate).  One thread per 8 elements.
__global__ void zero_rows_kernel(__nv_bfloat16* __restrict__ dst, Strided5 ds, int B, int G, int H, int S, int D) {
  const int64_t n8 = (int64_t)B * G * H * S * (D / 8);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(e % (D / 8));
    const int64_t row = e / (D / 8);
    const int q = (int)(row % S);
    const int64_t bgh = row / S;
    const int h = (int)(bgh % H), g = (int)((bgh / H) % G), b = (int)(bgh / ((int64_t)H * G));
    *reinterpret_cast<uint4*>(dst + b * ds.b + g * ds.g + h * ds.h + q * ds.s + c8 * 8) = make_uint4(0u, 0u, 0u, 0u);
  }
}

template <bool B>
struct BoolTag {
  static constexpr bool value = B;
};

// ---------------------------------------------------------------- shared configuration
template <int D>
struct BwdCfg {
  static constexpr int CH = D >= 64 ? 64 : 32;       // bf16 per swizzle row (128 B, or 64 B at D = 32)
  static constexpr int SWB = CH * 2;
  static constexpr int NCH = D / CH;
  static constexpr int CHUNK_BYTES = 128 * SWB;      // 128 rows x SWB bytes
  static constexpr int TILE_BYTES = 128 * D * 2;
  static constexpr uint32_t LAYOUT = SWB == 128 ? kLayoutSW128 : kLayoutSW64;
  static constexpr int SBO = 8 * SWB;
  static constexpr uint32_t IDESC_NN = idesc_bf16_f32(128, 128, 0);   // [128 x D] . [128 x D]^T (both K-major)
  static constexpr uint32_t IDESC_ND = idesc_bf16_f32(128, D, 1);     // TMEM A [128 x 128] . smem B [128 x D] MN-major
  static constexpr int NST = 2;                      // ring stages (pairs of tiles)
  // dK/dV kernel: 64-query items (Q and dO half tiles), two in flight (one per compute warpgroup)
  static constexpr int HCHUNK = 64 * SWB;            // 64 rows x SWB bytes
  static constexpr int HALF_BYTES = 64 * D * 2;
  static constexpr int NSTH = 4;                     // ring stages of (Q half, dO half)
  static constexpr uint32_t IDESC_N64 = idesc_bf16_f32(128, 64, 0);  // K [128 x D] . Q_half [64 x D]^T
  static constexpr int KV_RING = 2 * TILE_BYTES;
  static constexpr int KV_ROWS = KV_RING + NSTH * 2 * HALF_BYTES;
  static constexpr int KV_BAR = KV_ROWS + NSTH * 256 * 4;          // per stage: lse, dvec, lo, hi of 64 rows
  static constexpr int KV_SMEM = KV_BAR + 256 + 1024;
  // smem: two resident tiles | NST x two streamed tiles | per-stage LSE / Dvec rows (dkdv) | barriers
  static constexpr int SMEM_FIXED = 0;
  static constexpr int SMEM_RING = 2 * TILE_BYTES;
  static constexpr int SMEM_ROWS = SMEM_RING + NST * 2 * TILE_BYTES;
  static constexpr int SMEM_BAR = SMEM_ROWS + NST * 4 * 128 * 4;   // per stage: lse, dvec, lo, hi of 128 rows
  static constexpr int SMEM_TOTAL = SMEM_BAR + 128 + 1024;
};

// K-major 128 x D tile as UMMA operand, K step kk (16 elements)
template <int D>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t base, int kk) {
  using C = BwdCfg<D>;
  const uint32_t off = (kk * 16 / C::CH) * C::CHUNK_BYTES + (kk * 16 % C::CH) * 2;
  return smem_desc(base + off, 16, C::SBO, C::LAYOUT);
}
// K-major / MN-major descriptors for a tile whose 64-column chunks are `chunk` bytes apart (64-row half tiles)
template <int D>
__device__ __forceinline__ uint64_t kmajor_desc_c(uint32_t base, int kk, uint32_t chunk) {
  using C = BwdCfg<D>;
  return smem_desc(base + (kk * 16 / C::CH) * chunk + (kk * 16 % C::CH) * 2, 16, C::SBO, C::LAYOUT);
}
template <int D>
__device__ __forceinline__ uint64_t mnmajor_desc_c(uint32_t base, int kk, uint32_t chunk) {
  using C = BwdCfg<D>;
  return smem_desc(base + kk * 16 * C::SWB, chunk, C::SBO, C::LAYOUT);
}
// the same tile read as an MN-major B operand [K = its 128 rows, N = D], K step kk
template <int D>
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t base, int kk) {
  using C = BwdCfg<D>;
  return smem_desc(base + kk * 16 * C::SWB, C::CHUNK_BYTES, C::SBO, C::LAYOUT);
}

// Per-element score of the forward (natural units) for query row q (absolute q_abs), key k, head h:
// scale s (+ ALiBi) (-> softcap), plus the softcap derivative factor.
template <int MOD>
__device__ __forceinline__ float bwd_score(const AttnParams& p, float s_raw, float slope, int k, int q_abs, float& ft,
                                           float bias = 0.f) {
  float x = s_raw * p.scale;
  if (MOD == MOD_ALIBI) x = fmaf(slope, (float)(k - q_abs), x);
  x += bias;                                         // additive bias before the softcap (G16)
  ft = 1.f;
  if (MOD == MOD_SOFTCAP) {
    const float t = tanh_approx(x / p.softcap);
    ft = 1.f - t * t;
    x = p.softcap * t;
  }
  return x;
}

// additive score bias of (b, g, h, q, k) (bf16 or f32, any strides incl. broadcast), 0 when absent
__device__ __forceinline__ float bias_at(const AttnParams& p, int b, int g, int h, int q, int k) {
  if (!p.bias) return 0.f;
  const int64_t off = b * p.bs.b + g * p.bs.g + (int64_t)h * p.bs.h + (int64_t)q * p.bs.s + (int64_t)k * p.bs.d;
  return p.bias_dtype == 1 ? __ldg(static_cast<const float*>(p.bias) + off)
                           : __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(p.bias) + off));
}

__device__ __forceinline__ float head_slope(const AttnParams& p, int h) {
  return p.alibi ? p.alibi[h] : exp2f(-8.f * (float)(h + 1) / (float)p.Hq);
}

// ================================================================ dK / dV
// grid = B * G * Hkv * n_kvtile, 320 threads: warps 0-7 compute (thread = key row), warp 8 TMA producer,
// warp 9 MMA issuer + TMEM allocator.  Items are 64-query halves of the needed query tiles; warpgroup w
// takes items e = w (mod 2) in TMEM slot w (S^T [0, 64) and dP^T [64, 128) of slot w's 128 columns, P^T
// and dS^T written back over S^T), so the MMAs of item e + 1 (the other slot) run while warpgroup w works
// on item e -- the forward's ping-pong: S^T(e+2), dP^T(e+2) are issued right after dV(e), dK(e) consumed
// slot w.
template <int D, int MOD, bool BIAS>
__global__ void __launch_bounds__(kBwdThreads, 1)
    bwd_dkdv_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ TmaMaps maps,
                    const __grid_constant__ CUtensorMap tq64, const __grid_constant__ CUtensorMap tdo64,
                    const float* __restrict__ lse_g, Strided5 ls, const float* __restrict__ dvec,
                    __nv_bfloat16* __restrict__ dk, Strided5 dks, __nv_bfloat16* __restrict__ dv, Strided5 dvs) {
  using C = BwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;
  uint8_t* sV = smem + C::TILE_BYTES;
  uint8_t* sRing = smem + C::KV_RING;                // stage st: Q half, dO half
  float* sRows = reinterpret_cast<float*>(smem + C::KV_ROWS);   // stage st: lse_l2[64], dvec[64], lo[64], hi[64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::KV_BAR);
  uint64_t* kv_full = bars;
  uint64_t* full = bars + 1;                         // [NSTH]
  uint64_t* empty = full + C::NSTH;                  // [NSTH]
  uint64_t* s_full = empty + C::NSTH;                // [2] per slot / warpgroup
  uint64_t* p_full = s_full + 2;                     // [2]
  uint64_t* o_full = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int n_kt = (p.Sk + 127) / 128;
  const int kt = blockIdx.x % n_kt;
  const int hk = (blockIdx.x / n_kt) % p.Hkv;
  const int g = (blockIdx.x / (n_kt * p.Hkv)) % p.G;
  const int b = blockIdx.x / (n_kt * p.Hkv * p.G);
  const int k0 = kt * 128;
  const int n_qh = (p.Sq + 63) / 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // the 64-row query halves whose rows' key intervals meet [k0, k0 + 128)
  auto half_needed = [&](int qh) {
    const int q_first = qh * 64, q_last = min(p.Sq, q_first + 64) - 1;
    const Interval u = rows_union(p, b, q_first, q_last);
    return u.hi > k0 && u.lo < k0 + 128;
  };

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::NSTH; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 128);
    }
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t COL_DV = 256, COL_DK = 256 + D;

  if (warp == 8) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      const int gk = maps.k_bcast_g ? 0 : g, bk = maps.k_bcast_b ? 0 : b;
      const int gv = maps.v_bcast_g ? 0 : g, bv = maps.v_bcast_b ? 0 : b;
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE_BYTES);
      int krow, kb;
      kv_tile_coords(p, b, kt, bk, krow, kb);
      int vrow, vb;
      kv_tile_coords(p, b, kt, bv, vrow, vb);
      for (int c = 0; c < C::NCH; ++c) {
        tma_load_5d(sK + c * C::CHUNK_BYTES, &maps.k, kv_full, c * C::CH, krow, hk, gk, kb);
        tma_load_5d(sV + c * C::CHUNK_BYTES, &maps.v, kv_full, c * C::CH, vrow, hk, gv, vb);
      }
      const int bq = maps.q_bcast_b ? 0 : b, gq = maps.q_bcast_g ? 0 : g;
      int e = 0;
      for (int hh = hk * p.grp; hh < (hk + 1) * p.grp; ++hh)
        for (int qh = 0; qh < n_qh; ++qh) {
          if (!half_needed(qh)) continue;
          const int st = e % C::NSTH;
          if (e >= C::NSTH) mbar_wait(&empty[st], ((e / C::NSTH) - 1) & 1);
          mbar_arrive_expect_tx(&full[st], 2 * C::HALF_BYTES);
          uint8_t* dq_ = sRing + st * 2 * C::HALF_BYTES;
          for (int c = 0; c < C::NCH; ++c) {
            tma_load_5d(dq_ + c * C::HCHUNK, &tq64, &full[st], c * C::CH, qh * 64, hh, gq, bq);
            tma_load_5d(dq_ + C::HALF_BYTES + c * C::HCHUNK, &tdo64, &full[st], c * C::CH, qh * 64, hh, g, b);
          }
          ++e;
        }
    }
  } else if (warp == 9) {
    // ============================== MMA issuer ==============================
    if (lane == 0) {
      const uint32_t ka = smem_u32(sK), va = smem_u32(sV), ring = smem_u32(sRing);
      int n_items = 0;
      for (int hh = hk * p.grp; hh < (hk + 1) * p.grp; ++hh)
        for (int qh = 0; qh < n_qh; ++qh) n_items += half_needed(qh) ? 1 : 0;
      mbar_wait(kv_full, 0);
      auto issue_s = [&](int e) {                    // S^T(e) = K Q_e^T, dP^T(e) = V dO_e^T into slot e & 1
        const int st = e % C::NSTH, sl = e & 1;
        mbar_wait(&full[st], (e / C::NSTH) & 1);
        tc_fence_after();
        const uint32_t qa = ring + st * 2 * C::HALF_BYTES, doa = qa + C::HALF_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tmem + sl * 128, kmajor_desc<D>(ka, kk), kmajor_desc_c<D>(qa, kk, C::HCHUNK), C::IDESC_N64, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tmem + sl * 128 + 64, kmajor_desc<D>(va, kk), kmajor_desc_c<D>(doa, kk, C::HCHUNK), C::IDESC_N64,
                  kk > 0);
        umma_commit(&s_full[sl]);
      };
      if (n_items > 0) issue_s(0);
      if (n_items > 1) issue_s(1);
      for (int e = 0; e < n_items; ++e) {
        const int st = e % C::NSTH, sl = e & 1;
        mbar_wait(&p_full[sl], (e >> 1) & 1);
        tc_fence_after();
        const uint32_t qa = ring + st * 2 * C::HALF_BYTES, doa = qa + C::HALF_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)        // dV += P^T dO   (P^T bf16 at slot + [32, 64))
          umma_ts(tmem + COL_DV, tmem + sl * 128 + 32 + kk * 8, mnmajor_desc_c<D>(doa, kk, C::HCHUNK), C::IDESC_ND,
                  (e > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)        // dK += dS^T Q   (dS^T bf16 at slot + [0, 32))
          umma_ts(tmem + COL_DK, tmem + sl * 128 + kk * 8, mnmajor_desc_c<D>(qa, kk, C::HCHUNK), C::IDESC_ND,
                  (e > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty[st]);
        if (e + 2 < n_items) issue_s(e + 2);  // slot sl again: after dV(e), dK(e) read it (in order)
      }
      umma_commit(o_full);
    }
  } else {
    // ============================== compute (thread = key row) ==============================
    const int wg = warp >> 2;                       // warpgroup wg: items e = wg (mod 2), TMEM slot wg
    const int r = threadIdx.x & 127;                // key row == TMEM lane
    const int k = k0 + r;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col_s = wg * 128, col_dp = wg * 128 + 64;
    // MSA / key mask (G9): a masked key has P = 0 for every query -- its dK, dV rows stay 0
    const bool key_on = !p.keybits || k >= p.Sk ||
                        ((p.keybits[((int64_t)b * p.G + g) * p.keybits_words + (k >> 5)] >> (k & 31)) & 1u);
    int e = 0, ew = 0;
    for (int hh = hk * p.grp; hh < (hk + 1) * p.grp; ++hh) {
      const float slope_l2 = MOD == MOD_ALIBI ? head_slope(p, hh) : 0.f;
      for (int qh = 0; qh < n_qh; ++qh) {
        if (!half_needed(qh)) continue;
        if ((e & 1) != wg) {
          ++e;
          continue;
        }
        const int st = e % C::NSTH;
        const int q0 = qh * 64;
        // this half's rows, one per thread r < 64: LSE (log2 units), Dvec and the key interval [lo, hi) of
        // query q0 + r (rows past S_q get an empty interval: P = 0); the element loop reads them as broadcasts
        float* rl = sRows + st * 256;
        int* riv = reinterpret_cast<int*>(rl + 128);
        if (r < 64) {
          const int q = q0 + r;
          const bool ok = q < p.Sq;
          const int64_t li = (int64_t)b * ls.b + (int64_t)g * ls.g + (int64_t)hh * ls.h + (int64_t)(ok ? q : 0) * ls.s;
          rl[r] = ok ? lse_g[li] * kBwdLog2e : INFINITY;
          rl[64 + r] = ok ? dvec[(((int64_t)b * p.G + g) * p.Hq + hh) * p.Sq + q] : 0.f;
          const Interval iv = row_interval(p, b, q);
          riv[r] = ok ? iv.lo : 0;
          riv[64 + r] = ok ? iv.hi : 0;
        }
        named_bar_sync(1 + wg, 128);
        // tile class: mask-free when every row's interval covers [k0, k0 + 128) (intervals are monotone)
        const int q_last = min(p.Sq, q0 + 64) - 1;
        const Interval a0 = row_interval(p, b, q0), a1 = row_interval(p, b, q_last);
        const bool full_tile = q_last - q0 == 63 && a1.lo <= k0 && a0.hi >= k0 + 128 && k0 + 128 <= p.Sk;
        mbar_wait(&s_full[wg], ew & 1);
        tc_fence_after();
        uint32_t sv[64];
        tmem_ld32(tmem + lane_base + col_s, &sv[0]);
        tmem_ld32(tmem + lane_base + col_s + 32, &sv[32]);
        tmem_wait_ld();
        // P^T (bf16 pairs) and the softcap factor, query q0 + j = column j
        uint32_t pk[32], fk[32];
        // mask-free items (every element kept) take a loop without the per-element interval test
        auto p_loop = [&](auto fast_tag) {
          constexpr bool kFast = decltype(fast_tag)::value;
#pragma unroll
          for (int j = 0; j < 64; j += 4) {
            const float4 lse4 = *reinterpret_cast<const float4*>(rl + j);
            const float lsev[4] = {lse4.x, lse4.y, lse4.z, lse4.w};
            float pr[4], f[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int q = q0 + j + t;
              float ft;
              const bool keep = kFast || (key_on && (full_tile || (k >= riv[j + t] && k < riv[64 + j + t])));   // hi <= S_k
              const float bv = (BIAS && keep) ? bias_at(p, b, g, hh, q, k) : 0.f;
              const float s = bwd_score<MOD>(p, __uint_as_float(sv[j + t]), slope_l2, k, q + p.q_off, ft, bv);
              pr[t] = keep ? ex2(fmaf(s, kBwdLog2e, -lsev[t])) : 0.f;
              f[t] = ft;
            }
            pk[j >> 1] = pack_bf16(pr[0], pr[1]);
            pk[(j >> 1) + 1] = pack_bf16(pr[2], pr[3]);
            fk[j >> 1] = pack_bf16(f[0], f[1]);
            fk[(j >> 1) + 1] = pack_bf16(f[2], f[3]);
          }
        };
        if (full_tile && key_on)
          p_loop(BoolTag<true>{});
        else
          p_loop(BoolTag<false>{});
        tmem_st32(tmem + lane_base + col_s + 32, &pk[0]);
        // dS^T = P^T (dP^T - Dvec) * f, 32 queries at a time, into slot + [0, 32) (S^T is consumed)
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          uint32_t dp[32];
          tmem_ld32(tmem + lane_base + col_dp + c, dp);
          tmem_wait_ld();
          uint32_t ds[16];
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 dv4 = *reinterpret_cast<const float4*>(rl + 64 + c + j);
            const uint32_t pw0 = pk[(c + j) >> 1], pw1 = pk[((c + j) >> 1) + 1];
            const uint32_t fw0 = fk[(c + j) >> 1], fw1 = fk[((c + j) >> 1) + 1];
            float d0 = bf16_lo(pw0) * (__uint_as_float(dp[j]) - dv4.x);
            float d1 = bf16_hi(pw0) * (__uint_as_float(dp[j + 1]) - dv4.y);
            float d2 = bf16_lo(pw1) * (__uint_as_float(dp[j + 2]) - dv4.z);
            float d3 = bf16_hi(pw1) * (__uint_as_float(dp[j + 3]) - dv4.w);
            if (MOD == MOD_SOFTCAP) {
              d0 *= bf16_lo(fw0);
              d1 *= bf16_hi(fw0);
              d2 *= bf16_lo(fw1);
              d3 *= bf16_hi(fw1);
            }
            ds[j >> 1] = pack_bf16(d0, d1);
            ds[(j >> 1) + 1] = pack_bf16(d2, d3);
          }
          tmem_st16(tmem + lane_base + col_s + (c >> 1), ds);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[wg]);
        ++e;
        ++ew;
      }
    }
    // ---- epilogue: dK (x scale) and dV rows of this key tile
    if (e > 0) {
      mbar_wait(o_full, 0);
      tc_fence_after();
    }
    // tcgen05.ld is .sync.aligned: every lane of the warp loads, only valid key rows store
    {
      const bool k_ok = k < p.Sk;
      __nv_bfloat16* dkp = dk + b * dks.b + (int64_t)g * dks.g + (int64_t)hk * dks.h + (int64_t)(k_ok ? k : 0) * dks.s;
      __nv_bfloat16* dvp = dv + b * dvs.b + (int64_t)g * dvs.g + (int64_t)hk * dvs.h + (int64_t)(k_ok ? k : 0) * dvs.s;
      {
        const int which = wg;                         // warpgroup 0 stores dV, warpgroup 1 dK
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          if (e > 0) {
            tmem_ld32(tmem + lane_base + (which ? COL_DK : COL_DV) + c, o);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t) o[t] = 0u;
          }
          const float sc = which ? p.scale : 1.f;
          uint4* op = reinterpret_cast<uint4*>((which ? dkp : dvp) + c);
          if (k_ok && !which && p.grad_accum) {        // dV of the second diff map: add to the first map's
#pragma unroll
            for (int t8 = 0; t8 < 4; ++t8) {
              const uint4 u = op[t8];
              const uint32_t w[4] = {u.x, u.y, u.z, u.w};
              uint32_t r[4];
#pragma unroll
              for (int t = 0; t < 4; ++t)
                r[t] = pack_bf16(__uint_as_float(o[t8 * 8 + 2 * t]) + bf16_lo(w[t]),
                                 __uint_as_float(o[t8 * 8 + 2 * t + 1]) + bf16_hi(w[t]));
              op[t8] = make_uint4(r[0], r[1], r[2], r[3]);
            }
          } else if (k_ok)
#pragma unroll
          for (int t8 = 0; t8 < 4; ++t8)
            op[t8] = make_uint4(pack_bf16(__uint_as_float(o[t8 * 8 + 0]) * sc, __uint_as_float(o[t8 * 8 + 1]) * sc),
                                pack_bf16(__uint_as_float(o[t8 * 8 + 2]) * sc, __uint_as_float(o[t8 * 8 + 3]) * sc),
                                pack_bf16(__uint_as_float(o[t8 * 8 + 4]) * sc, __uint_as_float(o[t8 * 8 + 5]) * sc),
                                pack_bf16(__uint_as_float(o[t8 * 8 + 6]) * sc, __uint_as_float(o[t8 * 8 + 7]) * sc));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// ================================================================ dQ
// grid = B * G * Hq * n_qtile (query tile descending: causal's heaviest tiles first), 320 threads: warps 0-7
// compute, warp 8 TMA, warp 9 MMA + TMEM.  Items are the 64-key halves of the tile's KV tiles; warpgroup w
// takes items e = w (mod 2) in TMEM slot w (S [0, 64), dP [64, 128) of the slot, dS over S's upper half),
// so the MMAs of one item run while the other warpgroup computes (as in the dK/dV kernel).
template <int D, int MOD, bool BIAS>
__global__ void __launch_bounds__(kBwdThreads, 1)
    bwd_dq_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ TmaMaps maps,
                  const __grid_constant__ CUtensorMap tdo, const float* __restrict__ lse_g, Strided5 ls,
                  const float* __restrict__ dvec, __nv_bfloat16* __restrict__ dq, Strided5 dqs,
                  float* __restrict__ dbias, Strided5 dbs) {
  using C = BwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sDO = smem + C::TILE_BYTES;
  uint8_t* sRing = smem + C::SMEM_RING;              // stage st: K tile, V tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* q_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + C::NST;
  uint64_t* s_full = empty + C::NST;                 // [2] per slot / warpgroup
  uint64_t* p_full = s_full + 2;                     // [2]
  uint64_t* o_full = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int n_qt = (p.Sq + 127) / 128;
  const int qt = n_qt - 1 - (int)(blockIdx.x % n_qt);
  const int h = (blockIdx.x / n_qt) % p.Hq;
  const int g = (blockIdx.x / (n_qt * p.Hq)) % p.G;
  const int b = blockIdx.x / (n_qt * p.Hq * p.G);
  const int hk = h / p.grp;
  const int q0 = qt * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Interval u = rows_union(p, b, q0, min(p.Sq, q0 + 128) - 1);
  const int kt_lo = u.hi > u.lo ? u.lo / 128 : 0, kt_hi = u.hi > u.lo ? (u.hi + 127) / 128 : 0;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 128);
    }
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t COL_DQ = 256;

  if (warp == 8) {
    if (lane == 0) {
      const int bq = maps.q_bcast_b ? 0 : b, gq = maps.q_bcast_g ? 0 : g;
      mbar_arrive_expect_tx(q_full, 2 * C::TILE_BYTES);
      for (int c = 0; c < C::NCH; ++c) {
        tma_load_5d(sQ + c * C::CHUNK_BYTES, &maps.q, q_full, c * C::CH, q0, h, gq, bq);
        tma_load_5d(sDO + c * C::CHUNK_BYTES, &tdo, q_full, c * C::CH, q0, h, g, b);
      }
      const int bk = maps.k_bcast_b ? 0 : b, bv = maps.v_bcast_b ? 0 : b;
      const int gk = maps.k_bcast_g ? 0 : g, gv = maps.v_bcast_g ? 0 : g;
      for (int kt = kt_lo; kt < kt_hi; ++kt) {
        const int e = kt - kt_lo, st = e % C::NST;
        if (e >= C::NST) mbar_wait(&empty[st], ((e / C::NST) - 1) & 1);
        mbar_arrive_expect_tx(&full[st], 2 * C::TILE_BYTES);
        uint8_t* dst = sRing + st * 2 * C::TILE_BYTES;
        int krow, kb, vrow, vb;
        kv_tile_coords(p, b, kt, bk, krow, kb);
        kv_tile_coords(p, b, kt, bv, vrow, vb);
        for (int c = 0; c < C::NCH; ++c) {
          tma_load_5d(dst + c * C::CHUNK_BYTES, &maps.k, &full[st], c * C::CH, krow, hk, gk, kb);
          tma_load_5d(dst + C::TILE_BYTES + c * C::CHUNK_BYTES, &maps.v, &full[st], c * C::CH, vrow, hk, gv, vb);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      // items = 64-key halves of the KV tiles, e = 2 (kt - kt_lo) + half, in TMEM slot e & 1 (warpgroup e & 1)
      const uint32_t qa = smem_u32(sQ), doa = smem_u32(sDO), ring = smem_u32(sRing);
      const int n_items = 2 * (kt_hi - kt_lo);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int e) {                    // S = Q K_half^T, dP = dO V_half^T into slot e & 1
        const int t = e >> 1, st = t % C::NST, sl = e & 1;
        if ((e & 1) == 0) mbar_wait(&full[st], (t / C::NST) & 1);
        tc_fence_after();
        const uint32_t ka = ring + st * 2 * C::TILE_BYTES + (e & 1) * 64 * C::SWB, va = ka + C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tmem + sl * 128, kmajor_desc<D>(qa, kk), kmajor_desc_c<D>(ka, kk, C::CHUNK_BYTES), C::IDESC_N64, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_ss(tmem + sl * 128 + 64, kmajor_desc<D>(doa, kk), kmajor_desc_c<D>(va, kk, C::CHUNK_BYTES), C::IDESC_N64,
                  kk > 0);
        umma_commit(&s_full[sl]);
      };
      if (n_items > 0) issue_s(0);
      if (n_items > 1) issue_s(1);
      for (int e = 0; e < n_items; ++e) {
        const int t = e >> 1, st = t % C::NST, sl = e & 1;
        mbar_wait(&p_full[sl], (e >> 1) & 1);
        tc_fence_after();
        const uint32_t ka = ring + st * 2 * C::TILE_BYTES + (e & 1) * 64 * C::SWB;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)          // dQ += dS K_half   (dS bf16 at slot + [32, 64))
          umma_ts(tmem + COL_DQ, tmem + sl * 128 + 32 + kk * 8, mnmajor_desc_c<D>(ka, kk, C::CHUNK_BYTES),
                  C::IDESC_ND, (e > 0 || kk > 0) ? 1u : 0u);
        if (e & 1) umma_commit(&empty[st]);      // both halves of the K/V tile are done
        if (e + 2 < n_items) issue_s(e + 2);    // slot sl again, after dQ(e) read its dS (in order)
      }
      umma_commit(o_full);
    }
  } else {
    const int wg = warp >> 2;                       // warpgroup wg: items e = wg (mod 2), TMEM slot wg
    const int r = threadIdx.x & 127;
    const int q = q0 + r;
    const bool row_ok = q < p.Sq;
    const int q_abs = q + p.q_off;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col_s = wg * 128, col_dp = wg * 128 + 64;
    const float slope_l2 = MOD == MOD_ALIBI ? head_slope(p, h) : 0.f;
    const float lse_l2 =
        row_ok ? lse_g[(int64_t)b * ls.b + (int64_t)g * ls.g + (int64_t)h * ls.h + (int64_t)q * ls.s] * kBwdLog2e : INFINITY;
    const float dvr = row_ok ? dvec[(((int64_t)b * p.G + g) * p.Hq + h) * p.Sq + q] : 0.f;
    const uint32_t* kbits = p.keybits ? p.keybits + ((int64_t)b * p.G + g) * p.keybits_words : nullptr;
    const Interval iv = row_interval(p, b, q);
    const int n_items = 2 * (kt_hi - kt_lo);
    int ew = 0;
    for (int e = wg; e < n_items; e += 2, ++ew) {
      const int kh0 = kt_lo * 128 + e * 64;          // this item's first key
      const bool full_tile = kh0 >= iv.lo && kh0 + 64 <= iv.hi && kh0 + 64 <= p.Sk;
      uint32_t kw0 = 0xFFFFFFFFu, kw1 = 0xFFFFFFFFu; // key-mask words of the item's 64 keys
      if (kbits) {
        kw0 = __ldg(kbits + (kh0 >> 5));
        kw1 = __ldg(kbits + (kh0 >> 5) + 1);
      }
      mbar_wait(&s_full[wg], ew & 1);
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld32(tmem + lane_base + col_s, &sv[0]);
      tmem_ld32(tmem + lane_base + col_s + 32, &sv[32]);
      tmem_wait_ld();
      uint32_t pk[32], fk[32];
      // mask-free items (full tile, no masked key) take a loop without the per-element key / interval tests
      auto p_loop = [&](auto fast_tag) {
        constexpr bool kFast = decltype(fast_tag)::value;
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          float pr[2], f[2];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int k = kh0 + j + t;
            float ft;
            bool keep = true;
            if (!kFast) {
              const bool kon = (((j + t) < 32 ? kw0 : kw1) >> ((j + t) & 31)) & 1u;
              keep = kon && (full_tile || (k >= iv.lo && k < iv.hi && k < p.Sk));
            }
            const float bv = (BIAS && keep) ? bias_at(p, b, g, h, q, k) : 0.f;
            const float sc = bwd_score<MOD>(p, __uint_as_float(sv[j + t]), slope_l2, k, q_abs, ft, bv);
            pr[t] = keep ? ex2(fmaf(sc, kBwdLog2e, -lse_l2)) : 0.f;
            f[t] = ft;
          }
          pk[j >> 1] = pack_bf16(pr[0], pr[1]);
          fk[j >> 1] = pack_bf16(f[0], f[1]);
        }
      };
      if (full_tile && (kw0 & kw1) == 0xFFFFFFFFu)
        p_loop(BoolTag<true>{});
      else
        p_loop(BoolTag<false>{});
#pragma unroll
      for (int c = 0; c < 64; c += 32) {            // dS = P (dP - Dvec) f -> TMEM slot + [32 + c/2, ...)
        uint32_t dp[32];
        tmem_ld32(tmem + lane_base + col_dp + c, dp);
        tmem_wait_ld();
        uint32_t ds[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const uint32_t pw = pk[(c + j) >> 1], fw = fk[(c + j) >> 1];
          float d0 = bf16_lo(pw) * (__uint_as_float(dp[j]) - dvr);
          float d1 = bf16_hi(pw) * (__uint_as_float(dp[j + 1]) - dvr);
          if (MOD == MOD_SOFTCAP) {
            d0 *= bf16_lo(fw);
            d1 *= bf16_hi(fw);
          }
          ds[j >> 1] = pack_bf16(d0, d1);
          if (BIAS && dbias && row_ok) {            // dL/dbias = dS (fp32 atomics: broadcast dims accumulate)
            const int k = kh0 + c + j;
            const int64_t off = b * dbs.b + g * dbs.g + (int64_t)h * dbs.h + (int64_t)q * dbs.s + (int64_t)k * dbs.d;
            if (k < p.Sk && d0 != 0.f) atomicAdd(dbias + off, d0);
            if (k + 1 < p.Sk && d1 != 0.f) atomicAdd(dbias + off + dbs.d, d1);
          }
        }
        tmem_st16(tmem + lane_base + col_s + 32 + (c >> 1), ds);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[wg]);
    }
    if (kt_hi > kt_lo) {
      mbar_wait(o_full, 0);
      tc_fence_after();
    }
    {                                                // every lane loads (.sync.aligned), valid rows store
      __nv_bfloat16* qp = dq + b * dqs.b + (int64_t)g * dqs.g + (int64_t)h * dqs.h + (int64_t)(row_ok ? q : 0) * dqs.s;
      // warpgroup wg: dQ columns half wg (D = 32: warpgroup 0 stores the whole row)
      constexpr int kHalf = D >= 64 ? D / 2 : D;
#pragma unroll
      for (int c = wg * kHalf; c < (wg + 1) * kHalf && c < D; c += 32) {
        uint32_t o[32];
        if (kt_hi > kt_lo) {
          tmem_ld32(tmem + lane_base + COL_DQ + c, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = 0u;
        }
        const float sc = p.scale;
        uint4* op = reinterpret_cast<uint4*>(qp + c);
        if (row_ok)
#pragma unroll
        for (int t8 = 0; t8 < 4; ++t8)
          op[t8] = make_uint4(pack_bf16(__uint_as_float(o[t8 * 8 + 0]) * sc, __uint_as_float(o[t8 * 8 + 1]) * sc),
                              pack_bf16(__uint_as_float(o[t8 * 8 + 2]) * sc, __uint_as_float(o[t8 * 8 + 3]) * sc),
                              pack_bf16(__uint_as_float(o[t8 * 8 + 4]) * sc, __uint_as_float(o[t8 * 8 + 5]) * sc),
                              pack_bf16(__uint_as_float(o[t8 * 8 + 6]) * sc, __uint_as_float(o[t8 * 8 + 7]) * sc));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- launch
struct BwdLaunch {
  const CUtensorMap* tq64; const CUtensorMap* tdo64;   // 64-row boxes of q and dO (dK/dV kernel)
  const float* lse; Strided5 ls;
  float* dbias; Strided5 dbs;
  const __nv_bfloat16* dout; Strided5 dos;
  float* dvec;
  __nv_bfloat16 *dq, *dk, *dv;
  Strided5 dqs, dks, dvs;
};

template <int D, int MOD, bool BIAS>
static cudaError_t launch_bwd_dmb(const AttnParams& p, const TmaMaps& maps, const CUtensorMap& tdo, const BwdLaunch& L,
                                 cudaStream_t s) {
  using C = BwdCfg<D>;
  const int n_kt = (p.Sk + 127) / 128, n_qt = (p.Sq + 127) / 128;
  cudaError_t e = cudaFuncSetAttribute(bwd_dkdv_kernel<D, MOD, BIAS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::KV_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(bwd_dq_kernel<D, MOD, BIAS>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_TOTAL);
  if (e != cudaSuccess) return e;
  bwd_dkdv_kernel<D, MOD, BIAS><<<p.B * p.G * p.Hkv * n_kt, kBwdThreads, C::KV_SMEM, s>>>(p, maps, *L.tq64, *L.tdo64, L.lse, L.ls, L.dvec, L.dk, L.dks,
                                                                        L.dv, L.dvs);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  bwd_dq_kernel<D, MOD, BIAS><<<p.B * p.G * p.Hq * n_qt, kBwdThreads, C::SMEM_TOTAL, s>>>(p, maps, tdo, L.lse, L.ls, L.dvec, L.dq, L.dqs, L.dbias, L.dbs);
  return cudaGetLastError();
}

template <int D, int MOD>
static cudaError_t launch_bwd_dm(const AttnParams& p, const TmaMaps& maps, const CUtensorMap& tdo, const BwdLaunch& L,
                                 cudaStream_t s) {
  return p.bias ? launch_bwd_dmb<D, MOD, true>(p, maps, tdo, L, s) : launch_bwd_dmb<D, MOD, false>(p, maps, tdo, L, s);
}

template <int D>
static cudaError_t launch_bwd_d(const AttnParams& p, const TmaMaps& maps, const CUtensorMap& tdo, const BwdLaunch& L,
                                cudaStream_t s) {
  switch (p.mod) {
    case MOD_ALIBI: return launch_bwd_dm<D, MOD_ALIBI>(p, maps, tdo, L, s);
    case MOD_SOFTCAP: return launch_bwd_dm<D, MOD_SOFTCAP>(p, maps, tdo, L, s);
    default: return launch_bwd_dm<D, MOD_NONE>(p, maps, tdo, L, s);
  }
}

// The gate pre-pass (when p.gate_mode is sigmoid; `da` receives dO * s(g) and the caller's tdo map points
// at it) or the plain Dvec pass.
cudaError_t launch_bwd_prepass(const AttnParams& p, const void* dout, Strided5 dos, float* dvec, void* da, void* dgate,
                               Strided5 dgs, const void* aun, cudaStream_t s) {
  const int64_t rows = (int64_t)p.B * p.G * p.Hq * p.Sq;
  if (p.gate_mode == GATE_SIGMOID)
    bwd_gate_kernel<false><<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(
        p, static_cast<const __nv_bfloat16*>(dout), dos, static_cast<__nv_bfloat16*>(da),
        static_cast<__nv_bfloat16*>(dgate), dgs, dvec, nullptr);
  else if (p.gate_mode == GATE_MUL)
    bwd_gate_kernel<true><<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(
        p, static_cast<const __nv_bfloat16*>(dout), dos, static_cast<__nv_bfloat16*>(da),
        static_cast<__nv_bfloat16*>(dgate), dgs, dvec, static_cast<const __nv_bfloat16*>(aun));
  else
    bwd_dvec_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(p, static_cast<const __nv_bfloat16*>(dout), dos, dvec);
  return cudaGetLastError();
}

cudaError_t launch_zero_rows(void* dst, Strided5 ds, int B, int G, int H, int S, int D, cudaStream_t s) {
  const int64_t n8 = (int64_t)B * G * H * S * (D / 8);
  if (n8 == 0) return cudaSuccess;
  zero_rows_kernel<<<(unsigned)std::min<int64_t>((n8 + 255) / 256, 4 * 148), 256, 0, s>>>(
      static_cast<__nv_bfloat16*>(dst), ds, B, G, H, S, D);
  return cudaGetLastError();
}

cudaError_t launch_diff_bwd_seed(const AttnParams& p, const void* dout, Strided5 dos, const void* o1, void* do1,
                                 float* dlambda, cudaStream_t s) {
  const int64_t rows = (int64_t)p.B * p.G * p.Hq * p.Sq;
  diff_bwd_seed_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(
      p, static_cast<const __nv_bfloat16*>(dout), dos, static_cast<const __nv_bfloat16*>(o1),
      static_cast<__nv_bfloat16*>(do1), dlambda);
  return cudaGetLastError();
}

cudaError_t launch_attn_bwd(const AttnParams& p, const TmaMaps& maps, const CUtensorMap& tdo, const CUtensorMap& tq64,
                            const CUtensorMap& tdo64, const float* lse,
                            Strided5 ls, const void* dout, Strided5 dos, float* dvec, void* dq, Strided5 dqs, void* dk,
                            Strided5 dks, void* dv, Strided5 dvs, float* dbias, Strided5 dbs, cudaStream_t s) {
  BwdLaunch L{&tq64, &tdo64, lse, ls, dbias, dbs, static_cast<const __nv_bfloat16*>(dout), dos, dvec, static_cast<__nv_bfloat16*>(dq),
              static_cast<__nv_bfloat16*>(dk), static_cast<__nv_bfloat16*>(dv), dqs, dks, dvs};
  switch (p.Dqk) {
    case 128: return launch_bwd_d<128>(p, maps, tdo, L, s);
    case 64: return launch_bwd_d<64>(p, maps, tdo, L, s);
    case 32: return launch_bwd_d<32>(p, maps, tdo, L, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fl
