// decode.cu -- short-query path (S_q <= 16 rows per (b, g, h); RSA decode, G10/G12): split-KV
// attention and a SIMT block selection.  Decode is HBM-bound (each listed
// K/V block is read once per (b, h)), so the tensor-core tile of 128 query rows would idle 127/128
// of its MMA work and one CTA per (b, h) would leave SMs idle; instead
//
//  * attn_decode_split_kernel: grid (n_split, rows).  Each CTA walks `bps` KV blocks of one query
//    row (the row's RSA list, or the 128-key tiles of its mask interval): thread t scores key t of
//    the block (16-byte K loads, q in shared memory), block max/sum by warp shuffles (Alg.2's
//    online update, at block granularity), then 8 key-groups x D/8 column groups
//    accumulate P V with 16-byte V loads.  It writes the unnormalised partial (O_s, m_s, l_s).
//  * attn_decode_combine_kernel: O = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), M = max_s m_s
//    (the same closed form of the online softmax, applied across splits).
//  * rsa_select_small_kernel: the selection score of every KV block for a query block of <= 16 rows
//    as q+ . kmax + q- . kmin in fp32 on the FMA pipe (one thread per block j; the summaries are
//    read once), then the same rank top-k as the tensor-core selection.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "masks.cuh"
#include "params.h"
#include "ptx.cuh"

namespace fl {

constexpr int kDecThreads = 128;
constexpr float kDecLog2e = 1.4426950408889634f;

__device__ __forceinline__ float dec_warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float dec_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Number of 128-key blocks row (bgh, q) visits and the i-th of them.
struct DecRow {
  const int32_t* list;  // RSA list of the row's query block (nullptr: interval tiles)
  int lo_tile, n;
};

__device__ __forceinline__ DecRow dec_row(const AttnParams& p, int64_t bgh, int q, const Interval& iv) {
  DecRow r;
  if (p.mask == MASK_BLOCKLIST) {
    const int64_t row = bgh * p.n_qblk + q / p.blk_q;
    r.list = p.blk_idx + row * p.max_sel;
    r.n = min(p.blk_cnt[row], p.max_sel);
    r.lo_tile = 0;
  } else {
    r.list = nullptr;
    r.lo_tile = iv.lo / 128;
    r.n = iv.hi > iv.lo ? (iv.hi + 127) / 128 - r.lo_tile : 0;
  }
  return r;
}

template <int D>
__global__ void __launch_bounds__(kDecThreads) attn_decode_split_kernel(const __grid_constant__ AttnParams p,
                                                                         float* __restrict__ part, int bps) {
  constexpr int DG = D / 8;                 // 16-byte column groups
  constexpr int KG = kDecThreads / DG;      // key groups for P V
  constexpr int KPG = 128 / KG;             // keys per key group
  __shared__ __align__(16) float qs[D];
  __shared__ float ps[128];
  __shared__ float red[2][4];
  __shared__ __align__(16) float accs[KG][D];

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int split = blockIdx.x, n_split = gridDim.x;
  const int64_t row = blockIdx.y;                       // ((b*G + g)*Hq + h)*Sq + q
  const int q = (int)(row % p.Sq);
  const int64_t bgh = row / p.Sq;
  const int h = (int)(bgh % p.Hq), g = (int)((bgh / p.Hq) % p.G), b = (int)(bgh / ((int64_t)p.Hq * p.G));
  const int hkv = h / p.grp;
  const int q_abs = q + p.q_off;
  const Interval iv = row_interval(p, b, q);
  const DecRow dr = dec_row(p, bgh, q, iv);
  const unsigned short* kbase = static_cast<const unsigned short*>(p.k) + b * p.ks.b + g * p.ks.g + (int64_t)hkv * p.ks.h;
  const unsigned short* vbase = static_cast<const unsigned short*>(p.v) + b * p.vs.b + g * p.vs.g + (int64_t)hkv * p.vs.h;
  const uint32_t* kbits = p.keybits ? p.keybits + ((int64_t)b * p.G + g) * p.keybits_words : nullptr;
  float slope_l2 = 0.f;
  if (p.mod == MOD_ALIBI) slope_l2 = kDecLog2e * (p.alibi ? p.alibi[h] : exp2f(-8.f * (float)(h + 1) / (float)p.Hq));
  const float sc_l2 = p.scale * kDecLog2e;

  if (t < D) {
    const unsigned short* qp = static_cast<const unsigned short*>(p.q) + b * p.qs.b + g * p.qs.g +
                               (int64_t)h * p.qs.h + (int64_t)q * p.qs.s;
    qs[t] = __uint_as_float((uint32_t)qp[t] << 16);
  }
  __syncthreads();

  const int dg = t % DG, kg = t / DG;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  float m = -INFINITY, l = 0.f;
  const int i0 = split * bps, i1 = min(dr.n, i0 + bps);
  for (int i = i0; i < i1; ++i) {
    const int kb = dr.list ? dr.list[i] : dr.lo_tile + i;
    const int k = kb * 128 + t;
    // V rows of this thread's key group: issued first so they stream in while Q K^T and the block
    // reductions run (keys past S_k get p = 0; their row index is clamped to stay in bounds)
    uint4 vv[KPG];
#pragma unroll
    for (int t2 = 0; t2 < KPG; ++t2) {
      const int kr = min(max(kb, 0) * 128 + kg * KPG + t2, p.Sk - 1);
      vv[t2] = __ldg(reinterpret_cast<const uint4*>(vbase + (int64_t)kr * p.vs.s) + dg);
    }
    bool keep = kb >= 0 && k < p.Sk && k >= iv.lo && k < iv.hi;
    if (keep && kbits) keep = (kbits[k >> 5] >> (k & 31)) & 1u;
    float s = -INFINITY;
    if (keep) {
      const uint4* kr = reinterpret_cast<const uint4*>(kbase + (int64_t)k * p.ks.s);
      uint4 kv[DG];
#pragma unroll
      for (int c = 0; c < DG; ++c) kv[c] = __ldg(kr + c);
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int c = 0; c < DG; ++c) {
        const float4 qa = *reinterpret_cast<const float4*>(qs + c * 8);
        const float4 qb = *reinterpret_cast<const float4*>(qs + c * 8 + 4);
        const uint32_t w[4] = {kv[c].x, kv[c].y, kv[c].z, kv[c].w};
        d0 = fmaf(qa.x, bf16_lo(w[0]), d0);
        d1 = fmaf(qa.y, bf16_hi(w[0]), d1);
        d0 = fmaf(qa.z, bf16_lo(w[1]), d0);
        d1 = fmaf(qa.w, bf16_hi(w[1]), d1);
        d0 = fmaf(qb.x, bf16_lo(w[2]), d0);
        d1 = fmaf(qb.y, bf16_hi(w[2]), d1);
        d0 = fmaf(qb.z, bf16_lo(w[3]), d0);
        d1 = fmaf(qb.w, bf16_hi(w[3]), d1);
      }
      s = (d0 + d1) * sc_l2;                            // log2-domain score (G1, Eq.4)
      if (p.mod == MOD_ALIBI) s += slope_l2 * (float)(k - q_abs);
      if (p.mod == MOD_SOFTCAP) s = p.softcap * kDecLog2e * tanh_approx((d0 + d1) * p.scale / p.softcap);
    }
    float bm = dec_warp_max(s);
    if (lane == 0) red[0][warp] = bm;
    __syncthreads();
    bm = fmaxf(fmaxf(red[0][0], red[0][1]), fmaxf(red[0][2], red[0][3]));
    const float m_new = fmaxf(m, bm);
    if (m_new == -INFINITY) {                           // nothing kept so far (block-uniform)
      __syncthreads();
      continue;
    }
    const float corr = ex2(m - m_new);                  // 0 when m = -inf
    const float pe = s == -INFINITY ? 0.f : ex2(s - m_new);
    ps[t] = pe;
    const float ws = dec_warp_sum(pe);
    if (lane == 0) red[1][warp] = ws;
    __syncthreads();
    l = l * corr + ((red[1][0] + red[1][1]) + (red[1][2] + red[1][3]));
    m = m_new;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= corr;
    {
#pragma unroll
      for (int t2 = 0; t2 < KPG; ++t2) {
        const float pv = ps[kg * KPG + t2];
        const uint32_t w[4] = {vv[t2].x, vv[t2].y, vv[t2].z, vv[t2].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[2 * e] = fmaf(pv, bf16_lo(w[e]), acc[2 * e]);
          acc[2 * e + 1] = fmaf(pv, bf16_hi(w[e]), acc[2 * e + 1]);
        }
      }
    }
    __syncthreads();                                    // ps / red reuse
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) accs[kg][dg * 8 + e] = acc[e];
  __syncthreads();
  float* out = part + (row * n_split + split) * (D + 2);
  if (t < D) {
    float o = 0.f;
#pragma unroll
    for (int g2 = 0; g2 < KG; ++g2) o += accs[g2][t];
    out[t] = o;
  }
  if (t == 0) {
    out[D] = m;
    out[D + 1] = l;
  }
}

template <int D>
__global__ void __launch_bounds__(D) attn_decode_combine_kernel(const __grid_constant__ AttnParams p,
                                                                const float* __restrict__ part, int n_split) {
  const int t = threadIdx.x;
  const int64_t row = blockIdx.x;
  const int q = (int)(row % p.Sq);
  const int64_t bgh = row / p.Sq;
  const int h = (int)(bgh % p.Hq), g = (int)((bgh / p.Hq) % p.G), b = (int)(bgh / ((int64_t)p.Hq * p.G));
  const float* pr = part + row * n_split * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_split; ++s) M = fmaxf(M, pr[s * (D + 2) + D]);
  float L = 0.f, o = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < n_split; ++s) {
      const float ms = pr[s * (D + 2) + D];
      if (ms == -INFINITY) continue;
      const float f = ex2(ms - M);
      L = fmaf(pr[s * (D + 2) + D + 1], f, L);
      o = fmaf(pr[s * (D + 2) + t], f, o);
    }
  }
  const bool empty = M == -INFINITY || !(L > 0.f);     // G7: O = 0, lse = -inf
  o = empty ? 0.f : o / L;
  unsigned short* op = static_cast<unsigned short*>(p.o) + b * p.os.b + g * p.os.g + (int64_t)h * p.os.h +
                       (int64_t)q * p.os.s;
  const __nv_bfloat16 ob = __float2bfloat16_rn(o);
  op[t] = *reinterpret_cast<const unsigned short*>(&ob);
  if (t == 0 && p.lse)
    p.lse[b * p.lses.b + g * p.lses.g + (int64_t)h * p.lses.h + (int64_t)q * p.lses.s] =
        empty ? -INFINITY : (M + __log2f(L)) * 0.6931471805599453f;
}

// Split plan shared by the workspace query and the launch.
void decode_plan(const AttnParams& p, int n_sms, int* bps, int* n_split) {
  const int max_blocks = p.mask == MASK_BLOCKLIST ? p.max_sel : (p.Sk + 127) / 128 + 1;
  const long long rows = (long long)p.B * p.G * p.Hq * p.Sq;
  const long long target = (long long)n_sms * 8;        // ~8 resident CTAs per SM
  long long b = (rows * max_blocks + target - 1) / target;
  b = b < 1 ? 1 : b;
  *bps = (int)b;
  *n_split = (int)((max_blocks + b - 1) / b);
  if (*n_split < 1) *n_split = 1;
}

size_t decode_workspace_bytes(const AttnParams& p, int n_sms) {
  int bps, ns;
  decode_plan(p, n_sms, &bps, &ns);
  return (size_t)p.B * p.G * p.Hq * p.Sq * ns * (p.Dv + 2) * sizeof(float);
}

cudaError_t launch_attn_decode(const AttnParams& p, float* part, int n_sms, cudaStream_t stream) {
  int bps, ns;
  decode_plan(p, n_sms, &bps, &ns);
  const long long rows = (long long)p.B * p.G * p.Hq * p.Sq;
  if (rows > 65535LL * 32768LL) return cudaErrorInvalidValue;
  dim3 grid(ns, (unsigned)rows);
  if (p.Dqk == 128) {
    attn_decode_split_kernel<128><<<grid, kDecThreads, 0, stream>>>(p, part, bps);
    attn_decode_combine_kernel<128><<<(unsigned)rows, 128, 0, stream>>>(p, part, ns);
  } else {
    attn_decode_split_kernel<64><<<grid, kDecThreads, 0, stream>>>(p, part, bps);
    attn_decode_combine_kernel<64><<<(unsigned)rows, 64, 0, stream>>>(p, part, ns);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ small-query-block selection
// grid: B*G*Hkv*nqb, 256 threads.  Thread t scores blocks j = t, t + 256, ...; the group's query
// rows (<= 16 per head) are staged in shared memory as q+ / q- in fp32.
constexpr int kSelThreads = 256;
constexpr int kSelMaxRows = 16;

template <int D>
__global__ void __launch_bounds__(kSelThreads) rsa_select_small_kernel(const __grid_constant__ RsaSelParams p,
                                                                       const __nv_bfloat16* __restrict__ qg,
                                                                       int64_t qsb, int64_t qsg, int64_t qsh,
                                                                       int64_t qss, const __nv_bfloat16* __restrict__ kmin,
                                                                       const __nv_bfloat16* __restrict__ kmax) {
  extern __shared__ float sm[];
  float* qp = sm;                                      // [rows][D]  q+
  float* qn = qp + p.grp * kSelMaxRows * D;            // [rows][D]  q-
  float* sc = qn + p.grp * kSelMaxRows * D;            // [nkb] scores
  uint32_t* flags = reinterpret_cast<uint32_t*>(sc + p.nkb);
  const int t = threadIdx.x;
  const int i = blockIdx.x % p.nqb;
  const int bgk = blockIdx.x / p.nqb;
  const int hk = bgk % p.Hkv, g = (bgk / p.Hkv) % p.G, b = bgk / (p.Hkv * p.G);
  const int q0 = i * 128, nrow = min(p.Sq - q0, kSelMaxRows);
  const int n_q = p.grp * nrow;
  for (int e = t; e < n_q * D; e += kSelThreads) {
    const int r = e / D, d = e % D;
    const int hh = hk * p.grp + r / nrow, qq = q0 + r % nrow;
    const float v = __bfloat162float(qg[b * qsb + g * qsg + (int64_t)hh * qsh + (int64_t)qq * qss + d]);
    qp[e] = fmaxf(v, 0.f);
    qn[e] = fminf(v, 0.f);
  }
  const int q_last = min(p.Sq, (i + 1) * 128) - 1;
  const int q_last_abs = q_last + p.q_off;
  int c = q_last_abs < 0 ? 0 : q_last_abs / 128;
  c = min(c, p.nkb - 1);
  __syncthreads();
  for (int j = t; j < p.nkb; j += kSelThreads) {
    float best = -INFINITY;
    if (j >= 1 && j < c) {
      const uint4* mx = reinterpret_cast<const uint4*>(kmax + ((int64_t)bgk * p.nkb + j) * D);
      const uint4* mn = reinterpret_cast<const uint4*>(kmin + ((int64_t)bgk * p.nkb + j) * D);
      for (int r = 0; r < n_q; ++r) {
        const float* a = qp + r * D;
        const float* z = qn + r * D;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll 4
        for (int cc = 0; cc < D / 8; ++cc) {
          const uint4 u = __ldg(mx + cc), w = __ldg(mn + cc);
          const uint32_t uu[4] = {u.x, u.y, u.z, u.w}, ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            s0 = fmaf(a[cc * 8 + 2 * e], bf16_lo(uu[e]), s0);
            s1 = fmaf(a[cc * 8 + 2 * e + 1], bf16_hi(uu[e]), s1);
            s0 = fmaf(z[cc * 8 + 2 * e], bf16_lo(ww[e]), s0);
            s1 = fmaf(z[cc * 8 + 2 * e + 1], bf16_hi(ww[e]), s1);
          }
        }
        best = fmaxf(best, s0 + s1);
      }
    }
    sc[j] = best;
  }
  const int nwords = (p.nkb + 31) / 32;
  for (int w = t; w < nwords; w += kSelThreads) flags[w] = 0u;
  __syncthreads();
  for (int j0 = 0; j0 < p.nkb; j0 += kSelThreads) {
    const int j = j0 + t;
    bool sel = false;
    if (j < p.nkb && j <= c) {
      if (j == 0 || j == c) {
        sel = true;
      } else {
        const float s = sc[j];
        int rank = 0;
        for (int jj = 1; jj < c; ++jj) {
          const float o = sc[jj];
          rank += (o > s) || (o == s && jj < j);
        }
        sel = rank < p.topk;
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, sel);
    if ((t & 31) == 0 && j < p.nkb) flags[j >> 5] = bal;
  }
  __syncthreads();
  int cnt = 0;
  for (int w = 0; w < nwords; ++w) cnt += __popc(flags[w]);
  for (int hh = 0; hh < p.grp; ++hh) {
    const int64_t orow = (((int64_t)b * p.G + g) * p.Hq + hk * p.grp + hh) * p.nqb + i;
    int32_t* out = p.blk_idx + orow * p.max_sel;
    for (int j = t; j < p.nkb; j += kSelThreads) {
      const int w = j >> 5;
      if ((flags[w] >> (j & 31)) & 1u) {
        int pos = __popc(flags[w] & ((1u << (j & 31)) - 1u));
        for (int ww = 0; ww < w; ++ww) pos += __popc(flags[ww]);
        if (pos < p.max_sel) out[pos] = j;
      }
    }
    for (int e = cnt + t; e < p.max_sel; e += kSelThreads) out[e] = -1;
    if (t == 0) p.blk_cnt[orow] = min(cnt, p.max_sel);
  }
}

size_t rsa_select_small_smem(const RsaSelParams& p) {
  return sizeof(float) * (2 * (size_t)p.grp * kSelMaxRows * p.D + p.nkb) + sizeof(uint32_t) * ((p.nkb + 31) / 32);
}

bool rsa_select_small_ok(const RsaSelParams& p) {
  return p.Sq <= kSelMaxRows && rsa_select_small_smem(p) <= 200 * 1024;
}

cudaError_t launch_rsa_select_small(const RsaSelParams& p, const void* q, int64_t qsb, int64_t qsg, int64_t qsh,
                                    int64_t qss, const void* kmin, const void* kmax, cudaStream_t stream) {
  const size_t smem = rsa_select_small_smem(p);
  const unsigned grid = (unsigned)((long long)p.B * p.G * p.Hkv * p.nqb);
  auto qb = static_cast<const __nv_bfloat16*>(q);
  auto mn = static_cast<const __nv_bfloat16*>(kmin);
  auto mx = static_cast<const __nv_bfloat16*>(kmax);
  cudaError_t e;
  if (p.D == 128) {
    e = cudaFuncSetAttribute(rsa_select_small_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    rsa_select_small_kernel<128><<<grid, kSelThreads, smem, stream>>>(p, qb, qsb, qsg, qsh, qss, mn, mx);
  } else {
    e = cudaFuncSetAttribute(rsa_select_small_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    rsa_select_small_kernel<64><<<grid, kSelThreads, smem, stream>>>(p, qb, qsb, qsg, qsh, qss, mn, mx);
  }
  return cudaGetLastError();
}

}  // namespace fl
