// decode.cu -- short-query path (S_q <= 16 rows per (b, g, h); RSA decode, G10/G12): split-KV
// attention and a SIMT block selection.  Decode is HBM-bound (each listed
// K/V block is read once per (b, h)), so the tensor-core tile of 128 query rows would idle 127/128
// of its MMA work and one CTA per (b, h) would leave SMs idle; instead
//
//  * attn_decode_split_kernel: persistent (one CTA per SM) over items = (row, split of `bps` 128-key
//    blocks).  A producer warp resolves the blocks (the row's RSA list, or the tiles of its mask
//    interval) 32 at a time and streams each block's K and V tiles by TMA into a 3-stage shared-memory
//    ring; 256 compute threads score the keys (two threads per key, 128-B swizzled rows read
//    conflict-free), take the block max/sum by warp shuffles (Alg.2's online update, at
//    block granularity), accumulate P V (16 key groups x D/8 column groups) and write the item's
//    unnormalised partial (O_s, m_s, l_s).
//  * attn_decode_combine_kernel: O = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M), M = max_s m_s
//    (the same closed form of the online softmax, applied across splits).
//  * rsa_select_small_kernel: the selection score of every KV block for a query block of <= 16 rows
//    as q+ . kmax + q- . kmin in fp32 on the FMA pipe (one thread per block j; the summaries are
//    read once), then the same rank top-k as the tensor-core selection.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

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

// Persistent, TMA-fed split-KV kernel.  grid = min(items, SMs); item = (row, split) with `bps`
// consecutive 128-key blocks of that row.  Warp 4 (one lane) walks the CTA's items and streams every
// block's K and V tiles (128-B swizzled, the tcgen05 kernels' tensor maps) into an NST-stage
// shared-memory ring through full/empty mbarriers, so the next blocks are in flight while the 128
// compute threads work on the current one: thread t scores key t (chunk c of row r sits at
// (c ^ (r & 7)) * 16 -- conflict-free), block max/sum by warp shuffles (Alg.2 at block granularity),
// then 8 key groups x D/8 column groups accumulate P V.  The item's unnormalised partial
// (O_s, m_s, l_s) goes to the workspace for the combine kernel.
template <int D>
struct DecCfg {
  static constexpr int NST = D == 128 ? 3 : 6;            // ring stages (K + V of one block each)
  static constexpr int TILE = 128 * D * 2;
  static constexpr int SLAB = 128 * 128;                  // 128 rows x 64 columns (128-B swizzle)
  static constexpr int SMEM = NST * 2 * TILE + 1024;      // + alignment slack (1024-B swizzle atoms)
};

constexpr int kDecCompute = 256;            // compute threads: 2 per key for Q K^T
template <int D>
__global__ void __launch_bounds__(kDecCompute + 32, 1)
    attn_decode_split_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ TmaMaps maps,
                             float* __restrict__ part, int bps, int n_split, long long n_items) {
  using C = DecCfg<D>;
  constexpr int DG = D / 8;                 // 16-byte column groups
  constexpr int NW = kDecCompute / 32;
  constexpr int KPW = 128 / NW;             // keys per warp (16)
  constexpr int CPL = D / 32;               // P V columns per lane
  extern __shared__ uint8_t dec_smem_raw[];
  uint8_t* ring = dec_smem_raw + ((1024u - (smem_u32(dec_smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(16) float qs[D];
  __shared__ float wm_s[NW], wl_s[NW];
  __shared__ __align__(16) float accs[NW][D];
  __shared__ uint64_t full[C::NST], empty[C::NST];
  __shared__ int kbinfo[C::NST];

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDecCompute);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto split_of = [&](long long it) { return (int)(it % n_split); };
  auto row_coords = [&](int64_t row, int& q, int64_t& bgh, int& h, int& g, int& b) {
    q = (int)(row % p.Sq);
    bgh = row / p.Sq;
    h = (int)(bgh % p.Hq);
    g = (int)((bgh / p.Hq) % p.G);
    b = (int)(bgh / ((int64_t)p.Hq * p.G));
  };

  if (warp == NW) {
    // ============================== producer ==============================
    // The warp resolves 32 ring slots at a time in parallel (lane = slot: the row's list entry or
    // interval tile, one dependent global round trip per 32 slots instead of per item); lane 0 then
    // issues them in order.
    if (lane == 0) {
      tma_prefetch_desc(&maps.k);
      tma_prefetch_desc(&maps.v);
    }
    const long long my_items = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long n_slots = my_items * bps;
    for (long long e0 = 0; e0 < n_slots; e0 += 32) {
      const long long es = e0 + lane;
      int kb = -1, hkv = 0, gk = 0, bk = 0, gv = 0, bv = 0, kr = 0;
      if (es < n_slots) {
        const long long it = blockIdx.x + (es / bps) * gridDim.x;
        const int i = split_of(it) * bps + (int)(es % bps);
        const int64_t row = it / n_split;
        int q, h, g, b;
        int64_t bgh;
        row_coords(row, q, bgh, h, g, b);
        hkv = h / p.grp;
        gk = maps.k_bcast_g ? 0 : g; bk = maps.k_bcast_b ? 0 : b;
        gv = maps.v_bcast_g ? 0 : g; bv = maps.v_bcast_b ? 0 : b;
        const DecRow dr = dec_row(p, bgh, q, row_interval(p, b, q));
        if (i < dr.n) kb = dr.list ? dr.list[i] : dr.lo_tile + i;
        if (kb * 128 >= p.Sk) kb = -1;
        if (kb >= 0) {                                 // paged KV: the tile's page of the pools
          kv_tile_coords(p, b, kb, bk, kr, bk);
          bv = p.page_table ? bk : bv;
        }
      }
      const int cnt = (int)min(32ll, n_slots - e0);
      for (int j = 0; j < cnt; ++j) {
        const int kbj = __shfl_sync(0xffffffffu, kb, j), hj = __shfl_sync(0xffffffffu, hkv, j);
        const int gkj = __shfl_sync(0xffffffffu, gk, j), bkj = __shfl_sync(0xffffffffu, bk, j);
        const int gvj = __shfl_sync(0xffffffffu, gv, j), bvj = __shfl_sync(0xffffffffu, bv, j);
        const int krj = __shfl_sync(0xffffffffu, kr, j);
        if (lane == 0) {
          const int e = (int)(e0 + j);
          const int s = e % C::NST;
          if (e >= C::NST) mbar_wait(&empty[s], ((e / C::NST) - 1) & 1);
          kbinfo[s] = kbj;
          if (kbj >= 0) {
            uint8_t* ks = ring + s * 2 * C::TILE;
            mbar_arrive_expect_tx(&full[s], 2 * C::TILE);
            for (int c = 0; c < D / 64; ++c) {
              tma_load_5d(ks + c * C::SLAB, &maps.k, &full[s], c * 64, krj, hj, gkj, bkj);
              tma_load_5d(ks + C::TILE + c * C::SLAB, &maps.v, &full[s], c * 64, krj, hj, gvj, bvj);
            }
          } else {
            mbar_arrive(&full[s]);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // ============================== compute (256 threads) ==============================
  // Warp w owns keys [16 w, 16 w + 16) of every block and keeps its own online softmax (m, l, O over all
  // D columns): lane pair (2k, 2k + 1) splits key k's Q K^T dot product, then lane j accumulates P V for
  // columns [CPL j, CPL j + CPL) over the warp's 16 keys (P broadcast by shuffles).  No barrier per
  // block -- the eight warps meet once per item, when their partials are merged (Alg.2's closed form).
  const int key = warp * KPW + (lane >> 1), half = lane & 1;
  auto load_q = [&](long long it) -> unsigned short {  // element t of the item's query row
    int q, h, g, b;
    int64_t bgh;
    row_coords(it / n_split, q, bgh, h, g, b);
    return static_cast<const unsigned short*>(p.q)[b * p.qs.b + g * p.qs.g + (int64_t)h * p.qs.h + (int64_t)q * p.qs.s + t];
  };
  unsigned short q_next = 0;
  if (t < D && blockIdx.x < n_items) q_next = load_q(blockIdx.x);
  // lane's P V columns inside a 128-B swizzled V row: 16-B chunk cv, byte offset cb within it
  constexpr int BPL = CPL * 2;
  const int cv = lane * BPL / 16, cb = lane * BPL % 16;
  int e = 0;
  for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t row = it / n_split;
    const int split = (int)(it % n_split);
    int q, h, g, b;
    int64_t bgh;
    row_coords(row, q, bgh, h, g, b);
    const int q_abs = q + p.q_off;
    const Interval iv = row_interval(p, b, q);
    const uint32_t* kbits = p.keybits ? p.keybits + ((int64_t)b * p.G + g) * p.keybits_words : nullptr;
    float slope_l2 = 0.f;
    if (p.mod == MOD_ALIBI) slope_l2 = kDecLog2e * (p.alibi ? p.alibi[h] : exp2f(-8.f * (float)(h + 1) / (float)p.Hq));
    const float sc_l2 = p.scale * kDecLog2e;
    named_bar_sync(1, kDecCompute);                     // previous item done with qs / accs
    if (t < D) qs[t] = __uint_as_float((uint32_t)q_next << 16);
    named_bar_sync(1, kDecCompute);
    if (t < D && it + gridDim.x < n_items) q_next = load_q(it + gridDim.x);   // in flight during this item

    float acc[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc[i] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int i = 0; i < bps; ++i, ++e) {
      const int s = e % C::NST;
      mbar_wait(&full[s], (e / C::NST) & 1);
      const int kb = kbinfo[s];
      if (kb < 0) {                                     // no block in this slot (block-uniform)
        mbar_arrive(&empty[s]);
        continue;
      }
      const uint8_t* ks = ring + s * 2 * C::TILE;
      const uint8_t* vs = ks + C::TILE;
      const int k = kb * 128 + key;
      bool keep = k < p.Sk && k >= iv.lo && k < iv.hi;
      if (keep && kbits) keep = (kbits[k >> 5] >> (k & 31)) & 1u;
      float sv = -INFINITY, dot = 0.f;
      if (keep) {
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int cc = 0; cc < DG / 2; ++cc) {
          // this half's chunks (128-B swizzled tile: chunk c of row r at (c ^ (r & 7)) * 16), rotated by 4
          // for half 1 so the pair hits different bank groups
          const int c = half * (DG / 2) + ((cc + 4 * half) % (DG / 2));
          const uint4 kv = *reinterpret_cast<const uint4*>(ks + (c >> 3) * C::SLAB + key * 128 + (((c & 7) ^ (key & 7)) << 4));
          const float4 qa = *reinterpret_cast<const float4*>(qs + c * 8);
          const float4 qb = *reinterpret_cast<const float4*>(qs + c * 8 + 4);
          d0 = fmaf(qa.x, bf16_lo(kv.x), d0);
          d1 = fmaf(qa.y, bf16_hi(kv.x), d1);
          d0 = fmaf(qa.z, bf16_lo(kv.y), d0);
          d1 = fmaf(qa.w, bf16_hi(kv.y), d1);
          d0 = fmaf(qb.x, bf16_lo(kv.z), d0);
          d1 = fmaf(qb.y, bf16_hi(kv.z), d1);
          d0 = fmaf(qb.z, bf16_lo(kv.w), d0);
          d1 = fmaf(qb.w, bf16_hi(kv.w), d1);
        }
        dot = d0 + d1;
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);      // the pair's two halves of the dot product
      if (keep) {
        sv = dot * sc_l2;                               // log2-domain score (G1, Eq.4)
        if (p.mod == MOD_ALIBI) sv += slope_l2 * (float)(k - q_abs);
        if (p.mod == MOD_SOFTCAP) sv = p.softcap * kDecLog2e * tanh_approx(dot * p.scale / p.softcap);
      }
      const float m_new = fmaxf(m, dec_warp_max(sv));
      if (m_new == -INFINITY) {                         // nothing kept by this warp so far (warp-uniform)
        mbar_arrive(&empty[s]);
        continue;
      }
      const float corr = ex2(m - m_new);                // 0 when m = -inf
      const float pe = sv == -INFINITY ? 0.f : ex2(sv - m_new);
      l = l * corr + dec_warp_sum(half == 0 ? pe : 0.f);
      m = m_new;
#pragma unroll
      for (int i2 = 0; i2 < CPL; ++i2) acc[i2] *= corr;
#pragma unroll
      for (int kk = 0; kk < KPW; ++kk) {
        const int kr = warp * KPW + kk;
        const float pv = __shfl_sync(0xffffffffu, pe, 2 * kk);
        const uint8_t* vp = vs + (cv >> 3) * C::SLAB + kr * 128 + ((((cv & 7) ^ (kr & 7)) << 4) | cb);
        if constexpr (CPL == 4) {
          const uint2 vv = *reinterpret_cast<const uint2*>(vp);
          acc[0] = fmaf(pv, bf16_lo(vv.x), acc[0]);
          acc[1] = fmaf(pv, bf16_hi(vv.x), acc[1]);
          acc[2] = fmaf(pv, bf16_lo(vv.y), acc[2]);
          acc[3] = fmaf(pv, bf16_hi(vv.y), acc[3]);
        } else {
          const uint32_t vv = *reinterpret_cast<const uint32_t*>(vp);
          acc[0] = fmaf(pv, bf16_lo(vv), acc[0]);
          acc[1] = fmaf(pv, bf16_hi(vv), acc[1]);
        }
      }
      mbar_arrive(&empty[s]);                           // this thread is done with the stage
    }
    // merge the eight warps' partials: O_s = sum_w O_w 2^(m_w - M), l_s = sum_w l_w 2^(m_w - M)
#pragma unroll
    for (int i2 = 0; i2 < CPL; ++i2) accs[warp][lane * CPL + i2] = acc[i2];
    if (lane == 0) {
      wm_s[warp] = m;
      wl_s[warp] = l;
    }
    named_bar_sync(1, kDecCompute);
    float* out = part + (row * n_split + split) * (D + 2);
    if (t < D) {
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; ++w) M = fmaxf(M, wm_s[w]);
      float o = 0.f, L = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const float f = wm_s[w] == -INFINITY ? 0.f : ex2(wm_s[w] - M);
          o = fmaf(accs[w][t], f, o);
          L = fmaf(wl_s[w], f, L);
        }
      }
      out[t] = o;
      if (t == 0) {
        out[D] = M;
        out[D + 1] = L;
      }
    }
  }
}

template <int D>
__global__ void __launch_bounds__(D) attn_decode_combine_kernel(const __grid_constant__ AttnParams p,
                                                                const float* __restrict__ part, int n_split) {
  // The splits' (m_s, l_s) are staged in shared memory in one round of loads; every thread then
  // needs only its own column of the partial outputs (independent loads, unrolled).
  constexpr int kMaxStage = 512;
  __shared__ float sm_m[kMaxStage], sm_l[kMaxStage];
  const int t = threadIdx.x;
  const int64_t row = blockIdx.x;
  const int q = (int)(row % p.Sq);
  const int64_t bgh = row / p.Sq;
  const int h = (int)(bgh % p.Hq), g = (int)((bgh / p.Hq) % p.G), b = (int)(bgh / ((int64_t)p.Hq * p.G));
  const float* pr = part + row * n_split * (D + 2);
  const int ns = min(n_split, kMaxStage);
  for (int s = t; s < ns; s += D) {
    sm_m[s] = pr[s * (D + 2) + D];
    sm_l[s] = pr[s * (D + 2) + D + 1];
  }
  __syncthreads();
  float M = -INFINITY;
  for (int s = 0; s < n_split; ++s) M = fmaxf(M, s < ns ? sm_m[s] : pr[s * (D + 2) + D]);
  float L = 0.f, o = 0.f;
  if (M != -INFINITY) {
#pragma unroll 8
    for (int s = 0; s < n_split; ++s) {
      const float ms = s < ns ? sm_m[s] : pr[s * (D + 2) + D];
      const float ls = s < ns ? sm_l[s] : pr[s * (D + 2) + D + 1];
      const float f = ms == -INFINITY ? 0.f : ex2(ms - M);
      L = fmaf(ls, f, L);
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

cudaError_t launch_attn_decode(const AttnParams& p, const TmaMaps& maps, float* part, int n_sms, cudaStream_t stream) {
  int bps, ns;
  decode_plan(p, n_sms, &bps, &ns);
  const long long rows = (long long)p.B * p.G * p.Hq * p.Sq;
  const long long items = rows * ns;
  if (rows > 65535LL * 32768LL) return cudaErrorInvalidValue;
  const int grid = (int)std::min<long long>(items, n_sms > 0 ? n_sms : 148);   // persistent
  cudaError_t e;
  if (p.Dqk == 128) {
    e = cudaFuncSetAttribute(attn_decode_split_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DecCfg<128>::SMEM);
    if (e != cudaSuccess) return e;
    attn_decode_split_kernel<128><<<grid, kDecCompute + 32, DecCfg<128>::SMEM, stream>>>(p, maps, part, bps, ns, items);
    attn_decode_combine_kernel<128><<<(unsigned)rows, 128, 0, stream>>>(p, part, ns);
  } else {
    e = cudaFuncSetAttribute(attn_decode_split_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DecCfg<64>::SMEM);
    if (e != cudaSuccess) return e;
    attn_decode_split_kernel<64><<<grid, kDecCompute + 32, DecCfg<64>::SMEM, stream>>>(p, maps, part, bps, ns, items);
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
