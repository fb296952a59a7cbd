// rsa.cu -- the data-dependent half of Rectified Sparse Attention (reading G10;
// the paper only names RSA, as a variant beyond FlexAttention's
// template): per-KV-block key summaries and the per-query-block block list that
// the attention kernels then walk (mask FL_MASK_BLOCKLIST).
//
//  * rsa_summaries_kernel: kmin/kmax[bh, j, d] = element-wise min / max of the keys
//    of KV block j.  Exact (min/max of bf16 values is a bf16 value).  One pass over
//    K: HBM-bound, 16-byte loads, one CTA per (bh, block).
//
//  * rsa_select_kernel: score_j = max_{q in block} sum_d max(q_d kmax_jd, q_d kmin_jd).
//    Because kmax >= kmin the per-d maximum is exactly linear in the split
//    q = q+ + q-:  max(q_d kmax_d, q_d kmin_d) = q+_d kmax_d + q-_d kmin_d, so every
//    score of a (b, h) is ONE tensor-core GEMM over K = 2D:
//        D[j, q] = [kmax | kmin]_j . [q+ | q-]_q        (tcgen05, accumulator in TMEM)
//    issued with the summaries as the A operand (M = 128 blocks per tile) so that a
//    TMEM lane is one block j: the max over the 128 queries of the block is then a
//    register-local row max of that thread (no cross-thread reduction).  The top-k
//    (ties to the lower j) is a rank count over the candidates in shared memory, and
//    the ascending list {0} U {c} U top-k is written with a ballot prefix sum.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>

#include "params.h"
#include "ptx.cuh"

namespace fl {

// ------------------------------------------------------------------ summaries
// grid (n_kblk, BGH), 128 threads.  K row r of block j is K[bgh][j*blk + r][:].
__global__ void __launch_bounds__(128) rsa_summaries_kernel(const __nv_bfloat16* __restrict__ k, int64_t sb,
                                                            int64_t sg, int64_t sh, int64_t ss, int B, int G, int H,
                                                            int Sk, int D, int blk, int j0, __nv_bfloat16* __restrict__ kmin,
                                                            __nv_bfloat16* __restrict__ kmax) {
  __shared__ uint4 red_min[128], red_max[128];
  const int j = j0 + blockIdx.x;                       // blocks [j0, nkb): all of them, or the tail after a KV append
  const int bgh = blockIdx.y;
  const int h = bgh % H, g = (bgh / H) % G, b = bgh / (H * G);
  const int nkb = (Sk + blk - 1) / blk;
  const int nch = D / 8;                       // 16-byte chunks per row
  const int rows_par = 128 / nch;              // rows handled in parallel
  const int t = threadIdx.x;
  const int ch = t % nch, r0 = t / nch;
  const __nv_bfloat16* base = k + b * sb + g * sg + (int64_t)h * sh;
  __nv_bfloat162 mn[4], mx[4];
  const __nv_bfloat162 pinf = __floats2bfloat162_rn(INFINITY, INFINITY), ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mn[i] = pinf;
    mx[i] = ninf;
  }
  const int k_end = min(Sk, (j + 1) * blk);
  if (r0 < rows_par) {
    for (int kk = j * blk + r0; kk < k_end; kk += rows_par) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)kk * ss) + ch);
      const __nv_bfloat162* v = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mn[i] = __hmin2(mn[i], v[i]);
        mx[i] = __hmax2(mx[i], v[i]);
      }
    }
  }
  red_min[t] = *reinterpret_cast<uint4*>(mn);
  red_max[t] = *reinterpret_cast<uint4*>(mx);
  __syncthreads();
  if (t < nch) {
    for (int r = 1; r < rows_par; ++r) {
      const uint4 a = red_min[r * nch + t], z = red_max[r * nch + t];
      const __nv_bfloat162* va = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* vz = reinterpret_cast<const __nv_bfloat162*>(&z);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mn[i] = __hmin2(mn[i], va[i]);
        mx[i] = __hmax2(mx[i], vz[i]);
      }
    }
    const int64_t o = ((int64_t)bgh * nkb + j) * D;
    reinterpret_cast<uint4*>(kmin + o)[t] = *reinterpret_cast<uint4*>(mn);
    reinterpret_cast<uint4*>(kmax + o)[t] = *reinterpret_cast<uint4*>(mx);
  }
}

cudaError_t launch_rsa_summaries(const void* k, int64_t sb, int64_t sg, int64_t sh, int64_t ss, int B, int G, int H,
                                 int Sk, int D, int blk, int j0, void* kmin, void* kmax, cudaStream_t stream) {
  const int nkb = (Sk + blk - 1) / blk;
  if (j0 >= nkb) return cudaSuccess;
  dim3 grid(nkb - j0, B * G * H);
  rsa_summaries_kernel<<<grid, 128, 0, stream>>>(static_cast<const __nv_bfloat16*>(k), sb, sg, sh, ss, B, G, H, Sk,
                                                 D, blk, j0, static_cast<__nv_bfloat16*>(kmin),
                                                 static_cast<__nv_bfloat16*>(kmax));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ selection
// Pipelined, warp-specialised: 128 x (1 + kSelWG) threads, one CTA per SM, each CTA a contiguous range of
// (b, g, h_kv, q-block) pairs (x grp heads), so the summaries of a (b, g, h_kv) are loaded once
// per CTA per head it touches.
//   warps 4-7 ("split" WG): q+ / q- split of the landed Q tile into the operand buffers; its
//     thread 0 also issues the TMA loads (next Q tile into a separate raw buffer, summaries)
//     and the tcgen05 MMAs into a double-buffered TMEM accumulator;
//   warps 0-3, 8-11, 12-15, 16-19 ("select" WGs, thread = TMEM lane = KV block, round-robin items when GQA groups
//     do not span items): row max over the block's queries, running max over the heads of a GQA
//     group, exact radix top-k, ascending list.
// So the split of item n+1, the MMAs of item n+1 and the selection of item n overlap.
// Select warpgroups per CTA (up to kSelWG, as many as the shared memory admits): the accumulator is
// released right after the row max, so the top-k of several items runs concurrently; the radix passes
// are barrier / latency bound, not ALU bound.
#ifndef FL_SEL_WG
#define FL_SEL_WG 2
#endif
constexpr int kSelWG = FL_SEL_WG;
constexpr int kSelThreads = 128 * (kSelWG + 1);

template <int D>
struct SelCfg {
  static constexpr int CH = 64;                         // bf16 per 128-byte swizzle row
  static constexpr int NCH = D / CH;
  static constexpr int CHUNK = 128 * 128;               // one 128-row x 128-byte swizzle slab
  static constexpr int QTILE = NCH * CHUNK;             // one 128 x D tile
  static constexpr uint32_t IDESC = idesc_bf16_f32(128, 128, 0);
  // summaries (kmax, kmin) + raw Q + q+ / q- tiles + per-select-warpgroup scratch (256-bin histogram as
  // 16-bit counts, pass state, selection bitmap) + barriers + alignment slack
  static constexpr int SCR_WORDS = 128 + 16 + 16;
  static int scratch(int nsel) { return nsel * SCR_WORDS * 4; }
  static int smem(int n_mt, int nsel) { return 2 * n_mt * QTILE + 3 * QTILE + scratch(nsel) + 128 + 1024; }
};

template <int D>
__global__ void __launch_bounds__(kSelThreads, 1)
    rsa_select_kernel(const __grid_constant__ RsaSelParams p, const __grid_constant__ CUtensorMap tq,
                      const __grid_constant__ CUtensorMap tmin, const __grid_constant__ CUtensorMap tmax, int n_sel_wg) {
  using C = SelCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SW128 atoms); offset arithmetic on smem_raw keeps the shared address space visible
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int n_mt = (p.nkb + 127) / 128;
  const int nbuf = n_mt <= 2 ? 2 : 1;                   // TMEM accumulators in flight (512 columns)
  uint8_t* sMax = smem;                                 // [n_mt][NCH] slabs
  uint8_t* sMin = sMax + n_mt * C::QTILE;
  uint8_t* sQraw = sMin + n_mt * C::QTILE;              // TMA destination of the next Q tile
  uint8_t* sQp = sQraw + C::QTILE;
  uint8_t* sQn = sQp + C::QTILE;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sQn + C::QTILE);   // [n_sel_wg][SCR_WORDS], one per select WG
  uint64_t* bars = reinterpret_cast<uint64_t*>(scratch + n_sel_wg * C::SCR_WORDS);
  uint64_t* bar_sum = bars;                             // summaries landed
  uint64_t* bar_q = bars + 1;                           // raw Q tile landed
  uint64_t* bar_qfree = bars + 2;                       // MMAs of the previous item done (q+/q-, summaries free)
  // accumulator ready, one barrier per select warpgroup: with more select warpgroups than accumulator
  // buffers a per-buffer barrier would be waited phases ahead (parity aliasing); per warpgroup its k-th
  // item is its barrier's phase k
  uint64_t* mma_done = bars + 3;                        // [kSelWG]
  uint64_t* acc_empty = bars + 3 + kSelWG;              // [2] accumulator read by the select WG
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5 + kSelWG);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int64_t n_pairs = (int64_t)p.B * p.G * p.Hkv * p.nqb;
  const int64_t pb = n_pairs * blockIdx.x / gridDim.x, pe = n_pairs * (blockIdx.x + 1) / gridDim.x;
  const int n_items = (int)(pe - pb) * p.grp;           // (pair, head in group)
  const int n_mt0 = (p.nkb + 127) / 128;
  // select warpgroups taking items round-robin (each with its own TMEM buffer use and no GQA group
  // spanning items), else one warpgroup takes every item
  const int nsel_items = (n_mt0 <= 2 && p.grp == 1) ? n_sel_wg : 1;

  if (t == 0) {
    mbar_init(bar_sum, 1);
    mbar_init(bar_q, 1);
    mbar_init(bar_qfree, 1);
    for (int i = 0; i < 2; ++i) mbar_init(&acc_empty[i], 128);
    for (int i = 0; i < kSelWG; ++i) mbar_init(&mma_done[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto item_pair = [&](int n) { return pb + n / p.grp; };
  auto item_bgk = [&](int n) { return (int)(item_pair(n) / p.nqb); };
  auto item_qblk = [&](int n) { return (int)(item_pair(n) % p.nqb); };
  auto item_head = [&](int n) { return (item_bgk(n) % p.Hkv) * p.grp + n % p.grp; };
  // candidates 1 <= j < c, c = the diagonal block of the q-block's last row (reading G10)
  auto diag = [&](int i) {
    const int q_last = min(p.Sq, (i + 1) * 128) - 1;
    const int q_last_abs = q_last + p.q_off;
    const int c = q_last_abs < 0 ? 0 : q_last_abs / 128;
    return min(c, p.nkb - 1);
  };
  // candidates j = 1 .. c-1 live in accumulator tiles 0 .. (c-1)/128, i.e. ceil(c / 128) tiles
  auto n_mt_of = [&](int c) { return c >= 2 ? (c + 127) / 128 : 0; };

  if (warp >= 4 && warp < 8) {
    // ============================== split + TMA + MMA ==============================
    const int st = t - 128;
    int cur_bgk = -1, sum_phase = 0;
    auto load_q = [&](int n) {
      const int bgk = item_bgk(n);
      const int g = (bgk / p.Hkv) % p.G, b = bgk / (p.Hkv * p.G);
      const int gq = p.q_bcast_g ? 0 : g, bq = p.q_bcast_b ? 0 : b;
      mbar_arrive_expect_tx(bar_q, C::QTILE);
      for (int c = 0; c < C::NCH; ++c)
        tma_load_5d(sQraw + c * C::CHUNK, &tq, bar_q, c * C::CH, item_qblk(n) * 128, item_head(n), gq, bq);
    };
    if (st == 0 && n_items > 0) {
      tma_prefetch_desc(&tq);
      tma_prefetch_desc(&tmin);
      tma_prefetch_desc(&tmax);
      load_q(0);
    }
    for (int n = 0; n < n_items; ++n) {
      mbar_wait(bar_q, n & 1);                            // raw Q(n) landed
      if (n > 0) mbar_wait(bar_qfree, (n - 1) & 1);       // MMAs of n-1 have read q+ / q-
      {
        const uint4* src = reinterpret_cast<const uint4*>(sQraw);
        uint4* dp = reinterpret_cast<uint4*>(sQp);
        uint4* dn = reinterpret_cast<uint4*>(sQn);
        const __nv_bfloat162 z = __floats2bfloat162_rn(0.f, 0.f);
#pragma unroll 4
        for (int e = st; e < C::QTILE / 16; e += 128) {
          uint4 u = src[e], up, un;
          const __nv_bfloat162* v = reinterpret_cast<const __nv_bfloat162*>(&u);
          __nv_bfloat162* vp = reinterpret_cast<__nv_bfloat162*>(&up);
          __nv_bfloat162* vn = reinterpret_cast<__nv_bfloat162*>(&un);
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            vp[w] = __hmax2(v[w], z);
            vn[w] = __hmin2(v[w], z);
          }
          dp[e] = up;
          dn[e] = un;
        }
      }
      fence_proxy_async_smem();                           // generic writes -> tensor-core reads
      named_bar_sync(1, 128);
      if (st == 0) {
        if (n + 1 < n_items) load_q(n + 1);               // the raw buffer has been read
        const int bgk = item_bgk(n);
        if (bgk != cur_bgk) {                             // MMAs of n-1 are done (bar_qfree above)
          mbar_arrive_expect_tx(bar_sum, 2 * n_mt * C::QTILE);
          for (int m = 0; m < n_mt; ++m)
            for (int c = 0; c < C::NCH; ++c) {
              tma_load_5d(sMax + (m * C::NCH + c) * C::CHUNK, &tmax, bar_sum, c * C::CH, m * 128, bgk, 0, 0);
              tma_load_5d(sMin + (m * C::NCH + c) * C::CHUNK, &tmin, bar_sum, c * C::CH, m * 128, bgk, 0, 0);
            }
          mbar_wait(bar_sum, sum_phase & 1);
          ++sum_phase;
          cur_bgk = bgk;
        }
        const int buf = n % nbuf;
        if (n >= nbuf) mbar_wait(&acc_empty[buf], ((n / nbuf) - 1) & 1);
        tc_fence_after();
        const int n_mt_i = n_mt_of(diag(item_qblk(n)));
        const uint32_t acc = tmem + buf * n_mt * 128;
        const uint32_t ap = smem_u32(sMax), an = smem_u32(sMin), bp = smem_u32(sQp), bn = smem_u32(sQn);
        for (int m = 0; m < n_mt_i; ++m) {
#pragma unroll
          for (int kk = 0; kk < 2 * D / 16; ++kk) {
            const int kd = kk % (D / 16);                  // K step within the half
            const uint32_t off = (kd * 16 / C::CH) * C::CHUNK + (kd * 16 % C::CH) * 2;
            const uint32_t a = (kk < D / 16 ? ap : an) + m * C::QTILE + off;
            const uint32_t bb = (kk < D / 16 ? bp : bn) + off;
            umma_ss(acc + m * 128, smem_desc(a, 16, 1024, kLayoutSW128), smem_desc(bb, 16, 1024, kLayoutSW128),
                    C::IDESC, kk > 0);
          }
        }
        umma_commit(&mma_done[n % nsel_items]);
        umma_commit(bar_qfree);
      }
    }
  } else {
    // ============================== selection (thread = KV block) ==============================
    // kSelWG select warpgroups (warps 0-3, 8-11, ...) take items round-robin when each item has its own TMEM
    // accumulator buffer and no GQA group spans items; otherwise warps 0-3 take every item.
    const int sel = warp < 4 ? 0 : (warp - 4) / 4;      // warps 0-3, 8-11, 12-15, ...
    const int nsel = nsel_items;
    const int tt = t & 127, wq = warp & 3;              // thread / warp within the select warpgroup
    uint32_t* hist = scratch + sel * C::SCR_WORDS;      // [128] packed 16-bit bin counts
    uint32_t* rstate = hist + 128;                      // [16] digit / counts of the current pass
    uint32_t* flags = hist + 144;                       // [16] selection bitmap
    const uint32_t bar_id = 2 + sel;
    float run0 = -INFINITY, run1 = -INFINITY, run2 = -INFINITY, run3 = -INFINITY;  // block j = m*128 + tt
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    for (int n = sel; n < n_items && sel < nsel; n += nsel) {
      const int i = item_qblk(n);
      const int bgk = item_bgk(n);
      const int hk = bgk % p.Hkv, g = (bgk / p.Hkv) % p.G, b = bgk / (p.Hkv * p.G);
      const int h_in_grp = n % p.grp;
      const int c = diag(i);
      const int n_mt_i = n_mt_of(c);
      const int buf = n % nbuf;
      mbar_wait(&mma_done[sel], (n / nsel) & 1);
      tc_fence_after();
      // ---- row max over the block's valid queries: thread t owns blocks m*128 + t
      const int nvalid = min(128, p.Sq - i * 128);
      const uint32_t acc = tmem + buf * n_mt * 128;
      float mine[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (m >= n_mt_i) break;
        float mx0 = -INFINITY, mx1 = -INFINITY;
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(acc + lane_base + m * 128 + c0, r);
          tmem_wait_ld();
          if (c0 + 32 <= nvalid) {                        // warp-uniform: every query of the chunk is valid
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              mx0 = fmax3(mx0, __uint_as_float(r[e]), __uint_as_float(r[e + 1]));
              mx1 = fmax3(mx1, __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c0 + e < nvalid) mx0 = fmaxf(mx0, __uint_as_float(r[e]));
          }
        }
        mine[m] = fmaxf(mx0, mx1);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);                       // the accumulator may take item n + nbuf
      if (h_in_grp == 0) {
        run0 = mine[0]; run1 = mine[1]; run2 = mine[2]; run3 = mine[3];
      } else {
        run0 = fmaxf(run0, mine[0]); run1 = fmaxf(run1, mine[1]);
        run2 = fmaxf(run2, mine[2]); run3 = fmaxf(run3, mine[3]);
      }
      if (h_in_grp == p.grp - 1) {
        // ---- top-k over candidates 1 <= j < c (ties toward the lower j, G11) by an exact radix select:
        // order-preserving 32-bit keys of the scores, MSB-first 8-bit digits with a 256-bin histogram
        // per pass, stopping once the threshold bin is taken whole; exact ties at the threshold go to
        // the lowest j.  Thread t holds the scores of blocks m*128 + t in registers.
        const float runs[4] = {run0, run1, run2, run3};
        uint32_t key[4];
        bool cand[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int j = m * 128 + tt;
          cand[m] = m < n_mt && j >= 1 && j < c;
          const uint32_t bits = __float_as_uint(runs[m] + 0.f);     // -0 -> +0 (equal scores tie)
          key[m] = bits ^ ((bits >> 31) ? 0xFFFFFFFFu : 0x80000000u);
        }
        const int ncand = c >= 2 ? c - 1 : 0;
        const bool take_all = ncand <= p.topk, take_none = p.topk <= 0;
        uint32_t P = 0u, M = 0u;
        int krem = p.topk;
        if (!take_all && !take_none) {
          for (int pass = 0; pass < 4; ++pass) {
            const int shift = 24 - 8 * pass;
            hist[tt] = 0u;
            named_bar_sync(bar_id, 128);
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (cand[m] && (key[m] & M) == P) {
                const uint32_t d = (key[m] >> shift) & 255u;
                atomicAdd(&hist[d >> 1], 1u << ((d & 1u) * 16));   // two 16-bit bins per word (<= 512 keys)
              }
            named_bar_sync(bar_id, 128);
            if (wq == 0) {                                // lane l owns bins [8l, 8l + 8); count from the top
              uint32_t cnts[8], lsum = 0u;
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                cnts[e] = (hist[4 * lane + (e >> 1)] >> ((e & 1) * 16)) & 0xFFFFu;
                lsum += cnts[e];
              }
              uint32_t suf = lsum;                        // keys in bins of lanes >= lane
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 32) suf += v;
              }
              const uint32_t above = suf - lsum;
              if (above < (uint32_t)krem && (uint32_t)krem <= suf) {
                uint32_t acc = above, d = 0u, in_bin = 0u;
                bool found = false;
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                  if (!found && acc + cnts[e] >= (uint32_t)krem) {
                    d = 8u * lane + e;
                    in_bin = cnts[e];
                    found = true;
                  } else if (!found) {
                    acc += cnts[e];
                  }
                }
                rstate[0] = d;
                rstate[1] = acc;                          // keys above the threshold digit
                rstate[2] = in_bin;
              }
            }
            named_bar_sync(bar_id, 128);
            const uint32_t d = rstate[0];
            krem -= (int)rstate[1];
            const bool whole = rstate[2] == (uint32_t)krem;
            P |= d << shift;
            M |= 0xFFu << shift;
            if (whole) break;                             // the threshold bin is selected entirely
          }
        }
        // keys equal to the threshold prefix: the lowest-j krem of them (all of them unless exact ties)
        bool eq[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          eq[m] = !take_all && !take_none && cand[m] && (key[m] & M) == P;
          const uint32_t bal = __ballot_sync(0xffffffffu, eq[m]);
          if (lane == 0) hist[m * 4 + wq] = bal;          // the histogram is dead after the last pass
        }
        if (tt < 16) flags[tt] = 0u;
        named_bar_sync(bar_id, 128);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int j = m * 128 + tt;
          bool sel = false;
          if (m < n_mt && j < p.nkb && j <= c) {
            if (j == 0 || j == c) {
              sel = true;
            } else if (cand[m]) {
              if (take_all) {
                sel = true;
              } else if (!take_none) {
                const uint32_t pref = key[m] & M;
                if (pref > P) {
                  sel = true;
                } else if (eq[m]) {
                  const int w = j >> 5;
                  int tr = __popc(hist[w] & ((1u << (j & 31)) - 1u));
                  for (int ww = 0; ww < w; ++ww) tr += __popc(hist[ww]);
                  sel = tr < krem;
                }
              }
            }
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, sel);
          if (lane == 0) flags[m * 4 + wq] = bal;
        }
        named_bar_sync(bar_id, 128);
        int cnt = 0;
        for (int w = 0; w < 16; ++w) cnt += __popc(flags[w]);
        for (int hh = 0; hh < p.grp; ++hh) {
          const int64_t row = (((int64_t)b * p.G + g) * p.Hq + hk * p.grp + hh) * p.nqb + i;
          int32_t* out = p.blk_idx + row * p.max_sel;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int j = m * 128 + tt;
            const int w = j >> 5;
            if (m < n_mt && ((flags[w] >> (j & 31)) & 1u)) {
              int pos = __popc(flags[w] & ((1u << (j & 31)) - 1u));
              for (int ww = 0; ww < w; ++ww) pos += __popc(flags[ww]);
              if (pos < p.max_sel) out[pos] = j;
            }
          }
          for (int e = cnt + tt; e < p.max_sel; e += 128) out[e] = -1;
          if (tt == 0) p.blk_cnt[row] = min(cnt, p.max_sel);
        }
        named_bar_sync(bar_id, 128);                           // sc / flags reuse
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int rsa_select_max_blocks(int D) { return D == 128 ? 256 : 512; }

cudaError_t launch_rsa_select(const RsaSelParams& p0, const CUtensorMap& tq, const CUtensorMap& tmin,
                              const CUtensorMap& tmax, cudaStream_t stream) {
  RsaSelParams p = p0;
  p.parts = 1;
  const long long pairs = (long long)p.B * p.G * p.Hkv * p.nqb;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<long long>(pairs, sms > 0 ? sms : 148);   // persistent: one CTA per SM
  if (grid <= 0) return cudaSuccess;
  const int n_mt = (p.nkb + 127) / 128;
  int smem_max = 0;
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int nsel = kSelWG;
  auto fits = [&](int ns) { return (p.D == 128 ? SelCfg<128>::smem(n_mt, ns) : SelCfg<64>::smem(n_mt, ns)) <= smem_max; };
  while (nsel > 1 && !fits(nsel)) --nsel;
  const int threads = 128 * (nsel + 1);
  if (p.D == 128) {
    const int sm = SelCfg<128>::smem(n_mt, nsel);
    cudaError_t e = cudaFuncSetAttribute(rsa_select_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return e;
    rsa_select_kernel<128><<<grid, threads, sm, stream>>>(p, tq, tmin, tmax, nsel);
  } else {
    const int sm = SelCfg<64>::smem(n_mt, nsel);
    cudaError_t e = cudaFuncSetAttribute(rsa_select_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return e;
    rsa_select_kernel<64><<<grid, threads, sm, stream>>>(p, tq, tmin, tmax, nsel);
  }
  return cudaGetLastError();
}

}  // namespace fl
