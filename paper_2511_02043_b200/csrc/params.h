// params.h -- device-side problem description built by host.cu from fl_attn_args
// (include/fl_attn.h).  One struct for every kernel of the attention family; it is
// passed by value as a __grid_constant__ kernel parameter.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace fl {

enum Mod : int32_t { MOD_NONE = 0, MOD_ALIBI = 1, MOD_SOFTCAP = 2 };
enum Mask : int32_t { MASK_NONE = 0, MASK_CAUSAL = 1, MASK_SLIDING = 2, MASK_PREFIX = 3, MASK_DOCUMENT = 4,
                      MASK_BLOCKLIST = 5 };
enum Gate : int32_t { GATE_NONE = 0, GATE_MUL = 1, GATE_SIGMOID = 2 };

struct Strided5 {          // element strides of a [B,G,H,S,D] view
  int64_t b, g, h, s, d;
};

struct AttnParams {
  // ---- shape (rank-4 inputs have G = 1)
  int32_t B, G, Hq, Hkv, Sq, Sk, Dqk, Dv;
  int32_t maps;            // 2 for differential attention, else 1
  int32_t grp;             // Hq / Hkv (G15)
  int32_t q_off;           // Sk - Sq for bottom-right alignment (G12), 0 for top-left
  // ---- data (device pointers) and strides
  const void* q; const void* k; const void* v; void* o;
  Strided5 qs, ks, vs, os;
  float* lse; Strided5 lses;       // lse [B,G,H,S] (d unused)
  // ---- score modification (Eq.4), in the log2 domain where noted
  float scale;             // softmax scale (G1)
  float scale_log2;        // scale * log2(e)
  int32_t mod;
  float softcap;           // cap
  const float* alibi;      // [Hq] slopes or nullptr (default 2^(-8(h+1)/Hq))
  // ---- masking
  int32_t mask, window, prefix;
  const int32_t* doc_offsets; int32_t n_docs; int64_t doc_stride_b; int32_t doc_causal;
  const void* bias; int32_t bias_dtype; int32_t bias_vec; Strided5 bs;  // bias [B,G,H,Sq,Sk] (d = key stride);
                                                               // bias_vec: bf16, key-contiguous, 16-B aligned rows
  const uint32_t* keybits; int32_t keybits_words;              // packed key mask [B*G][words] (workspace)
  // ---- gate / diff
  int32_t gate_mode; const void* gate; Strided5 gs; int32_t gate_dtype;
  float lambda; const float* lambda_h;
  // DIFF-Transformer epilogue (NEXT-2): lambda re-parameterisation [4][Dqk] and per-head RMSNorm
  const float* lambda_qk; float lambda_init; int32_t diff_norm; float diff_norm_eps; const float* diff_norm_w;
  // ---- block list (RSA)
  const int32_t* blk_idx; const int32_t* blk_cnt; int32_t blk_q, blk_k, max_sel, n_qblk;
  // ---- paged KV: logical KV tile t of batch b is page page_table[b * page_stride + t] of the k/v pools
  const int32_t* page_table; int64_t page_stride;
  int32_t in_dtype;        // 0 bf16, 1 f32
  int32_t* tile_ctr;       // bf16 path: persistent-scheduler ticket counter (workspace, zeroed per call)
  // bf16 small heads (attn_tc.cuh): 0 = (b, g, h)-major units claimed by tickets; 1 = pair bias resident in
  // TMEM (Evoformer rows): (b, h, q-block) segments with the G pairs minor, static contiguous chunks per CTA
  int32_t unit_order;
  // backward only: add this call's dV and dgate to the values already in dv / dgate (the second map of a
  // differential attention: the maps share V and the gate) instead of overwriting them
  int32_t grad_accum;
};

// lambda of head h (Listing 4's lambda_full, G8): re-parameterised from lambda_qk when given (NEXT-2:
// exp(q1 . k1) - exp(q2 . k2) + lambda_init), else the per-head or scalar value.
#ifdef __CUDACC__
__device__ inline float diff_lambda(const AttnParams& p, int h) {
  if (p.lambda_qk) {
    float d1 = 0.f, d2 = 0.f;
    for (int d = 0; d < p.Dqk; ++d) {
      d1 = fmaf(p.lambda_qk[d], p.lambda_qk[p.Dqk + d], d1);
      d2 = fmaf(p.lambda_qk[2 * p.Dqk + d], p.lambda_qk[3 * p.Dqk + d], d2);
    }
    return expf(d1) - expf(d2) + p.lambda_init;
  }
  return p.lambda_h ? p.lambda_h[h] : p.lambda;
}
#endif

// TMA (row, batch) coordinates of logical KV tile `tile` of batch b: contiguous K/V -> (128 tile, b);
// paged K/V -> (0, page) with page = page_table[b, tile] (the pool's batch dim indexes pages).
#ifdef __CUDACC__
__device__ __forceinline__ void kv_tile_coords(const AttnParams& p, int b, int tile, int bb, int& row, int& bcoord) {
  if (p.page_table) {
    row = 0;
    bcoord = __ldg(p.page_table + (int64_t)b * p.page_stride + tile);
  } else {
    row = tile * 128;
    bcoord = bb;
  }
}
#endif

// TMA tensor maps for the tcgen05 kernel family (5-D: D, S, H, G, B).
struct TmaMaps {
  CUtensorMap q, k, v;
  // dims whose tensor-map extent was collapsed to 1 because the view broadcasts
  // them (stride 0): the kernel passes coordinate 0 there.
  int32_t q_bcast_g, q_bcast_b, k_bcast_g, k_bcast_b, v_bcast_g, v_bcast_b;
  // additive bias through TMA (D = 32 kernels, bf16 key-contiguous bias): dims (S_k, S_q, H, G, B)
  CUtensorMap bias;
  int32_t bias_tma, bias_bcast_g, bias_bcast_b;
};

// Fused LayerNorm-prologue linear layer (linear.cu, NEXT-2), built by host.cu's fl_linear.
struct LinParams {
  int32_t M, N, K, NT;       // NT: output columns per tile (multiple of 16, <= 128)
  const float* bias;         // [N] or nullptr
  const float* ln_g;         // [K] or nullptr (no LayerNorm)
  const float* ln_b;         // [K] or nullptr
  float eps;
  void* y;                   // bf16
  int64_t ys_m, ys_n;        // element strides of y
};

// Invariant Point Attention core (ipa.cu, NEXT-4), built by host.cu's fl_ipa_fwd.
struct IpaParams {
  int N, H, c, Pq, Pv, cz;
  const __nv_bfloat16 *q, *k, *qp, *kp, *vp, *bias, *z;   // contiguous: [N,H,c], [N,H,P,3], [H,N,N], [N,N,cz]
  const float *R, *t, *gamma;                              // [N,3,3] (x_global = R x + t), [N,3], [H]
  __nv_bfloat16 *qa, *ka;                                  // augmented Q', K' [N,H,64]
  float* gv;                                               // global value points T_j v_jp [N,H,Pv*3]
  __nv_bfloat16* bias_s;                                   // w_L b [H,N,N] (bf16: the attention's vector bias path)
};

// RSA block selection (rsa.cu), built by host.cu's fl_rsa_select.
struct RsaSelParams {
  int B, G, Hq, Hkv, grp, Sq, Sk, D, nkb, nqb, topk, max_sel, q_off, parts;
  int32_t* blk_idx;  // [B*G*Hq][nqb][max_sel]
  int32_t* blk_cnt;  // [B*G*Hq][nqb]
  int q_bcast_g, q_bcast_b;
};

}  // namespace fl
