/*
 * fl_attn.h -- C ABI of the B200-native (sm_100a) fused attention-variant
 * forward: the data-parallel hot path of Flashlight (arXiv 2511.02043).
 *
 * "P:Lnnn" cites /root/reference/PAPER.md line nnn (section / equation /
 * listing named beside it); "Gnn" is a reading of an ambiguous passage listed
 * in DESIGN.md §Readings.
 *
 * What one call computes (per output row b, g, h, q; the kernel fuses all of
 * it, one pass over K/V with the online softmax of Alg.2):
 *   s_k  = scale * <Q[b,g,h,q,:], K[b,g,h_kv,k,:]>      Eq.3, Listing 1
 *   s_k  = score_mod(s_k)                              Eq.4 P:L251-257 (ALiBi, softcap, bias)
 *   s_k  = -inf where masked                           Listing 1, Listing 2
 *   P    = softmax_k(s)   ;   O = P V                  Eq.2/Eq.3
 *   diff : O = A_0 - lambda_h A_1                      Listing 4 P:L412-424 (G8)
 *   gate : O = O * sigmoid(G)  |  O * G                Evoformer P:L865 (G9)
 *
 * Conventions (all functions):
 *  - All symbols are extern "C"; structs are POD; no exception crosses the ABI.
 *  - OWNERSHIP: the caller owns every buffer.  The library never allocates or
 *    frees device memory, never synchronises, never changes the current device.
 *    Device pointers must be on the current device.
 *  - ASYNCHRONY: work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and the call returns.  Launch failures return FL_ERR_CUDA
 *    with the CUDA error text in fl_last_error(); device faults surface at the
 *    caller's next synchronisation.
 *  - VALIDATION is all-or-nothing: on any non-OK status nothing is enqueued and
 *    no output is touched.  Unsupported combinations return FL_ERR_UNSUPPORTED
 *    and a reason in fl_last_error().  There is NO fallback path of any kind
 *    (no CPU path, no second backend).
 *  - Thread safety: every call is re-entrant; the only global state is the
 *    once-resolved driver entry point (cuTensorMapEncodeTiled) and the
 *    thread-local error string.
 */
#ifndef FL_ATTN_H
#define FL_ATTN_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define FL_ABI_VERSION 4

typedef enum {
  FL_OK = 0,
  FL_ERR_INVALID_ARGUMENT = 1, /* null/inconsistent descriptor, bad enum, pointer not on device */
  FL_ERR_UNSUPPORTED = 2,      /* valid but not implemented (reason in fl_last_error) */
  FL_ERR_MISALIGNED = 3,       /* TMA needs 16-B aligned base and 16-B multiple strides */
  FL_ERR_SHAPE_MISMATCH = 4,   /* q/k/v/o/bias/gate/lse shapes disagree */
  FL_ERR_WORKSPACE = 5,        /* workspace too small */
  FL_ERR_CUDA = 6,             /* CUDA runtime/driver error (text in fl_last_error) */
  FL_ERR_ABI_VERSION = 7       /* abi_version != FL_ABI_VERSION */
} fl_status;

typedef enum { FL_BF16 = 0, FL_F32 = 1, FL_U8 = 2, FL_I32 = 3 } fl_dtype;

/* A strided view.  rank <= 5, sizes/strides in ELEMENTS, stride 0 broadcasts a
 * dim.  data == NULL means "absent".  The last dim of q/k/v/o/gate must be
 * contiguous (stride 1). */
typedef struct {
  void* data;
  int32_t dtype;     /* fl_dtype */
  int32_t rank;
  int64_t size[5];
  int64_t stride[5];
} fl_tensor;

typedef enum { FL_MOD_NONE = 0, FL_MOD_ALIBI = 1, FL_MOD_SOFTCAP = 2 } fl_mod;
typedef enum {
  FL_MASK_NONE = 0,
  FL_MASK_CAUSAL = 1,    /* keep k <= q_abs                                  */
  FL_MASK_SLIDING = 2,   /* keep k <= q_abs && q_abs - k <= window  (G4) */
  FL_MASK_PREFIX = 3,    /* keep k < prefix_len || k <= q_abs       (G5)       */
  FL_MASK_DOCUMENT = 4,  /* keep doc(k) == doc(q_abs) [&& k <= q_abs]  (G6)    */
  FL_MASK_BLOCKLIST = 5  /* keep floor(k/blk_k) in list[b,h,floor(q/blk_q)] && k <= q_abs (RSA, G10) */
} fl_mask;
typedef enum { FL_GATE_NONE = 0, FL_GATE_MUL = 1, FL_GATE_SIGMOID = 2 } fl_gate;

/* The variant descriptor (BASELINE.json north_star: "mod type, mask,
 * bias/gate tensors, diff-lambda, sparse block list").  Zero-initialise it
 * and set abi_version; every field's zero value means "off". */
typedef struct {
  uint32_t abi_version;      /* must equal FL_ABI_VERSION */
  float scale;               /* 0 -> 1/sqrt(D_qk)  (Listing 1, G1) */
  int32_t mod;               /* fl_mod; acts on the SCALED score (Eq.4) */
  float softcap;             /* FL_MOD_SOFTCAP: s <- softcap * tanh(s / softcap)   (G3) */
  fl_tensor alibi_slopes;    /* FL_MOD_ALIBI: f32 [Hq]; absent -> 2^(-8(h+1)/Hq); s += slope_h (k - q_abs) (G2) */
  int32_t mask;              /* fl_mask */
  int32_t window;            /* FL_MASK_SLIDING window w (inclusive: w+1 keys incl. the diagonal) */
  int32_t prefix_len;        /* FL_MASK_PREFIX P */
  fl_tensor doc_offsets;     /* FL_MASK_DOCUMENT: i32 [B, n_docs+1], 0 = off[0] < ... < off[n_docs] = S_k */
  int32_t doc_causal;        /* FL_MASK_DOCUMENT: also require k <= q_abs */
  int32_t causal_align;      /* 0: bottom-right q_abs = q + S_k - S_q (G12); 1: top-left q_abs = q */
  fl_tensor bias;            /* optional additive score bias, same rank as q: [B,Hq,S_q,S_k] or [B,G,Hq,S_q,S_k],
                                bf16 or f32, broadcast by stride 0 (Evoformer pair bias [b,h,i,j] broadcast over
                                G = s) */
  fl_tensor key_mask;        /* optional u8, rank(q)-2: [B,S_k] or [B,G,S_k]; 1 = keep (Evoformer MSA mask, G9) */
  int32_t gate_mode;         /* fl_gate */
  fl_tensor gate;            /* gate logits/values, same logical shape as o */
  int32_t diff;              /* differential attention: q,k carry 2*H heads, map i = heads [iH,(i+1)H) (G8) */
  float lambda;              /* diff: lambda_full (Listing 4 P:L431 uses 0.2) */
  fl_tensor lambda_h;        /* diff: optional f32 [Hq] per-head lambda (overrides lambda) */
  fl_tensor blk_idx;         /* FL_MASK_BLOCKLIST: i32 [B*(G)*Hq, n_qblk, max_sel], ascending, -1 padded */
  fl_tensor blk_cnt;         /* FL_MASK_BLOCKLIST: i32 [B*(G)*Hq, n_qblk] */
  int32_t blk_q;             /* FL_MASK_BLOCKLIST query block (must be 128) */
  int32_t blk_k;             /* FL_MASK_BLOCKLIST key block (must be 128) */
  /* Paged KV (serving-side RSA): when kv_page_table.data != NULL, k and v are page
   * POOLS of rank 4 [n_pages, Hkv(x2 if diff), 128, D] (one 128-key page per KV tile, any page order),
   * and logical KV tile t of batch b (keys [128 t, 128 t + 128)) is page kv_page_table[b, t].  i32
   * [B, n_pages_per_seq], contiguous rows; the logical key count S_k is kv_len (<= 128 n_pages_per_seq).
   * bf16 only, rank-4 q only (G = 1); every mask incl. block lists, and the split-KV decode path. */
  fl_tensor kv_page_table;
  int32_t kv_len;
  /* DIFF-Transformer epilogue (reading G8b, external: Ye et al. 2024), diff only:
   *   lambda_qk (optional f32 [4, D_qk] = lambda_q1, lambda_k1, lambda_q2, lambda_k2): the re-parameterised
   *     lambda = exp(lambda_q1 . lambda_k1) - exp(lambda_q2 . lambda_k2) + lambda_init, overriding
   *     lambda / lambda_h;
   *   diff_norm = 1: O <- (1 - lambda_init) * RMSNorm(A_0 - lambda A_1) per output row and head, over D_v,
   *     RMSNorm(x) = x / sqrt(mean_d x_d^2 + diff_norm_eps) * w, w = diff_norm_w f32 [D_v] (absent: ones). */
  fl_tensor lambda_qk;
  float lambda_init;
  int32_t diff_norm;
  float diff_norm_eps;
  fl_tensor diff_norm_w;
} fl_variant;

typedef struct {
  /* rank 4 [B,H,S,D] or rank 5 [B,G,H,S,D]; any strides with a contiguous last dim.
   * q [..,Hq(x2 if diff),S_q,D_qk]; k [..,Hkv(x2 if diff),S_k,D_qk]; v [..,Hkv,S_k,D_v];
   * o [..,Hq,S_q,D_v].  Hq % Hkv == 0; query head h reads KV head floor(h/(Hq/Hkv)) (G15). */
  fl_tensor q, k, v, o;
  fl_tensor lse;             /* optional f32 [B,(G,)Hq,S_q]: natural-log LSE of the scaled, modified scores (G19) */
  fl_variant var;
  void* stream;              /* cudaStream_t */
  void* workspace;           /* device scratch (see fl_attn_workspace_size); never allocated here */
  size_t workspace_bytes;
} fl_attn_args;

/* Supported set (ABI v2 = v1 + paged KV; v3 = v2 + the backward's dgate and fl_linear):
 *   f32 q/k/v/o  : exact-fp32 SIMT path, every variant, D_qk, D_v <= 128.
 *   bf16 q/k/v/o : tcgen05/TMEM/TMA persistent kernel, D_qk == D_v in {32, 64, 128}; every mask,
 *                  mod, bias, key_mask, gate; diff (lse must be absent with diff).  FL_MASK_BLOCKLIST
 *                  on bf16: blk_q == blk_k == 128, max_sel <= 256, no diff, no bias.
 *                  Short query blocks (S_q <= 16, no diff / bias / gate, D in {64, 128}) take the
 *                  split-KV decode kernels (a split pass + a combine pass) instead.
 * Launches per call: 1 attention kernel (2 on the split-KV path), +1 key-mask pack kernel when a
 * key mask is given, + a 4-byte stream-ordered memset of the scheduler counter (bf16).
 * Empty work (B*G*Hq*S_q == 0) returns FL_OK without a launch; S_k == 0 gives O = 0,
 * lse = -inf (G7); a fully masked row likewise gives O = 0, lse = -inf.  A tensor with zero elements
 * may carry data == NULL. */
fl_status fl_attn_fwd(const fl_attn_args* args);

/* ---- backward (the training half, §2.4) ------------------------------
 * dQ, dK, dV of L = sum(O * dout) for the forward fl_attn_fwd computes with the same q, k, v, variant,
 * given its output o and natural-log LSE (G19).  A rowsum pass (or, with a sigmoid gate, the gate pre-pass:
 * dA = dO s(g) into the workspace, dgate = dO o (1 - s(g)), Dvec = rowsum(dO o)), then two tcgen05 kernels
 * (a KV-tile-major dK/dV pass and a query-tile-major dQ pass, two compute warpgroups each, no atomics).
 * Supported (v3): bf16, rank-4 or rank-5 q/k/v (G), D_qk == D_v in {32, 64, 128}, GQA, masks none /
 * causal / sliding / prefix / document (either alignment), mods none / ALiBi / softcap, key_mask (MSA
 * mask), sigmoid gate (+ dgate), additive bias (+ dbias), differential attention (v4, Listing 4 P:L412-424,
 * G8: lambda, lambda_h or lambda_qk; + dlambda), mul gate (v4; + dgate = dO * A, A recomputed by the forward
 * kernel without the gate into the workspace: 2 B G Hq S_q D_v bytes + that forward's workspace).  Not yet:
 * the diff_norm epilogue, dbias or the mul gate with diff, block lists, paged KV, fp32 (FL_ERR_UNSUPPORTED).  Workspace (fl_attn_bwd_workspace_size): 4 B G Hq S_q
 * bytes (Dvec) + the packed key mask + 2 B G Hq S_q D_v bytes with a sigmoid gate, each 256-byte rounded.
 * Diff: the forward keeps neither map's output, so the call recomputes both maps (o_i, lse_i: the forward
 * kernel per map), seeds map 1 with -lambda_h dO, runs the single-map backward per map and sums dV (and
 * dgate) over the maps; lse must be absent, o (the diff output) is validated but not read, and the workspace
 * holds o_0, o_1, lse_0, lse_1 and dO_1 plus one forward and one backward workspace.
 * Degenerate shapes: no queries -> dK = dV = 0; no keys -> dQ = 0 and dgate = 0 (zero-fill launches). */
typedef struct {
  fl_tensor q, k, v, o;      /* the forward's inputs and output (bf16) */
  fl_tensor lse;             /* the forward's LSE, f32 [B, Hq, S_q] (required) */
  fl_tensor dout;            /* dL/dO, bf16, o's shape */
  fl_tensor dq, dk, dv;      /* outputs, bf16, the shapes of q, k, v; written in full */
  fl_variant var;
  void* stream;
  void* workspace;
  size_t workspace_bytes;
  fl_tensor dgate;           /* optional (a gate): dL/dgate (sigmoid: of the logits), bf16, the gate's shape (ABI v3) */
  fl_tensor dbias;           /* optional (with a bias): dL/dbias, f32, the bias's shape; dims the bias broadcasts
                                (stride 0 or size 1) are summed over; must be compact -- the call zeroes it and
                                accumulates with fp32 atomics (ABI v3) */
  fl_tensor dlambda;         /* optional (diff): dL/dlambda_h, f32 [Hq] (sum it over h for a scalar lambda; with
                                lambda_qk, the gradient of the lambda it yields); zeroed and accumulated (ABI v4) */
} fl_attn_bwd_args;

fl_status fl_attn_bwd(const fl_attn_bwd_args* args);
fl_status fl_attn_bwd_workspace_size(const fl_attn_bwd_args* args, size_t* bytes);

/* Bytes of device workspace fl_attn_fwd needs for these args (caller-owned, >= 16-byte aligned, not
 * shared by concurrent calls): bf16 path: 256 bytes for the persistent kernel's work-unit ticket
 * counter (reset by the call itself with a stream-ordered memset), then -- when key_mask is present --
 * the key mask packed to one bit per key (ceil(S_k/128)*16 bytes per (b, g), 256-byte rounded), then
 * -- on the split-KV short-query path -- the per-split partials (rows x splits x (D_v + 2) floats).
 * f32 path: the packed key mask only.  0 when the call has no work. */
fl_status fl_attn_workspace_size(const fl_attn_args* args, size_t* bytes);

/* Host-buffer entry (the end-to-end path): same as fl_attn_fwd, but q/k/v (and
 * bias/gate/key_mask/doc_offsets/blk_* if present) and o/lse point to HOST
 * memory (pinned for overlap).  `device_scratch` holds device copies laid out
 * by the library: size from fl_attn_host_scratch_size.  The call enqueues
 * H2D copies, the kernel and the D2H copy of o (and lse) on `stream`, and
 * returns without synchronising.  Host tensors must be contiguous.  With B >= 2
 * and only q / k / v / doc_offsets batched (no bias, key mask, gate, block lists,
 * paged KV), the batch is split into up to 8 chunks whose H2D (an internal copy-in
 * stream), kernel (`stream`) and D2H (an internal copy-out stream) overlap; events
 * order them after `stream`'s prior work and `stream` waits for the last D2H. */
fl_status fl_attn_host_scratch_size(const fl_attn_args* args, size_t* bytes);
fl_status fl_attn_fwd_host(const fl_attn_args* host_args, void* device_scratch, size_t scratch_bytes);

/* RSA block summaries (reading G10; the paper only names RSA).
 *   k    : bf16 [B,Hkv,S_k,D] or [B,G,Hkv,S_k,D], contiguous last dim, 16-byte aligned rows, D % 8 == 0, D <= 1024.
 *   kmin, kmax : bf16 [B*G*Hkv, n_kblk, D] contiguous, n_kblk = ceil(S_k / blk_k); device memory owned by
 *          the caller.  kmin[bh, j, d] = min over the keys of block j (keys [j*blk_k, min((j+1)*blk_k, S_k)))
 *          of K[bh, key, d]; kmax likewise.  Exact (min/max of bf16 values).
 *   blk_k > 0.  One launch, HBM-bound (one pass over K). */
fl_status fl_rsa_build_summaries(const fl_tensor* k, fl_tensor* kmin, fl_tensor* kmax,
                                 int32_t blk_k, void* stream);

/* Incremental summary maintenance after a KV append (RSA's decode loop, P:L47,
 * P:L443 name only): k is the whole cache after the append (S_k keys), kmin/kmax as for
 * fl_rsa_build_summaries with n_kblk = ceil(S_k / blk_k), already valid for keys [0, k_begin).
 * Recomputes exactly the blocks floor(k_begin / blk_k) .. n_kblk - 1 (the one the append started
 * in, which may have been partial, and every new one); the rest is untouched.  The result equals
 * fl_rsa_build_summaries on the whole cache bit for bit.  k_begin >= 0 (no launch when
 * floor(k_begin / blk_k) >= n_kblk).
 * Same argument checks, errors and ownership as fl_rsa_build_summaries; one launch (none if no block). */
fl_status fl_rsa_update_summaries(const fl_tensor* k, fl_tensor* kmin, fl_tensor* kmax,
                                  int32_t blk_k, int64_t k_begin, void* stream);

/* RSA selection (reading G10/G11): for each (b, g, h, q-block i of blk_q rows) with diagonal block
 *   c = min(floor(q_abs(last row of block i) / blk_k), n_kblk - 1)   (q_abs per causal_align, G12),
 *   score_j = max_{q in block i, h' in h's KV group} sum_d max(q_d kmax_jd, q_d kmin_jd),  0 < j < c;
 *   list = {0} U {c} U top-k(score) (ties to the lower j), ascending, -1 padded (all of 0..c if c <= topk+1).
 *   q    : bf16 [B,(G,)Hq,S_q,D], D in {64, 128}, TMA-aligned as for fl_attn_fwd.
 *   kmin, kmax : as written by fl_rsa_build_summaries for the same K (Hkv = kmin.size[0] / (B*G)).
 *   s_k  : number of keys the summaries cover (n_kblk == ceil(s_k / blk_k)); tensor-core path (S_q > 16):
 *          n_kblk <= 256 (D=128) / 512 (D=64); SIMT path (S_q <= 16): n_kblk bounded by shared memory.
 *   blk_q == blk_k == 128; 0 <= topk; topk + 2 <= max_sel <= 512.
 *   blk_idx : i32 [B*G*Hq, n_qblk, max_sel] contiguous; blk_cnt : i32 [B*G*Hq, n_qblk] contiguous.
 *   The scores are one tcgen05 GEMM per (b, h) over K = 2D (q+ . kmax + q- . kmin, exact identity for
 *   kmax >= kmin), fp32 accumulation; near-ties may resolve differently from an fp64 evaluation (G11). */
fl_status fl_rsa_select(const fl_tensor* q, const fl_tensor* kmin, const fl_tensor* kmax, int32_t s_k,
                        int32_t topk, int32_t blk_q, int32_t blk_k, int32_t causal_align,
                        fl_tensor* blk_idx, fl_tensor* blk_cnt, void* stream);

/* ---- fused LayerNorm-prologue linear layer (the memory passes on either side of
 * the attention kernel -- Flashlight fuses "complex element-wise prologues", §3.1; AF2 Alg.7
 * lines 1-4 and 7 of the Evoformer row attention, the paper's second workload P:L865) ----------------
 *   y[m, n] = sum_k xhat[m, k] w[n, k] + bias[n],
 *   xhat[m, :] = LN(x[m, :]) = (x - mean) / sqrt(var + ln_eps) * ln_gamma + ln_beta   (ln_gamma present),
 *              = x[m, :]                                                            (ln_gamma absent)
 *   with mean / var (biased) over the K entries of row m, in fp32; xhat is rounded to bf16 before the
 *   tensor-core product (fp32 accumulation).
 *   x        : bf16 [M, K] (rank 2), contiguous last dim, 16-byte aligned base and row stride; K in
 *              {64, 128, 192, 256} (the whole row is one tile).
 *   w        : bf16 [N, K] (rank 2; the PyTorch Linear weight layout), contiguous last dim, aligned rows.
 *   bias     : optional f32 [N], contiguous.   ln_gamma / ln_beta : optional f32 [K] (beta needs gamma).
 *   y        : bf16 [M, N] (rank 2), ANY element strides (e.g. a head-major [H, i, j] pair bias written
 *              from [i*j, H] rows); must not overlap x / w.
 *   M >= 0, 1 <= N.  One tcgen05 kernel: one CTA per 128 rows of x (read and normalised once, in place
 *   in shared memory), looping over 128-column tiles of w (double-buffered) into two TMEM accumulators,
 *   fused bias epilogue.  Asynchronous on `stream`; no workspace.
 *   Errors: FL_ERR_INVALID_ARGUMENT (missing / non-device tensors, dtype), FL_ERR_SHAPE_MISMATCH,
 *   FL_ERR_UNSUPPORTED (K not in the set), FL_ERR_MISALIGNED. */
typedef struct {
  fl_tensor x, w, bias, ln_gamma, ln_beta, y;
  float ln_eps;
  void* stream;
} fl_linear_args;
fl_status fl_linear(const fl_linear_args* args);

/* ---- Invariant Point Attention core (the paper names IPA among the variants
 * FlexAttention cannot express, P:L47 / P:L443, with 12 heads of dimension 16; formula: reading
 * G23 = AF2 Suppl. Alg.22 lines 7-10, after the linear projections) -------------------------------------
 *   logit_ij^h = w_L ( c^-1/2 q_i.k_j + b_ij^h - (gamma_h w_C / 2) sum_p |T_i q_ip - T_j k_jp|^2 ),
 *   w_L = sqrt(1/3), w_C = sqrt(2 / (9 Pq)), T x = R x + t,  a = softmax_j(logit),
 *   o_i = sum_j a_ij v_j,  opair_i = sum_j a_ij z_ij,  op_ip = T_i^-1 sum_j a_ij T_j v_jp.
 * Inputs (device, contiguous): q, k, v bf16 [N, H, c]; qp, kp bf16 [N, H, Pq, 3]; vp bf16 [N, H, Pv, 3];
 * R f32 [N, 3, 3] (row-major, global = R local + t); t f32 [N, 3]; bias bf16 [H, N, N] (the projected pair
 * bias b); z bf16 [N, N, cz]; gamma f32 [H] (already softplus'ed).  Outputs: o bf16 [N, H, c]; op f32
 * [N, H, Pv, 3] (local frames); opair bf16 [N, H, cz].  Limits: c + 9 Pq + 2 <= 64, Pv in {0, 4, 8},
 * cz % 8 == 0, N <= 8600 (a row's probabilities for 6 heads staged in shared memory; FL_ERR_UNSUPPORTED
 * otherwise).  Launches: a prep
 * kernel (the augmented 64-column Q' / K' of the point term's expansion, hi/lo bf16 pairs), a bias-scale
 * kernel, the fused attention forward (tensor cores, softmax, o and the LSE), a probabilities kernel
 * (a_ij^h = exp(logit - LSE) in fp32, 16 query rows per CTA) and an output kernel (CTA per row i and group of
 * 6 heads: z_i streamed once per group for the pair output, the point sums back-transformed by T_i^-1).
 * Workspace: fl_ipa_workspace_size.  Asynchronous on `stream`. */
typedef struct {
  fl_tensor q, k, v, qp, kp, vp, R, t, bias, z, gamma;
  fl_tensor o, op, opair;
  void* stream;
  void* workspace;
  size_t workspace_bytes;
} fl_ipa_args;
fl_status fl_ipa_fwd(const fl_ipa_args* args);
fl_status fl_ipa_workspace_size(const fl_ipa_args* args, size_t* bytes);

/* Contiguous range [begin, end) of `units` independent work units owned by
 * `rank` of `world` (multi-GPU batch x head sharding; no collective). */
void fl_shard_range(int64_t units, int32_t world, int32_t rank, int64_t* begin, int64_t* end);

/* Diagnostic: one bf16 tcgen05 GEMM C[M,N] (f32) = A[M,K] B[N,K]^T (or B[K,N] when
 * b_mn_major), M = 128, N in {32,64,128}, K in {32,64,128}, through the same
 * TMA/UMMA descriptor helpers the attention kernels use; `a_from_tmem` routes
 * A through TMEM (the P operand path).  For bring-up tests only. */
fl_status fl_diag_umma_gemm(const void* a, const void* b, float* c, int32_t n, int32_t k,
                            int32_t b_mn_major, int32_t a_from_tmem, void* stream);

/* Diagnostic: the bf16 tcgen05 kernel's work decomposition and tile classification
 * for `args` (interval masks only), computed on the device by the kernel's own decode_work / needs /
 * tile_inside functions.  One record per (unit, softmax warpgroup): 8 int32 [unit, wg, b, g, h, q0,
 * lo, hi] followed by max_tiles int32 codes per KV tile j: -1 = not run by that warpgroup, else a 4-bit
 * mask of its warps (32 rows each) that apply the element-wise mask on tile j (0 = mask-free tile).
 * With out == NULL only *n_records / *max_tiles are set.  out: device buffer of >= n_records *
 * (8 + max_tiles) words, on args->stream.  FL_ERR_UNSUPPORTED for block lists, decode shapes, fp32. */
fl_status fl_debug_schedule(const fl_attn_args* args, int32_t* out, int64_t out_words, int64_t* n_records,
                            int32_t* max_tiles);

/* Diagnostic: measured pipe throughput for the MUFU-bound rooflines.  Enqueues one kernel
 * (one CTA of 512 threads per SM, 8 independent chains per thread, `iters` steps each) of op
 * 0 = ex2.approx.ftz.f32, 1 = ex2.approx.ftz.bf16x2, 2 = tanh.approx.f32, 3 = fma.rn.f32x2; *ops receives
 * the number of elementary operations it performs (bf16x2 / f32x2: 2 per instruction).  The caller
 * times the launch on `stream` (rate = ops / time).  sink: device buffer of >= n_SM*512 floats (never
 * written in practice; keeps the chains live).  Asynchronous. */
fl_status fl_diag_pipe_rate(int32_t op, int32_t iters, float* sink, int64_t* ops, void* stream);

/* Diagnostic: cycle counters of the bf16 kernel's pipeline phases, only in a library built with
 * -DFL_TIMING (FL_ERR_UNSUPPORTED otherwise).  out48 receives [3][16] uint64 sums over CTAs:
 * rows 0/1 = softmax warpgroups (slots 0..8: bookkeeping, S wait, S load, score+mask+max, O rescale,
 * ping-pong wait, exp loop, P store, tail; slot 15 = tiles), row 2 reserved.  Synchronises. */
fl_status fl_debug_timing(uint64_t* out48, int32_t reset);

const char* fl_status_string(fl_status s);
const char* fl_last_error(void);   /* thread-local detail of the last non-OK status */
int32_t fl_abi_version(void);
/* sizeof(fl_attn_args) of this build: bindings compare it with their own mirror at load time. */
size_t fl_attn_args_size(void);
size_t fl_attn_bwd_args_size(void);      /* sizeof(fl_attn_bwd_args), for the same check (ABI v4) */
/* Number of kernel launches enqueued by the calling thread since the last reset. */
int64_t fl_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* FL_ATTN_H */
