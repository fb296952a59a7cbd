/*
 * fl_oracle.h -- plain fp64 CPU oracle for the fused attention-variant forward
 * of Flashlight (arXiv 2511.02043).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2511_02043_b200/csrc, include/fl_attn.h); neither side includes or
 * links the other.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (section/eq/listing
 * named beside it).  Readings of ambiguous passages are G1..G20 in DESIGN.md.
 *
 * All tensors are 5-D strided views [B, G, H, S, D] (G = extra batch dim, e.g.
 * the Evoformer MSA row or residue column; G=1 for plain LLM attention).
 * Strides are in ELEMENTS; a stride of 0 broadcasts.  Element types: FLO_F64,
 * FLO_F32, FLO_BF16 (raw uint16 bits), FLO_U8 (key masks).  Every input value
 * is converted exactly to double before use; nothing is ever rounded.
 */
#ifndef FL_ORACLE_H
#define FL_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { FLO_F64 = 0, FLO_F32 = 1, FLO_BF16 = 2, FLO_U8 = 3 };
enum { FLO_MOD_NONE = 0, FLO_MOD_ALIBI = 1, FLO_MOD_SOFTCAP = 2 };
enum { FLO_MASK_NONE = 0, FLO_MASK_CAUSAL = 1, FLO_MASK_SLIDING = 2,
       FLO_MASK_PREFIX = 3, FLO_MASK_DOCUMENT = 4, FLO_MASK_BLOCKLIST = 5 };
enum { FLO_GATE_NONE = 0, FLO_GATE_MUL = 1, FLO_GATE_SIGMOID = 2 };

typedef struct {
  const void* data;      /* NULL = absent */
  int32_t dtype;
  int64_t size[5];       /* [B, G, H, S, D] (key_mask: [B, G, 1, 1, S_k] style, see below) */
  int64_t stride[5];
} flo_tensor;

typedef struct {
  /* q [B,G,Hq*maps,Sq,Dqk]; k [B,G,Hkv*maps,Sk,Dqk]; v [B,G,Hkv,Sk,Dv]; maps = diff ? 2 : 1 */
  flo_tensor q, k, v;
  double scale;                 /* 0 -> 1/sqrt(Dqk)            (Listing 1, G1) */
  int32_t mod;                  /* FLO_MOD_*                   (Eq.4) */
  double softcap;               /* cap for FLO_MOD_SOFTCAP     (G3) */
  const double* alibi_slopes;   /* [Hq] or NULL -> 2^(-8(h+1)/Hq)  (G2) */
  int32_t mask;                 /* FLO_MASK_* */
  int64_t window;               /* sliding window w            (Listing 2, G4) */
  int64_t prefix;               /* PrefixLM length P           (G5) */
  const int32_t* doc_offsets;   /* [B][n_docs+1], 0=off[0] < ... < off[n_docs]=Sk  (G6) */
  int32_t n_docs;
  int32_t doc_causal;
  int32_t causal_align;         /* 0: bottom-right q_abs = q + Sk - Sq; 1: top-left (G12) */
  flo_tensor bias;              /* additive, logical [B,G,Hq,Sq,Sk] (stride 0 broadcasts) */
  flo_tensor key_mask;          /* u8 logical [B,G,Sk] given as size/stride[0..2]; 1 = keep */
  int32_t gate_mode;            /* FLO_GATE_* */
  flo_tensor gate;              /* logical [B,G,Hq,Sq,Dv] */
  int32_t diff;                 /* differential attention      (Listing 4, G8) */
  double lambda;                /* lambda_full */
  const double* lambda_h;       /* [Hq] or NULL */
  const int32_t* blk_idx;       /* [B*G*Hq][n_qblk][max_sel]   (G10) */
  const int32_t* blk_cnt;       /* [B*G*Hq][n_qblk] */
  int32_t blk_q, blk_k, max_sel;
  /* DIFF-Transformer epilogue (reading G8b, external Ye et al. 2024) */
  const double* lambda_qk;      /* [4][Dqk]: lambda = exp(q1.k1) - exp(q2.k2) + lambda_init, or NULL */
  double lambda_init;
  int32_t diff_norm;            /* 1: O <- (1 - lambda_init) * w * O / sqrt(mean_d O_d^2 + eps) */
  double diff_norm_eps;
  const double* diff_norm_w;    /* [Dv] or NULL (ones) */
} flo_problem;

/* Output rows.  rows[i] = ((b*G + g)*Hq + h)*Sq + q; rows == NULL means all
 * B*G*Hq*Sq rows in that order.  out: nrows x Dv doubles.  lse (may be NULL):
 * nrows doubles, natural-log LSE of the scaled, modified scores (G19); -inf for
 * an empty row (G7); NaN for diff (two maps, no single LSE).
 * Returns 0, or a negative code for an invalid problem. */
int flo_attn(const flo_problem* p, const int64_t* rows, int64_t nrows,
             double* out, double* lse);

/* The kept-key predicate of output row (b, g, h, q) (definition step 2: mask AND key mask) as
 * S_k bytes 0/1 -- the scheduler / tile-classifier test compares the kernel's tiles against it. */
int flo_keep_row(const flo_problem* p, int64_t b, int64_t g, int64_t h, int64_t q, uint8_t* keep_out);

/* Alg.1: two serial loops, m_N = max x, d_N = sum e^{x_j - m_N}.
 * Writes sigma(x) (Eq.2) into y and returns d_N; *m gets m_N. */
double flo_stable_softmax(const double* x, int64_t n, double* y, double* m);

/* RSA block summaries: for each (bh, KV block j), kmin[d] / kmax[d] over the
 * keys of block j (exact).  k is [BH][Sk][D] as a flo_tensor with dims
 * [B,G,H,S,D]; outputs [B*G*H][n_kblk][D]. */
int flo_rsa_summaries(const flo_tensor* k, int32_t blk_k, double* kmin, double* kmax);

/* RSA selection (reading G10/G11): per (b,g,h,q-block i) with diagonal block
 * c, score_j = max_{q in block i} sum_d max(q_d*kmax_jd, q_d*kmin_jd) for
 * 0 < j < c; list = {0} U {c} U top-k(score), ties to lower j, ascending.
 * If c <= topk + 1 the list is all of 0..c.  Scores (optional, may be NULL):
 * [B*G*Hq][n_qblk][n_kblk] (NaN where not admissible).  q dims [B,G,Hq,Sq,D],
 * k dims [B,G,Hkv,Sk,D]; with Hkv < Hq the per-group score is the max over the
 * group's query heads (G10), so every head of a group gets the same list. */
int flo_rsa_select(const flo_tensor* q, const flo_tensor* k, int32_t blk_q, int32_t blk_k,
                   int32_t topk, int32_t causal_align, int32_t max_sel,
                   int32_t* blk_idx, int32_t* blk_cnt, double* scores);

/* Backward: dQ, dK, dV (fp64, logical shapes of q, k, v, row-major) of
 * L = sum O * dO for the problem's forward, by the plain chain rule through the definition (see the
 * comment at the definition).  dout: logical [B,G,Hq,Sq,Dv].  -11 when diff_norm is set (not derived).
 * dgate / dbias / dlambda: optional (NULL), see the definition's comment. */
int flo_attn_bwd(const flo_problem* p, const flo_tensor* dout, double* dq, double* dk, double* dv, double* dgate,
                 double* dbias, double* dlambda);

int flo_num_threads(void);

#ifdef __cplusplus
}
#endif
/* NEXT-2: y = [LayerNorm(x)] w^T + bias (see fl_oracle.c). */
int flo_linear_ln(int64_t M, int64_t N, int64_t K, const double* x, const double* w, const double* bias,
                  const double* gamma, const double* beta, double eps, double* y, double* yabs);
/* NEXT-4: Invariant Point Attention core (AF2 Alg.22 lines 7-10, reading G23; see fl_oracle.c). */
int flo_ipa(int64_t N, int64_t H, int64_t c, int64_t Pq, int64_t Pv, int64_t cz, const double* q, const double* k,
            const double* v, const double* qp, const double* kp, const double* vp, const double* R, const double* t,
            const double* bias, const double* z, const double* gamma, double* o, double* op, double* opair);
#endif
