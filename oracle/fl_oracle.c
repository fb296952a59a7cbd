/*
 * fl_oracle.c -- plain, unfused fp64 CPU oracle of the attention-variant
 * forward that Flashlight (arXiv 2511.02043) fuses into one kernel.
 *
 * TEST INFRASTRUCTURE ONLY (see fl_oracle.h).  The product path never loads it.
 *
 * What it computes: the PLAIN DEFINITION, not the fused method.  Flashlight's
 * kernel is exact in real arithmetic (§2.2; §3.7) and the
 * online rewrite is proved equal to the two-pass form (§3.3), so per
 * output row this file evaluates
 *     s_k  = scale * <Q_q, K_k>                    Eq.3  P:L186-189, Listing 1
 *     s_k  = score_mod(s_k)                        Eq.4  P:L251-257 (ALiBi / bias / softcap)
 *     keep = mask predicate                        Listing 1, Listing 2
 *     m    = max_k s_k ;  d = sum_k e^{s_k - m}    Alg.1 P:L146-160 (two serial loops)
 *     O_q  = sum_k (e^{s_k - m} / d) V_k           Eq.2  P:L134-141, Listing 1
 *     diff:  O = A_0 - lambda * A_1                Listing 4
 *            [ (1 - lambda_init) RMSNorm(O), lambda re-parameterised ]   reading G8b (NEXT-2)
 *     gate:  O = O * sigmoid(G) | O * G            Evoformer P:L865 (reading G9)
 * with every intermediate in fp64, one row at a time, no blocking, no online
 * rescaling, no reordering beyond the definition.  OpenMP splits rows only.
 */
#include "fl_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- element access: exact conversion of the stored value to double ---- */
static double elem(const flo_tensor* t, int64_t off) {
  switch (t->dtype) {
    case FLO_F64: return ((const double*)t->data)[off];
    case FLO_F32: return (double)((const float*)t->data)[off];
    case FLO_BF16: {
      uint32_t bits = (uint32_t)((const uint16_t*)t->data)[off] << 16;
      float f;
      memcpy(&f, &bits, 4);
      return (double)f;
    }
    case FLO_U8: return (double)((const uint8_t*)t->data)[off];
  }
  return NAN;
}

static int64_t off5(const flo_tensor* t, int64_t b, int64_t g, int64_t h, int64_t s, int64_t d) {
  return b * t->stride[0] + g * t->stride[1] + h * t->stride[2] + s * t->stride[3] + d * t->stride[4];
}

/* Alg.1: first loop m_k = maximum(m_{k-1}, x_k); second loop
 * d_j = d_{j-1} + e^{x_j - m_N}.  Returns d_N; y = e^{x - m_N} / d_N (Eq.2). */
double flo_stable_softmax(const double* x, int64_t n, double* y, double* m_out) {
  double m = -INFINITY;
  for (int64_t k = 0; k < n; ++k) m = x[k] > m ? x[k] : m;
  double d = 0.0;
  for (int64_t j = 0; j < n; ++j) d += exp(x[j] - m);
  if (y)
    for (int64_t j = 0; j < n; ++j) y[j] = exp(x[j] - m) / d;
  if (m_out) *m_out = m;
  return d;
}

/* ---- mask predicates (reading G4-G6, G10, G12) ---- */
static int doc_of(const int32_t* offs, int32_t n_docs, int64_t pos) {
  for (int32_t j = 0; j < n_docs; ++j)
    if (pos >= offs[j] && pos < offs[j + 1]) return j;
  return -1;
}

static int keep_key(const flo_problem* p, int64_t bgh, int64_t b, int64_t q, int64_t q_abs, int64_t k) {
  switch (p->mask) {
    case FLO_MASK_NONE: return 1;
    case FLO_MASK_CAUSAL: return k <= q_abs;
    /* Listing 2: keep = (q >= kv) & ((q - kv) <= window_size) */
    case FLO_MASK_SLIDING: return k <= q_abs && (q_abs - k) <= p->window;
    case FLO_MASK_PREFIX: return k < p->prefix || k <= q_abs;
    case FLO_MASK_DOCUMENT: {
      const int32_t* offs = p->doc_offsets + b * (int64_t)(p->n_docs + 1);
      int same = doc_of(offs, p->n_docs, k) == doc_of(offs, p->n_docs, q_abs);
      return same && (!p->doc_causal || k <= q_abs);
    }
    case FLO_MASK_BLOCKLIST: {
      int64_t qb = q / p->blk_q;
      int64_t sq = p->q.size[3];
      int64_t nqb = (sq + p->blk_q - 1) / p->blk_q;
      const int32_t* idx = p->blk_idx + (bgh * nqb + qb) * p->max_sel;
      int32_t cnt = p->blk_cnt[bgh * nqb + qb];
      int64_t kb = k / p->blk_k;
      int listed = 0;
      for (int32_t i = 0; i < cnt; ++i)
        if (idx[i] == kb) listed = 1;
      return listed && k <= q_abs;
    }
  }
  return 0;
}

static int check_problem(const flo_problem* p, int64_t* maps_out) {
  if (!p || !p->q.data || !p->k.data || !p->v.data) return -1;
  int64_t maps = p->diff ? 2 : 1;
  const int64_t* qs = p->q.size; const int64_t* ks = p->k.size; const int64_t* vs = p->v.size;
  if (qs[0] != ks[0] || qs[0] != vs[0] || qs[1] != ks[1] || qs[1] != vs[1]) return -2;
  if (qs[4] != ks[4]) return -3;
  if (ks[3] != vs[3]) return -4;
  if (qs[2] % maps || ks[2] % maps) return -5;
  int64_t hq = qs[2] / maps, hkv = ks[2] / maps;
  if (hkv != vs[2] || hkv == 0 || hq % hkv) return -6;
  if (p->mask == FLO_MASK_DOCUMENT && (!p->doc_offsets || p->n_docs < 1)) return -7;
  if (p->mask == FLO_MASK_BLOCKLIST && (!p->blk_idx || !p->blk_cnt || p->blk_q <= 0 || p->blk_k <= 0)) return -8;
  if (p->mod == FLO_MOD_SOFTCAP && !(p->softcap > 0)) return -9;
  *maps_out = maps;
  return 0;
}

/* Step 2 of the definition: is key k kept for output row (b, g, h, q)?  The mask
 * predicate (Listing 1, Listing 2, readings G4-G6, G10, G12) AND the key mask. */
static int kept(const flo_problem* p, int64_t bgh, int64_t b, int64_t g, int64_t q, int64_t q_abs, int64_t k) {
  int keep = keep_key(p, bgh, b, q, q_abs, k);
  if (keep && p->key_mask.data) {
    int64_t mo = b * p->key_mask.stride[0] + g * p->key_mask.stride[1] + k * p->key_mask.stride[2];
    keep = elem(&p->key_mask, mo) != 0.0;
  }
  return keep;
}

/* One output row (b, g, h, q): the plain definition, map by map. */
static void one_row(const flo_problem* p, int64_t maps, int64_t b, int64_t g, int64_t h, int64_t q,
                    double* s, double* acc, double* out, double* lse_out) {
  const int64_t G = p->q.size[1];
  const int64_t Hq = p->q.size[2] / maps, Hkv = p->k.size[2] / maps;
  const int64_t Sq = p->q.size[3], Sk = p->k.size[3], Dqk = p->q.size[4], Dv = p->v.size[4];
  const double scale = p->scale != 0.0 ? p->scale : 1.0 / sqrt((double)Dqk); /* G1 */
  const int64_t h_kv = h / (Hq / Hkv);                                      /* G15 */
  const int64_t q_abs = p->causal_align ? q : q + (Sk - Sq);                /* G12 */
  const int64_t bgh = (b * G + g) * Hq + h;
  double lam = p->lambda_h ? p->lambda_h[h] : p->lambda;
  if (maps == 2 && p->lambda_qk) {               /* lambda re-parameterisation (G8b) */
    double d1 = 0.0, d2 = 0.0;
    for (int64_t d = 0; d < Dqk; ++d) {
      d1 += p->lambda_qk[d] * p->lambda_qk[Dqk + d];
      d2 += p->lambda_qk[2 * Dqk + d] * p->lambda_qk[3 * Dqk + d];
    }
    lam = exp(d1) - exp(d2) + p->lambda_init;
  }

  for (int64_t d = 0; d < Dv; ++d) out[d] = 0.0;
  double lse = NAN;
  for (int64_t map = 0; map < maps; ++map) {
    const int64_t qh = h + map * Hq, kh = h_kv + map * Hkv;
    int any = 0;
    for (int64_t k = 0; k < Sk; ++k) {
      if (!kept(p, bgh, b, g, q, q_abs, k)) { s[k] = -INFINITY; continue; }
      any = 1;
      double dot = 0.0;                         /* QK^T, Eq.3 */
      for (int64_t d = 0; d < Dqk; ++d)
        dot += elem(&p->q, off5(&p->q, b, g, qh, q, d)) * elem(&p->k, off5(&p->k, b, g, kh, k, d));
      double x = scale * dot;                   /* Listing 1: attn_scores *= 1/sqrt(d) */
      /* score_mod on the scaled score (Eq.4), fixed order G16 */
      if (p->mod == FLO_MOD_ALIBI) {
        double slope = p->alibi_slopes ? p->alibi_slopes[h] : pow(2.0, -8.0 * (double)(h + 1) / (double)Hq);
        x += slope * (double)(k - q_abs);
      }
      if (p->bias.data) x += elem(&p->bias, off5(&p->bias, b, g, h, q, k));
      if (p->mod == FLO_MOD_SOFTCAP) x = p->softcap * tanh(x / p->softcap);
      s[k] = x;
    }
    if (!any) {                                 /* empty row: O = 0, lse = -inf (G7) */
      if (maps == 1) lse = -INFINITY;
      continue;
    }
    /* Alg.1: loop 1 = max over kept scores; loop 2 = sum of e^{x - m} */
    double m = -INFINITY;
    for (int64_t k = 0; k < Sk; ++k) m = s[k] > m ? s[k] : m;
    double dsum = 0.0;
    for (int64_t k = 0; k < Sk; ++k) dsum += exp(s[k] - m);
    /* O = softmax(s) V  (Listing 1: torch.matmul(attn_weights, v)) */
    for (int64_t d = 0; d < Dv; ++d) acc[d] = 0.0;
    for (int64_t k = 0; k < Sk; ++k) {
      if (s[k] == -INFINITY) continue;
      double w = exp(s[k] - m) / dsum;
      for (int64_t d = 0; d < Dv; ++d) acc[d] += w * elem(&p->v, off5(&p->v, b, g, h_kv, k, d));
    }
    /* Listing 4: output = attn0 - lambda_full * attn1 */
    double coef = map == 0 ? 1.0 : -lam;
    for (int64_t d = 0; d < Dv; ++d) out[d] += coef * acc[d];
    if (maps == 1) lse = m + log(dsum);
  }
  if (maps == 2 && p->diff_norm) {               /* per-head RMSNorm of the diff output (G8b) */
    double ms = 0.0;
    for (int64_t d = 0; d < Dv; ++d) ms += out[d] * out[d];
    ms /= (double)Dv;
    const double k = (1.0 - p->lambda_init) / sqrt(ms + p->diff_norm_eps);
    for (int64_t d = 0; d < Dv; ++d) out[d] *= k * (p->diff_norm_w ? p->diff_norm_w[d] : 1.0);
  }
  if (p->gate_mode != FLO_GATE_NONE) {
    for (int64_t d = 0; d < Dv; ++d) {
      double gv = elem(&p->gate, off5(&p->gate, b, g, h, q, d));
      out[d] *= p->gate_mode == FLO_GATE_SIGMOID ? 1.0 / (1.0 + exp(-gv)) : gv;
    }
  }
  if (lse_out) *lse_out = lse;
}

int flo_attn(const flo_problem* p, const int64_t* rows, int64_t nrows, double* out, double* lse) {
  int64_t maps;
  int rc = check_problem(p, &maps);
  if (rc) return rc;
  const int64_t B = p->q.size[0], G = p->q.size[1], Hq = p->q.size[2] / maps, Sq = p->q.size[3];
  const int64_t Sk = p->k.size[3], Dv = p->v.size[4];
  const int64_t total = B * G * Hq * Sq;
  if (!rows) nrows = total;
  int bad = 0;
#pragma omp parallel
  {
    double* s = (double*)malloc(sizeof(double) * (size_t)(Sk > 0 ? Sk : 1));
    double* acc = (double*)malloc(sizeof(double) * (size_t)(Dv > 0 ? Dv : 1));
#pragma omp for schedule(dynamic, 16)
    for (int64_t i = 0; i < nrows; ++i) {
      int64_t r = rows ? rows[i] : i;
      if (r < 0 || r >= total) { bad = 1; continue; }
      int64_t q = r % Sq, t = r / Sq;
      int64_t h = t % Hq; t /= Hq;
      int64_t g = t % G, b = t / G;
      one_row(p, maps, b, g, h, q, s, acc, out + i * Dv, lse ? lse + i : NULL);
    }
    free(s);
    free(acc);
  }
  return bad ? -10 : 0;
}

int flo_keep_row(const flo_problem* p, int64_t b, int64_t g, int64_t h, int64_t q, uint8_t* keep_out) {
  int64_t maps;
  int rc = check_problem(p, &maps);
  if (rc) return rc;
  const int64_t G = p->q.size[1], Hq = p->q.size[2] / maps, Sq = p->q.size[3], Sk = p->k.size[3];
  const int64_t q_abs = p->causal_align ? q : q + (Sk - Sq);                /* G12 */
  const int64_t bgh = (b * G + g) * Hq + h;
  for (int64_t k = 0; k < Sk; ++k) keep_out[k] = (uint8_t)kept(p, bgh, b, g, q, q_abs, k);
  return 0;
}

/* ---- backward (the training half of the same program, §2.4 AOTAutograd) ----
 * The plain chain rule through the definition evaluated by one_row, per output row (b, g, h, q):
 *   P_k = e^{s_k - m} / d over the kept keys,   O = sum_k P_k V_k  (map by map; diff: O = A_0 - lambda A_1)
 *   dA_map = dO * gate' (gate' = sigma(G) or G) * (map 0: 1, map 1: -lambda)
 *   dV_k += P_k dA ;  dP_k = <dA, V_k> ;  dS_k = P_k (dP_k - <dA, A_map>)      (softmax Jacobian)
 *   dx_k = dS_k * (softcap: 1 - (s_k / cap)^2, else 1)                          (s = cap tanh(x / cap))
 *   dQ += scale dx_k K_k ;  dK_k += scale dx_k Q                                (x = scale <Q, K_k> + ...)
 * dK, dV of a KV head accumulate over its GQA group (G15).  Outputs are fp64 arrays with the logical shapes
 * of q, k, v ([B,G,H,S,D], row-major).  diff_norm is not differentiated here (returns -11). */
/* dgate (optional, may be NULL): dL/dgate for the Evoformer gate of reading G9 (O = gate'(g) * A, AF2
 * Alg.7 line 6): dgate = dO * A * sigma(g) (1 - sigma(g)) (sigmoid) or dO * A (mul), A the map-combined
 * attention output before the gate (sum over maps of coef * P V). */
/* dbias (optional, may be NULL): dL/dbias for the additive score bias of Eq.4 / G16 (s = scale q.k + bias
 * before the softcap), logical [B, G, Hq, Sq, Sk] contiguous: the score gradient dx of each kept (q, k) --
 * the caller sums it over the dims its bias broadcasts (e.g. the MSA rows s of the Evoformer pair bias). */
/* dlambda (optional, may be NULL; diff only): dL/dlambda_h [Hq] of Listing 4's O = A_0 - lambda_h A_1 (P:L412-424,
 * G8): -sum over (b, g, q, d) of dO * gate' * A_1 -- with lambda_qk the lambda the re-parameterisation yields
 * (the caller chains into lambda_qk), with a scalar lambda the caller sums it over h. */
int flo_attn_bwd(const flo_problem* p, const flo_tensor* dout, double* dq, double* dk, double* dv, double* dgate,
                 double* dbias, double* dlambda) {
  int64_t maps;
  int rc = check_problem(p, &maps);
  if (rc) return rc;
  if (p->diff_norm) return -11;
  const int64_t B = p->q.size[0], G = p->q.size[1], Hq = p->q.size[2] / maps, Hkv = p->k.size[2] / maps;
  const int64_t Sq = p->q.size[3], Sk = p->k.size[3], Dqk = p->q.size[4], Dv = p->v.size[4];
  const int64_t grp = Hq / Hkv;
  const double scale = p->scale != 0.0 ? p->scale : 1.0 / sqrt((double)Dqk);     /* G1 */
  const int64_t nq = B * G * Hq * maps * Sq * Dqk, nk = B * G * Hkv * maps * Sk * Dqk, nv = B * G * Hkv * Sk * Dv;
  for (int64_t i = 0; i < nq; ++i) dq[i] = 0.0;
  for (int64_t i = 0; i < nk; ++i) dk[i] = 0.0;
  for (int64_t i = 0; i < nv; ++i) dv[i] = 0.0;
  if (dgate)
    for (int64_t i = 0; i < B * G * Hq * Sq * Dv; ++i) dgate[i] = 0.0;
  if (dbias)
    for (int64_t i = 0; i < B * G * Hq * Sq * Sk; ++i) dbias[i] = 0.0;
  if (dlambda)
    for (int64_t i = 0; i < Hq; ++i) dlambda[i] = 0.0;
  /* one task per (b, g, kv head): every write of the task stays inside it */
#pragma omp parallel
  {
    double* sc = (double*)malloc(sizeof(double) * (size_t)(Sk > 0 ? Sk : 1));
    double* pr = (double*)malloc(sizeof(double) * (size_t)(Sk > 0 ? Sk : 1));
    double* a = (double*)malloc(sizeof(double) * (size_t)(Dv > 0 ? Dv : 1));
    double* da = (double*)malloc(sizeof(double) * (size_t)(Dv > 0 ? Dv : 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t task = 0; task < B * G * Hkv; ++task) {
      const int64_t hk = task % Hkv, g = (task / Hkv) % G, b = task / (Hkv * G);
      for (int64_t h = hk * grp; h < (hk + 1) * grp; ++h) {
        const int64_t bgh = (b * G + g) * Hq + h;
        double lam = p->lambda_h ? p->lambda_h[h] : p->lambda;
        if (maps == 2 && p->lambda_qk) {
          double d1 = 0.0, d2 = 0.0;
          for (int64_t d = 0; d < Dqk; ++d) {
            d1 += p->lambda_qk[d] * p->lambda_qk[Dqk + d];
            d2 += p->lambda_qk[2 * Dqk + d] * p->lambda_qk[3 * Dqk + d];
          }
          lam = exp(d1) - exp(d2) + p->lambda_init;
        }
        for (int64_t q = 0; q < Sq; ++q) {
          const int64_t q_abs = p->causal_align ? q : q + (Sk - Sq);            /* G12 */
          for (int64_t map = 0; map < maps; ++map) {
            const int64_t qh = h + map * Hq, kh = hk + map * Hkv;
            /* forward of this map: kept scores, P (Alg.1 two-pass), A = P V */
            int any = 0;
            for (int64_t k = 0; k < Sk; ++k) {
              if (!kept(p, bgh, b, g, q, q_abs, k)) { sc[k] = -INFINITY; continue; }
              any = 1;
              double dot = 0.0;
              for (int64_t d = 0; d < Dqk; ++d)
                dot += elem(&p->q, off5(&p->q, b, g, qh, q, d)) * elem(&p->k, off5(&p->k, b, g, kh, k, d));
              double x = scale * dot;
              if (p->mod == FLO_MOD_ALIBI) {
                double slope = p->alibi_slopes ? p->alibi_slopes[h] : pow(2.0, -8.0 * (double)(h + 1) / (double)Hq);
                x += slope * (double)(k - q_abs);
              }
              if (p->bias.data) x += elem(&p->bias, off5(&p->bias, b, g, h, q, k));
              if (p->mod == FLO_MOD_SOFTCAP) x = p->softcap * tanh(x / p->softcap);
              sc[k] = x;
            }
            if (!any) continue;                                                   /* G7: O = 0, no gradient */
            double m = -INFINITY, den = 0.0;
            for (int64_t k = 0; k < Sk; ++k) m = sc[k] > m ? sc[k] : m;
            for (int64_t k = 0; k < Sk; ++k) den += exp(sc[k] - m);
            for (int64_t d = 0; d < Dv; ++d) a[d] = 0.0;
            for (int64_t k = 0; k < Sk; ++k) {
              pr[k] = sc[k] == -INFINITY ? 0.0 : exp(sc[k] - m) / den;
              if (pr[k] != 0.0)
                for (int64_t d = 0; d < Dv; ++d) a[d] += pr[k] * elem(&p->v, off5(&p->v, b, g, hk, k, d));
            }
            /* dA = dO * gate' * (1 or -lambda) */
            double coef = map == 0 ? 1.0 : -lam;
            double dot_da_a = 0.0, dlam = 0.0;
            for (int64_t d = 0; d < Dv; ++d) {
              double gv = 1.0;
              if (p->gate_mode != FLO_GATE_NONE) {
                double gl = elem(&p->gate, off5(&p->gate, b, g, h, q, d));
                gv = p->gate_mode == FLO_GATE_SIGMOID ? 1.0 / (1.0 + exp(-gl)) : gl;
              }
              da[d] = coef * gv * elem(dout, off5(dout, b, g, h, q, d));
              dot_da_a += da[d] * a[d];
              if (map == 1) dlam -= gv * elem(dout, off5(dout, b, g, h, q, d)) * a[d];    /* dO/dlambda = -gate' A_1 */
              if (dgate && p->gate_mode != FLO_GATE_NONE) {
                const double gl = elem(&p->gate, off5(&p->gate, b, g, h, q, d));
                const double dgl = p->gate_mode == FLO_GATE_SIGMOID ? gv * (1.0 - gv) : 1.0;   /* gate'(g) */
                (void)gl;
                dgate[(((b * G + g) * Hq + h) * Sq + q) * Dv + d] += coef * a[d] * dgl * elem(dout, off5(dout, b, g, h, q, d));
              }
            }
            if (dlambda && map == 1) {
#pragma omp atomic
              dlambda[h] += dlam;                       /* heads of one group meet across the b, g tasks */
            }
            for (int64_t k = 0; k < Sk; ++k) {
              if (pr[k] == 0.0 && sc[k] == -INFINITY) continue;
              double dp = 0.0;
              for (int64_t d = 0; d < Dv; ++d) {
                const double vv = elem(&p->v, off5(&p->v, b, g, hk, k, d));
                dp += da[d] * vv;
                dv[(((b * G + g) * Hkv + hk) * Sk + k) * Dv + d] += pr[k] * da[d];
              }
              double dx = pr[k] * (dp - dot_da_a);
              if (p->mod == FLO_MOD_SOFTCAP) {
                const double t = sc[k] / p->softcap;
                dx *= 1.0 - t * t;
              }
              if (dbias) dbias[(((b * G + g) * Hq + h) * Sq + q) * Sk + k] += dx;   /* maps share the bias */
              for (int64_t d = 0; d < Dqk; ++d) {
                dq[((((b * G + g) * Hq * maps) + qh) * Sq + q) * Dqk + d] +=
                    scale * dx * elem(&p->k, off5(&p->k, b, g, kh, k, d));
                dk[((((b * G + g) * Hkv * maps) + kh) * Sk + k) * Dqk + d] +=
                    scale * dx * elem(&p->q, off5(&p->q, b, g, qh, q, d));
              }
            }
          }
        }
      }
    }
    free(sc);
    free(pr);
    free(a);
    free(da);
  }
  return 0;
}

/* ---- RSA (reading G10/G11; the paper only names RSA) ---- */
int flo_rsa_summaries(const flo_tensor* k, int32_t blk_k, double* kmin, double* kmax) {
  const int64_t B = k->size[0], G = k->size[1], H = k->size[2], Sk = k->size[3], D = k->size[4];
  if (blk_k <= 0) return -1;
  const int64_t nkb = (Sk + blk_k - 1) / blk_k;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t bgh = 0; bgh < B * G * H; ++bgh)
    for (int64_t j = 0; j < nkb; ++j) {
      int64_t h = bgh % H, g = (bgh / H) % G, b = bgh / (H * G);
      for (int64_t d = 0; d < D; ++d) {
        double lo = INFINITY, hi = -INFINITY;
        for (int64_t kk = j * blk_k; kk < (j + 1) * blk_k && kk < Sk; ++kk) {
          double x = elem(k, off5(k, b, g, h, kk, d));
          lo = x < lo ? x : lo;
          hi = x > hi ? x : hi;
        }
        kmin[(bgh * nkb + j) * D + d] = lo;
        kmax[(bgh * nkb + j) * D + d] = hi;
      }
    }
  return 0;
}

int flo_rsa_select(const flo_tensor* q, const flo_tensor* k, int32_t blk_q, int32_t blk_k,
                   int32_t topk, int32_t causal_align, int32_t max_sel,
                   int32_t* blk_idx, int32_t* blk_cnt, double* scores) {
  const int64_t B = q->size[0], G = q->size[1], Hq = q->size[2], Sq = q->size[3], D = q->size[4];
  const int64_t Hkv = k->size[2], Sk = k->size[3];
  if (blk_q <= 0 || blk_k <= 0 || topk < 0 || Hkv <= 0 || Hq % Hkv || k->size[4] != D) return -1;
  if (max_sel < topk + 2) return -2;
  const int64_t nqb = (Sq + blk_q - 1) / blk_q, nkb = (Sk + blk_k - 1) / blk_k;
  const int64_t grp = Hq / Hkv;
  double* kmin = (double*)malloc(sizeof(double) * (size_t)(B * G * Hkv * nkb * D));
  double* kmax = (double*)malloc(sizeof(double) * (size_t)(B * G * Hkv * nkb * D));
  flo_rsa_summaries(k, blk_k, kmin, kmax);
  int bad = 0;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int64_t bgk = 0; bgk < B * G * Hkv; ++bgk)
    for (int64_t i = 0; i < nqb; ++i) {
      int64_t hk = bgk % Hkv, g = (bgk / Hkv) % G, b = bgk / (Hkv * G);
      int64_t q_last = (i + 1) * blk_q - 1;
      if (q_last > Sq - 1) q_last = Sq - 1;
      int64_t q_last_abs = causal_align ? q_last : q_last + (Sk - Sq);
      int64_t c = q_last_abs / blk_k;            /* diagonal (local) block */
      if (c > nkb - 1) c = nkb - 1;
      if (c < 0) c = 0;
      double* sc = (double*)malloc(sizeof(double) * (size_t)(nkb > 0 ? nkb : 1));
      for (int64_t j = 0; j < nkb; ++j) sc[j] = NAN;
      /* score_j = max over the group's query heads and the block's queries of
       * sum_d max(q_d * kmax_jd, q_d * kmin_jd)   (Quest-style bound, G10) */
      for (int64_t j = 1; j < c; ++j) {
        double best = -INFINITY;
        const double* mx = kmax + ((bgk * nkb) + j) * D;
        const double* mn = kmin + ((bgk * nkb) + j) * D;
        for (int64_t hh = hk * grp; hh < (hk + 1) * grp; ++hh)
          for (int64_t qq = i * blk_q; qq < (i + 1) * blk_q && qq < Sq; ++qq) {
            double tot = 0.0;
            for (int64_t d = 0; d < D; ++d) {
              double qd = elem(q, off5(q, b, g, hh, qq, d));
              double a = qd * mx[d], bb = qd * mn[d];
              tot += a > bb ? a : bb;
            }
            best = tot > best ? tot : best;
          }
        sc[j] = best;
      }
      /* list = {0} U {c} U top-k(score), ties toward lower j, sorted ascending */
      char* sel = (char*)calloc((size_t)(nkb > 0 ? nkb : 1), 1);
      sel[0] = 1;
      sel[c] = 1;
      if (c <= (int64_t)topk + 1) {
        for (int64_t j = 0; j <= c; ++j) sel[j] = 1;
      } else {
        for (int32_t t = 0; t < topk; ++t) {
          int64_t arg = -1;
          for (int64_t j = 1; j < c; ++j)
            if (!sel[j] && (arg < 0 || sc[j] > sc[arg])) arg = j;
          if (arg >= 0) sel[arg] = 1;
        }
      }
      int32_t cnt = 0;
      for (int64_t j = 0; j < nkb; ++j)
        if (sel[j]) {
          if (cnt >= max_sel) { bad = 1; break; }
          for (int64_t hh = hk * grp; hh < (hk + 1) * grp; ++hh)
            blk_idx[((((b * G + g) * Hq + hh) * nqb) + i) * max_sel + cnt] = (int32_t)j;
          ++cnt;
        }
      for (int64_t hh = hk * grp; hh < (hk + 1) * grp; ++hh) {
        int64_t base = (((b * G + g) * Hq + hh) * nqb) + i;
        blk_cnt[base] = cnt;
        for (int32_t t = cnt; t < max_sel; ++t) blk_idx[base * max_sel + t] = -1;
        if (scores)
          for (int64_t j = 0; j < nkb; ++j) scores[base * nkb + j] = sc[j];
      }
      free(sel);
      free(sc);
    }
  free(kmin);
  free(kmax);
  return bad ? -3 : 0;
}

int flo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* SURVEY §8(f) NEXT-2, the memory passes on either side of the attention kernel (Flashlight fuses
 * "complex element-wise prologues", §3.1; the Evoformer row attention of the paper's second
 * workload, is AF2 Alg.7: line 1 m <- LayerNorm(m), lines 2-4 q, k, v, g = Linear(m), line 7
 * the output Linear).  Written out as defined, fp64, in this order per row m:
 *   mean = (1/K) sum_k x[m,k];  var = (1/K) sum_k (x[m,k] - mean)^2          (LayerNorm, biased variance)
 *   xhat[k] = (x[m,k] - mean) / sqrt(var + eps) * gamma[k] + beta[k]        (gamma == NULL: xhat = x[m,:];
 *                                                                           beta == NULL: beta = 0)
 *   y[m,n] = sum_k xhat[k] w[n,k] + bias[n]                                 (bias == NULL: 0)
 *   yabs[m,n] = sum_k |xhat[k]| |w[n,k]|   (if yabs != NULL: the scale the tests derive a rounding bound from)
 * x [M][K], w [N][K], y / yabs [M][N], all contiguous fp64. */
int flo_linear_ln(int64_t M, int64_t N, int64_t K, const double* x, const double* w, const double* bias,
                  const double* gamma, const double* beta, double eps, double* y, double* yabs) {
  if (M < 0 || N < 1 || K < 1) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t m = 0; m < M; ++m) {
    double* xhat = (double*)malloc(sizeof(double) * K);
    const double* xr = x + m * K;
    if (gamma) {
      double mean = 0.0, var = 0.0;
      for (int64_t k = 0; k < K; ++k) mean += xr[k];
      mean /= (double)K;
      for (int64_t k = 0; k < K; ++k) var += (xr[k] - mean) * (xr[k] - mean);
      var /= (double)K;
      const double inv = 1.0 / sqrt(var + eps);
      for (int64_t k = 0; k < K; ++k) xhat[k] = (xr[k] - mean) * inv * gamma[k] + (beta ? beta[k] : 0.0);
    } else {
      for (int64_t k = 0; k < K; ++k) xhat[k] = xr[k];
    }
    for (int64_t n = 0; n < N; ++n) {
      double acc = 0.0, aabs = 0.0;
      for (int64_t k = 0; k < K; ++k) {
        acc += xhat[k] * w[n * K + k];
        aabs += fabs(xhat[k]) * fabs(w[n * K + k]);
      }
      y[m * N + n] = acc + (bias ? bias[n] : 0.0);
      if (yabs) yabs[m * N + n] = aabs;
    }
    free(xhat);
  }
  return 0;
}

/* AlphaFold's Invariant Point Attention (IPA), named by the paper among the variants
 * FlexAttention cannot express with 12 heads of dimension 16.  The paper
 * gives no formula; this is AF2 (Jumper et al. 2021) Suppl. Alg.22 lines 7-10 (the attention core, after
 * the linear projections), written out per (i, h) in fp64 (reading G23):
 *   logit_ij = w_L ( c^-1/2 q_i . k_j + b_ij - (gamma_h w_C / 2) sum_p || T_i q_ip - T_j k_jp ||^2 ),
 *   w_L = sqrt(1/3), w_C = sqrt(2 / (9 Pq)), T x = R x + t;
 *   a_ij = softmax_j(logit_ij) (two-pass, Alg.1);
 *   o_i = sum_j a_ij v_j;   opair_i = sum_j a_ij z_ij;   op_ip = T_i^-1 ( sum_j a_ij T_j v_jp ) = R_i^T (g - t_i).
 * Layouts (contiguous fp64): q, k, v [N][H][c]; qp, kp [N][H][Pq][3]; vp [N][H][Pv][3]; R [N][3][3]
 * (row-major, x_global = R x_local + t); t [N][3]; bias [H][N][N]; z [N][N][cz]; gamma [H];
 * outputs o [N][H][c], op [N][H][Pv][3], opair [N][H][cz]. */
int flo_ipa(int64_t N, int64_t H, int64_t c, int64_t Pq, int64_t Pv, int64_t cz, const double* q, const double* k,
            const double* v, const double* qp, const double* kp, const double* vp, const double* R, const double* t,
            const double* bias, const double* z, const double* gamma, double* o, double* op, double* opair) {
  if (N < 1 || H < 1 || c < 1 || Pq < 0 || Pv < 0 || cz < 0) return -1;
  const double wL = sqrt(1.0 / 3.0), wC = Pq > 0 ? sqrt(2.0 / (9.0 * (double)Pq)) : 0.0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t task = 0; task < N * H; ++task) {
    const int64_t i = task / H, h = task % H;
    double* lg = (double*)malloc(sizeof(double) * N);
    double* g = (double*)malloc(sizeof(double) * (Pv > 0 ? Pv * 3 : 1));
    /* logits */
    for (int64_t j = 0; j < N; ++j) {
      double dot = 0.0;
      for (int64_t d = 0; d < c; ++d) dot += q[(i * H + h) * c + d] * k[(j * H + h) * c + d];
      double dist = 0.0;
      for (int64_t pp = 0; pp < Pq; ++pp) {
        double xi[3], yj[3];
        for (int a = 0; a < 3; ++a) {
          xi[a] = t[i * 3 + a];
          yj[a] = t[j * 3 + a];
          for (int bq = 0; bq < 3; ++bq) {
            xi[a] += R[(i * 3 + a) * 3 + bq] * qp[((i * H + h) * Pq + pp) * 3 + bq];
            yj[a] += R[(j * 3 + a) * 3 + bq] * kp[((j * H + h) * Pq + pp) * 3 + bq];
          }
        }
        for (int a = 0; a < 3; ++a) dist += (xi[a] - yj[a]) * (xi[a] - yj[a]);
      }
      lg[j] = wL * (dot / sqrt((double)c) + bias[(h * N + i) * N + j] - gamma[h] * wC / 2.0 * dist);
    }
    /* softmax (two-pass) */
    double m = -INFINITY, den = 0.0;
    for (int64_t j = 0; j < N; ++j) m = lg[j] > m ? lg[j] : m;
    for (int64_t j = 0; j < N; ++j) den += exp(lg[j] - m);
    for (int64_t j = 0; j < N; ++j) lg[j] = exp(lg[j] - m) / den;
    /* outputs */
    for (int64_t d = 0; d < c; ++d) {
      double acc = 0.0;
      for (int64_t j = 0; j < N; ++j) acc += lg[j] * v[(j * H + h) * c + d];
      o[(i * H + h) * c + d] = acc;
    }
    for (int64_t e = 0; e < cz; ++e) {
      double acc = 0.0;
      for (int64_t j = 0; j < N; ++j) acc += lg[j] * z[(i * N + j) * cz + e];
      opair[(i * H + h) * cz + e] = acc;
    }
    for (int64_t pp = 0; pp < Pv; ++pp) {
      for (int a = 0; a < 3; ++a) g[pp * 3 + a] = 0.0;
      for (int64_t j = 0; j < N; ++j)
        for (int a = 0; a < 3; ++a) {
          double y = t[j * 3 + a];
          for (int bq = 0; bq < 3; ++bq) y += R[(j * 3 + a) * 3 + bq] * vp[((j * H + h) * Pv + pp) * 3 + bq];
          g[pp * 3 + a] += lg[j] * y;
        }
      for (int a = 0; a < 3; ++a) {                   /* R_i^T (g - t_i) */
        double acc = 0.0;
        for (int bq = 0; bq < 3; ++bq) acc += R[(i * 3 + bq) * 3 + a] * (g[pp * 3 + bq] - t[i * 3 + bq]);
        op[((i * H + h) * Pv + pp) * 3 + a] = acc;
      }
    }
    free(lg);
    free(g);
  }
  return 0;
}
