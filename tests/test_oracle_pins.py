"""Pins for the fp64 oracle (-m "not gpu"): the oracle is checked against things
other than itself -- closed forms, invariants, library routines (torch SDPA /
torch.softmax run in fp64), the paper's own Listing 1/4 programs executed
eagerly, a hand-derived golden example and brute force.  Each test names the
paper passage or DESIGN.md reading it pins.  A plausible slip in the oracle
(dropped term, wrong sign or index, transposed operand) fails at least one.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from paper_2511_02043_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
D64 = torch.float64


def rnd(*shape, seed=0, lo=-1.0, hi=1.0):
    g = torch.Generator().manual_seed(seed)
    return torch.rand(*shape, generator=g, dtype=D64) * (hi - lo) + lo


def listing1(q, k, v, attn_mask=None):
    """Listing 1 executed eagerly with torch in fp64; attn_mask True = masked."""
    attn_scores = torch.matmul(q, k.transpose(-2, -1))
    attn_scores *= 1 / math.sqrt(q.size(-1))
    if attn_mask is not None:
        attn_scores = attn_scores.masked_fill(attn_mask, -float("inf"))
    attn_weights = torch.softmax(attn_scores, dim=-1)
    return torch.matmul(attn_weights, v)


def O(out, like):
    return torch.from_numpy(out).reshape(like)


# ----------------------------------------------------------------- softmax (Alg.1/Alg.2, §3.3)
def online_softmax_alg2(x):
    """Alg.2, written independently: returns all prefixes (m_j, d_j)."""
    m, d, ms, ds = -math.inf, 0.0, [], []
    for xj in x:
        mj = max(m, xj)
        d = d * math.exp(m - mj) + math.exp(xj - mj) if m != -math.inf else math.exp(xj - mj)
        m = mj
        ms.append(m)
        ds.append(d)
    return ms, ds


@pytest.mark.parametrize("case", ["random", "ascending", "descending", "equal", "dupmax", "single", "wide"])
def test_alg1_matches_library_and_alg2_closed_form(case):
    """P1: Alg.1's asserts, Alg.2 == Alg.1, do[j] closed form at every prefix."""
    r = np.random.default_rng(abs(hash(case)) % 2**32)
    x = {"random": r.normal(size=257), "ascending": np.arange(50.0), "descending": np.arange(50.0)[::-1].copy(),
         "equal": np.full(33, 3.25), "dupmax": np.array([1.0, 7.0, -2.0, 7.0, 0.5]), "single": np.array([-4.0]),
         "wide": r.uniform(-700, 700, size=64)}[case]
    y, m, d = oracle.stable_softmax(x)
    # library routine
    ref = torch.softmax(torch.from_numpy(x), dim=0).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-300)
    assert m == x.max()                                          # Alg.1 Assert m_N = max x
    np.testing.assert_allclose(d, math.fsum(math.exp(v - x.max()) for v in x), rtol=1e-13)
    assert abs(y.sum() - 1.0) < 1e-12 and (y >= 0).all() and (case == "wide" or (y > 0).all())  # Eq.1
    ms, ds = online_softmax_alg2(list(x))
    np.testing.assert_allclose(ds[-1], d, rtol=1e-12)            # ds[N] = do[N]
    for j in range(len(x)):                                       # do[j] = (sum_{i<=j} e^x_i) * e^{-m_j}
        closed = math.fsum(math.exp(v - ms[j]) for v in x[: j + 1])
        np.testing.assert_allclose(ds[j], closed, rtol=1e-12)


def test_softmax_of_zeros_is_uniform():
    y, m, d = oracle.stable_softmax(np.zeros(4))
    np.testing.assert_array_equal(y, np.full(4, 0.25))
    assert m == 0.0 and d == 4.0


# ----------------------------------------------------------------- golden (hand-derived)
def test_golden_hand_computed_2x2():
    """tests/golden/hand_2x2.json: Eq.3 expanded by hand for a 2x2 case (S:L74 idea)."""
    g = json.load(open(os.path.join(GOLDEN, "hand_2x2.json")))
    q, k, v = (torch.tensor(g[n], dtype=D64).reshape(1, 1, 2, 2) for n in ("Q", "K", "V"))
    out, lse = oracle.attn(q, k, v)
    np.testing.assert_allclose(out, np.array(g["O"]), rtol=0, atol=1e-15)
    np.testing.assert_allclose(lse, np.array(g["LSE"]), rtol=0, atol=1e-15)
    out, _ = oracle.attn(q, k, v, mask="causal")
    np.testing.assert_allclose(out, np.array(g["O_causal"]), rtol=0, atol=1e-15)


# ----------------------------------------------------------------- library routines
@pytest.mark.parametrize("sq,sk", [(17, 17), (9, 23), (64, 64)])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_vanilla_and_causal_vs_sdpa(sq, sk, dtype):
    """Eq.3 against torch SDPA (fp64); bf16/fp32 storage read exactly."""
    q, k, v = (rnd(2, 3, s, 16, seed=i).to(dtype) for i, s in enumerate((sq, sk, sk)))
    qd, kd, vd = (t.to(D64) for t in (q, k, v))
    out, lse = oracle.attn(q, k, v)
    ref = F.scaled_dot_product_attention(qd, kd, vd)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)
    s = (qd @ kd.transpose(-1, -2)) / math.sqrt(16)
    torch.testing.assert_close(torch.from_numpy(lse).reshape(2, 3, sq), torch.logsumexp(s, -1), rtol=1e-12, atol=1e-12)
    out, _ = oracle.attn(q, k, v, mask="causal")
    # bottom-right causal (G12): keep k <= q + (Sk - Sq); torch tril with diagonal offset
    keep = torch.ones(sq, sk, dtype=torch.bool).tril(sk - sq)
    ref = F.scaled_dot_product_attention(qd, kd, vd, attn_mask=keep)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)
    if sq == sk:
        ref2 = F.scaled_dot_product_attention(qd, kd, vd, is_causal=True)
        torch.testing.assert_close(O(out, ref.shape), ref2, rtol=1e-12, atol=1e-13)
    # top-left alignment (causal_align = 1, the G12 flag): keep k <= q, which is torch's is_causal
    # convention (tril with diagonal 0) for any S_q, S_k; and a top-left sliding window / prefix
    out, _ = oracle.attn(q, k, v, mask="causal", causal_align=1)
    ref3 = F.scaled_dot_product_attention(qd, kd, vd, is_causal=True)
    torch.testing.assert_close(O(out, ref.shape), ref3, rtol=1e-12, atol=1e-13)
    qi, ki = torch.arange(sq).view(-1, 1), torch.arange(sk).view(1, -1)
    out, _ = oracle.attn(q, k, v, mask="sliding", window=3, causal_align=1)
    ref4 = F.scaled_dot_product_attention(qd, kd, vd, attn_mask=(ki <= qi) & (qi - ki <= 3))
    torch.testing.assert_close(O(out, ref.shape), ref4, rtol=1e-12, atol=1e-13)
    out, _ = oracle.attn(q, k, v, mask="prefix", prefix=5, causal_align=1)
    ref5 = F.scaled_dot_product_attention(qd, kd, vd, attn_mask=(ki < 5) | (ki <= qi))
    torch.testing.assert_close(O(out, ref.shape), ref5, rtol=1e-12, atol=1e-13)


def test_gqa_vs_sdpa_enable_gqa():
    """G15: h_kv = floor(h / (Hq/Hkv)) == PyTorch enable_gqa (P:L858, 16 Q : 2 KV)."""
    q, k, v = rnd(2, 16, 20, 8, seed=1), rnd(2, 2, 20, 8, seed=2), rnd(2, 2, 20, 8, seed=3)
    out, _ = oracle.attn(q, k, v, mask="causal")
    ref = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)


def test_listing1_sliding_window_predicate():
    """G4: Listing 2 predicate keep = (q >= kv) & (q - kv <= w); Listing 3's
    garbled mask read as its complement, fed to Listing 1."""
    S, w = 40, 7
    q, k, v = rnd(1, 2, S, 8, seed=4), rnd(1, 2, S, 8, seed=5), rnd(1, 2, S, 8, seed=6)
    qi = torch.arange(S).view(S, 1)
    kv = torch.arange(S).view(1, S)
    mask = (qi < kv) | ((qi - kv) > w)        # True = masked (Listing 1 convention)
    ref = listing1(q, k, v, mask)
    out, _ = oracle.attn(q, k, v, mask="sliding", window=w)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)


def test_listing4_differential():
    """P:L412-424 Listing 4 run eagerly: chunk on dim=1, shared v, attn0 - lambda*attn1 (G8)."""
    H = 3
    q, k, v = rnd(2, 2 * H, 15, 8, seed=7), rnd(2, 2 * H, 15, 8, seed=8), rnd(2, H, 15, 8, seed=9)
    q0, q1 = q.chunk(2, dim=1)
    k0, k1 = k.chunk(2, dim=1)
    ref = listing1(q0, k0, v) - 0.2 * listing1(q1, k1, v)
    out, lse = oracle.attn(q, k, v, diff=True, lam=0.2)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)
    assert np.isnan(lse).all()
    lam_h = np.array([0.1, 0.5, 0.9])
    ref = listing1(q0, k0, v) - torch.tensor(lam_h).view(1, H, 1, 1) * listing1(q1, k1, v)
    out, _ = oracle.attn(q, k, v, diff=True, lambda_h=lam_h)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)


def test_prefix_and_document_vs_sdpa_bool_masks():
    """G5/G6 predicates fed as bool masks to SDPA (library softmax/matmul)."""
    S = 48
    q, k, v = rnd(2, 2, S, 8, seed=10), rnd(2, 2, S, 8, seed=11), rnd(2, 2, S, 8, seed=12)
    P = 10
    qi, ki = torch.arange(S).view(S, 1), torch.arange(S).view(1, S)
    out, _ = oracle.attn(q, k, v, mask="prefix", prefix=P)
    ref = F.scaled_dot_product_attention(q, k, v, attn_mask=(ki < P) | (ki <= qi))
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)
    offs = synth.doc_offsets(2, S, 5, seed=3)
    for causal in (False, True):
        out, _ = oracle.attn(q, k, v, mask="document", doc_offsets=offs, doc_causal=causal)
        for b in range(2):
            doc = torch.from_numpy(np.searchsorted(offs[b], np.arange(S), side="right") - 1)
            keep = doc.view(S, 1) == doc.view(1, S)
            if causal:
                keep &= ki <= qi
            ref = F.scaled_dot_product_attention(q[b:b + 1], k[b:b + 1], v[b:b + 1], attn_mask=keep)
            torch.testing.assert_close(O(out, (2, 2, S, 8))[b:b + 1], ref, rtol=1e-12, atol=1e-13)


def test_alibi_and_softcap_vs_explicit_torch_ops():
    """Eq.4: score_mod on the SCALED score (G1); ALiBi slope_h*(k-q) (G2), softcap tanh (G3)."""
    H, S = 4, 24
    q, k, v = rnd(1, H, S, 8, seed=13), rnd(1, H, S, 8, seed=14), rnd(1, H, S, 8, seed=15)
    s = (q @ k.transpose(-1, -2)) * (1 / math.sqrt(8))
    slopes = torch.tensor([2.0 ** (-8.0 * (h + 1) / H) for h in range(H)], dtype=D64)
    ref = torch.softmax(s + slopes.view(1, H, 1, 1) * (torch.arange(S).view(1, S) - torch.arange(S).view(S, 1)), -1) @ v
    out, _ = oracle.attn(q, k, v, mod="alibi")
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)
    ref = torch.softmax(20.0 * torch.tanh(s / 20.0), -1) @ v
    out, _ = oracle.attn(q, k, v, mod="softcap", softcap=20.0)
    torch.testing.assert_close(O(out, ref.shape), ref, rtol=1e-12, atol=1e-13)


def test_evoformer_row_and_column_vs_explicit_torch():
    """G9: row attention adds pair bias [b,h,i,j] broadcast over s plus the MSA
    key mask; sigmoid gate.  Column attention = row attention of the transposed MSA."""
    Bn, Ns, Nr, H, c = 1, 5, 7, 2, 4
    m = lambda s: rnd(Bn, Ns, Nr, H, c, seed=s)
    Q, K, V, Gt = m(20), m(21), m(22), m(23)
    bias = rnd(Bn, H, Nr, Nr, seed=24, lo=-4, hi=4)
    msa_mask = torch.ones(Bn, Ns, Nr, dtype=torch.uint8)
    msa_mask[0, 1, 3] = 0
    msa_mask[0, 4, 0] = 0
    # row: views [B, G=s, H, S=i, D=c]
    rv = lambda t: t.permute(0, 1, 3, 2, 4)
    out, _ = oracle.attn(rv(Q), rv(K), rv(V), bias=bias.unsqueeze(1).expand(Bn, Ns, H, Nr, Nr),
                         key_mask=msa_mask, gate_mode="sigmoid", gate=rv(Gt))
    s = torch.einsum("bsihc,bsjhc->bshij", Q, K) / math.sqrt(c) + bias.unsqueeze(1)
    s = s.masked_fill(msa_mask.view(Bn, Ns, 1, 1, Nr) == 0, -float("inf"))
    ref = torch.einsum("bshij,bsjhc->bsihc", torch.softmax(s, -1), V) * torch.sigmoid(Gt)
    torch.testing.assert_close(O(out, (Bn, Ns, H, Nr, c)), rv(ref), rtol=1e-12, atol=1e-13)
    # column: views [B, G=i, H, S=s, D=c]; key mask msa_mask[b, s', i] -> [B, G=i, S=s']
    cv = lambda t: t.permute(0, 2, 3, 1, 4)
    out, _ = oracle.attn(cv(Q), cv(K), cv(V), key_mask=msa_mask.permute(0, 2, 1),
                         gate_mode="sigmoid", gate=cv(Gt))
    s = torch.einsum("bsihc,btihc->bihst", Q, K) / math.sqrt(c)
    s = s.masked_fill(msa_mask.permute(0, 2, 1).reshape(Bn, Nr, 1, 1, Ns) == 0, -float("inf"))
    ref = torch.einsum("bihst,btihc->bsihc", torch.softmax(s, -1), V) * torch.sigmoid(Gt)
    torch.testing.assert_close(O(out, (Bn, Nr, H, Ns, c)), cv(ref), rtol=1e-12, atol=1e-13)
    # and column == row of a transposed copy (P9)
    Qt, Kt, Vt, Gtt = (t.transpose(1, 2).contiguous() for t in (Q, K, V, Gt))
    out2, _ = oracle.attn(rv(Qt), rv(Kt), rv(Vt), key_mask=msa_mask.transpose(1, 2).contiguous(),
                          gate_mode="sigmoid", gate=rv(Gtt))
    np.testing.assert_allclose(out2, out, rtol=0, atol=0)


# ----------------------------------------------------------------- closed forms
MASKS = [("none", {}), ("causal", {}), ("sliding", {"window": 5}), ("prefix", {"prefix": 6}),
         ("document", {"doc_offsets": np.array([[0, 4, 11, 30]], dtype=np.int32)})]


def kept_sets(mask, kw, S):
    """Admissible key sets per row, straight from the predicates (G4-G6)."""
    out = []
    for q in range(S):
        if mask == "none":
            ks = range(S)
        elif mask == "causal":
            ks = range(q + 1)
        elif mask == "sliding":
            ks = range(max(0, q - kw["window"]), q + 1)
        elif mask == "prefix":
            ks = [k for k in range(S) if k < kw["prefix"] or k <= q]
        else:
            o = kw["doc_offsets"][0]
            j = np.searchsorted(o, q, side="right") - 1
            ks = range(o[j], o[j + 1])
        out.append(list(ks))
    return out


@pytest.mark.parametrize("mask,kw", MASKS)
@pytest.mark.parametrize("mod", ["none", "softcap"])
def test_uniform_scores_give_mean_of_kept_v(mask, kw, mod):
    """P2: Q = 0 => every kept score equal => O = mean of the kept V rows (also under softcap)."""
    S = 30
    q = torch.zeros(1, 1, S, 8, dtype=D64)
    k, v = rnd(1, 1, S, 8, seed=30), rnd(1, 1, S, 6, seed=31)
    out, _ = oracle.attn(q, k, v, mask=mask, mod=mod, softcap=3.0, **kw)
    for qi, ks in enumerate(kept_sets(mask, kw, S)):
        np.testing.assert_allclose(out[qi], v[0, 0, ks].mean(0).numpy(), rtol=0, atol=1e-14)


@pytest.mark.parametrize("mask,kw", MASKS + [("blocklist", {})])
@pytest.mark.parametrize("mod", ["none", "alibi", "softcap"])
def test_constant_v_gives_constant(mask, kw, mod):
    """P13: V[k,:] = c  =>  O = c for every non-empty row, every mask and mod."""
    S = 40
    q, k = rnd(1, 2, S, 8, seed=32), rnd(1, 2, S, 8, seed=33)
    c = torch.linspace(-0.9, 0.8, 6, dtype=D64)
    v = c.view(1, 1, 1, 6).expand(1, 2, S, 6).contiguous()
    if mask == "blocklist":
        nqb = 3
        idx = np.array([[[0, 2, -1], [1, -1, -1], [0, 1, 2]]] * 2, dtype=np.int32)
        cnt = np.array([[2, 1, 3]] * 2, dtype=np.int32)
        kw = dict(blk_idx=idx, blk_cnt=cnt, blk_q=16, blk_k=16)
        assert nqb == idx.shape[1]
    out, _ = oracle.attn(q, k, v, mask=mask, mod=mod, softcap=5.0, **kw)
    for r in range(out.shape[0]):
        np.testing.assert_allclose(out[r], c.numpy(), rtol=0, atol=1e-14)


def test_causal_row0_is_v0_and_window0_is_identity():
    """P3: causal row 0 attends only key 0; SW with w=0 attends only the diagonal."""
    S = 19
    q, k, v = rnd(2, 2, S, 8, seed=34), rnd(2, 2, S, 8, seed=35), rnd(2, 2, S, 8, seed=36)
    out, _ = oracle.attn(q, k, v, mask="causal")
    np.testing.assert_array_equal(O(out, (2, 2, S, 8))[:, :, 0], v[:, :, 0])
    out, _ = oracle.attn(q, k, v, mask="sliding", window=0)
    np.testing.assert_array_equal(O(out, (2, 2, S, 8)), v)


def test_empty_rows_give_zero_and_neg_inf_lse():
    """G7: a fully masked row gives O = 0, LSE = -inf."""
    q, k, v = rnd(1, 1, 4, 8, seed=37), rnd(1, 1, 6, 8, seed=38), rnd(1, 1, 6, 8, seed=39)
    km = torch.zeros(1, 1, 6, dtype=torch.uint8)
    out, lse = oracle.attn(q, k, v, key_mask=km)
    assert (out == 0).all() and np.isneginf(lse).all()


def test_diff_lambda_zero_and_equal_maps():
    """P4: lambda=0 => A_0; Q_1=Q_0, K_1=K_0 => (1-lambda) A_0."""
    q0, k0, v = rnd(1, 2, 12, 8, seed=40), rnd(1, 2, 12, 8, seed=41), rnd(1, 2, 12, 8, seed=42)
    q1, k1 = rnd(1, 2, 12, 8, seed=43), rnd(1, 2, 12, 8, seed=44)
    a0, _ = oracle.attn(q0, k0, v, mask="causal")
    out, _ = oracle.attn(torch.cat([q0, q1], 1), torch.cat([k0, k1], 1), v, diff=True, lam=0.0, mask="causal")
    np.testing.assert_array_equal(out, a0)
    out, _ = oracle.attn(torch.cat([q0, q0], 1), torch.cat([k0, k0], 1), v, diff=True, lam=0.3, mask="causal")
    np.testing.assert_allclose(out, 0.7 * a0, rtol=1e-15, atol=1e-16)


def test_gate_identities():
    """P5: gate mul with ones is the identity; sigmoid(+40) ~ 1 and sigmoid(-40) ~ 0."""
    q, k, v = rnd(1, 2, 9, 8, seed=45), rnd(1, 2, 9, 8, seed=46), rnd(1, 2, 9, 8, seed=47)
    base, _ = oracle.attn(q, k, v)
    out, _ = oracle.attn(q, k, v, gate_mode="mul", gate=torch.ones(1, 2, 9, 8, dtype=D64))
    np.testing.assert_array_equal(out, base)
    out, _ = oracle.attn(q, k, v, gate_mode="sigmoid", gate=torch.full((1, 2, 9, 8), 40.0, dtype=D64))
    np.testing.assert_allclose(out, base, rtol=1e-16, atol=1e-17)
    out, _ = oracle.attn(q, k, v, gate_mode="sigmoid", gate=torch.full((1, 2, 9, 8), -40.0, dtype=D64))
    assert np.abs(out).max() < 1e-17
    g = rnd(1, 2, 9, 8, seed=48, lo=-4, hi=4)
    out, _ = oracle.attn(q, k, v, gate_mode="mul", gate=g)
    np.testing.assert_allclose(out, base * g.numpy().reshape(-1, 8), rtol=1e-15)


def test_full_blocklist_is_dense_causal():
    """P6: RSA with every admissible block listed == dense causal attention (BJ north_star)."""
    S, blk = 50, 8
    q, k, v = rnd(1, 2, S, 8, seed=49), rnd(1, 2, S, 8, seed=50), rnd(1, 2, S, 8, seed=51)
    nqb = (S + blk - 1) // blk
    idx = np.full((2, nqb, nqb), -1, dtype=np.int32)
    cnt = np.zeros((2, nqb), dtype=np.int32)
    for i in range(nqb):
        idx[:, i, : i + 1] = np.arange(i + 1)
        cnt[:, i] = i + 1
    out, _ = oracle.attn(q, k, v, mask="blocklist", blk_idx=idx, blk_cnt=cnt, blk_q=blk, blk_k=blk)
    ref, _ = oracle.attn(q, k, v, mask="causal")
    np.testing.assert_array_equal(out, ref)
    idx1 = np.full((2, nqb, 1), -1, dtype=np.int32)
    idx1[:, :, 0] = np.arange(nqb)
    out, _ = oracle.attn(q, k, v, mask="blocklist", blk_idx=idx1, blk_cnt=np.ones((2, nqb), np.int32),
                         blk_q=blk, blk_k=blk)
    # P3: list = {diagonal} => causal attention inside each block
    for i in range(nqb):
        sl = slice(i * blk, min(S, (i + 1) * blk))
        ref, _ = oracle.attn(q[:, :, sl], k[:, :, sl], v[:, :, sl], mask="causal")
        np.testing.assert_allclose(O(out, (2, S, 8))[:, sl].reshape(-1, 8).numpy(), ref, rtol=1e-14, atol=1e-15)


# ----------------------------------------------------------------- invariances (P9)
def test_invariances():
    S = 32
    q, k, v = rnd(1, 2, S, 8, seed=52), rnd(1, 2, S, 8, seed=53), rnd(1, 2, S, 8, seed=54)
    base, lse = oracle.attn(q, k, v)
    # a per-row constant added to scores changes O, shifts LSE by the constant
    row_c = rnd(1, 2, S, 1, seed=55, lo=-3, hi=3)
    out, lse2 = oracle.attn(q, k, v, bias=row_c.expand(1, 2, S, S))
    np.testing.assert_allclose(out, base, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(lse2, lse + row_c.reshape(-1).numpy(), rtol=1e-13)
    # ALiBi == additive bias slope_h * k (the -slope*q part is per-row constant)
    sl = synth.alibi_slopes(2).astype(np.float64)
    al, _ = oracle.attn(q, k, v, mod="alibi")
    bias = torch.from_numpy(sl).view(1, 2, 1, 1) * torch.arange(S, dtype=D64).view(1, 1, 1, S)
    out, _ = oracle.attn(q, k, v, bias=bias.expand(1, 2, S, S))
    np.testing.assert_allclose(out, al, rtol=1e-12, atol=1e-13)
    # key permutation invariance (no position-dependent mod or mask)
    perm = torch.randperm(S, generator=torch.Generator().manual_seed(1))
    out, _ = oracle.attn(q, k[:, :, perm], v[:, :, perm])
    np.testing.assert_allclose(out, base, rtol=1e-12, atol=1e-13)
    # softcap with a huge cap == vanilla
    out, _ = oracle.attn(q, k, v, mod="softcap", softcap=1e6)
    np.testing.assert_allclose(out, base, rtol=1e-9, atol=1e-10)
    # causal perturbation invariance: row q ignores keys > q
    causal, _ = oracle.attn(q, k, v, mask="causal")
    k2, v2 = k.clone(), v.clone()
    k2[:, :, 20:] += 5
    v2[:, :, 20:] -= 7
    out, _ = oracle.attn(q, k2, v2, mask="causal")
    rows = np.array([h * S + r for h in range(2) for r in range(20)])
    np.testing.assert_array_equal(out[rows], causal[rows])
    # SW with w >= S-1 == causal; prefix 0 == causal; prefix S == vanilla
    for kw in (dict(mask="sliding", window=S - 1), dict(mask="prefix", prefix=0)):
        out, _ = oracle.attn(q, k, v, **kw)
        np.testing.assert_array_equal(out, causal)
    out, _ = oracle.attn(q, k, v, mask="prefix", prefix=S)
    np.testing.assert_array_equal(out, base)
    # 1 document == vanilla; 12 documents == per-segment vanilla
    out, _ = oracle.attn(q, k, v, mask="document", doc_offsets=np.array([[0, S]], np.int32))
    np.testing.assert_array_equal(out, base)
    offs = synth.doc_offsets(1, S, 12, seed=4)
    out, _ = oracle.attn(q, k, v, mask="document", doc_offsets=offs)
    for j in range(12):
        a, b = offs[0, j], offs[0, j + 1]
        seg, _ = oracle.attn(q[:, :, a:b], k[:, :, a:b], v[:, :, a:b])
        np.testing.assert_allclose(O(out, (2, S, 8))[:, a:b].reshape(-1, 8).numpy(), seg, rtol=1e-14, atol=1e-15)
    # GQA (G15, consecutive groups) == MHA on K/V heads repeated group by group, bit for bit
    q4 = rnd(1, 4, S, 8, seed=59)
    out, _ = oracle.attn(q4, k, v, mask="causal")
    rep, _ = oracle.attn(q4, k.repeat_interleave(2, dim=1), v.repeat_interleave(2, dim=1), mask="causal")
    np.testing.assert_array_equal(out, rep)
    wrong, _ = oracle.attn(q4, k.repeat(1, 2, 1, 1), v.repeat(1, 2, 1, 1), mask="causal")
    assert not np.allclose(out, wrong)                  # the interleaved map is a different operator


def test_row_subset_equals_full_run():
    """P10: the oracle's row-subset API returns exactly the rows of a full run."""
    q, k, v = rnd(2, 3, 21, 8, seed=56), rnd(2, 3, 21, 8, seed=57), rnd(2, 3, 21, 8, seed=58)
    full, lse = oracle.attn(q, k, v, mask="causal")
    rows = np.array([0, 5, 20, 21, 63, 125])
    sub, lse_s = oracle.attn(q, k, v, mask="causal", rows=rows)
    np.testing.assert_array_equal(sub, full[rows])
    np.testing.assert_array_equal(lse_s, lse[rows])


# ----------------------------------------------------------------- brute force (P7)
def brute(q, k, v, keep, mod=None, gate=None):
    """Quadruple loop in plain Python with math.fsum, tiny shapes only."""
    B, H, Sq, D = q.shape
    Sk, Dv = k.shape[2], v.shape[3]
    out = np.zeros((B, H, Sq, Dv))
    for b in range(B):
        for h in range(H):
            for i in range(Sq):
                s = {}
                for j in range(Sk):
                    if keep(b, h, i, j):
                        x = math.fsum(float(q[b, h, i, d]) * float(k[b, h, j, d]) for d in range(D)) / math.sqrt(D)
                        s[j] = mod(h, i, j, x) if mod else x
                if not s:
                    continue
                mx = max(s.values())
                den = math.fsum(math.exp(x - mx) for x in s.values())
                for d in range(Dv):
                    out[b, h, i, d] = math.fsum(math.exp(x - mx) / den * float(v[b, h, j, d]) for j, x in s.items())
                    if gate is not None:
                        out[b, h, i, d] /= 1.0 + math.exp(-float(gate[b, h, i, d]))
    return out


@pytest.mark.parametrize("name", ["vanilla", "causal", "sliding", "prefix", "alibi", "softcap", "gate"])
def test_brute_force_tiny(name):
    q, k, v = rnd(1, 2, 6, 4, seed=60), rnd(1, 2, 6, 4, seed=61), rnd(1, 2, 6, 3, seed=62)
    keep = lambda b, h, i, j: True
    mod = None
    kw = {}
    gate = None
    if name == "causal":
        keep, kw = (lambda b, h, i, j: j <= i), dict(mask="causal")
    if name == "sliding":
        keep, kw = (lambda b, h, i, j: j <= i and i - j <= 2), dict(mask="sliding", window=2)
    if name == "prefix":
        keep, kw = (lambda b, h, i, j: j < 3 or j <= i), dict(mask="prefix", prefix=3)
    if name == "alibi":
        mod, kw = (lambda h, i, j, x: x + 2.0 ** (-8.0 * (h + 1) / 2) * (j - i)), dict(mod="alibi")
    if name == "softcap":
        mod, kw = (lambda h, i, j, x: 0.5 * math.tanh(x / 0.5)), dict(mod="softcap", softcap=0.5)
    if name == "gate":
        gate = rnd(1, 2, 6, 3, seed=63, lo=-4, hi=4)
        kw = dict(gate_mode="sigmoid", gate=gate)
    ref = brute(q.numpy(), k.numpy(), v.numpy(), keep, mod, None if gate is None else gate.numpy())
    out, _ = oracle.attn(q, k, v, **kw)
    np.testing.assert_allclose(out.reshape(ref.shape), ref, rtol=1e-13, atol=1e-15)


# ----------------------------------------------------------------- RSA selection (G10/G11, P14)
def test_rsa_summaries_and_bound_identity():
    q, k = synth.clustered_qk((1, 2, 64, 16), (1, 1, 64, 16), blk=16, dtype=torch.float32)
    kmin, kmax = oracle.rsa_summaries(k.to(D64), 16)
    kk = k.to(D64).reshape(1, 4, 16, 16)
    np.testing.assert_array_equal(kmin[0], kk[0].amin(1).numpy())
    np.testing.assert_array_equal(kmax[0], kk[0].amax(1).numpy())
    # P14: sum_d max(q_d x_d, q_d y_d) == q+ . x + q- . y when x >= y
    qq = q.to(D64)[0, 0].numpy()
    lhs = np.maximum(qq[:, None, :] * kmax[0][None], qq[:, None, :] * kmin[0][None]).sum(-1)
    rhs = np.maximum(qq, 0) @ kmax[0].T + np.minimum(qq, 0) @ kmin[0].T
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("Sq,Sk,align", [(256, 256, 0), (64, 256, 0), (100, 256, 0), (1, 256, 0), (100, 256, 1),
                                        (256, 256, 1)])
def test_rsa_selection_matches_sort_reference(Sq, Sk, align):
    """G10 selection incl. S_q < S_k (the C5 decode / chunked-prefill shapes) with bottom-right
    (G12) and top-left alignment: diagonal block c of q-block i from the last query's absolute
    position, scores by the q+/q- identity (P14), top-k by a sort with ties to the lower j."""
    blk, topk = 16, 4
    qf, k = synth.clustered_qk((1, 4, Sk, 16), (1, 2, Sk, 16), blk=blk, dtype=torch.bfloat16)
    q = qf[:, :, Sk - Sq:].contiguous()
    idx, cnt, sc = oracle.rsa_select(q, k, blk_q=blk, blk_k=blk, topk=topk, causal_align=align, want_scores=True)
    kmin, kmax = oracle.rsa_summaries(k, blk)
    qd = q.to(D64).numpy()
    nqb = (Sq + blk - 1) // blk
    assert idx.shape[1] == nqb
    for h in range(4):
        hk = h // 2
        for i in range(nqb):
            q_last = min(Sq, (i + 1) * blk) - 1
            c = (q_last + (0 if align else Sk - Sq)) // blk
            if c <= topk + 1:
                assert list(idx[h, i, : cnt[h, i]]) == list(range(c + 1))
                continue
            # independent score via the q+/q- identity (P14), max over the group's heads
            qs = qd[0, hk * 2:(hk + 1) * 2, i * blk:(i + 1) * blk].reshape(-1, 16)
            score = (np.maximum(qs, 0) @ kmax[hk].T + np.minimum(qs, 0) @ kmin[hk].T).max(0)
            np.testing.assert_allclose(sc[h, i, 1:c], score[1:c], rtol=1e-12, atol=1e-12)
            order = sorted(range(1, c), key=lambda j: (-score[j], j))[:topk]
            want = sorted({0, c, *order})
            assert list(idx[h, i, : cnt[h, i]]) == want
            assert cnt[h, i] == topk + 2


def test_keep_rows_is_the_mask_predicate():
    """oracle.keep_rows (definition step 2, used by the T2 schedule test) against the predicates written
    out: Listing 2's window (G4), causal / prefix (G5, G12 both alignments), documents (G6),
    key mask, block list (G10)."""
    Sq, Sk = 37, 50
    q, k, v = rnd(2, 2, Sq, 4, seed=70), rnd(2, 2, Sk, 4, seed=71), rnd(2, 2, Sk, 4, seed=72)
    rows = np.arange(2 * 2 * Sq)
    b, h, qq = rows // (2 * Sq), (rows // Sq) % 2, rows % Sq
    kk = np.arange(Sk)[None, :]
    qa = (qq + Sk - Sq)[:, None]
    offs = np.array([[0, 7, 30, 50], [0, 20, 21, 50]], dtype=np.int32)
    doc = lambda b_, x: np.searchsorted(offs[b_], x, side="right") - 1
    km = (torch.arange(Sk) % 3 != 1).to(torch.uint8).view(1, Sk).expand(2, Sk)
    expect = {
        "causal": (dict(mask="causal"), kk <= qa),
        "topleft": (dict(mask="causal", causal_align=1), kk <= qq[:, None]),
        "sliding": (dict(mask="sliding", window=5), (kk <= qa) & (qa - kk <= 5)),
        "prefix": (dict(mask="prefix", prefix=9), (kk < 9) | (kk <= qa)),
        "document": (dict(mask="document", doc_offsets=offs),
                     np.stack([doc(bb, np.arange(Sk)) == doc(bb, a) for bb, a in zip(b, qa[:, 0])])),
        "keymask": (dict(key_mask=km), np.broadcast_to(km[0].numpy().astype(bool), (len(rows), Sk))),
    }
    for name, (kw, want) in expect.items():
        got = oracle.keep_rows(q, k, v, rows, **kw).astype(bool)
        assert np.array_equal(got, want), name
    idx = np.array([[[0, 2, -1]] * 3] * 4, dtype=np.int32)
    cnt = np.array([[2] * 3] * 4, dtype=np.int32)
    got = oracle.keep_rows(q, k, v, rows, mask="blocklist", blk_idx=idx, blk_cnt=cnt, blk_q=16, blk_k=16).astype(bool)
    listed = ((kk // 16) == 0) | ((kk // 16) == 2)
    assert np.array_equal(got, listed & (kk <= qa))


def test_diff_transformer_epilogue_brute_force_and_closed_forms():
    """Reading G8b (NEXT-2, DIFF Transformer): lambda = exp(q1.k1) - exp(q2.k2) + lambda_init and
    O = (1 - lambda_init) w * x / sqrt(mean(x^2) + eps), x = A_0 - lambda A_1 -- checked against an
    independent math.fsum loop, and closed forms (mean square of a unit-weight row = ms/(ms+eps))."""
    H, S, D = 2, 6, 4
    q, k, v = rnd(1, 2 * H, S, D, seed=80), rnd(1, 2 * H, S, D, seed=81), rnd(1, H, S, D, seed=82)
    lq = rnd(4, D, seed=83, lo=-0.5, hi=0.5).numpy()
    w = rnd(D, seed=84, lo=0.5, hi=1.5).numpy()
    out, _ = oracle.attn(q, k, v, diff=True, lambda_qk=lq, lambda_init=0.7, diff_norm=True, diff_norm_eps=1e-3,
                         diff_norm_w=w)
    lam = math.exp(math.fsum(lq[0] * lq[1])) - math.exp(math.fsum(lq[2] * lq[3])) + 0.7
    a0 = brute(q[:, :H].numpy(), k[:, :H].numpy(), v.numpy(), lambda b, h, i, j: True)
    a1 = brute(q[:, H:].numpy(), k[:, H:].numpy(), v.numpy(), lambda b, h, i, j: True)
    x = a0 - lam * a1
    want = np.zeros_like(x)
    for h in range(H):
        for i in range(S):
            ms = math.fsum(float(t) ** 2 for t in x[0, h, i]) / D
            want[0, h, i] = (1 - 0.7) * w * x[0, h, i] / math.sqrt(ms + 1e-3)
    np.testing.assert_allclose(out.reshape(want.shape), want, rtol=1e-12, atol=1e-14)
    # unit weight, lambda_init 0: every row's mean square is ms / (ms + eps)
    plain, _ = oracle.attn(q, k, v, diff=True, lam=0.4)
    normed, _ = oracle.attn(q, k, v, diff=True, lam=0.4, diff_norm=True, diff_norm_eps=1e-3)
    ms = (plain ** 2).mean(1)
    np.testing.assert_allclose((normed ** 2).mean(1), ms / (ms + 1e-3), rtol=1e-12)
    # q2 = k2 = 0: lambda = exp(q1.k1) - 1 + lambda_init
    lq2 = lq.copy()
    lq2[2:] = 0
    a, _ = oracle.attn(q, k, v, diff=True, lambda_qk=lq2, lambda_init=0.3)
    b, _ = oracle.attn(q, k, v, diff=True, lam=math.exp(float(lq[0] @ lq[1])) - 1 + 0.3)
    np.testing.assert_allclose(a, b, rtol=1e-14, atol=1e-15)


# ----------------------------------------------------------------- backward (NEXT-3)
@pytest.mark.parametrize("kw", [dict(), dict(mask="causal"), dict(mask="sliding", window=2), dict(mod="alibi"),
                                dict(mod="softcap", softcap=0.7), dict(mask="prefix", prefix=2),
                                dict(gate_mode="sigmoid"), dict(gate_mode="mul"), dict(diff=True, lam=0.4),
                                dict(diff=True, lam=0.4, gate_mode="sigmoid"), dict(gqa=True),
                                dict(bias=True, mod="softcap", softcap=0.9), dict(bias="bcast", mask="causal")])
def test_backward_matches_central_differences(kw):
    """The oracle's dQ, dK, dV (plain chain rule) against central differences of the oracle's own
    FORWARD (an independent route: no derivative formula involved), L = sum(O * dO), h = 1e-6."""
    kw = dict(kw)
    gqa = kw.pop("gqa", False)
    maps = 2 if kw.get("diff") else 1
    H, Hkv, S, D = 2, (1 if gqa else 2), 5, 3
    q = rnd(1, H * maps, S, D, seed=90)
    k = rnd(1, Hkv * maps, S, D, seed=91)
    v = rnd(1, Hkv, S, D, seed=92)
    do = rnd(1, H, S, D, seed=93)
    if kw.get("gate_mode"):
        kw["gate"] = rnd(1, H, S, D, seed=94, lo=-2, hi=2)
    gated = bool(kw.get("gate_mode"))
    bias_kind = kw.pop("bias", None)
    if bias_kind:                  # additive bias (G16); "bcast": one [H, S, S] bias broadcast over B = 2
        if bias_kind == "bcast":
            q, k, v, do = (torch.cat([t, t * 0.5 + 0.1]) for t in (q, k, v, do))
            base = rnd(1, H, S, S, seed=95, lo=-1, hi=1)
            kw["bias"] = base.expand(2, H, S, S)
        else:
            base = rnd(1, H, S, S, seed=95, lo=-1, hi=1)
            kw["bias"] = base
    outs = oracle.attn_bwd(q, k, v, do, with_dgate=gated, with_dbias=bool(bias_kind), **kw)
    dq, dk, dv = outs[:3]
    L = lambda q_, k_, v_: float((oracle.attn(q_, k_, v_, **kw)[0].reshape(do.shape) * do.numpy()).sum())
    h = 1e-6
    pairs = [(q, dq), (k, dk), (v, dv)] + ([(kw["gate"], outs[3])] if gated else [])   # the gate is read through kw
    if bias_kind:              # dbias summed over the dims the bias broadcasts (B for "bcast"), shaped like base
        db = outs[-1].sum(axis=0, keepdims=True) if bias_kind == "bcast" else outs[-1]
        pairs.append((base, db.reshape(base.shape)))
    for t, grad in pairs:
        num = np.zeros(grad.shape)
        flat = t.view(-1)
        for i in range(flat.numel()):
            old = flat[i].item()
            flat[i] = old + h
            lp = L(q, k, v)
            flat[i] = old - h
            lm = L(q, k, v)
            flat[i] = old
            num.reshape(-1)[i] = (lp - lm) / (2 * h)
        np.testing.assert_allclose(grad, num, rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("gated", [False, True])
def test_backward_dlambda_matches_central_differences(gated):
    """dL/dlambda_h of Listing 4 (G8) against central differences of the oracle forward in the
    per-head lambda_h and in the scalar lambda (whose gradient is the sum over heads), with and without the
    sigmoid gate, causal, GQA 2:1."""
    H, Hkv, S, D = 2, 1, 6, 4
    q, k, v, do = rnd(1, 2 * H, S, D, seed=80), rnd(1, 2 * Hkv, S, D, seed=81), rnd(1, Hkv, S, D, seed=82), rnd(1, H, S, D, seed=83)
    kw = dict(diff=True, mask="causal")
    if gated:
        kw.update(gate_mode="sigmoid", gate=rnd(1, H, S, D, seed=84, lo=-2, hi=2))
    lh = np.array([0.3, -0.45])
    dl = oracle.attn_bwd(q, k, v, do, with_dgate=gated, with_dlambda=True, lambda_h=torch.tensor(lh), **kw)[-1]
    L = lambda **x: float((oracle.attn(q, k, v, **kw, **x)[0].reshape(do.shape) * do.numpy()).sum())
    h = 1e-6
    for i in range(H):
        lp, lm = lh.copy(), lh.copy()
        lp[i] += h
        lm[i] -= h
        num = (L(lambda_h=torch.tensor(lp)) - L(lambda_h=torch.tensor(lm))) / (2 * h)
        assert abs(dl[i] - num) <= 1e-6 * max(1.0, abs(num)), (i, dl[i], num)
    dl_s = oracle.attn_bwd(q, k, v, do, with_dgate=gated, with_dlambda=True, lam=0.25, **kw)[-1]
    num = (L(lam=0.25 + h) - L(lam=0.25 - h)) / (2 * h)
    assert abs(dl_s.sum() - num) <= 1e-6 * max(1.0, abs(num))
    assert np.all(dl_s != 0.0)


def test_backward_matches_torch_autograd_listing1():
    """Listing 1 executed eagerly in fp64 under torch.autograd, causal and GQA via repeats."""
    q, k, v, do = rnd(2, 4, 33, 8, seed=95), rnd(2, 2, 33, 8, seed=96), rnd(2, 2, 33, 8, seed=97), rnd(2, 4, 33, 8, seed=98)
    qt, kt, vt = (t.clone().requires_grad_(True) for t in (q, k, v))
    mask = ~torch.ones(33, 33, dtype=torch.bool).tril()
    out = listing1(qt, kt.repeat_interleave(2, dim=1), vt.repeat_interleave(2, dim=1), attn_mask=mask)
    (out * do).sum().backward()
    dq, dk, dv = oracle.attn_bwd(q, k, v, do, mask="causal")
    np.testing.assert_allclose(dq, qt.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dk, kt.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dv, vt.grad.numpy(), rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- NEXT-2: LayerNorm-prologue linear
def _ln_case(M=37, K=128, N=48, seed=3):
    g = torch.Generator().manual_seed(seed)
    x = torch.rand(M, K, generator=g, dtype=torch.float64) * 4 - 2
    w = (torch.rand(N, K, generator=g, dtype=torch.float64) * 2 - 1) / np.sqrt(K)
    gam = torch.rand(K, generator=g, dtype=torch.float64) + 0.5
    bet = torch.rand(K, generator=g, dtype=torch.float64) - 0.5
    bias = torch.rand(N, generator=g, dtype=torch.float64) - 0.5
    return x, w, gam, bet, bias


def test_linear_ln_plain_is_matmul():
    """No LayerNorm: y = x w^T + bias, the library matmul (special case that is a library routine)."""
    x, w, _, _, bias = _ln_case()
    y = oracle.linear_ln(x, w, bias=bias)
    assert np.abs(y - (x.numpy() @ w.numpy().T + bias.numpy())).max() < 1e-12


def test_linear_ln_matches_torch_layer_norm():
    """LayerNorm prologue (AF2 Alg.7 line 1): torch.nn.functional.layer_norm (biased variance, eps inside
    the square root) followed by the product."""
    x, w, gam, bet, bias = _ln_case()
    y = oracle.linear_ln(x, w, bias=bias, ln_gamma=gam, ln_beta=bet, eps=1e-5)
    ref = torch.nn.functional.layer_norm(x, (x.shape[1],), gam, bet, 1e-5) @ w.T + bias
    assert np.abs(y - ref.numpy()).max() < 1e-11


def test_linear_ln_invariants():
    """With gamma = 1, beta = 0 and w = I: every output row has mean 0 and variance var / (var + eps)
    (closed form); LayerNorm is invariant under x -> a x + c for a > 0 up to eps; a constant row
    normalises to beta (so y = w beta + bias)."""
    x, _, _, bet, _ = _ln_case(K=64, N=64)
    K = x.shape[1]
    eye = torch.eye(K, dtype=torch.float64)
    ones = torch.ones(K, dtype=torch.float64)
    y = oracle.linear_ln(x, eye, ln_gamma=ones, eps=1e-5)
    var = x.var(dim=1, unbiased=False).numpy()
    assert np.abs(y.mean(axis=1)).max() < 1e-12
    assert np.abs(y.var(axis=1) - var / (var + 1e-5)).max() < 1e-12
    y0 = oracle.linear_ln(x, eye, ln_gamma=ones, eps=0.0)
    y1 = oracle.linear_ln(3.5 * x - 1.25, eye, ln_gamma=ones, eps=0.0)
    assert np.abs(y0 - y1).max() < 1e-12
    xc = torch.full((2, K), 0.7, dtype=torch.float64)
    _, w, _, _, bias = _ln_case(K=K, N=5)
    yc = oracle.linear_ln(xc, w, bias=bias, ln_gamma=ones, ln_beta=bet, eps=1e-5)
    assert np.abs(yc - (w.numpy() @ bet.numpy() + bias.numpy())).max() < 1e-12


def test_linear_ln_abs_scale():
    """yabs = sum_k |xhat| |w| bounds |y - bias| (triangle inequality) and equals it for non-negative data."""
    x, w, gam, bet, bias = _ln_case()
    y, ya = oracle.linear_ln(x, w, bias=bias, ln_gamma=gam, ln_beta=bet, with_abs=True)
    assert (np.abs(y - bias.numpy()) <= ya + 1e-12).all()
    xp, wp = x.abs(), w.abs()
    y2, ya2 = oracle.linear_ln(xp, wp, with_abs=True)
    assert np.abs(y2 - ya2).max() < 1e-12


# ---------------------------------------------------------------- NEXT-4: Invariant Point Attention (G23)
def _ipa(N=7, H=2, c=4, Pq=2, Pv=3, cz=5, seed=4):
    from paper_2511_02043_b200 import synth
    return {k: v.double() for k, v in synth.ipa_inputs(N, H, c, Pq, Pv, cz, seed=seed, dtype=torch.float64).items()}


def test_ipa_invariant_under_global_rigid_motion():
    """IPA's defining property (AF2 Suppl. 1.8.2): a global rotation + translation of every frame leaves
    the scalar, local-point and pair outputs unchanged."""
    x = _ipa()
    o, op, opair = oracle.ipa(**x)
    g = torch.Generator().manual_seed(9)
    qq = torch.randn(4, generator=g, dtype=torch.float64)
    a, b, c, d = (qq / qq.norm()).tolist()
    G = torch.tensor([[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                      [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                      [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]], dtype=torch.float64)
    y = dict(x, R=G @ x["R"], t=x["t"] @ G.T + torch.tensor([5.0, -3.0, 11.0], dtype=torch.float64))
    o2, op2, opair2 = oracle.ipa(**y)
    np.testing.assert_allclose(o2, o, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(op2, op, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(opair2, opair, rtol=1e-10, atol=1e-12)


def test_ipa_without_points_is_biased_attention():
    """gamma = 0 removes the point term: o = softmax(w_L (q.k / sqrt(c) + b)) v, i.e. the attention oracle
    with scale w_L / sqrt(c) and additive bias w_L b (w_L = sqrt(1/3))."""
    x = _ipa()
    x["gamma"] = torch.zeros_like(x["gamma"])
    o, _, _ = oracle.ipa(**x)
    wl = math.sqrt(1 / 3)
    q4 = x["q"].permute(1, 0, 2).unsqueeze(0)
    k4 = x["k"].permute(1, 0, 2).unsqueeze(0)
    v4 = x["v"].permute(1, 0, 2).unsqueeze(0)
    ref, _ = oracle.attn(q4, k4, v4, scale=wl / math.sqrt(x["q"].shape[2]), bias=(wl * x["bias"]).unsqueeze(0))
    np.testing.assert_allclose(o, np.asarray(ref).reshape(q4.shape).transpose(0, 2, 1, 3)[0], rtol=1e-12, atol=1e-13)


def test_ipa_brute_force():
    """Every output against a separate math.fsum transcription of AF2 Alg.22 lines 7-10 on a tiny case."""
    x = _ipa(N=4, H=2, c=3, Pq=2, Pv=2, cz=3, seed=6)
    o, op, opair = oracle.ipa(**x)
    X = {k: v.numpy() for k, v in x.items()}
    N, H, c = X["q"].shape
    Pq, Pv = X["qp"].shape[2], X["vp"].shape[2]
    wl, wc = math.sqrt(1 / 3), math.sqrt(2 / (9 * Pq))
    glob = lambda i, pt: X["R"][i] @ pt + X["t"][i]
    for i in range(N):
        for h in range(H):
            lg = []
            for j in range(N):
                dot = math.fsum(X["q"][i, h, d] * X["k"][j, h, d] for d in range(c))
                dist = math.fsum(float(((glob(i, X["qp"][i, h, p]) - glob(j, X["kp"][j, h, p])) ** 2).sum())
                                 for p in range(Pq))
                lg.append(wl * (dot / math.sqrt(c) + X["bias"][h, i, j] - X["gamma"][h] * wc / 2 * dist))
            m = max(lg)
            e = [math.exp(v - m) for v in lg]
            s = math.fsum(e)
            a = [v / s for v in e]
            for d in range(c):
                assert abs(o[i, h, d] - math.fsum(a[j] * X["v"][j, h, d] for j in range(N))) < 1e-12
            for f in range(X["z"].shape[2]):
                assert abs(opair[i, h, f] - math.fsum(a[j] * X["z"][i, j, f] for j in range(N))) < 1e-12
            for p in range(Pv):
                gsum = sum(a[j] * glob(j, X["vp"][j, h, p]) for j in range(N))
                loc = X["R"][i].T @ (gsum - X["t"][i])
                np.testing.assert_allclose(op[i, h, p], loc, rtol=1e-10, atol=1e-12)
