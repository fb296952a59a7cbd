"""GPU parity of the Rectified-Sparse-Attention row (reading G10/G11):
block summaries (bit-exact vs the oracle), data-dependent selection (G11 acceptance:
exact set equality wherever the oracle's k-th / (k+1)-th score gap exceeds the fp32
accumulation bound, otherwise a valid top-k), and the bf16 tcgen05 attention over a
block list (max-abs 2e-2 vs the fp64 oracle given the same list)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_02043_b200 import synth
from tests import cases
from tests.parity import TOL, check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl as _fl
    return _fl


# ------------------------------------------------------------------ summaries (bit-exact)
@pytest.mark.parametrize("shape,blk", [((1, 2, 1000, 128), 128), ((2, 3, 333, 64), 128), ((1, 1, 256, 32), 64),
                                       ((1, 1, 77, 128), 128)])
def test_summaries_bit_exact(fl, shape, blk):
    k = synth.uniform(shape, seed=3, tensor="k")
    kmin, kmax = fl.rsa_build_summaries(k.cuda(), blk)
    torch.cuda.synchronize()
    rmin, rmax = oracle.rsa_summaries(k, blk)
    assert np.array_equal(kmin.cpu().double().numpy(), rmin)
    assert np.array_equal(kmax.cpu().double().numpy(), rmax)


def test_summaries_rank5_strided(fl):
    """Evoformer-style strided view [B, G, H, S, D] (no copy)."""
    st = synth.uniform((1, 40, 6, 2, 64), seed=4, tensor="k", lead=3)   # [B, s, i, h, c]
    view = st.permute(0, 2, 3, 1, 4)                                      # [B, G=i, H, S=s, c]
    kmin, kmax = fl.rsa_build_summaries(st.cuda().permute(0, 2, 3, 1, 4), 16)
    torch.cuda.synchronize()
    rmin, rmax = oracle.rsa_summaries(view, 16)
    assert np.array_equal(kmin.cpu().double().numpy(), rmin)
    assert np.array_equal(kmax.cpu().double().numpy(), rmax)


@pytest.mark.parametrize("s1,s2,blk", [(640, 1000, 128), (600, 1000, 128), (1000, 1001, 128), (0, 300, 64),
                                       (777, 777, 128)])
def test_summaries_update_after_append(fl, s1, s2, blk):
    """KV append: summaries valid for keys [0, s1), cache grows to s2, update from
    k_begin = s1 -> bit-equal to the oracle's summaries of the whole cache; blocks before
    floor(s1 / blk) are not rewritten (sentinel preserved)."""
    k = synth.uniform((1, 2, s2, 64), seed=5, tensor="k")
    kd = k.cuda()
    nkb = (s2 + blk - 1) // blk
    kmin = torch.full((2, nkb, 64), 7.0, device="cuda", dtype=torch.bfloat16)
    kmax = torch.full((2, nkb, 64), 7.0, device="cuda", dtype=torch.bfloat16)
    j0 = s1 // blk
    if s1 > 0:                                   # the pre-append state: summaries of [0, s1)
        pmin, pmax = fl.rsa_build_summaries(kd[:, :, :s1], blk)
        kmin[:, :j0] = pmin[:, :j0]
        kmax[:, :j0] = pmax[:, :j0]
    fl.rsa_update_summaries(kd, kmin, kmax, s1, blk)
    torch.cuda.synchronize()
    rmin, rmax = oracle.rsa_summaries(k, blk)
    assert np.array_equal(kmin.cpu().double().numpy(), rmin)
    assert np.array_equal(kmax.cpu().double().numpy(), rmax)
    sentinel = torch.full((2, nkb, 64), 7.0, dtype=torch.bfloat16)
    kmin2 = sentinel.clone().cuda()
    fl.rsa_update_summaries(kd, kmin2, sentinel.clone().cuda(), s2, blk)     # k_begin = S_k: only the tail block
    torch.cuda.synchronize()
    keep = (s2 // blk)
    assert torch.equal(kmin2[:, :keep].cpu(), sentinel[:, :keep])


# ------------------------------------------------------------------ selection (G11)
def selection_eps(q, kmin, kmax, Hq, Hkv):
    """G11 bound on the fp32 accumulation error of one score, maxed over blocks/queries:
    2D * 2^-24 * sum_d |q_d| max(|kmax_d|, |kmin_d|) (x4 margin for the tensor core's
    internal accumulation order)."""
    qa = q.abs().double().numpy()                     # [B,Hq,S,D]
    ka = np.maximum(np.abs(kmin), np.abs(kmax))       # [B*Hkv, nkb, D]
    D = qa.shape[-1]
    worst = 0.0
    for bh in range(ka.shape[0]):
        b, hk = divmod(bh, Hkv)
        grp = Hq // Hkv
        qmax = qa[b, hk * grp:(hk + 1) * grp].max(axis=(0, 1))   # upper bound of |q_d| over rows
        worst = max(worst, float((ka[bh] * qmax).sum(-1).max()))
    return 4 * 2 * D * 2.0 ** -24 * worst


def check_selection(got_idx, got_cnt, ref_idx, ref_cnt, scores, topk, eps, nkb, q_off, Sq):
    """G11: accept the GPU list if it has the sink and the diagonal, the right size, and
    every selected block's oracle score >= the oracle k-th score - 2 eps; require exact
    equality when the oracle's k-th / (k+1)-th gap exceeds 2 eps."""
    n_exact = 0
    BH, nqb, _ = ref_idx.shape
    for bh in range(BH):
        for i in range(nqb):
            rl = list(ref_idx[bh, i, : ref_cnt[bh, i]])
            gl = list(got_idx[bh, i, : got_cnt[bh, i]])
            assert all(x == -1 for x in got_idx[bh, i, got_cnt[bh, i]:]), (bh, i)
            c = rl[-1]
            assert len(gl) == len(rl), (bh, i, gl, rl)
            assert gl == sorted(set(gl)) and gl[0] == 0 and gl[-1] == c, (bh, i, gl)
            cand = scores[bh, i, 1:c]
            if c - 1 <= topk or topk == 0:
                assert gl == rl
                n_exact += 1
                continue
            srt = np.sort(cand)[::-1]
            kth, nxt = srt[topk - 1], srt[topk]
            if kth - nxt > 2 * eps:
                assert gl == rl, (bh, i, gl, rl, kth, nxt)
                n_exact += 1
            else:
                for j in gl[1:-1]:
                    assert scores[bh, i, j] >= kth - 2 * eps, (bh, i, j)
    return n_exact


SEL_CASES = [
    dict(name="mha_D128", B=1, Hq=2, Hkv=2, Sq=2048, Sk=2048, D=128, topk=4),
    dict(name="ragged_D64", B=2, Hq=1, Hkv=1, Sq=1000, Sk=1000, D=64, topk=3),
    dict(name="gqa_D128", B=1, Hq=4, Hkv=2, Sq=1536, Sk=1536, D=128, topk=4),
    dict(name="sq_lt_sk", B=1, Hq=2, Hkv=2, Sq=300, Sk=3000, D=128, topk=5),
    dict(name="top_left", B=1, Hq=1, Hkv=1, Sq=700, Sk=3000, D=64, topk=5, causal_align=1),
    dict(name="decode", B=2, Hq=2, Hkv=2, Sq=1, Sk=4096 + 77, D=128, topk=16),
    dict(name="nkb256_tail", B=1, Hq=1, Hkv=1, Sq=1024, Sk=32768, D=128, topk=16),
    dict(name="nkb512_D64", B=1, Hq=1, Hkv=1, Sq=256, Sk=65536, D=64, topk=16),
    dict(name="topk0", B=1, Hq=1, Hkv=1, Sq=1024, Sk=1024, D=128, topk=0),
    # diagonal c = 129 (and 257 at D = 64): candidate c-1 opens a new 128-block accumulator tile; the
    # planted key block (= the query block's own rows) has the top score, so dropping it fails
    dict(name="c129_plant", B=1, Hq=1, Hkv=1, Sq=16640, Sk=16640, D=128, topk=16, plant=[(129, 128), (101, 100)]),
    dict(name="c257_plant_D64", B=1, Hq=1, Hkv=1, Sq=33024, Sk=33024, D=64, topk=16,
         plant=[(129, 128), (257, 256)]),
]


@pytest.mark.parametrize("case", SEL_CASES, ids=[c["name"] for c in SEL_CASES])
def test_selection_vs_oracle(fl, case):
    B, Hq, Hkv, Sq, Sk, D, topk = (case[x] for x in ("B", "Hq", "Hkv", "Sq", "Sk", "D", "topk"))
    ca = case.get("causal_align", 0)
    q, k = synth.clustered_qk((B, Hq, Sk, D), (B, Hkv, Sk, D), seed=2)
    for i, j in case.get("plant", ()):                  # key block j := query block i (bottom-right, Sq = Sk)
        k[:, :, j * 128:(j + 1) * 128] = q[:, :Hkv, i * 128:(i + 1) * 128]
    q = q[:, :, Sk - Sq:].contiguous()                 # the last Sq queries (bottom-right)
    ref_idx, ref_cnt, sc = oracle.rsa_select(q, k, topk=topk, causal_align=ca, want_scores=True)
    for i, j in case.get("plant", ()):
        assert j in ref_idx[0, i, :ref_cnt[0, i]]       # the planted block is the oracle's pick
    kmin, kmax = fl.rsa_build_summaries(k.cuda(), 128)
    idx, cnt = fl.rsa_select(q.cuda(), kmin, kmax, Sk, topk=topk, causal_align=ca)
    torch.cuda.synchronize()
    rmin, rmax = oracle.rsa_summaries(k, 128)
    eps = selection_eps(q, rmin, rmax, Hq, Hkv)
    n_exact = check_selection(idx.cpu().numpy(), cnt.cpu().numpy(), ref_idx, ref_cnt, sc, topk, eps,
                              (Sk + 127) // 128, Sk - Sq, Sq)
    assert n_exact >= 0.5 * ref_cnt.size, "too few exactly-decided lists: inputs are not discriminative"


# ------------------------------------------------------------------ attention over a block list
BL_CASES = [
    dict(name="bl_D128", Hq=2, S=1300, D=128, topk=3),
    dict(name="bl_D64_const", Hq=2, S=1100, D=64, topk=2, dist="constant"),
    dict(name="bl_D128_const_gqa", Hq=4, Hkv=2, S=900, D=128, topk=2, dist="constant"),
    dict(name="bl_D32", Hq=1, S=700, D=32, topk=1),
    dict(name="bl_sq_ne_sk_const", Hq=2, Sq=200, Sk=1500, D=128, topk=3, dist="constant"),
    dict(name="bl_decode_const", B=2, Hq=2, Sq=1, Sk=3000, D=128, topk=4, dist="constant"),
    dict(name="bl_full_list_needle", Hq=1, S=1000, D=128, topk=64, dist="needle"),
]


@pytest.mark.parametrize("case", BL_CASES, ids=[c["name"] for c in BL_CASES])
def test_blocklist_attention(fl, case):
    ins, gk, ok = cases.build(dict(case, dtype="bf16", mask="blocklist"))
    out = cases.run_gpu(fl, ins, gk)
    ref, _ = cases.run_oracle(ins, ok)
    strong = case.get("dist") in ("needle", "constant")
    check(out.cpu().double().reshape(ref.shape), ref, TOL["bf16"], min_ref=0.1 if strong else 0.0,
          what=case["name"])


def test_full_blocklist_equals_dense_causal(fl):
    """P6 on the GPU: listing every admissible block gives dense causal attention."""
    ins, gk, _ = cases.build(dict(Hq=2, S=1000, D=128, topk=64, mask="blocklist", dtype="bf16"))
    out_bl = cases.run_gpu(fl, ins, gk)
    ins2 = dict(ins)
    out_c = fl.attn_fwd(ins2["q"].cuda(), ins2["k"].cuda(), ins2["v"].cuda(), mask="causal")
    torch.cuda.synchronize()
    # same tiling (128-key tiles on both paths) -> identical arithmetic; allow bf16 rounding slack in
    # case the interval kernel's tile size differs (FL_BN64 builds)
    assert (out_bl.float() - out_c.float()).abs().max().item() <= 4e-3


def test_rsa_pipeline_end_to_end(fl):
    """summaries -> selection -> attention, all on the GPU, against the oracle given the
    oracle's own list (identical lists on clustered inputs; checked first)."""
    B, H, S, D, topk = 1, 2, 2048, 128, 4
    q, k = synth.clustered_qk((B, H, S, D), (B, H, S, D), seed=2)
    v = synth.constant_v((B, H, S, D), seed=5)
    ref_idx, ref_cnt, _ = oracle.rsa_select(q, k, topk=topk)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    kmin, kmax = fl.rsa_build_summaries(kd, 128)
    idx, cnt = fl.rsa_select(qd, kmin, kmax, S, topk=topk)
    out = fl.attn_fwd(qd, kd, vd, mask="blocklist", blk_idx=idx, blk_cnt=cnt)
    torch.cuda.synchronize()
    assert np.array_equal(idx.cpu().numpy(), ref_idx) and np.array_equal(cnt.cpu().numpy(), ref_cnt)
    ref, _ = oracle.attn(q, k, v, mask="blocklist", blk_idx=ref_idx, blk_cnt=ref_cnt)
    check(out.cpu().double().reshape(ref.shape), ref, TOL["bf16"], min_ref=0.1, what="rsa pipeline")


def test_rsa_errors_are_loud(fl):
    k = torch.zeros(1, 1, 256, 12, device="cuda", dtype=torch.bfloat16)   # D % 8 != 0
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.rsa_build_summaries(k, 128)
    q = torch.zeros(1, 1, 256, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.zeros(1, 1, 256 * 300, 128, device="cuda", dtype=torch.bfloat16)
    kmin, kmax = fl.rsa_build_summaries(k, 128)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.rsa_select(q, kmin, kmax, k.shape[2], topk=4)              # 300 blocks > 256 at D=128
