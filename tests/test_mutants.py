"""T4 mutation tests (-m "not gpu", SPEC's injected-bug idea S:L469): the parity
checker (tests/parity.py) must FAIL on plausible kernel bugs, evaluated on the very inputs the GPU
parity tests use.  Each mutant is a synthetic "GPU output": the fp64 oracle run on a mutated
problem (mask off by one, wrong head map, dropped or swapped map, missing gate / bias / mod, shifted
block list, a wrong K tile) or, for the online-softmax rescale, an independent buggy tile loop.
A mutant that the checker accepted would mean the GPU test cannot see that bug."""
import math

import numpy as np
import pytest
import torch

import oracle
from tests import cases
from tests.parity import TOL, check
from tests.test_gpu_parity import BF16_CASES
from tests.test_gpu_rsa import BL_CASES

CASES = {c["name"]: c for c in BF16_CASES + [dict(b, mask="blocklist") for b in BL_CASES]}


def must_fail(got, ref, what, strong=True):
    with pytest.raises(AssertionError):
        check(got.reshape(ref.shape), ref, TOL["bf16"], min_ref=0.1 if strong else 0.0, what=what)


def setup(name):
    case = dict(CASES[name], dtype="bf16")
    if case.get("mask") == "document":
        from paper_2511_02043_b200 import synth
        S = case.get("Sk", case.get("S", 128))
        case["doc_offsets"] = synth.doc_offsets(case.get("B", 1), S, case.get("n_docs", 12), seed=case.get("seed", 0) + 1)
    ins, gk, ok = cases.build(case)
    ref, _ = cases.run_oracle(ins, ok)
    # the unmutated oracle passes its own check with the GPU test's strength requirement
    strong = case.get("dist") in ("needle", "constant")
    check(ref, ref, TOL["bf16"], min_ref=0.1 if strong else 0.0, what=name)
    return case, ins, ok, ref


def keep_matrix(case, Sq, Sk, b=0):
    lo, hi = cases.admissible(case, Sq, Sk)(np.arange(Sq), b)
    k = np.arange(Sk)
    return (k[None, :] >= lo[:, None]) & (k[None, :] < hi[:, None])


def as_bias(keep, B, H):
    """A boolean keep matrix [Sq, Sk] as an additive fp64 bias (0 / -inf) for the oracle."""
    b = torch.from_numpy(np.where(keep, 0.0, -np.inf))
    return b.view(1, 1, *keep.shape).expand(B, H, *keep.shape)


@pytest.mark.parametrize("name", ["causal_needle_D128", "diff_needle_D64", "keymask_needle_D32",
                                  "gqa_needle_D64", "bl_full_list_needle"])
def test_zeros_output_fails(name):
    _, _, _, ref = setup(name)
    must_fail(np.zeros_like(ref), ref, f"zeros {name}")


@pytest.mark.parametrize("name,mut", [
    ("sliding_needle_D128", dict(window=199)),           # window one key too short
    ("sliding_leak_D64", dict(window=201)),              # window one key too long
    ("sliding_leak_D128", dict(mask="causal")),          # window ignored
])
def test_window_off_by_one_fails(name, mut):
    case, ins, ok, ref = setup(name)
    got, _ = cases.run_oracle(ins, dict(ok, **mut))
    must_fail(got, ref, f"{name} {mut}", strong=False)


@pytest.mark.parametrize("name,shift", [("causal_leak_D128", 1), ("causal_leak_D32", 1), ("causal_needle_D64", -1),
                                        ("prefix_leak_D64", "prefix+1"), ("document_leak_D128", "doc+1")])
def test_mask_boundary_off_by_one_fails(name, shift):
    case, ins, ok, ref = setup(name)
    q = ins["q"]
    B, H, Sq, _ = q.shape
    Sk = ins["k"].shape[2]
    keep = keep_matrix(case, Sq, Sk)
    if shift == 1:                                        # causal admits k = q + 1
        keep |= np.eye(Sq, Sk, k=1, dtype=bool)
    elif shift == -1:                                     # causal drops the diagonal
        keep &= ~np.eye(Sq, Sk, dtype=bool)
    elif shift == "prefix+1":
        keep[:, case["prefix"]] = True
    elif shift == "doc+1":                                # each document also sees the next one's first key
        lo, hi = cases.admissible(case, Sq, Sk)(np.arange(Sq), 0)
        keep[np.arange(Sq), np.minimum(hi, Sk - 1)] = True
    okm = {x: y for x, y in ok.items() if x not in ("mask", "window", "prefix", "doc_offsets")}
    got, _ = cases.run_oracle(ins, dict(okm, bias=as_bias(keep, B, H)))
    must_fail(got, ref, f"{name} {shift}", strong=False)


def buggy_online(q, k, v, keep, flip_rescale=False, tile=128):
    """Independent tile-wise online softmax (Alg.2 at tile granularity) with an optional bug:
    the running O / l are rescaled by exp(m_new - m_old) instead of exp(m_old - m_new)."""
    q, k, v = (t.double().numpy()[0, 0] for t in (q, k, v))
    Sq, D = q.shape
    Sk = k.shape[0]
    out = np.zeros((Sq, v.shape[1]))
    s_all = q @ k.T / math.sqrt(D)
    for r in range(Sq):
        m, l, o = -np.inf, 0.0, np.zeros(v.shape[1])
        for t0 in range(0, Sk, tile):
            s = np.where(keep[r, t0:t0 + tile], s_all[r, t0:t0 + tile], -np.inf)
            mt = max(m, s.max())
            if mt == -np.inf:
                continue
            corr = math.exp(m - mt) if m != -np.inf else 0.0
            if flip_rescale and m != -np.inf:
                corr = math.exp(mt - m)
            p = np.exp(s - mt)
            l = l * corr + p.sum()
            o = o * corr + p @ v[t0:t0 + tile]
            m = mt
        out[r] = o / l if l > 0 else 0.0
    return out


def test_flipped_rescale_sign_fails_and_correct_loop_passes():
    case, ins, ok, ref = setup("causal_needle_D128")
    keep = keep_matrix(case, 700, 700)
    good = buggy_online(ins["q"], ins["k"], ins["v"], keep, flip_rescale=False)
    check(good.reshape(ref.shape), ref, 1e-9, what="correct online loop")
    bad = buggy_online(ins["q"], ins["k"], ins["v"], keep, flip_rescale=True)
    must_fail(bad, ref, "flipped rescale")


def test_wrong_kv_tile_fails():
    """K/V tile j read from tile j + 1 (a TMA coordinate bug) on the causal needle case."""
    case, ins, ok, ref = setup("causal_needle_D128")
    k = ins["k"].clone()
    k[:, :, 128:256] = ins["k"][:, :, 256:384]
    got, _ = cases.run_oracle(dict(ins, k=k), ok)
    must_fail(got, ref, "wrong K tile")


@pytest.mark.parametrize("name", ["gqa_needle_D128", "gqa_needle_D32"])
def test_wrong_gqa_head_map_fails(name):
    case, ins, ok, ref = setup(name)
    Hq, Hkv = case["Hq"], case["Hkv"]
    wrong = [h % Hkv for h in range(Hq)]                  # interleaved instead of consecutive groups (G15)
    got, _ = cases.run_oracle(dict(ins, k=ins["k"][:, wrong], v=ins["v"][:, wrong]), ok)
    must_fail(got, ref, f"{name} head map")


DIFF = ["diff_needle_D128", "diff_needle_D64", "diff_needle_D32", "diff_needle_lambda_h_causal_D64"]


@pytest.mark.parametrize("name", DIFF)
@pytest.mark.parametrize("mut", ["lambda_sign", "map1_dropped", "map_swap", "k1_is_k0", "q1_is_q0", "v_of_map1"])
def test_differential_mutants_fail(name, mut):
    case, ins, ok, ref = setup(name)
    H = case["Hq"]
    q, k, v = ins["q"], ins["k"], ins["v"]
    okm = dict(ok)
    if mut == "lambda_sign":
        if "lambda_h" in okm:
            okm["lambda_h"] = -okm["lambda_h"]
        else:
            okm["lam"] = -okm["lam"]
    elif mut == "map1_dropped":
        okm.pop("lambda_h", None)
        okm["lam"] = 0.0
    elif mut == "map_swap":
        sw = list(range(H, 2 * H)) + list(range(H))
        q, k = q[:, sw], k[:, sw]
    elif mut == "k1_is_k0":
        k = torch.cat([k[:, :H], k[:, :H]], 1)
    elif mut == "q1_is_q0":
        q = torch.cat([q[:, :H], q[:, :H]], 1)
    elif mut == "v_of_map1":                             # map 1 weights applied to a shifted V head
        vv = torch.roll(v, 1, dims=1)
        a0, _ = cases.run_oracle(dict(ins, q=q[:, :H], k=k[:, :H]), {x: y for x, y in ok.items()
                                                                     if x not in ("diff", "lam", "lambda_h")})
        a1, _ = cases.run_oracle(dict(ins, q=q[:, H:], k=k[:, H:], v=vv), {x: y for x, y in ok.items()
                                                                           if x not in ("diff", "lam", "lambda_h")})
        lam = np.repeat(ok["lambda_h"], ref.shape[0] // H // case.get("B", 1))[:, None] if "lambda_h" in ok \
            else ok["lam"]
        must_fail(a0 - lam * a1, ref, f"{name} {mut}")
        return
    got, _ = cases.run_oracle(dict(ins, q=q, k=k, v=v), okm)
    must_fail(got, ref, f"{name} {mut}")


@pytest.mark.parametrize("name,drop", [
    ("gate_const_D128", "gate"), ("gate_const_D32", "gate"), ("bias_f32_gate_mul_D64", "gate"),
    ("bias_needle_D128", "bias"), ("bias_needle_D32", "bias"), ("softcap_bias_D64", "bias"),
    ("softcap2_needle_D128", "softcap"), ("softcap2_needle_D32", "softcap"), ("alibi_needle_D64", "alibi"), ("keymask_needle_D128", "key_mask"),
    ("alibi_bias_causal_D32", "alibi"),
])
def test_dropped_mod_gate_bias_fails(name, drop):
    case, ins, ok, ref = setup(name)
    okm = dict(ok)
    if drop == "gate":
        okm.pop("gate_mode")
        okm.pop("gate")
    elif drop in ("softcap", "alibi"):
        okm.pop("mod")
    else:
        okm.pop(drop)
    got, _ = cases.run_oracle(ins, okm)
    must_fail(got, ref, f"{name} without {drop}", strong=False)


def test_alibi_sign_flip_fails():
    case, ins, ok, ref = setup("alibi_needle_D128")
    from paper_2511_02043_b200 import synth
    got, _ = cases.run_oracle(ins, dict(ok, alibi_slopes=-synth.alibi_slopes(case["Hq"]).astype(np.float64)))
    must_fail(got, ref, "alibi sign")


@pytest.mark.parametrize("name", ["bl_full_list_needle", "bl_D128"])
def test_rsa_list_shifted_by_one_block_fails(name):
    case, ins, ok, ref = setup(name)
    idx, cnt = ok["blk_idx"].copy(), ok["blk_cnt"].copy()
    # every listed block j -> j + 1, dropping blocks past the query block's diagonal
    nqb = idx.shape[1]
    for bh in range(idx.shape[0]):
        for i in range(nqb):
            lst = [j + 1 for j in idx[bh, i, :cnt[bh, i]] if j + 1 <= i]
            idx[bh, i, :] = -1
            idx[bh, i, :len(lst)] = lst
            cnt[bh, i] = len(lst)
    got, _ = cases.run_oracle(ins, dict(ok, blk_idx=idx, blk_cnt=cnt))
    must_fail(got, ref, f"{name} shifted list", strong=False)


@pytest.mark.parametrize("kind", ["row", "col"])
@pytest.mark.parametrize("drop", ["gate", "key_mask", "bias", "transpose_bias"])
def test_evoformer_mutants_fail(kind, drop):
    if kind == "col" and "bias" in drop:
        pytest.skip("column attention has no pair bias (G9)")
    case = dict(kind=kind, B=1, Ns=24, Nr=40, H=2, c=32, p_zero=0.1, dtype="bf16")
    ins, gk, ok = cases.evoformer(case)
    ref, _ = cases.run_oracle(ins, ok)
    okm = dict(ok)
    if drop == "gate":
        okm.pop("gate_mode")
        okm.pop("gate")
    elif drop == "transpose_bias":                          # pair bias [b,h,j,i] instead of [b,h,i,j]
        okm["bias"] = ok["bias"].transpose(-1, -2)
    else:
        okm.pop(drop)
    got, _ = cases.run_oracle(ins, okm)
    must_fail(got, ref, f"evoformer {kind} without {drop}", strong=False)


@pytest.mark.parametrize("name", ["diff_norm_needle_D128", "diff_norm_needle_D64", "diff_norm_causal_D32"])
@pytest.mark.parametrize("mut", ["no_norm", "no_lambda_init_scale", "no_weight", "reparam_sign"])
def test_diff_transformer_epilogue_mutants_fail(name, mut):
    case, ins, ok, ref = setup(name)
    okm = dict(ok)
    if mut == "no_norm":
        okm.pop("diff_norm")
    elif mut == "no_lambda_init_scale":                    # (1 - lambda_init) factor dropped
        if "lambda_qk" in okm:
            pytest.skip("lambda_init also enters lambda here")
        okm["lambda_init"] = 0.0
    elif mut == "no_weight":
        if "diff_norm_w" not in okm:
            pytest.skip("unit weight")
        okm.pop("diff_norm_w")
    elif mut == "reparam_sign":                            # exp(q2.k2) - exp(q1.k1) + lambda_init
        if "lambda_qk" not in okm:
            pytest.skip("no re-parameterisation")
        lq = okm["lambda_qk"]
        okm["lambda_qk"] = np.concatenate([lq[2:], lq[:2]])
    got, _ = cases.run_oracle(ins, okm)
    must_fail(got, ref, f"{name} {mut}", strong=False)
