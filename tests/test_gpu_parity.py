"""GPU parity (-m gpu): the CUDA path through the C ABI against the fp64 oracle,
element by element on the same seeded inputs.  bf16 inputs: max-abs <= 2e-2;
fp32 path: <= 1e-5 (BASELINE.json north_star).  Uniform inputs give tiny
outputs at long S (SURVEY finding 3), so every family also runs needle and
constant-V inputs where max|ref| >= 0.1 (P12, P13)."""
import math

import numpy as np
import pytest
import torch

from tests import cases
from tests.parity import TOL, check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl as _fl
    return _fl


# ------------------------------------------------------------ descriptor bring-up
@pytest.mark.parametrize("n", [32, 64, 128])
@pytest.mark.parametrize("k", [32, 64, 128])
@pytest.mark.parametrize("b_mn,a_tmem", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_diag_umma_gemm(fl, n, k, b_mn, a_tmem):
    g = torch.Generator().manual_seed(n * 1000 + k)
    a = (torch.rand(128, k, generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(k, n, generator=g) * 2 - 1).to(torch.bfloat16) if b_mn else \
        (torch.rand(n, k, generator=g) * 2 - 1).to(torch.bfloat16)
    c = fl.diag_umma_gemm(a.cuda(), b.cuda(), n, k, bool(b_mn), bool(a_tmem)).cpu().double()
    ref = a.double() @ (b.double() if b_mn else b.double().t())
    assert torch.allclose(c, ref, atol=1e-3, rtol=1e-3), (c - ref).abs().max()


# ------------------------------------------------------------ fp32 SIMT path (1e-5)
F32_CASES = [
    dict(name="C1_causal", S=128, D=64, mask="causal"),                       # BASELINE config 1
    dict(name="vanilla_ragged", S=131, D=48, Dv=40),
    dict(name="sq_ne_sk", Sq=37, Sk=100, D=32, mask="causal"),
    dict(name="alibi", Hq=4, S=96, D=32, mod="alibi"),
    dict(name="alibi_custom", Hq=4, S=96, D=32, mod="alibi", alibi_custom=True),
    dict(name="softcap", S=96, D=32, mod="softcap", softcap=3.0),
    dict(name="sliding", S=200, D=32, mask="sliding", window=37),
    dict(name="prefix", S=150, D=32, mask="prefix", prefix=40),
    dict(name="document", B=2, S=300, D=32, mask="document", n_docs=5),
    dict(name="document_causal", B=2, S=300, D=32, mask="document", n_docs=5, doc_causal=True),
    dict(name="gqa", Hq=8, Hkv=2, S=70, D=32, mask="causal"),
    dict(name="diff", Hq=2, S=90, D=32, diff=True, lam=0.3),
    dict(name="diff_lambda_h", Hq=3, S=90, D=32, diff=True, lambda_h=True, mask="causal"),
    dict(name="diff_norm_reparam", Hq=2, S=90, D=64, diff=True, lambda_qk=True, lambda_init=0.8, diff_norm=True,
         diff_norm_w=True, mask="causal"),
    dict(name="diff_norm_lambda_h", Hq=3, S=77, D=48, diff=True, lambda_h=True, lambda_init=0.2, diff_norm=True),
    dict(name="gate_sigmoid", S=64, D=32, gate_mode="sigmoid"),
    dict(name="gate_mul", S=64, D=32, gate_mode="mul"),
    dict(name="bias", Hq=2, S=64, D=32, bias="f32"),
    dict(name="key_mask", S=100, D=32, key_mask=True, p_zero=0.3),
    dict(name="blocklist", Hq=2, Hkv=1, S=600, D=32, mask="blocklist", topk=1),
    dict(name="needle_causal", S=256, D=64, mask="causal", dist="needle"),
    dict(name="constant_sliding", S=256, D=64, mask="sliding", window=10, dist="constant"),
]


@pytest.mark.parametrize("case", F32_CASES, ids=[c["name"] for c in F32_CASES])
def test_f32_path(fl, case):
    ins, gk, ok = cases.build(dict(case, dtype="f32"))
    out = cases.run_gpu(fl, ins, gk)
    ref, _ = cases.run_oracle(ins, ok)
    check(out.cpu().double().reshape(ref.shape), ref, TOL["f32"], what=case["name"])


def test_f32_lse_and_empty_rows(fl):
    ins, gk, ok = cases.build(dict(S=50, D=16, dtype="f32", key_mask=True, p_zero=1.0))
    out, lse = cases.run_gpu(fl, ins, gk, return_lse=True)
    assert (out == 0).all() and torch.isneginf(lse).all()
    ins, gk, ok = cases.build(dict(S=50, D=16, dtype="f32", mask="causal"))
    out, lse = cases.run_gpu(fl, ins, gk, return_lse=True)
    ref, rl = cases.run_oracle(ins, ok)
    check(lse.cpu().double().reshape(-1), rl, 1e-5, what="lse")


# ------------------------------------------------------------ bf16 tcgen05 path (2e-2)
BF16_CASES = []
for D in (128, 64, 32):
    for S in (1, 17, 128, 129, 300):
        BF16_CASES.append(dict(name=f"vanilla_D{D}_S{S}", S=S, D=D))
    BF16_CASES += [
        dict(name=f"causal_D{D}", S=520, D=D, mask="causal", Hq=2),
        dict(name=f"causal_needle_D{D}", S=700, D=D, mask="causal", dist="needle"),
        dict(name=f"causal_const_D{D}", S=700, D=D, mask="causal", dist="constant"),
        dict(name=f"alibi_needle_D{D}", S=400, D=D, mod="alibi", Hq=4, dist="needle"),
        dict(name=f"softcap_needle_D{D}", S=400, D=D, mod="softcap", softcap=20.0, dist="needle"),
        # cap 2: the cap bends the needle score as well as the rest (cap 20 leaves needle rows unchanged)
        dict(name=f"softcap2_needle_D{D}", S=400, D=D, mod="softcap", softcap=2.0, dist="needle"),
        dict(name=f"sliding_needle_D{D}", S=900, D=D, mask="sliding", window=200, dist="needle"),
        dict(name=f"sliding_const_D{D}", S=900, D=D, mask="sliding", window=200, dist="constant"),
        dict(name=f"prefix_needle_D{D}", S=640, D=D, mask="prefix", prefix=200, dist="needle"),
        dict(name=f"document_const_D{D}", B=2, S=1000, D=D, mask="document", n_docs=6, dist="constant"),
        dict(name=f"document_D{D}", B=2, S=1000, D=D, mask="document", n_docs=6),
        dict(name=f"gqa_needle_D{D}", Hq=4, Hkv=2, S=300, D=D, mask="causal", dist="needle"),
        dict(name=f"diff_D{D}", Hq=2, S=400, D=D, diff=True, lam=0.2),
        dict(name=f"diff_causal_const_D{D}", Hq=2, S=400, D=D, diff=True, lambda_h=True, mask="causal",
             dist="constant"),
        dict(name=f"gate_const_D{D}", S=300, D=D, gate_mode="sigmoid", dist="constant"),
        dict(name=f"bias_needle_D{D}", Hq=2, S=260, D=D, bias="bf16", dist="needle"),
        dict(name=f"keymask_const_D{D}", S=300, D=D, key_mask=True, p_zero=0.2, dist="constant"),
        dict(name=f"sq_ne_sk_D{D}", Sq=200, Sk=333, D=D, mask="causal", dist="needle"),
        # score-mod combinations (raw-score domain for ALiBi + bias, log2 domain for softcap + bias, G16)
        dict(name=f"alibi_bias_causal_D{D}", Hq=2, S=300, D=D, mod="alibi", bias="bf16", mask="causal",
             dist="needle"),
        dict(name=f"softcap_bias_D{D}", Hq=2, S=260, D=D, mod="softcap", softcap=5.0, bias="bf16", dist="needle"),
        dict(name=f"alibi_custom_keymask_D{D}", Hq=4, S=300, D=D, mod="alibi", alibi_custom=True, key_mask=True,
             p_zero=0.2, dist="constant"),
        dict(name=f"bias_f32_gate_mul_D{D}", Hq=2, S=200, D=D, bias="f32", gate_mode="mul", dist="constant"),
        # differential attention with per-map needles (map 1's needle moves O by lambda x O(1), so a kernel
        # that drops, swaps or mis-indexes map 1 fails: tests/test_mutants.py)
        dict(name=f"diff_needle_D{D}", Hq=2, S=400, D=D, diff=True, lam=0.7, dist="needle"),
        dict(name=f"diff_needle_lambda_h_causal_D{D}", Hq=3, S=333, D=D, diff=True, lambda_h=True, mask="causal",
             dist="needle"),
        # "leak" inputs: each row's needle sits one key past its admissible interval
        dict(name=f"causal_leak_D{D}", S=700, D=D, mask="causal", dist="leak"),
        dict(name=f"sliding_leak_D{D}", S=900, D=D, mask="sliding", window=200, dist="leak"),
        dict(name=f"prefix_leak_D{D}", S=640, D=D, mask="prefix", prefix=200, dist="leak"),
        dict(name=f"document_leak_D{D}", S=1000, D=D, mask="document", n_docs=6, dist="leak"),
        dict(name=f"keymask_needle_D{D}", S=300, D=D, key_mask=True, p_zero=0.2, dist="needle"),
        # DIFF-Transformer epilogue (NEXT-2, G8b): lambda re-parameterised, per-head RMSNorm x (1 - lambda_init)
        dict(name=f"diff_norm_needle_D{D}", Hq=2, S=400, D=D, diff=True, lambda_qk=True, lambda_init=0.5,
             diff_norm=True, diff_norm_w=True, dist="needle"),
        dict(name=f"diff_norm_causal_D{D}", Hq=2, S=333, D=D, diff=True, lam=0.6, lambda_init=0.3,
             diff_norm=True, mask="causal"),
        dict(name=f"document_needle_B2_D{D}", B=2, S=1000, D=D, mask="document", n_docs=6, dist="needle"),
    ]


# short query blocks (S_q <= 16) take the split-KV decode kernels (decode.cu)
for D in (128, 64):
    BF16_CASES += [
        dict(name=f"dec_causal_needle_D{D}", Hq=2, Sq=1, Sk=3000, D=D, mask="causal", dist="needle"),
        dict(name=f"dec_causal_const_D{D}", B=2, Hq=2, Sq=7, Sk=5000, D=D, mask="causal", dist="constant"),
        dict(name=f"dec_vanilla_D{D}", Hq=3, Sq=16, Sk=777, D=D),
        dict(name=f"dec_sliding_needle_D{D}", Hq=1, Sq=3, Sk=4000, D=D, mask="sliding", window=300, dist="needle"),
        dict(name=f"dec_alibi_needle_D{D}", Hq=4, Sq=2, Sk=1000, D=D, mod="alibi", dist="needle"),
        dict(name=f"dec_softcap_needle_D{D}", Hq=2, Sq=1, Sk=1500, D=D, mod="softcap", softcap=20.0, dist="needle"),
        dict(name=f"dec_gqa_needle_D{D}", Hq=8, Hkv=2, Sq=4, Sk=2000, D=D, mask="causal", dist="needle"),
        dict(name=f"dec_keymask_const_D{D}", Hq=2, Sq=5, Sk=900, D=D, key_mask=True, p_zero=0.5, dist="constant"),
        dict(name=f"dec_doc_const_D{D}", B=2, Hq=1, Sq=9, Sk=3000, D=D, mask="document", n_docs=5, dist="constant"),
        dict(name=f"dec_topleft_needle_D{D}", Hq=1, Sq=12, Sk=600, D=D, mask="causal", causal_align=1, dist="needle"),
    ]


@pytest.mark.parametrize("case", BF16_CASES, ids=[c["name"] for c in BF16_CASES])
def test_bf16_path(fl, case):
    ins, gk, ok = cases.build(dict(case, dtype="bf16"))
    out = cases.run_gpu(fl, ins, gk)
    ref, _ = cases.run_oracle(ins, ok)
    strong = case.get("dist") in ("needle", "constant")
    check(out.cpu().double().reshape(ref.shape), ref, TOL["bf16"], min_ref=0.1 if strong else 0.0,
          what=case["name"])


def test_decode_lse_and_empty_rows(fl):
    """split-KV path: LSE across splits (combine) and fully-masked rows (G7: O = 0, lse = -inf)."""
    ins, gk, ok = cases.build(dict(Sq=4, Sk=3000, D=128, mask="causal", dist="needle"))
    out, lse = cases.run_gpu(fl, ins, gk, return_lse=True)
    ref, rl = cases.run_oracle(ins, ok)
    check(lse.cpu().double().reshape(-1), rl, 1e-2, what="decode lse")
    ins, gk, ok = cases.build(dict(Sq=3, Sk=700, D=64, key_mask=True, p_zero=1.0))
    out, lse = cases.run_gpu(fl, ins, gk, return_lse=True)
    assert (out == 0).all() and torch.isneginf(lse).all()


def test_bf16_lse(fl):
    ins, gk, ok = cases.build(dict(S=333, D=128, mask="causal", dist="needle"))
    out, lse = cases.run_gpu(fl, ins, gk, return_lse=True)
    _, rl = cases.run_oracle(ins, ok)
    check(lse.cpu().double().reshape(-1), rl, 1e-2, what="bf16 lse")


@pytest.mark.parametrize("kind", ["row", "col"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("dist", ["uniform", "needle"])
def test_evoformer(fl, kind, dtype, dist):
    """Needle Q/K (peaked rows, max|ref| >= 0.1 asserted) so that a wrong key, head, MSA row or bias
    placement moves the output; the uniform case keeps the bench's value distribution."""
    case = dict(kind=kind, B=1, Ns=24, Nr=40, H=2, c=32, p_zero=0.1, dtype=dtype, dist=dist)
    ins, gk, ok = cases.evoformer(case)
    out = cases.run_gpu(fl, ins, gk)
    ref, _ = cases.run_oracle(ins, ok)
    check(out.cpu().double().reshape(ref.shape), ref, TOL[dtype], min_ref=0.1 if dist == "needle" else 0.0,
          what=f"evoformer {kind} {dtype} {dist}")


@pytest.mark.parametrize("B,Ns,Nr", [(1, 25, 300), (1, 7, 130), (1, 3, 384), (1, 2, 200), (1, 9, 640), (2, 6, 257),
                                     (2, 3, 100)])
def test_evoformer_row_pairs(fl, B, Ns, Nr):
    """Row attention at S_q % 256 <= 128 runs the paired-G kernel (two MSA rows per unit): odd G (last
    pair half empty), several query tiles, ragged tails; S_q % 256 > 128 keeps the 256-row units.  Up to
    N_res = 384 the pair bias is resident in TMEM (static segment schedule, bias refilled per (b, h,
    q-block)); N_res = 640 keeps the TMA'd bias tiles."""
    case = dict(kind="row", B=B, Ns=Ns, Nr=Nr, H=2, c=32, p_zero=0.1, dtype="bf16", seed=Ns, dist="needle")
    ins, gk, ok = cases.evoformer(case)
    out = cases.run_gpu(fl, ins, gk)
    ref, _ = cases.run_oracle(ins, ok)
    check(out.cpu().double().reshape(ref.shape), ref, TOL["bf16"], min_ref=0.1, what=f"evoformer row pairs Ns{Ns} Nr{Nr}")


def test_determinism(fl):
    ins, gk, _ = cases.build(dict(S=700, D=128, mask="causal", Hq=2))
    a = cases.run_gpu(fl, ins, gk)
    b = cases.run_gpu(fl, ins, gk)
    assert torch.equal(a, b)


def test_host_entry_matches_device_entry(fl):
    ins, gk, _ = cases.build(dict(S=384, D=128, mask="causal", Hq=2))
    dev = cases.run_gpu(fl, ins, gk)
    runner = fl.HostRunner()
    out = torch.empty(dev.shape, dtype=dev.dtype).pin_memory()
    runner(ins["q"].pin_memory(), ins["k"].pin_memory(), ins["v"].pin_memory(), out, **gk)
    torch.cuda.synchronize()
    assert torch.equal(out, dev.cpu())


@pytest.mark.parametrize("case", [dict(B=4, S=300, D=128, mask="document", n_docs=3, Hq=2),
                                  dict(B=3, S=200, D=64, mask="causal", mod="alibi")])
def test_host_entry_pipelined_matches_device_entry(fl, case):
    """B >= 2: fl_attn_fwd_host pipelines batch chunks (H2D / kernel / D2H on three streams); the result
    (O and LSE) must equal the device entry's bit for bit."""
    ins, gk, _ = cases.build(case)
    dev, dlse = cases.run_gpu(fl, ins, gk, return_lse=True)
    runner = fl.HostRunner()
    out = torch.empty(dev.shape, dtype=dev.dtype).pin_memory()
    lse = torch.empty(dlse.shape, dtype=torch.float32).pin_memory()
    hk = {k: (v.pin_memory() if torch.is_tensor(v) else v) for k, v in gk.items()}
    runner(ins["q"].pin_memory(), ins["k"].pin_memory(), ins["v"].pin_memory(), out, lse, **hk)
    torch.cuda.synchronize()
    assert torch.equal(out, dev.cpu())
    assert torch.equal(lse, dlse.cpu())


def test_errors_are_loud(fl):
    q = torch.zeros(1, 1, 8, 48, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.attn_fwd(q, q, q)
    q = torch.zeros(1, 1, 8, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(fl.FlError):
        fl.attn_fwd(q, q, q, out=q)          # o aliases inputs
    with pytest.raises(fl.FlError, match="INVALID"):
        fl.attn_fwd(q.cpu(), q.cpu(), q.cpu(), out=torch.empty(1, 1, 8, 64, dtype=torch.bfloat16))
