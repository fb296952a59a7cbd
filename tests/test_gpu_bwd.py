"""Backward parity (-m gpu): fl_attn_bwd's dQ, dK, dV against the fp64 oracle's plain
chain rule (oracle.attn_bwd, itself pinned to central differences and torch.autograd of Listing 1).
The forward's O and LSE come from fl_attn_fwd on the same inputs (as in training).  Tolerance: max-abs
2e-2 per gradient with |Q|, |K|, |V|, |dO| <= 1 (the north_star's bf16 bar, applied to each gradient),
and max|ref| >= 0.05 so the comparison is not vacuous."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_02043_b200 import synth
from tests import cases
from tests.parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl as _fl
    return _fl


BWD = []
for D in (128, 64):
    BWD += [
        dict(name=f"vanilla_D{D}", Hq=2, S=300, D=D),
        dict(name=f"causal_needle_D{D}", Hq=2, S=520, D=D, mask="causal", dist="needle"),
        dict(name=f"sliding_D{D}", S=700, D=D, mask="sliding", window=150, dist="needle"),
        dict(name=f"prefix_D{D}", S=400, D=D, mask="prefix", prefix=100),
        dict(name=f"document_D{D}", B=2, S=600, D=D, mask="document", n_docs=5),
        dict(name=f"alibi_D{D}", Hq=4, S=260, D=D, mod="alibi", dist="needle"),
        dict(name=f"softcap_D{D}", S=300, D=D, mod="softcap", softcap=2.0, dist="needle"),
        dict(name=f"gqa_causal_D{D}", Hq=4, Hkv=2, S=333, D=D, mask="causal", dist="needle"),
        dict(name=f"sq_lt_sk_D{D}", Sq=100, Sk=450, D=D, mask="causal"),
        dict(name=f"keymask_D{D}", Hq=2, S=300, D=D, key_mask=True, dist="needle"),
        dict(name=f"gate_sigmoid_D{D}", Hq=2, S=260, D=D, mask="causal", gate_mode="sigmoid", dist="needle"),
        dict(name=f"gate_mul_D{D}", Hq=2, S=260, D=D, mask="causal", gate_mode="mul", gate_unit=True, dist="needle"),
    ]
BWD += [
    dict(name="vanilla_D32", Hq=2, S=300, D=32),
    dict(name="causal_needle_D32", Hq=2, S=520, D=32, mask="causal", dist="needle"),
    dict(name="gate_keymask_D32", Hq=2, S=200, D=32, key_mask=True, gate_mode="sigmoid", dist="needle"),
    dict(name="gate_mul_keymask_D32", Hq=2, S=200, D=32, key_mask=True, gate_mode="mul", gate_unit=True, dist="needle"),
]


@pytest.mark.parametrize("case", BWD, ids=[c["name"] for c in BWD])
def test_backward_vs_oracle(fl, case):
    ins, gk, ok = cases.build(dict(case, dtype="bf16"))
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    out, lse = fl.attn_fwd(q, k, v, return_lse=True, **kw)
    dout = synth.uniform(tuple(out.shape), seed=17, tensor="gate")
    _compare(fl, case["name"], (ins["q"], ins["k"], ins["v"]), (q, k, v), out, lse, dout, kw, ok)


def _compare(fl, name0, host_qkv, dev_qkv, out, lse, dout, kw, ok):
    gated = kw.get("gate_mode") in ("sigmoid", "mul")
    grads = fl.attn_bwd(*dev_qkv, out, lse, dout.cuda(), **kw)
    torch.cuda.synchronize()
    refs = oracle.attn_bwd(*host_qkv, dout, with_dgate=gated, **ok)
    names = ("dq", "dk", "dv", "dgate") if gated else ("dq", "dk", "dv")
    for name, got, ref in zip(names, grads, refs):
        case = {"name": name0}
        r = check(got.cpu().double().numpy(), ref, 2e-2, min_ref=0.05 if name == "dv" else 0.0,
                  what=f"{case['name']} {name}")
        # where a gradient's scale is >= 0.05 it must also hold 5 % of that scale (G22); on peaked rows dQ
        # cancels (dS = P (dP - Dvec) with Dvec from the bf16 O) and only the absolute bar applies
        if r["max_ref"] >= 0.05:
            assert r["max_abs"] <= 0.05 * r["max_ref"], f"{case['name']} {name}: {r}"


@pytest.mark.parametrize("Nr", [130, 300])
def test_backward_evoformer_column(fl, Nr):
    """Rank-5 strided views, D = 32, sigmoid gate (+ dgate) and MSA key mask: the Evoformer column
    attention (AF2 Alg.8, reading G9), all of whose steps the backward now covers."""
    ins, gk, ok = cases.evoformer(dict(kind="col", B=1, Ns=Nr, Nr=5, H=2, c=32, p_zero=0.1))
    q, k, v = (ins[n].cuda().contiguous() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    kw["gate"] = kw["gate"].contiguous()
    ok = dict(ok, gate=ok["gate"].contiguous())
    out, lse = fl.attn_fwd(q, k, v, return_lse=True, **kw)
    dout = synth.uniform(tuple(out.shape), seed=18, tensor="gate", lead=3)
    _compare(fl, f"evo_col_Nr{Nr}", tuple(ins[n].contiguous() for n in ("q", "k", "v")), (q, k, v), out, lse, dout,
             kw, ok)


@pytest.mark.parametrize("bias_dtype,D", [("bf16", 64), ("f32", 128)])
def test_backward_bias(fl, bias_dtype, D):
    """Additive score bias (G16) with dL/dbias (f32 atomics) against the oracle's dbias."""
    case = dict(Hq=2, S=260, D=D, bias=bias_dtype, mask="causal", dist="needle")
    ins, gk, ok = cases.build(dict(case, dtype="bf16"))
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    out, lse = fl.attn_fwd(q, k, v, return_lse=True, **kw)
    dout = synth.uniform(tuple(out.shape), seed=19, tensor="gate")
    dbias = torch.empty(kw["bias"].shape, dtype=torch.float32, device="cuda")
    dq, dk, dv = fl.attn_bwd(q, k, v, out, lse, dout.cuda(), dbias=dbias, **kw)
    torch.cuda.synchronize()
    rq, rk, rv, rb = oracle.attn_bwd(ins["q"], ins["k"], ins["v"], dout, with_dbias=True, **ok)
    for name, got, ref in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv), ("dbias", dbias, rb.reshape(dbias.shape))):
        r = check(got.cpu().double().numpy(), ref, 2e-2, what=f"bias {bias_dtype} D{D} {name}")
        if r["max_ref"] >= 0.05:
            assert r["max_abs"] <= 0.05 * r["max_ref"], f"bias {name}: {r}"


@pytest.mark.parametrize("Nr", [100, 300])
def test_backward_evoformer_row(fl, Nr):
    """The Evoformer row attention (AF2 Alg.7, reading G9): rank-5 views, D = 32, the pair bias broadcast
    over the MSA rows s (dbias = sum over s of dS, accumulated by the atomics), sigmoid gate (+ dgate),
    MSA key mask."""
    Ns = 6
    ins, gk, ok = cases.evoformer(dict(kind="row", B=1, Ns=Ns, Nr=Nr, H=2, c=32, p_zero=0.1))
    q, k, v = (ins[n].cuda().contiguous() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    kw["gate"] = kw["gate"].contiguous()
    ok = dict(ok, gate=ok["gate"].contiguous())
    out, lse = fl.attn_fwd(q, k, v, return_lse=True, **kw)
    dout = synth.uniform(tuple(out.shape), seed=20, tensor="gate", lead=3)
    dbias = torch.empty(1, 1, 2, Nr, Nr, dtype=torch.float32, device="cuda").expand(kw["bias"].shape)
    dq, dk, dv, dg = fl.attn_bwd(q, k, v, out, lse, dout.cuda(), dbias=dbias, **kw)
    torch.cuda.synchronize()
    host = tuple(ins[n].contiguous() for n in ("q", "k", "v"))
    rq, rk, rv, rg, rb = oracle.attn_bwd(*host, dout, with_dgate=True, with_dbias=True, **ok)
    rb = rb.sum(axis=1, keepdims=True)                 # the pair bias broadcasts over s
    for name, got, ref in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv), ("dgate", dg, rg),
                           ("dbias", dbias[:, :1], rb)):
        r = check(got.cpu().double().numpy(), ref, 2e-2 * (Ns if name == "dbias" else 1), what=f"evo row {name}")
        if r["max_ref"] >= 0.05:
            assert r["max_abs"] <= 0.05 * r["max_ref"], f"evo row {name}: {r}"


def test_backward_unsupported_is_loud(fl):
    q = torch.zeros(1, 2, 128, 64, device="cuda", dtype=torch.bfloat16)
    o, lse = fl.attn_fwd(q, q, q[:, :1].expand(1, 2, 128, 64).contiguous(), return_lse=True)
    q2 = torch.zeros(1, 4, 128, 64, device="cuda", dtype=torch.bfloat16)
    od, ld = fl.attn_fwd(q2, q2, q, diff=True, lam=0.3), None
    with pytest.raises(fl.FlError):
        fl.attn_bwd(q2, q2, q, od, torch.zeros(1, 2, 128, device="cuda"), od.clone(), diff=True, lam=0.3)


DIFF_BWD = [
    dict(name="diff_needle_D64", Hq=2, S=300, D=64, diff=True, lam=0.7, dist="needle"),
    dict(name="diff_lambda_h_causal_gqa_D128", Hq=4, Hkv=2, S=333, D=128, diff=True, lambda_h=True, mask="causal",
         dist="needle"),
    dict(name="diff_gate_causal_D32", Hq=2, S=260, D=32, diff=True, lam=0.5, gate_mode="sigmoid", mask="causal",
         dist="needle"),
    dict(name="diff_reparam_sliding_D64", Hq=2, S=200, D=64, diff=True, lambda_qk=True, lambda_init=0.8,
         mask="sliding", window=64, dist="needle"),
]
_DIFF_KEYS = ("diff", "lam", "lambda_h", "lambda_qk", "lambda_init")


@pytest.mark.parametrize("case", DIFF_BWD, ids=[c["name"] for c in DIFF_BWD])
def test_backward_diff(fl, case):
    """Differential attention (Listing 4, G8): dQ, dK (both maps), dV (summed over the maps),
    dgate and dL/dlambda_h against the oracle's chain rule (pinned to central differences).  dlambda_h is a
    sum of B S D terms dO * o_1: its bar is 8 x 2^-8 x sqrt(sum (dO o_1)^2) (bf16 rounding of o_1, independent
    per element, 8 sigma), o_1 = the oracle's map-1 output."""
    ins, gk, ok = cases.build(dict(case, dtype="bf16"))
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    out = fl.attn_fwd(q, k, v, **kw)
    dout = synth.uniform(tuple(out.shape), seed=21, tensor="gate")
    Hq = out.shape[-3]
    dl = torch.empty(Hq, dtype=torch.float32, device="cuda")
    gated = kw.get("gate_mode") == "sigmoid"
    grads = fl.attn_bwd(q, k, v, out, None, dout.cuda(), dlambda=dl, **kw)
    torch.cuda.synchronize()
    refs = oracle.attn_bwd(ins["q"], ins["k"], ins["v"], dout, with_dgate=gated, with_dlambda=True, **ok)
    names = ("dq", "dk", "dv", "dgate") if gated else ("dq", "dk", "dv")
    # map 0 alone (lambda = 0): the value dV / dgate hold, rounded to bf16, before map 1 adds to them
    ok0 = dict({x: y for x, y in ok.items() if x not in _DIFF_KEYS}, diff=True, lam=0.0)
    refs0 = oracle.attn_bwd(ins["q"], ins["k"], ins["v"], dout, with_dgate=gated, **ok0)
    for i, (name, got, ref) in enumerate(zip(names, grads, refs)):
        g64 = got.cpu().double().numpy()
        if name in ("dv", "dgate"):
            # summed over the maps: the map-0 value is stored in bf16, map 1 adds in fp32 and the sum is
            # rounded again -- up to 2^-9 (|map-0 value| + |sum|) on top of the 2e-2 bar (|dV| reaches ~8 with
            # GQA over needle rows, where one bf16 ulp is 2^-5)
            ref = ref.reshape(g64.shape)
            err = np.abs(g64 - ref)
            bound = 2e-2 + 2.0 ** -9 * (np.abs(refs0[i].reshape(g64.shape)) + np.abs(ref))
            assert np.all(err <= bound), f"{case['name']} {name}: worst excess {(err - bound).max():.3e}"
            assert np.abs(ref).max() >= 0.05 and err.max() <= 0.05 * np.abs(ref).max()
            continue
        r = check(g64, ref, 2e-2, what=f"{case['name']} {name}")
        if r["max_ref"] >= 0.05:
            assert r["max_abs"] <= 0.05 * r["max_ref"], f"{case['name']} {name}: {r}"
    # dlambda: the map-1 output from the oracle (gate included), per head
    ok1 = {x: y for x, y in ok.items() if x not in _DIFF_KEYS}
    Hkv = ins["k"].shape[1] // 2
    o1, _ = oracle.attn(ins["q"][:, Hq:], ins["k"][:, Hkv:], ins["v"], **ok1)
    terms = dout.double().numpy() * o1.reshape(dout.shape)
    ref_dl = refs[-1]
    assert np.allclose(ref_dl, -terms.sum(axis=(0, 2, 3)), rtol=1e-9, atol=1e-9)     # the oracle agrees with itself
    bar = 8 * 2.0 ** -8 * np.sqrt((terms ** 2).sum(axis=(0, 2, 3))) + 1e-3
    err = np.abs(dl.cpu().double().numpy() - ref_dl)
    assert np.all(err <= bar), (case["name"], err, bar, ref_dl)
    assert np.abs(ref_dl).max() > 4 * bar.max(), "dlambda check not discriminating"


def test_backward_diff_unsupported_is_loud(fl):
    q = torch.zeros(1, 4, 128, 64, device="cuda", dtype=torch.bfloat16)
    v = torch.zeros(1, 2, 128, 64, device="cuda", dtype=torch.bfloat16)
    o = fl.attn_fwd(q, q, v, diff=True, lam=0.3)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.attn_bwd(q, q, v, o, None, o.clone(), diff=True, lam=0.3, diff_norm=True, diff_norm_eps=1e-5)
    with pytest.raises(fl.FlError):
        fl.attn_bwd(q, q, v, o, torch.zeros(1, 2, 128, device="cuda"), o.clone(), diff=True, lam=0.3)


def test_backward_degenerate_shapes(fl):
    """Edge cases of the definition: no queries -> dK = dV = 0; no keys -> O = 0 (G7), so dQ = 0 and dgate = 0.
    The gradient buffers start as NaN so an unwritten gradient fails."""
    bf = torch.bfloat16
    nan = lambda *s: torch.full(s, float("nan"), device="cuda", dtype=bf)
    # S_q = 0
    q = torch.zeros(1, 2, 0, 64, device="cuda", dtype=bf)
    k = torch.rand(1, 2, 50, 64, device="cuda", dtype=bf)
    o, lse = fl.attn_fwd(q, k, k, return_lse=True)
    dq, dk, dv = fl.attn_bwd(q, k, k, o, lse, o.clone(), dq=torch.empty_like(q), dk=nan(1, 2, 50, 64), dv=nan(1, 2, 50, 64))
    torch.cuda.synchronize()
    assert dk.abs().max().item() == 0 and dv.abs().max().item() == 0
    # S_k = 0, sigmoid gate
    q = torch.rand(1, 2, 40, 64, device="cuda", dtype=bf)
    k = torch.zeros(1, 2, 0, 64, device="cuda", dtype=bf)
    g = torch.rand(1, 2, 40, 64, device="cuda", dtype=bf)
    o, lse = fl.attn_fwd(q, k, k, return_lse=True, gate_mode="sigmoid", gate=g)
    assert o.abs().max().item() == 0
    dq, dk, dv, dg = fl.attn_bwd(q, k, k, o, lse, torch.rand_like(o), dq=nan(1, 2, 40, 64), dgate=nan(1, 2, 40, 64),
                                 gate_mode="sigmoid", gate=g)
    torch.cuda.synchronize()
    assert dq.abs().max().item() == 0 and dg.abs().max().item() == 0
    # differential attention, S_q = 0: both maps' dK slices and the shared dV are zeroed
    q = torch.zeros(1, 4, 0, 64, device="cuda", dtype=bf)
    k = torch.rand(1, 4, 30, 64, device="cuda", dtype=bf)
    v = torch.rand(1, 2, 30, 64, device="cuda", dtype=bf)
    o = fl.attn_fwd(q, k, v, diff=True, lam=0.3)
    dq, dk, dv = fl.attn_bwd(q, k, v, o, None, o.clone(), dq=torch.empty_like(q), dk=nan(1, 4, 30, 64),
                             dv=nan(1, 2, 30, 64), diff=True, lam=0.3)
    torch.cuda.synchronize()
    assert dk.abs().max().item() == 0 and dv.abs().max().item() == 0
