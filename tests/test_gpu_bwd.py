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
    ]
BWD += [
    dict(name="vanilla_D32", Hq=2, S=300, D=32),
    dict(name="causal_needle_D32", Hq=2, S=520, D=32, mask="causal", dist="needle"),
    dict(name="gate_keymask_D32", Hq=2, S=200, D=32, key_mask=True, gate_mode="sigmoid", dist="needle"),
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
    gated = kw.get("gate_mode") == "sigmoid"
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


def test_backward_unsupported_is_loud(fl):
    q = torch.zeros(1, 2, 128, 64, device="cuda", dtype=torch.bfloat16)
    o, lse = fl.attn_fwd(q, q, q[:, :1].expand(1, 2, 128, 64).contiguous(), return_lse=True)
    g = torch.ones_like(o)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.attn_bwd(q, q, q, o, lse, o.clone(), gate_mode="mul", gate=g)
    bias = torch.zeros(1, 2, 128, 128, device="cuda", dtype=torch.bfloat16)
    ob, lb = fl.attn_fwd(q, q, q, return_lse=True, bias=bias)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.attn_bwd(q, q, q, ob, lb, ob.clone(), bias=bias)
