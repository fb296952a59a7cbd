"""Paged KV (-m gpu, the serving side of RSA, reading G10): K/V held in a pool of
128-key pages in shuffled order behind a page table.  The page-table indirection lives in the TMA
producers of the tcgen05 kernel (interval masks and RSA block lists) and of the split-KV decode kernel.
Checks: parity with the fp64 oracle on the CONTIGUOUS K/V (needle inputs, max|ref| >= 0.1), and bit
equality with the same call on contiguous K/V (identical arithmetic, only the addressing differs)."""
import numpy as np
import pytest
import torch

import oracle
from tests import cases
from tests.parity import TOL, check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl as _fl
    return _fl


PAGED = [
    dict(name="prefill_causal_D128", B=2, Hq=2, S=1000, D=128, mask="causal", dist="needle"),
    dict(name="prefill_sliding_D64", B=2, Hq=2, S=1100, D=64, mask="sliding", window=300, dist="needle"),
    dict(name="prefill_gqa_D128", B=1, Hq=4, Hkv=2, S=777, D=128, mask="causal", dist="needle"),
    dict(name="chunk_sq_lt_sk_D128", B=2, Hq=2, Sq=64, Sk=2000, D=128, mask="causal", dist="needle"),
    dict(name="blocklist_D128", B=1, Hq=2, S=1300, D=128, mask="blocklist", topk=3, v="blockconst"),
    dict(name="decode_D128", B=2, Hq=2, Sq=1, Sk=3000, D=128, mask="causal", dist="needle"),
    dict(name="decode_gqa_D64", B=2, Hq=4, Hkv=2, Sq=4, Sk=2500, D=64, mask="causal", dist="needle"),
    dict(name="decode_blocklist_D128", B=2, Hq=2, Sq=1, Sk=4000, D=128, mask="blocklist", topk=4,
         v="blockconst"),
    dict(name="vanilla_ragged_D32", B=2, Hq=1, S=300, D=32),
]


@pytest.mark.parametrize("case", PAGED, ids=[c["name"] for c in PAGED])
def test_paged_kv_matches_oracle_and_contiguous(fl, case):
    ins, gk, ok = cases.build(dict(case, dtype="bf16"))
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    Sk = k.shape[2]
    ref_dev = fl.attn_fwd(q, k, v, **kw)
    npb = (Sk + 127) // 128
    kp, vp, table = fl.paged_kv(k, v, n_pages_total=k.shape[0] * npb + 5, seed=hash(case["name"]) % 1000)
    out = fl.attn_fwd(q, kp, vp, kv_page_table=table.cuda(), kv_len=Sk, **kw)
    torch.cuda.synchronize()
    assert torch.equal(out, ref_dev), "paged and contiguous K/V give different bits"
    ref, _ = cases.run_oracle(ins, ok)
    strong = case.get("dist") == "needle" or case.get("v") == "blockconst"
    check(out.cpu().double().reshape(ref.shape), ref, TOL["bf16"], min_ref=0.1 if strong else 0.0,
          what=case["name"])


def test_paged_kv_validation(fl):
    q = torch.zeros(1, 1, 64, 128, device="cuda", dtype=torch.bfloat16)
    kp = torch.zeros(4, 1, 128, 128, device="cuda", dtype=torch.bfloat16)
    table = torch.zeros(1, 2, dtype=torch.int32, device="cuda")
    with pytest.raises(fl.FlError, match="INVALID"):
        fl.attn_fwd(q, kp, kp, kv_page_table=table, kv_len=300)          # kv_len > 128 * pages
    with pytest.raises(fl.FlError, match="SHAPE"):
        fl.attn_fwd(q, kp[:, :, :64], kp[:, :, :64], kv_page_table=table, kv_len=100)   # 64-key pages
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.attn_fwd(q.float(), kp.float(), kp.float(), kv_page_table=table, kv_len=100)  # fp32 path
