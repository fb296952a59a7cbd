"""T7 (-m gpu) without compute-sanitizer (closed on this GPU pool: runs under it left
GPUs needing a reset).  Guard bands of our own instead, over one small call of every kernel family --
tcgen05 attention (interval mask, block list, Evoformer small head with key mask / bias / gate, both
Evoformer layouts, differential attention), split-KV decode, fp32 SIMT, paged KV, RSA summaries /
selection:

* every floating-point input lives in the middle of a larger buffer whose margins hold NaN, so a read
  past either end of a tensor (a wrong stride, an unclamped ragged tail, a bad bias / gate / key-mask
  offset) turns into a NaN or a changed output;
* every output (O, LSE, summaries, lists) lives in the middle of a buffer whose margins hold a canary
  pattern, so a write past either end is seen;
* the guarded call's output must equal, bit for bit, the same call on plain tensors (the kernels are
  deterministic: tests/test_gpu_parity.py::test_determinism)."""
import pytest
import torch

from tests import cases

pytestmark = pytest.mark.gpu
PAD = 4096          # elements of margin on each side


def _guarded_like(t, fill):
    """A tensor equal to t (same shape and strides) inside a buffer with `fill` margins.  Returns
    (view, buffer, (lo, hi)) where buffer[:lo] and buffer[hi:] are the margins."""
    t = t.cuda()
    span = max(1, 1 + sum((s - 1) * st for s, st in zip(t.shape, t.stride()) if s > 0))
    buf = torch.full((span + 2 * PAD,), fill, dtype=t.dtype, device="cuda")
    view = buf.as_strided(t.shape, t.stride(), PAD)
    view.copy_(t)
    return view, buf, (PAD, PAD + span)


def _nan_guard(t):
    if torch.is_tensor(t) and t.is_floating_point():
        return _guarded_like(t, float("nan"))[0]
    return t.cuda() if torch.is_tensor(t) else t


def _canary_out(shape, dtype):
    z = torch.zeros(shape, dtype=dtype)
    return _guarded_like(z, 1234.5 if dtype != torch.int32 else 0x5A5A5A5A)


def _check_margins(buf, lo, hi, fill):
    m = torch.cat([buf[:lo], buf[hi:]])
    assert bool((m == fill).all()), "write outside the output tensor"


ATTN_CASES = [
    dict(S=300, D=128, mask="causal"),
    dict(S=333, D=64, mask="sliding", window=40),
    dict(S=260, D=128, mod="softcap", softcap=2.0, mask="document", n_docs=3, B=2),
    dict(S=300, D=64, Hq=2, diff=True, lam=0.3),
    dict(S=200, D=32, bias="bf16", key_mask=True, gate_mode="sigmoid"),
    dict(S=700, D=128, mask="blocklist", topk=2),
    dict(Sq=1, Sk=2000, D=128, mask="causal"),
    dict(Sq=5, Sk=900, D=64, Hq=4, Hkv=2, mask="causal"),
    dict(S=100, D=64, mask="sliding", window=20, dtype="f32"),
]


@pytest.mark.parametrize("case", ATTN_CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_guard_attn(case):
    from paper_2511_02043_b200 import fl
    ins, gk, _ = cases.build(case)
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    with_lse = not case.get("diff")                    # differential attention has no single LSE
    ref, ref_lse = fl.attn_fwd(q, k, v, return_lse=True, **kw) if with_lse else (fl.attn_fwd(q, k, v, **kw), None)
    gq, gk_, gv = (_nan_guard(t) for t in (q, k, v))
    gkw = {x: _nan_guard(y) for x, y in kw.items()}
    out, obuf, (olo, ohi) = _canary_out(ref.shape, ref.dtype)
    if with_lse:
        lse, lbuf, (llo, lhi) = _canary_out(ref_lse.shape, torch.float32)
        fl.attn_fwd(gq, gk_, gv, out=out, lse=lse, return_lse=True, **gkw)
    else:
        fl.attn_fwd(gq, gk_, gv, out=out, **gkw)
    torch.cuda.synchronize()
    _check_margins(obuf, olo, ohi, 1234.5)
    assert torch.equal(out.view(torch.int16) if out.dtype == torch.bfloat16 else out,
                       ref.view(torch.int16) if ref.dtype == torch.bfloat16 else ref)
    if with_lse:
        _check_margins(lbuf, llo, lhi, 1234.5)
        assert torch.equal(lse, ref_lse)


@pytest.mark.parametrize("kind,Nr", [("row", 130), ("row", 384), ("col", 130)])
def test_guard_evoformer(kind, Nr):
    from paper_2511_02043_b200 import fl
    ins, gk, _ = cases.evoformer(dict(kind=kind, B=1, Ns=5, Nr=Nr, H=2, c=32, p_zero=0.1))
    Q, K, V = (t.cuda() for t in ins["storage"])
    view = (lambda t: t.permute(0, 1, 3, 2, 4)) if kind == "row" else (lambda t: t.permute(0, 2, 3, 1, 4))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    ref = fl.attn_fwd(view(Q), view(K), view(V), **kw)
    gQ, gK, gV = (_nan_guard(t) for t in (Q, K, V))
    gkw = dict(kw)
    unview = (lambda t: t.permute(0, 1, 3, 2, 4)) if kind == "row" else (lambda t: t.permute(0, 3, 1, 2, 4))
    gkw["gate"] = view(_nan_guard(unview(gk["gate"]).contiguous()))
    if "bias" in kw:
        pb = _nan_guard(kw["bias"][:, 0].contiguous())
        gkw["bias"] = pb.unsqueeze(1).expand(kw["bias"].shape)
    out, obuf, (olo, ohi) = _canary_out(ref.shape, ref.dtype)
    fl.attn_fwd(view(gQ), view(gK), view(gV), out=out, **gkw)
    torch.cuda.synchronize()
    _check_margins(obuf, olo, ohi, 1234.5)
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def test_guard_paged():
    from paper_2511_02043_b200 import fl
    torch.manual_seed(0)
    q = torch.randn(1, 2, 1000, 128, device="cuda").to(torch.bfloat16)
    k = torch.randn(1, 2, 1000, 128, device="cuda").to(torch.bfloat16)
    kp, vp, t = fl.paged_kv(k, k, seed=1)
    ref = fl.attn_fwd(q, kp, vp, kv_page_table=t.cuda(), kv_len=1000, mask="causal")
    out, obuf, (olo, ohi) = _canary_out(ref.shape, ref.dtype)
    fl.attn_fwd(_nan_guard(q), _nan_guard(kp), _nan_guard(vp), out=out, kv_page_table=t.cuda(), kv_len=1000,
                mask="causal")
    torch.cuda.synchronize()
    _check_margins(obuf, olo, ohi, 1234.5)
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("Sq", [1000, 1])
def test_guard_rsa(Sq):
    from paper_2511_02043_b200 import fl
    torch.manual_seed(1)
    k = torch.randn(1, 2, 1000, 128, device="cuda").to(torch.bfloat16)
    q = torch.randn(1, 2, 1000, 128, device="cuda").to(torch.bfloat16)[:, :, -Sq:]
    kmin, kmax = fl.rsa_build_summaries(k, 128)
    gkmin, bmin, (lo0, hi0) = _canary_out(kmin.shape, kmin.dtype)
    gkmax, bmax, (lo1, hi1) = _canary_out(kmax.shape, kmax.dtype)
    fl.rsa_build_summaries(_nan_guard(k), 128, kmin=gkmin, kmax=gkmax)
    torch.cuda.synchronize()
    _check_margins(bmin, lo0, hi0, 1234.5)
    _check_margins(bmax, lo1, hi1, 1234.5)
    assert torch.equal(gkmin.view(torch.int16), kmin.view(torch.int16))
    assert torch.equal(gkmax.view(torch.int16), kmax.view(torch.int16))
    idx, cnt = fl.rsa_select(q, kmin, kmax, 1000, topk=2)
    gidx, bidx, (lo2, hi2) = _canary_out(idx.shape, torch.int32)
    gcnt, bcnt, (lo3, hi3) = _canary_out(cnt.shape, torch.int32)
    fl.rsa_select(_nan_guard(q), _nan_guard(kmin), _nan_guard(kmax), 1000, topk=2, blk_idx=gidx, blk_cnt=gcnt)
    torch.cuda.synchronize()
    _check_margins(bidx, lo2, hi2, 0x5A5A5A5A)
    _check_margins(bcnt, lo3, hi3, 0x5A5A5A5A)
    assert torch.equal(gidx, idx) and torch.equal(gcnt, cnt)
