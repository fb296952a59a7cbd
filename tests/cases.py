"""Test-case builder: one seeded input set (synth) fed to both the CUDA path
(through the C ABI binding) and the fp64 oracle.  Inputs are generated on the
CPU, rounded once to the storage dtype, copied to the GPU; the oracle reads the
same CPU tensors, so no oracle input ever comes from the CUDA path."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2511_02043_b200 import synth

DT = {"bf16": torch.bfloat16, "f32": torch.float32}


def admissible(case, Sq, Sk, b=0):
    """Admissible key interval [lo, hi) per query row (for needle inputs)."""
    mask = case.get("mask", "none")
    off = 0 if case.get("causal_align") else Sk - Sq
    def f(q, b=b):
        qa = q + off
        if mask in ("causal", "blocklist"):
            return np.zeros_like(q), np.minimum(qa + 1, Sk)
        if mask == "sliding":
            return np.maximum(qa - case["window"], 0), np.minimum(qa + 1, Sk)
        if mask == "prefix":
            return np.zeros_like(q), np.minimum(np.maximum(case["prefix"], qa + 1), Sk)
        if mask == "document":
            o = case["doc_offsets"][b]
            j = np.searchsorted(o, qa, side="right") - 1
            return o[j], o[j + 1]
        return np.zeros_like(q), np.full_like(q, Sk)
    return f


def build(case: dict):
    """Returns (inputs, gpu_kwargs, oracle_kwargs).  inputs: q,k,v CPU tensors."""
    c = dict(case)
    dt = DT[c.get("dtype", "bf16")]
    B, Hq, Hkv = c.get("B", 1), c.get("Hq", 1), c.get("Hkv", c.get("Hq", 1))
    Sq, Sk = c.get("Sq", c.get("S", 128)), c.get("Sk", c.get("S", 128))
    D = c.get("D", 64)
    Dv = c.get("Dv", D)
    seed = c.get("seed", 0)
    maps = 2 if c.get("diff") else 1
    dist = c.get("dist", "uniform")
    if c.get("mask") == "document" and "doc_offsets" not in c:
        c["doc_offsets"] = synth.doc_offsets(B, Sk, c.get("n_docs", 12), seed=seed + 1)
    qs, ks, vs = (B, Hq * maps, Sq, D), (B, Hkv * maps, Sk, D), (B, Hkv, Sk, Dv)
    if dist == "needle":
        q, k = synth.needle(qs, ks, seed=seed, dtype=dt, interval=admissible(c, Sq, Sk))
    elif dist == "leak":
        # needle one key past each row's admissible interval (window start - 1 for sliding windows,
        # the first key after the interval otherwise): a mask that admits one key too many is
        # dominated by that key (T4 mutants in tests/test_mutants.py)
        lo, hi = admissible(c, Sq, Sk)(np.arange(Sq), 0)
        pick = lo - 1 if c.get("mask") == "sliding" else hi
        q, k = synth.needle_at(qs, ks, pick, seed=seed, dtype=dt)
    else:
        q = synth.uniform(qs, seed=seed, tensor="q", dtype=dt)
        k = synth.uniform(ks, seed=seed, tensor="k", dtype=dt)
    if dist == "constant":
        v = synth.constant_v(vs, seed=seed, dtype=dt)
    elif c.get("v") == "blockconst":
        v = synth.block_constant_v(vs, seed=seed, dtype=dt)
    else:
        v = synth.uniform(vs, seed=seed, tensor="v", dtype=dt)
    gk, ok = {}, {}
    for key in ("scale", "mod", "softcap", "mask", "window", "prefix", "doc_causal", "causal_align", "diff"):
        if key in c:
            gk[key] = c[key]
            ok[key] = c[key]
    if "doc_offsets" in c:
        gk["doc_offsets"] = torch.as_tensor(c["doc_offsets"])
        ok["doc_offsets"] = c["doc_offsets"]
    if c.get("alibi_custom"):
        sl = np.linspace(0.05, 0.9, Hq).astype(np.float32)
        gk["alibi_slopes"] = torch.from_numpy(sl)
        ok["alibi_slopes"] = sl.astype(np.float64)
    if c.get("diff"):
        lam = c.get("lam", 0.2)
        gk["lam"] = ok["lam"] = lam
        if c.get("lambda_h"):
            lh = np.linspace(0.1, 0.9, Hq).astype(np.float32)
            gk["lambda_h"] = torch.from_numpy(lh)
            ok["lambda_h"] = lh.astype(np.float64)
    if c.get("diff") and c.get("lambda_qk"):          # DIFF-Transformer lambda re-parameterisation (G8b)
        lq = (np.random.default_rng(seed + 7).random((4, D)) * 0.2 - 0.1).astype(np.float32)
        gk["lambda_qk"] = torch.from_numpy(lq)
        ok["lambda_qk"] = lq.astype(np.float64)
    if c.get("diff") and ("lambda_init" in c):
        gk["lambda_init"] = ok["lambda_init"] = c["lambda_init"]
    if c.get("diff") and c.get("diff_norm"):           # per-head RMSNorm epilogue (G8b)
        gk["diff_norm"] = ok["diff_norm"] = True
        gk["diff_norm_eps"] = ok["diff_norm_eps"] = c.get("diff_norm_eps", 1e-5)
        if c.get("diff_norm_w"):
            w = (np.random.default_rng(seed + 8).random(Dv) * 1.5 + 0.25).astype(np.float32)
            gk["diff_norm_w"] = torch.from_numpy(w)
            ok["diff_norm_w"] = w.astype(np.float64)
    if c.get("gate_mode"):
        g = synth.gate_logits((B, Hq, Sq, Dv), seed=seed, dtype=torch.bfloat16 if dt == torch.bfloat16 else dt)
        if c.get("gate_unit"):          # a mul gate in [-1, 1] (exact: / 4), the |inputs| <= 1 regime of the bar
            g = g / 4
        gk["gate_mode"] = ok["gate_mode"] = c["gate_mode"]
        gk["gate"] = g
        ok["gate"] = g
    if c.get("bias"):
        bshape = (B, Hq, Sq, Sk)
        bias = synth.pair_bias(bshape, seed=seed, dtype=torch.bfloat16 if c.get("bias") == "bf16" else torch.float32)
        gk["bias"] = bias
        ok["bias"] = bias
    if c.get("key_mask"):
        km = synth.key_mask((B, Sk), seed=seed, p_zero=c.get("p_zero", 0.1))
        gk["key_mask"] = km
        ok["key_mask"] = km
    if c.get("mask") == "blocklist":
        blk = 128
        idx, cnt, _ = oracle.rsa_select(q, k, blk_q=blk, blk_k=blk, topk=c.get("topk", 2), causal_align=0)
        gk.update(blk_idx=torch.from_numpy(idx), blk_cnt=torch.from_numpy(cnt), blk_q=blk, blk_k=blk)
        ok.update(blk_idx=idx, blk_cnt=cnt, blk_q=blk, blk_k=blk)
    return {"q": q, "k": k, "v": v}, gk, ok


def evoformer(case: dict):
    """Evoformer row/column gated attention with pair bias on MSA storage
    [B, N_seq, N_res, H, c] (reading G9).  Returns (inputs5, gpu_kwargs, oracle_kwargs, out_shape)."""
    B, Ns, Nr, H, c = case["B"], case["Ns"], case["Nr"], case["H"], case["c"]
    seed = case.get("seed", 0)
    dt = DT[case.get("dtype", "bf16")]
    m = lambda t: synth.uniform((B, Ns, Nr, H, c), seed=seed, tensor=t, dtype=dt, lead=3)
    Q, K, V = m("q"), m("k"), m("v")
    if case.get("dist") == "needle":                    # needle rows in the attention view (peaked softmax)
        if case["kind"] == "row":                       # view rows: (b, s, h) x keys i
            q, k = synth.needle((B * Ns, H, Nr, c), (B * Ns, H, Nr, c), seed=seed, dtype=dt)
            to = lambda t: t.reshape(B, Ns, H, Nr, c).permute(0, 1, 3, 2, 4).contiguous()
        else:                                           # view rows: (b, i, h) x keys s
            q, k = synth.needle((B * Nr, H, Ns, c), (B * Nr, H, Ns, c), seed=seed, dtype=dt)
            to = lambda t: t.reshape(B, Nr, H, Ns, c).permute(0, 3, 1, 2, 4).contiguous()
        Q, K = to(q), to(k)
    Gt = synth.uniform((B, Ns, Nr, H, c), seed=seed, tensor="gate", dtype=torch.bfloat16 if dt == torch.bfloat16 else dt,
                       lo=-4, hi=4, lead=3)
    msa_mask = synth.key_mask((B, Ns, Nr), seed=seed, p_zero=case.get("p_zero", 0.0), lead=2)
    if case["kind"] == "row":
        view = lambda t: t.permute(0, 1, 3, 2, 4)               # [B, G=s, H, S=i, c]
        pb = synth.pair_bias((B, H, Nr, Nr), seed=seed, dtype=torch.bfloat16 if dt == torch.bfloat16 else dt)
        bias = pb.unsqueeze(1).expand(B, Ns, H, Nr, Nr)        # broadcast over s (stride 0)
        km = msa_mask                                           # [B, G=s, S_k=j]
    else:
        view = lambda t: t.permute(0, 2, 3, 1, 4)               # [B, G=i, H, S=s, c]
        bias = None
        km = msa_mask.permute(0, 2, 1)                          # [B, G=i, S_k=s'] (strided)
    ins = {"q": view(Q), "k": view(K), "v": view(V), "storage": (Q, K, V)}
    gk = dict(gate_mode="sigmoid", gate=view(Gt), key_mask=km)
    ok = dict(gate_mode="sigmoid", gate=view(Gt), key_mask=km)
    if bias is not None:
        gk["bias"] = bias
        ok["bias"] = bias
    return ins, gk, ok


def to_dev(x, dev):
    """Copy to the device keeping broadcast (stride-0) dims broadcast: .to() would materialise an
    expanded tensor, and the kernels take different paths for a broadcast bias (resident pair bias)."""
    if torch.is_tensor(x):
        bdims = [i for i, (n, st) in enumerate(zip(x.shape, x.stride())) if st == 0 and n > 1]
        if bdims:
            sl = tuple(slice(0, 1) if i in bdims else slice(None) for i in range(x.dim()))
            return x[sl].to(dev).expand(x.shape)
        return x.to(dev)
    return x


def run_gpu(fl, ins, gk, dev="cuda", **extra):
    q, k, v = (ins[n].to(dev) for n in ("q", "k", "v"))
    kw = {kk: to_dev(vv, dev) for kk, vv in gk.items()}
    kw.update(extra)
    out = fl.attn_fwd(q, k, v, **kw)
    torch.cuda.synchronize()
    return out


def run_oracle(ins, ok, rows=None):
    return oracle.attn(ins["q"], ins["k"], ins["v"], rows=rows, **ok)


def sample_rows(B, G, H, Sq, n=512, seed=0, extra_q=()):
    """Deterministic row sample over (b,g,h,q): tile boundaries + random rows."""
    rng = np.random.default_rng(seed)
    total = B * G * H * Sq
    qs = sorted({0, 1, 127, 128, 129, 255, 256, Sq // 2, Sq - 2, Sq - 1, *extra_q} & set(range(Sq)))
    rows = []
    for bgh in rng.choice(B * G * H, size=min(8, B * G * H), replace=False):
        rows += [int(bgh) * Sq + q for q in qs]
    rows += list(rng.choice(total, size=max(0, n - len(rows)), replace=False))
    return np.unique(np.array(rows, dtype=np.int64))
