"""fp64 CPU oracle of the Flashlight attention-variant forward (arXiv 2511.02043).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2511_02043_b200``) never imports it and it
never imports the product path: the two share no code.

The arithmetic lives in ``fl_oracle.c`` (plain C, fp64, OpenMP over rows); this
module only marshals tensors into its ``flo_problem`` struct.  See the header of
``fl_oracle.c`` for the paper passages each step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fl_oracle.c")
_SO = os.path.join(_HERE, "libfl_oracle.so")

F64, F32, BF16, U8 = 0, 1, 2, 3
MOD = {"none": 0, "alibi": 1, "softcap": 2}
MASK = {"none": 0, "causal": 1, "sliding": 2, "prefix": 3, "document": 4, "blocklist": 5}
GATE = {"none": 0, "mul": 1, "sigmoid": 2}


def build(force: bool = False) -> str:
    """Compile libfl_oracle.so with gcc (-O2, no fast-math: exact IEEE fp64)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
               "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


class _Tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32),
                ("size", C.c_int64 * 5), ("stride", C.c_int64 * 5)]


class _Problem(C.Structure):
    _fields_ = [
        ("q", _Tensor), ("k", _Tensor), ("v", _Tensor),
        ("scale", C.c_double), ("mod", C.c_int32), ("softcap", C.c_double),
        ("alibi_slopes", C.POINTER(C.c_double)),
        ("mask", C.c_int32), ("window", C.c_int64), ("prefix", C.c_int64),
        ("doc_offsets", C.POINTER(C.c_int32)), ("n_docs", C.c_int32), ("doc_causal", C.c_int32),
        ("causal_align", C.c_int32),
        ("bias", _Tensor), ("key_mask", _Tensor),
        ("gate_mode", C.c_int32), ("gate", _Tensor),
        ("diff", C.c_int32), ("lambda_", C.c_double), ("lambda_h", C.POINTER(C.c_double)),
        ("blk_idx", C.POINTER(C.c_int32)), ("blk_cnt", C.POINTER(C.c_int32)),
        ("blk_q", C.c_int32), ("blk_k", C.c_int32), ("max_sel", C.c_int32),
        ("lambda_qk", C.POINTER(C.c_double)), ("lambda_init", C.c_double), ("diff_norm", C.c_int32),
        ("diff_norm_eps", C.c_double), ("diff_norm_w", C.POINTER(C.c_double)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.flo_attn.argtypes = [C.POINTER(_Problem), C.POINTER(C.c_int64), C.c_int64,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.flo_attn.restype = C.c_int
        _lib.flo_stable_softmax.argtypes = [C.POINTER(C.c_double), C.c_int64,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.flo_stable_softmax.restype = C.c_double
        _lib.flo_rsa_summaries.argtypes = [C.POINTER(_Tensor), C.c_int32,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.flo_rsa_select.argtypes = [C.POINTER(_Tensor), C.POINTER(_Tensor), C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        _lib.flo_num_threads.restype = C.c_int
        _lib.flo_keep_row.argtypes = [C.POINTER(_Problem), C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                      C.POINTER(C.c_uint8)]
        _lib.flo_keep_row.restype = C.c_int
        _lib.flo_attn_bwd.argtypes = [C.POINTER(_Problem), C.POINTER(_Tensor), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.flo_attn_bwd.restype = C.c_int
        dp = C.POINTER(C.c_double)
        _lib.flo_linear_ln.argtypes = [C.c_int64, C.c_int64, C.c_int64, dp, dp, dp, dp, dp, C.c_double, dp, dp]
        _lib.flo_linear_ln.restype = C.c_int
        _lib.flo_ipa.argtypes = [C.c_int64] * 6 + [dp] * 14
        _lib.flo_ipa.restype = C.c_int
    return _lib


def num_threads() -> int:
    return int(lib().flo_num_threads())


_DT = {torch.float64: F64, torch.float32: F32, torch.bfloat16: BF16, torch.uint8: U8, torch.bool: U8}


def _as5(t: torch.Tensor, keep: list) -> torch.Tensor:
    if t.device.type != "cpu":
        raise ValueError("oracle inputs must be CPU tensors")
    if t.dtype not in _DT:
        t = t.to(torch.float64)
    keep.append(t)
    return t


def _tensor(t, keep, rank5=True) -> _Tensor:
    out = _Tensor()
    if t is None:
        out.data = None
        return out
    t = _as5(t, keep)
    if rank5 and t.dim() == 4:
        t = t.unsqueeze(1)
        keep.append(t)
    if rank5 and t.dim() != 5:
        raise ValueError(f"expected rank 4 or 5, got {t.dim()}")
    out.data = t.data_ptr()
    out.dtype = _DT[t.dtype]
    sz = list(t.shape) + [1] * (5 - t.dim())
    st = list(t.stride()) + [0] * (5 - t.dim())
    for i in range(5):
        out.size[i] = sz[i]
        out.stride[i] = st[i] if sz[i] > 1 else 0
    return out


def _dptr(a, keep, ctype=C.c_double, np_dtype=np.float64):
    if a is None:
        return None
    arr = np.ascontiguousarray(np.asarray(a, dtype=np_dtype))
    keep.append(arr)
    return arr.ctypes.data_as(C.POINTER(ctype))


def attn(q, k, v, *, scale=0.0, mod="none", softcap=0.0, alibi_slopes=None,
         mask="none", window=0, prefix=0, doc_offsets=None, doc_causal=False,
         causal_align=0, bias=None, key_mask=None, gate_mode="none", gate=None,
         diff=False, lam=0.0, lambda_h=None, blk_idx=None, blk_cnt=None,
         blk_q=128, blk_k=128, lambda_qk=None, lambda_init=0.0, diff_norm=False, diff_norm_eps=1e-5,
         diff_norm_w=None, rows=None):
    """Evaluate the plain definition on CPU in fp64.

    q/k/v/bias/gate: torch CPU tensors [B,H,S,D] or [B,G,H,S,D] (any strides,
    bf16/fp32/fp64 values are read exactly).  bias is logical [B,G,Hq,Sq,Sk]
    (use expand() for broadcast dims); key_mask is logical [B,G,Sk] (u8/bool,
    1 = keep).  Returns (out [nrows, Dv] float64, lse [nrows] float64) where
    rows are flat ((b*G+g)*Hq+h)*Sq+q ids (None = all rows in that order).
    """
    keep: list = []
    p = _problem(q, k, v, keep, scale=scale, mod=mod, softcap=softcap, alibi_slopes=alibi_slopes, mask=mask,
                 window=window, prefix=prefix, doc_offsets=doc_offsets, doc_causal=doc_causal,
                 causal_align=causal_align, bias=bias, key_mask=key_mask, gate_mode=gate_mode, gate=gate, diff=diff,
                 lam=lam, lambda_h=lambda_h, blk_idx=blk_idx, blk_cnt=blk_cnt, blk_q=blk_q, blk_k=blk_k,
                 lambda_qk=lambda_qk, lambda_init=lambda_init, diff_norm=diff_norm, diff_norm_eps=diff_norm_eps,
                 diff_norm_w=diff_norm_w)
    maps = 2 if diff else 1
    qs = p.q.size
    total = qs[0] * qs[1] * (qs[2] // maps) * qs[3]
    if rows is None:
        rows_arr, n = None, total
    else:
        ra = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        keep.append(ra)
        rows_arr, n = ra.ctypes.data_as(C.POINTER(C.c_int64)), ra.size
    dv = p.v.size[4]
    out = np.zeros((n, dv), dtype=np.float64)
    lse = np.zeros((n,), dtype=np.float64)
    rc = lib().flo_attn(C.byref(p), rows_arr, n, out.ctypes.data_as(C.POINTER(C.c_double)),
                        lse.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        raise ValueError(f"flo_attn rejected the problem (code {rc})")
    return out, lse


def attn_bwd(q, k, v, dout, with_dgate=False, with_dbias=False, with_dlambda=False, **variant):
    """Gradients (dq, dk, dv) of L = sum(O * dout), fp64 numpy arrays shaped like q, k, v (NEXT-3); with
    with_dgate also dL/dgate (shaped like dout) for a gated variant, with with_dbias also dL/dbias as the
    full logical [B, G, Hq, Sq, Sk] array (sum it over the dims the bias broadcasts), with with_dlambda (diff)
    also dL/dlambda_h [Hq] (sum it over h for a scalar lambda)."""
    keep: list = []
    p = _problem(q, k, v, keep, **variant)
    dt = _tensor(dout, keep)
    dq = np.zeros(tuple(q.shape), dtype=np.float64)
    dk = np.zeros(tuple(k.shape), dtype=np.float64)
    dv = np.zeros(tuple(v.shape), dtype=np.float64)
    dg = np.zeros(tuple(dout.shape), dtype=np.float64) if with_dgate else None
    qs = tuple(q.shape) if q.dim() == 5 else (q.shape[0], 1) + tuple(q.shape[1:])
    maps = 2 if variant.get("diff") else 1
    B, G, Hq, Sq = qs[0], qs[1], qs[2] // maps, qs[3]
    Sk = tuple(k.shape)[-2]
    db = np.zeros((B, G, Hq, Sq, Sk), dtype=np.float64) if with_dbias else None
    dl = np.zeros(Hq, dtype=np.float64) if with_dlambda else None
    dpp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None
    rc = lib().flo_attn_bwd(C.byref(p), C.byref(dt), dpp(dq), dpp(dk), dpp(dv), dpp(dg), dpp(db), dpp(dl))
    if rc != 0:
        raise ValueError(f"flo_attn_bwd rejected the problem (code {rc})")
    out = (dq, dk, dv) + ((dg,) if with_dgate else ()) + ((db,) if with_dbias else ()) + ((dl,) if with_dlambda else ())
    return out


def keep_rows(q, k, v, rows, **variant):
    """Kept-key predicate (definition step 2: mask AND key mask) of each flat output row id
    ((b*G+g)*Hq+h)*Sq+q: returns uint8 [len(rows), S_k]."""
    keep: list = []
    p = _problem(q, k, v, keep, **variant)
    maps = 2 if variant.get("diff") else 1
    _, G, H2, Sq = (p.q.size[i] for i in range(4))
    Hq = H2 // maps
    Sk = p.k.size[3]
    out = np.zeros((len(rows), Sk), dtype=np.uint8)
    for i, r in enumerate(rows):
        qq, t = r % Sq, r // Sq
        h, t = t % Hq, t // Hq
        g, b = t % G, t // G
        rc = lib().flo_keep_row(C.byref(p), b, g, h, qq, out[i].ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc != 0:
            raise ValueError(f"flo_keep_row rejected the problem (code {rc})")
    return out


def _problem(q, k, v, keep, *, scale=0.0, mod="none", softcap=0.0, alibi_slopes=None,
             mask="none", window=0, prefix=0, doc_offsets=None, doc_causal=False,
             causal_align=0, bias=None, key_mask=None, gate_mode="none", gate=None,
             diff=False, lam=0.0, lambda_h=None, blk_idx=None, blk_cnt=None,
             blk_q=128, blk_k=128, lambda_qk=None, lambda_init=0.0, diff_norm=False, diff_norm_eps=1e-5,
             diff_norm_w=None):
    p = _Problem()
    p.q, p.k, p.v = _tensor(q, keep), _tensor(k, keep), _tensor(v, keep)
    p.scale = float(scale)
    p.mod = MOD[mod]
    p.softcap = float(softcap)
    p.alibi_slopes = _dptr(alibi_slopes, keep)
    p.mask = MASK[mask]
    p.window, p.prefix = int(window), int(prefix)
    if doc_offsets is not None:
        do = np.ascontiguousarray(np.asarray(doc_offsets, dtype=np.int32))
        keep.append(do)
        p.doc_offsets = do.ctypes.data_as(C.POINTER(C.c_int32))
        p.n_docs = do.shape[-1] - 1
    p.doc_causal = int(bool(doc_causal))
    p.causal_align = int(causal_align)
    if bias is not None:
        b5 = bias if bias.dim() == 5 else bias.unsqueeze(1)
        p.bias = _tensor(b5, keep)
    if key_mask is not None:
        km = key_mask.to(torch.uint8) if key_mask.dtype == torch.bool else key_mask
        km = km if km.dim() == 3 else km.unsqueeze(1)
        keep.append(km)
        t = _Tensor()
        t.data = km.data_ptr()
        t.dtype = U8
        for i in range(3):
            t.size[i] = km.shape[i]
            t.stride[i] = km.stride(i) if km.shape[i] > 1 else 0
        p.key_mask = t
    p.gate_mode = GATE[gate_mode]
    if gate is not None:
        p.gate = _tensor(gate, keep)
    p.diff = int(bool(diff))
    p.lambda_ = float(lam)
    p.lambda_h = _dptr(lambda_h, keep)
    if blk_idx is not None:
        bi = np.ascontiguousarray(np.asarray(blk_idx, dtype=np.int32))
        bc = np.ascontiguousarray(np.asarray(blk_cnt, dtype=np.int32))
        keep += [bi, bc]
        p.blk_idx = bi.ctypes.data_as(C.POINTER(C.c_int32))
        p.blk_cnt = bc.ctypes.data_as(C.POINTER(C.c_int32))
        p.max_sel = bi.shape[-1]
    p.blk_q, p.blk_k = int(blk_q), int(blk_k)
    p.lambda_qk = _dptr(None if lambda_qk is None else np.asarray(lambda_qk, dtype=np.float64).reshape(-1), keep)
    p.lambda_init = float(lambda_init)
    p.diff_norm = int(bool(diff_norm))
    p.diff_norm_eps = float(diff_norm_eps)
    p.diff_norm_w = _dptr(diff_norm_w, keep)
    return p


def stable_softmax(x):
    """Alg.1 on one vector: returns (sigma(x), m_N, d_N)."""
    keep: list = []
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    y = np.empty_like(x)
    m = C.c_double()
    d = lib().flo_stable_softmax(_dptr(x, keep), x.size, y.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.byref(m))
    return y, m.value, d


def rsa_summaries(k, blk_k):
    keep: list = []
    kt = _tensor(k, keep)
    B, G, H, S, D = (kt.size[i] for i in range(5))
    nkb = (S + blk_k - 1) // blk_k
    kmin = np.zeros((B * G * H, nkb, D))
    kmax = np.zeros((B * G * H, nkb, D))
    lib().flo_rsa_summaries(C.byref(kt), blk_k, kmin.ctypes.data_as(C.POINTER(C.c_double)),
                            kmax.ctypes.data_as(C.POINTER(C.c_double)))
    return kmin, kmax


def rsa_select(q, k, *, blk_q=128, blk_k=128, topk=16, causal_align=0, max_sel=None,
               want_scores=False):
    """Reading G10/G11 selection; returns (blk_idx [BGH,nqb,max_sel], blk_cnt [BGH,nqb], scores)."""
    keep: list = []
    qt, kt = _tensor(q, keep), _tensor(k, keep)
    B, G, Hq, Sq = (qt.size[i] for i in range(4))
    Sk = kt.size[3]
    nqb, nkb = (Sq + blk_q - 1) // blk_q, (Sk + blk_k - 1) // blk_k
    max_sel = topk + 2 if max_sel is None else max_sel
    idx = np.full((B * G * Hq, nqb, max_sel), -1, dtype=np.int32)
    cnt = np.zeros((B * G * Hq, nqb), dtype=np.int32)
    sc = np.zeros((B * G * Hq, nqb, nkb)) if want_scores else None
    rc = lib().flo_rsa_select(C.byref(qt), C.byref(kt), blk_q, blk_k, topk, causal_align, max_sel,
                              idx.ctypes.data_as(C.POINTER(C.c_int32)),
                              cnt.ctypes.data_as(C.POINTER(C.c_int32)),
                              sc.ctypes.data_as(C.POINTER(C.c_double)) if sc is not None else None)
    if rc != 0:
        raise ValueError(f"flo_rsa_select failed ({rc})")
    return idx, cnt, sc


def linear_ln(x, w, bias=None, ln_gamma=None, ln_beta=None, eps=1e-5, with_abs=False):
    """NEXT-2 oracle (fl_oracle.c flo_linear_ln): y = [LayerNorm(x)] w^T + bias in fp64.  x [..., K],
    w [N, K]; returns y [..., N] (and yabs = sum_k |xhat| |w| when with_abs)."""
    xt = torch.as_tensor(x).double().reshape(-1, np.shape(x)[-1]).contiguous()
    wt = torch.as_tensor(w).double().contiguous()
    M, K = xt.shape
    N = wt.shape[0]
    keep = []

    def ptr(a):
        if a is None:
            return None
        arr = np.ascontiguousarray(torch.as_tensor(a).double().numpy(), dtype=np.float64)
        keep.append(arr)
        return arr.ctypes.data_as(C.POINTER(C.c_double))
    y = np.empty((M, N), dtype=np.float64)
    ya = np.empty((M, N), dtype=np.float64) if with_abs else None
    rc = lib().flo_linear_ln(M, N, K, ptr(xt), ptr(wt), ptr(bias), ptr(ln_gamma), ptr(ln_beta), float(eps),
                             y.ctypes.data_as(C.POINTER(C.c_double)),
                             ya.ctypes.data_as(C.POINTER(C.c_double)) if with_abs else None)
    assert rc == 0, rc
    shp = tuple(np.shape(x)[:-1]) + (N,)
    return (y.reshape(shp), ya.reshape(shp)) if with_abs else y.reshape(shp)


def ipa(q, k, v, qp, kp, vp, R, t, bias, z, gamma):
    """NEXT-4 oracle (fl_oracle.c flo_ipa): the Invariant Point Attention core of AF2 Alg.22 (reading G23).
    q, k, v [N, H, c]; qp, kp [N, H, Pq, 3]; vp [N, H, Pv, 3]; R [N, 3, 3]; t [N, 3]; bias [H, N, N];
    z [N, N, cz]; gamma [H].  Returns (o [N, H, c], op [N, H, Pv, 3] in the local frames, opair [N, H, cz])."""
    arr = lambda x: np.ascontiguousarray(torch.as_tensor(x).double().numpy(), dtype=np.float64)
    ins = [arr(x) for x in (q, k, v, qp, kp, vp, R, t, bias, z, gamma)]
    N, H, c = ins[0].shape
    Pq, Pv, cz = ins[3].shape[2], ins[5].shape[2], ins[9].shape[2]
    o = np.zeros((N, H, c))
    op = np.zeros((N, H, Pv, 3))
    opair = np.zeros((N, H, cz))
    pp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    rc = lib().flo_ipa(N, H, c, Pq, Pv, cz, *[pp(a) for a in ins], pp(o), pp(op), pp(opair))
    assert rc == 0, rc
    return o, op, opair
