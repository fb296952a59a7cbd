"""Python binding of the C ABI (include/fl_attn.h) -- argument marshalling only.

Every step of the attention path runs in the CUDA kernels behind
``libfl_attn.so``; this module turns torch tensors (device memory, streams) into
``fl_tensor`` views and raises :class:`FlError` on any non-OK status.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from ._lib import AttnArgs, FlError, Tensor, Variant  # noqa: F401  (re-export)

MOD = {"none": 0, "alibi": 1, "softcap": 2}
MASK = {"none": 0, "causal": 1, "sliding": 2, "prefix": 3, "document": 4, "blocklist": 5}
GATE = {"none": 0, "mul": 1, "sigmoid": 2}
_DT = {torch.bfloat16: _lib.FL_BF16, torch.float32: _lib.FL_F32, torch.uint8: _lib.FL_U8,
       torch.int32: _lib.FL_I32, torch.bool: _lib.FL_U8}


def tensor(t: Optional[torch.Tensor]) -> Tensor:
    out = Tensor()
    if t is None:
        return out
    if t.dim() > 5:
        raise ValueError("rank > 5")
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype}")
    out.data = t.data_ptr()
    out.dtype = _DT[t.dtype]
    out.rank = t.dim()
    for i, (s, st) in enumerate(zip(t.shape, t.stride())):
        out.size[i] = s
        out.stride[i] = st
    return out


def _f32vec(x, device):
    if x is None:
        return None
    if not torch.is_tensor(x):
        x = torch.tensor(x, dtype=torch.float32)
    return x.to(device=device, dtype=torch.float32).contiguous()


def make_args(q, k, v, o, lse=None, *, scale=0.0, mod="none", softcap=0.0, alibi_slopes=None, mask="none",
              window=0, prefix=0, doc_offsets=None, doc_causal=False, causal_align=0, bias=None, key_mask=None,
              gate_mode="none", gate=None, diff=False, lam=0.0, lambda_h=None, blk_idx=None, blk_cnt=None,
              blk_q=128, blk_k=128, kv_page_table=None, kv_len=0, lambda_qk=None, lambda_init=0.0,
              diff_norm=False, diff_norm_eps=1e-5, diff_norm_w=None, stream=None, keep=None):
    """Fill an fl_attn_args.  ``keep`` collects temporaries that must outlive the call."""
    keep = [] if keep is None else keep
    dev = q.device
    a = AttnArgs()
    a.q, a.k, a.v, a.o, a.lse = tensor(q), tensor(k), tensor(v), tensor(o), tensor(lse)
    var = a.var
    var.abi_version = _lib.ABI_VERSION
    var.scale = float(scale)
    var.mod = MOD[mod]
    var.softcap = float(softcap)
    sl = _f32vec(alibi_slopes, dev)
    keep.append(sl)
    var.alibi_slopes = tensor(sl)
    var.mask = MASK[mask]
    var.window = int(window)
    var.prefix_len = int(prefix)
    if doc_offsets is not None:
        do = doc_offsets if torch.is_tensor(doc_offsets) else torch.as_tensor(doc_offsets)
        do = do.to(device=dev, dtype=torch.int32).contiguous()
        keep.append(do)
        var.doc_offsets = tensor(do)
    var.doc_causal = int(bool(doc_causal))
    var.causal_align = int(causal_align)
    var.bias = tensor(bias)
    if key_mask is not None and key_mask.dtype == torch.bool:
        key_mask = key_mask.to(torch.uint8)
        keep.append(key_mask)
    var.key_mask = tensor(key_mask)
    var.gate_mode = GATE[gate_mode]
    var.gate = tensor(gate)
    var.diff = int(bool(diff))
    var.lambda_ = float(lam)
    lh = _f32vec(lambda_h, dev)
    keep.append(lh)
    var.lambda_h = tensor(lh)
    for name, t in (("blk_idx", blk_idx), ("blk_cnt", blk_cnt)):
        if t is not None:
            t = (t if torch.is_tensor(t) else torch.as_tensor(t)).to(device=dev, dtype=torch.int32).contiguous()
            keep.append(t)
            setattr(var, name, tensor(t))
    var.blk_q, var.blk_k = int(blk_q), int(blk_k)
    lq = _f32vec(lambda_qk, dev)            # DIFF-Transformer epilogue (NEXT-2): [4, D_qk] flattened
    lq = lq.reshape(-1) if lq is not None else None
    keep.append(lq)
    var.lambda_qk = tensor(lq)
    var.lambda_init = float(lambda_init)
    var.diff_norm = int(bool(diff_norm))
    var.diff_norm_eps = float(diff_norm_eps)
    nw = _f32vec(diff_norm_w, dev)
    keep.append(nw)
    var.diff_norm_w = tensor(nw)
    if kv_page_table is not None:          # paged KV: k / v are page pools [n_pages, H, 128, D]
        t = (kv_page_table if torch.is_tensor(kv_page_table) else torch.as_tensor(kv_page_table))
        t = t.to(device=dev, dtype=torch.int32).contiguous()
        keep.append(t)
        var.kv_page_table = tensor(t)
        var.kv_len = int(kv_len)
    if stream is None and q.is_cuda:
        stream = torch.cuda.current_stream(q.device)
    a.stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    return a


def paged_kv(k: torch.Tensor, v: torch.Tensor, n_pages_total=None, seed=0):
    """Scatter contiguous K/V [B, H, S_k, D] into page pools [n_pages, H, 128, D] in a shuffled page
    order; returns (k_pool, v_pool, page_table i32 [B, ceil(S_k / 128)]).  A test / serving helper
    (data movement only)."""
    B, H, S, D = k.shape
    npb = (S + 127) // 128
    n_pages = n_pages_total or B * npb
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(n_pages, generator=g)[:B * npb].view(B, npb)
    kp = torch.zeros(n_pages, H, 128, D, dtype=k.dtype, device=k.device)
    vp = torch.zeros(n_pages, H, 128, v.shape[-1], dtype=v.dtype, device=v.device)
    for b in range(B):
        for t in range(npb):
            n = min(128, S - 128 * t)
            kp[perm[b, t], :, :n] = k[b, :, 128 * t:128 * t + n]
            vp[perm[b, t], :, :n] = v[b, :, 128 * t:128 * t + n]
    return kp, vp, perm.to(torch.int32)


def out_shape(q, v, diff):
    shp = list(q.shape)
    if diff:
        shp[-3] //= 2
    shp[-1] = v.shape[-1]
    return shp


def attn_fwd(q, k, v, *, out=None, return_lse=False, lse=None, workspace=None, **variant):
    """Fused attention forward on the current CUDA stream.

    q/k/v: CUDA tensors [B,H,S,D] or [B,G,H,S,D] (bf16 -> tcgen05 path, f32 ->
    exact SIMT path).  Variant keywords follow fl_variant (see make_args).
    Returns ``out`` (and ``lse`` when ``return_lse``)."""
    diff = variant.get("diff", False)
    if out is None:
        out = torch.empty(out_shape(q, v, diff), device=q.device, dtype=q.dtype)
    if return_lse and lse is None:
        lse = torch.empty(out_shape(q, v, diff)[:-1], device=q.device, dtype=torch.float32)
    keep: list = []
    a = make_args(q, k, v, out, lse, keep=keep, **variant)
    need = C.c_size_t(0)
    _lib.check(_lib.lib().fl_attn_workspace_size(C.byref(a), C.byref(need)))
    if need.value:
        if workspace is None or workspace.numel() * workspace.element_size() < need.value:
            workspace = torch.empty(need.value, dtype=torch.uint8, device=q.device)
        keep.append(workspace)
        a.workspace = workspace.data_ptr()
        a.workspace_bytes = need.value
    _lib.check(_lib.lib().fl_attn_fwd(C.byref(a)))
    _keep_alive_on(variant.get("stream"), keep)
    return (out, lse) if return_lse else out


def _keep_alive_on(stream, tensors):
    """The kernel may still read temporaries (workspace, slopes, offsets, lists) on a caller-given stream
    after this call returns: tell the caching allocator they are in use there."""
    if stream is None or not hasattr(stream, "cuda_stream"):
        return
    for t in tensors:
        if torch.is_tensor(t) and t.is_cuda:
            t.record_stream(stream)


def _bwd_args(q, k, v, out, lse, dout, dq, dk, dv, dgate, dbias, dlambda, variant):
    keep: list = []
    fa = make_args(q, k, v, out, lse, keep=keep, **variant)
    a = _lib.BwdArgs()
    a.q, a.k, a.v, a.o, a.lse = fa.q, fa.k, fa.v, fa.o, fa.lse
    a.dout, a.dq, a.dk, a.dv = tensor(dout), tensor(dq), tensor(dk), tensor(dv)
    a.dgate = tensor(dgate)
    a.dbias = tensor(dbias)        # optional: pass an f32 tensor shaped like the bias to receive dL/dbias
    a.dlambda = tensor(dlambda)
    a.var = fa.var
    a.stream = fa.stream
    need = C.c_size_t(0)
    _lib.check(_lib.lib().fl_attn_bwd_workspace_size(C.byref(a), C.byref(need)))
    return a, keep, need


def attn_bwd_workspace_bytes(q, k, v, out, lse, dout, **variant) -> int:
    """fl_attn_bwd_workspace_size for these arguments (gradient buffers are not needed to size it)."""
    gated = variant.get("gate_mode") in ("sigmoid", "mul")
    dg = torch.empty(out.shape, dtype=torch.bfloat16, device=q.device) if gated else None
    return _bwd_args(q, k, v, out, lse, dout, torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), dg,
                     None, None, variant)[2].value


def attn_bwd(q, k, v, out, lse, dout, *, dq=None, dk=None, dv=None, dgate=None, dbias=None, dlambda=None,
             workspace=None, **variant):
    """Backward of attn_fwd (fl_attn_bwd, NEXT-3): returns (dq, dk, dv) of L = sum(out * dout), given the
    forward's output and natural-log LSE (attn_fwd(..., return_lse=True)); with a gate also dgate
    (dL/dgate, of the logits for the sigmoid gate): (dq, dk, dv, dgate).  Differential attention (diff=True): lse=None (the call recomputes
    the maps); pass an f32 [Hq] `dlambda` to receive dL/dlambda_h."""
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    gated = variant.get("gate_mode") in ("sigmoid", "mul")
    if gated and dgate is None:
        dgate = torch.empty(out.shape, dtype=torch.bfloat16, device=q.device)
    a, keep, need = _bwd_args(q, k, v, out, lse, dout, dq, dk, dv, dgate, dbias, dlambda, variant)
    if workspace is None or workspace.numel() * workspace.element_size() < need.value:
        workspace = torch.empty(max(need.value, 1), dtype=torch.uint8, device=q.device)
    keep.append(workspace)
    a.workspace = workspace.data_ptr()
    a.workspace_bytes = need.value
    _lib.check(_lib.lib().fl_attn_bwd(C.byref(a)))
    _keep_alive_on(variant.get("stream"), keep)
    return (dq, dk, dv, dgate) if gated else (dq, dk, dv)


class HostRunner:
    """End-to-end entry over HOST buffers (fl_attn_fwd_host): H2D copies of the
    inputs, the kernel and the D2H copy of the output, all enqueued by the C ABI
    on one stream.  Device scratch is allocated once and reused."""

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self.scratch = None

    def __call__(self, q, k, v, out, lse=None, stream=None, **variant):
        keep: list = []
        a = make_args(q, k, v, out, lse, keep=keep, stream=stream or torch.cuda.current_stream(self.device),
                      **variant)
        need = C.c_size_t(0)
        _lib.check(_lib.lib().fl_attn_host_scratch_size(C.byref(a), C.byref(need)))
        if self.scratch is None or self.scratch.numel() < need.value:
            self.scratch = torch.empty(max(need.value, 1), dtype=torch.uint8, device=self.device)
        _lib.check(_lib.lib().fl_attn_fwd_host(C.byref(a), self.scratch.data_ptr(), self.scratch.numel()))
        _keep_alive_on(stream, keep)
        return out


def _stream_handle(device, stream=None):
    stream = stream or torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream


def rsa_build_summaries(k: torch.Tensor, blk_k: int = 128, kmin=None, kmax=None, stream=None):
    """RSA per-KV-block key summaries (fl_rsa_build_summaries): returns (kmin, kmax),
    bf16 [B*G*Hkv, ceil(S_k/blk_k), D], the exact element-wise min / max of each block."""
    rank = k.dim()
    bgh = 1
    for s_ in k.shape[:rank - 2]:
        bgh *= s_
    Sk, D = k.shape[-2], k.shape[-1]
    nkb = (Sk + blk_k - 1) // blk_k
    if kmin is None:
        kmin = torch.empty(bgh, nkb, D, device=k.device, dtype=torch.bfloat16)
    if kmax is None:
        kmax = torch.empty(bgh, nkb, D, device=k.device, dtype=torch.bfloat16)
    tk, tmn, tmx = tensor(k), tensor(kmin), tensor(kmax)
    _lib.check(_lib.lib().fl_rsa_build_summaries(C.byref(tk), C.byref(tmn), C.byref(tmx), int(blk_k),
                                                 _stream_handle(k.device, stream)))
    return kmin, kmax


def rsa_update_summaries(k: torch.Tensor, kmin: torch.Tensor, kmax: torch.Tensor, k_begin: int, blk_k: int = 128,
                         stream=None):
    """Refresh the summaries of the blocks from floor(k_begin / blk_k) on after a KV append
    (fl_rsa_update_summaries); k is the whole cache, kmin / kmax sized for it.  Returns (kmin, kmax)."""
    tk, tmn, tmx = tensor(k), tensor(kmin), tensor(kmax)
    _lib.check(_lib.lib().fl_rsa_update_summaries(C.byref(tk), C.byref(tmn), C.byref(tmx), int(blk_k), int(k_begin),
                                                  _stream_handle(k.device, stream)))
    return kmin, kmax


def rsa_select(q: torch.Tensor, kmin: torch.Tensor, kmax: torch.Tensor, s_k: int, *, topk: int = 16,
               blk_q: int = 128, blk_k: int = 128, causal_align: int = 0, max_sel=None, blk_idx=None,
               blk_cnt=None, stream=None):
    """RSA data-dependent block selection (fl_rsa_select): returns (blk_idx i32
    [B*G*Hq, n_qblk, max_sel], blk_cnt i32 [B*G*Hq, n_qblk]) ready for mask="blocklist"."""
    bgh = 1
    for s_ in q.shape[:-2]:
        bgh *= s_
    nqb = (q.shape[-2] + blk_q - 1) // blk_q
    max_sel = topk + 2 if max_sel is None else max_sel
    if blk_idx is None:
        blk_idx = torch.empty(bgh, nqb, max_sel, device=q.device, dtype=torch.int32)
    if blk_cnt is None:
        blk_cnt = torch.empty(bgh, nqb, device=q.device, dtype=torch.int32)
    tq, tmn, tmx, ti, tc = tensor(q), tensor(kmin), tensor(kmax), tensor(blk_idx), tensor(blk_cnt)
    _lib.check(_lib.lib().fl_rsa_select(C.byref(tq), C.byref(tmn), C.byref(tmx), int(s_k), int(topk), int(blk_q),
                                        int(blk_k), int(causal_align), C.byref(ti), C.byref(tc),
                                        _stream_handle(q.device, stream)))
    return blk_idx, blk_cnt


def linear(x: torch.Tensor, w: torch.Tensor, bias=None, ln_gamma=None, ln_beta=None, eps: float = 1e-5, out=None,
           stream=None):
    """Fused LayerNorm-prologue linear layer (fl_linear, NEXT-2): out = [LN(x)] w^T + bias.  x bf16
    [..., K] (rows flattened), w bf16 [N, K], bias / ln_gamma / ln_beta f32; out bf16 [..., N] or any
    rank-2 [M, N] view (e.g. a transposed one)."""
    x2 = x.reshape(-1, x.shape[-1])
    if out is None:
        out = torch.empty(*x.shape[:-1], w.shape[0], device=x.device, dtype=torch.bfloat16)
    y2 = out if out.dim() == 2 else out.view(-1, w.shape[0])
    a = _lib.LinearArgs()
    a.x, a.w, a.y = tensor(x2), tensor(w), tensor(y2)
    a.bias, a.ln_gamma, a.ln_beta = tensor(bias), tensor(ln_gamma), tensor(ln_beta)
    a.ln_eps = float(eps)
    a.stream = _stream_handle(x.device, stream)
    _lib.check(_lib.lib().fl_linear(C.byref(a)))
    return out


def ipa_fwd(q, k, v, qp, kp, vp, R, t, bias, z, gamma, *, workspace=None, stream=None):
    """Invariant Point Attention core (fl_ipa_fwd, NEXT-4, reading G23): q, k, v bf16 [N, H, c]; qp, kp bf16
    [N, H, Pq, 3]; vp bf16 [N, H, Pv, 3]; R f32 [N, 3, 3]; t f32 [N, 3]; bias bf16 [H, N, N]; z bf16
    [N, N, cz]; gamma f32 [H].  Returns (o bf16 [N, H, c], op f32 [N, H, Pv, 3], opair bf16 [N, H, cz])."""
    N, H, c = q.shape
    Pv, cz = vp.shape[2], z.shape[2]
    o = torch.empty(N, H, c, device=q.device, dtype=torch.bfloat16)
    op = torch.empty(N, H, Pv, 3, device=q.device, dtype=torch.float32)
    opair = torch.empty(N, H, cz, device=q.device, dtype=torch.bfloat16)
    a = _lib.IpaArgs()
    for name, tt in (("q", q), ("k", k), ("v", v), ("qp", qp), ("kp", kp), ("vp", vp), ("R", R), ("t", t),
                     ("bias", bias), ("z", z), ("gamma", gamma), ("o", o), ("op", op), ("opair", opair)):
        setattr(a, name, tensor(tt))
    a.stream = _stream_handle(q.device, stream)
    need = C.c_size_t(0)
    _lib.check(_lib.lib().fl_ipa_workspace_size(C.byref(a), C.byref(need)))
    if workspace is None or workspace.numel() * workspace.element_size() < need.value:
        workspace = torch.empty(need.value, dtype=torch.uint8, device=q.device)
    a.workspace, a.workspace_bytes = workspace.data_ptr(), need.value
    _lib.check(_lib.lib().fl_ipa_fwd(C.byref(a)))
    _keep_alive_on(stream, [workspace])
    return o, op, opair


def diag_umma_gemm(a: torch.Tensor, b: torch.Tensor, n: int, k: int, b_mn_major=False, a_from_tmem=False):
    c = torch.empty(128, n, device=a.device, dtype=torch.float32)
    s = torch.cuda.current_stream(a.device).cuda_stream
    _lib.check(_lib.lib().fl_diag_umma_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, k, int(b_mn_major),
                                            int(a_from_tmem), s))
    return c


def debug_schedule(q, k, v, **variant):
    """The bf16 kernel's (unit, warpgroup) work and tile classes for this problem (fl_debug_schedule):
    int32 numpy array [n_records, 8 + max_tiles] (see include/fl_attn.h)."""
    import numpy as np
    out = torch.empty(out_shape(q, v, variant.get("diff", False)), device=q.device, dtype=q.dtype)
    keep: list = []
    a = make_args(q, k, v, out, None, keep=keep, **variant)
    n, mt = C.c_int64(0), C.c_int32(0)
    _lib.check(_lib.lib().fl_debug_schedule(C.byref(a), None, 0, C.byref(n), C.byref(mt)))
    buf = torch.empty(n.value * (8 + mt.value), dtype=torch.int32, device=q.device)
    _lib.check(_lib.lib().fl_debug_schedule(C.byref(a), buf.data_ptr(), buf.numel(), C.byref(n), C.byref(mt)))
    torch.cuda.synchronize(q.device)
    return buf.cpu().numpy().reshape(n.value, 8 + mt.value)


PIPE_OPS = {"ex2_f32": 0, "ex2_bf16x2": 1, "tanh_f32": 2, "ffma2": 3}


def pipe_rate(op: str, device=None, iters: int = 4096, reps: int = 5) -> float:
    """Measured throughput (elementary ops / s) of one MUFU / FMA operation (fl_diag_pipe_rate), the
    best of `reps` launches timed with CUDA events on the current stream."""
    device = torch.device(device or "cuda")
    sink = torch.empty(1 << 20, dtype=torch.float32, device=device)
    s = torch.cuda.current_stream(device)
    ops = C.c_int64(0)
    best = 0.0
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        _lib.check(_lib.lib().fl_diag_pipe_rate(PIPE_OPS[op], iters, sink.data_ptr(), C.byref(ops), s.cuda_stream))
        e1.record(s)
        torch.cuda.synchronize(device)
        if r:
            best = max(best, ops.value / (e0.elapsed_time(e1) * 1e-3))
    return best


def shard_range(units: int, world: int, rank: int):
    b, e = C.c_int64(), C.c_int64()
    _lib.lib().fl_shard_range(units, world, rank, C.byref(b), C.byref(e))
    return b.value, e.value


def launch_count(reset=False) -> int:
    return int(_lib.lib().fl_launch_count(int(reset)))
