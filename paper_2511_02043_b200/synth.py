"""Seeded synthetic inputs for the attention-variant forward (no method arithmetic).

This module is the ONE piece shared by the CUDA path's callers (bench, tests)
and the oracle's callers: it only draws numbers.  It contains none of the
method's arithmetic (no scores, softmax, masks applied to data, ...).

Shard consistency: every tensor is drawn slab by slab, each slab from its own
numpy Philox stream keyed by (seed, tensor id, slab index) where a slab is one
index of the leading ``lead`` dims.  Any rank can therefore regenerate exactly
its slice of the global tensor (SURVEY §8(d) "Input distributions").

Recipes:
  uniform   U[-1,1) -> bf16 (round to nearest even) or fp32
  needle    K in {+-1}^D, Q[q] = K[pi(q)], pi(q) uniform over the row's admissible keys
  constant  V[k,:] = c for every key k, c ~ U[-1,1)^D per slab  (closed form O = c)
  docs      11 distinct cut points uniform on (1, S-1) per batch b, seed (1, b)
  clustered RSA: 32 centroids in {+-0.6}^D per slab; a KV block of 128 keys
            gets cluster z(j), its keys clip(c_z + 0.4 U[-1,1), +-1); q-blocks likewise
"""
from __future__ import annotations

import numpy as np
import torch

TENSOR_IDS = {"q": 1, "k": 2, "v": 3, "gate": 4, "bias": 5, "key_mask": 6, "lambda": 7, "doc": 8}


def _rng(seed: int, tensor: str, slab: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed) & 0xFFFFFFFF, TENSOR_IDS[tensor] * (1 << 40) + slab]))


def _to(a: np.ndarray, dtype: torch.dtype) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return t.to(dtype)


def _slabs(shape, lead):
    n = 1
    for s in shape[:lead]:
        n *= s
    inner = shape[lead:]
    return n, inner


def _slab_ids(n, slab_range, slabs):
    if slabs is not None:
        return list(slabs)
    b, e = (0, n) if slab_range is None else slab_range
    return list(range(b, e))


def uniform(shape, *, seed=0, tensor="q", dtype=torch.bfloat16, lo=-1.0, hi=1.0, lead=2,
            slab_range=None, slabs=None) -> torch.Tensor:
    """U[lo,hi) drawn slab by slab over the first ``lead`` dims.

    slab_range=(begin, end) -- or an explicit list ``slabs`` of flattened slab ids -- returns only
    those slabs (flattened over the lead dims), identical to the same slabs of the full tensor."""
    n, inner = _slabs(shape, lead)
    ids = _slab_ids(n, slab_range, slabs)
    out = np.empty((len(ids),) + tuple(inner), dtype=np.float32)
    for j, i in enumerate(ids):
        out[j] = _rng(seed, tensor, i).random(tuple(inner), dtype=np.float32) * (hi - lo) + lo
    t = _to(out, dtype)
    return t.reshape(tuple(shape)) if slab_range is None and slabs is None else t


def constant_v(shape, *, seed=0, dtype=torch.bfloat16, lead=2, slab_range=None, slabs=None) -> torch.Tensor:
    """V[..., k, :] = c (one c ~ U[-1,1)^Dv per slab) -- the closed-form check O = c (P13)."""
    n, inner = _slabs(shape, lead)
    ids = _slab_ids(n, slab_range, slabs)
    out = np.empty((len(ids),) + tuple(inner), dtype=np.float32)
    for j, i in enumerate(ids):
        c = _rng(seed, "v", i).random((inner[-1],), dtype=np.float32) * 2 - 1
        out[j] = np.broadcast_to(c, tuple(inner))
    t = _to(out, dtype)
    return t.reshape(tuple(shape)) if slab_range is None and slabs is None else t


def _pm1_keys(k_shape, seed):
    B, Hkv, Sk, D = k_shape
    k = np.empty(k_shape, dtype=np.float32)
    for i in range(B * Hkv):
        r = _rng(seed, "k", i)
        k.reshape(B * Hkv, Sk, D)[i] = np.where(r.random((Sk, D)) < 0.5, -1.0, 1.0)
    return k


def _interval_of(interval, b, Sq):
    if interval is None:
        return None
    import inspect
    if len(inspect.signature(interval).parameters) >= 2:
        return interval(np.arange(Sq), b)
    return interval(np.arange(Sq))


def needle(q_shape, k_shape, *, seed=0, dtype=torch.bfloat16, interval=None, sq_sk=None):
    """Peaked inputs: K in {+-1}^D; Q[b,h,q] = K[b,h_kv,pi(q)] with pi(q) drawn
    uniformly from the admissible keys [lo(q), hi(q)) of row q.

    ``interval(q[, b]) -> (lo, hi)`` gives the admissible key range of the rows of
    batch b (None = all keys).  Shapes are [B,H,S,D]; GQA groups copy from their
    shared KV head."""
    B, Hq, Sq, D = q_shape
    _, Hkv, Sk, _ = k_shape
    k = _pm1_keys(k_shape, seed)
    q = np.empty(q_shape, dtype=np.float32)
    grp = Hq // Hkv
    for b in range(B):
        iv = _interval_of(interval, b, Sq)
        if iv is None:
            lo = np.zeros(Sq, dtype=np.int64)
            hi = np.full(Sq, Sk, dtype=np.int64)
        else:
            lo, hi = (np.asarray(a, dtype=np.int64) for a in iv)
        hi = np.maximum(hi, lo + 1)
        for h in range(Hq):
            r = _rng(seed, "q", b * Hq + h)
            u = r.random(Sq)
            pick = np.clip(lo + np.floor(u * (hi - lo)).astype(np.int64), 0, Sk - 1)
            q[b, h] = k[b, h // grp][pick]
    return _to(q, dtype), _to(k, dtype)


def needle_at(q_shape, k_shape, pick, *, seed=0, dtype=torch.bfloat16):
    """Needle inputs with an explicit key per row: K in {+-1}^D, Q[b,h,q] = K[b,h_kv,pick[q]]
    (pick clipped to [0, S_k)).  With pick just outside a row's admissible keys ("leak"
    inputs) a mask that admits one key too many is dominated by that key."""
    B, Hq, Sq, D = q_shape
    _, Hkv, Sk, _ = k_shape
    k = _pm1_keys(k_shape, seed)
    pick = np.clip(np.asarray(pick, dtype=np.int64), 0, Sk - 1)
    q = np.empty(q_shape, dtype=np.float32)
    grp = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            q[b, h] = k[b, h // grp][pick]
    return _to(q, dtype), _to(k, dtype)


def block_constant_v(shape, *, blk=128, seed=0, dtype=torch.bfloat16, lead=2):
    """V[..., k, :] = c_(slab, k // blk), one c ~ U[-1,1)^Dv per key block: O is the mixture of
    the block vectors weighted by each block's softmax mass, so a wrong block list or a wrong
    K/V tile moves it by O(1) while the normalisation is pinned as for constant V."""
    n, inner = _slabs(shape, lead)
    S, Dv = inner[-2], inner[-1]
    nb = (S + blk - 1) // blk
    out = np.empty((n,) + tuple(inner), dtype=np.float32)
    for i in range(n):
        c = _rng(seed, "v", i).random((nb, Dv), dtype=np.float32) * 2 - 1
        out[i] = np.repeat(c, blk, axis=0)[:S]
    return _to(out, dtype).reshape(tuple(shape))


def doc_offsets(B, S, n_docs=12, *, seed=1) -> np.ndarray:
    """[B, n_docs+1] int32: 0 = off[0] < ... < off[n_docs] = S; cut points
    uniform on (1, S-1) per batch b, drawn from stream (seed, b) (reading G6)."""
    out = np.zeros((B, n_docs + 1), dtype=np.int32)
    for b in range(B):
        r = _rng(seed, "doc", b)
        cuts = np.sort(r.choice(np.arange(1, S), size=n_docs - 1, replace=False))
        out[b, 1:-1] = cuts
        out[b, -1] = S
    return out


def alibi_slopes(H: int) -> np.ndarray:
    """Geometric schedule 2^(-8(h+1)/H), h 0-based (reading G2)."""
    return np.array([2.0 ** (-8.0 * (h + 1) / H) for h in range(H)], dtype=np.float32)


def clustered_qk(q_shape, k_shape, *, seed=2, blk=128, n_clusters=32, dtype=torch.bfloat16, b_range=None,
                 kv_head_range=None):
    """RSA inputs: per slab 32 centroids in {+-0.6}^D; each KV block / q block
    draws a cluster and its rows are clip(c_z + 0.4 U[-1,1), +-1).

    Shapes are the GLOBAL [B,H,S,D]; b_range=(b0, b1) returns only batches
    [b0, b1) and kv_head_range=(g0, g1) only KV heads [g0, g1) with their query
    heads (identical to that slice of the full tensors: streams are keyed by
    the global batch and head indices)."""
    b0, b1 = (0, q_shape[0]) if b_range is None else b_range
    grp = q_shape[1] // k_shape[1]
    g0, g1 = (0, k_shape[1]) if kv_head_range is None else kv_head_range

    def one(shape, tensor, heads_per_centroid_slab):
        _, H, S, D = shape
        h0, h1 = g0 * heads_per_centroid_slab, g1 * heads_per_centroid_slab
        out = np.empty((b1 - b0, h1 - h0, S, D), dtype=np.float32)
        nb = (S + blk - 1) // blk
        for b in range(b0, b1):
            for h in range(h0, h1):
                r = _rng(seed, tensor, b * H + h)
                cr = _rng(seed + 1000, "k", b * (H // heads_per_centroid_slab) + h // heads_per_centroid_slab)
                cents = np.where(cr.random((n_clusters, D)) < 0.5, -0.6, 0.6).astype(np.float32)
                z = r.integers(0, n_clusters, size=nb)
                x = cents[np.repeat(z, blk)[:S]]
                x += 0.4 * (r.random((S, D), dtype=np.float32) * 2 - 1)
                np.clip(x, -1.0, 1.0, out=out[b - b0, h - h0])
        return _to(out, dtype)
    return one(q_shape, "q", grp), one(k_shape, "k", 1)


def gate_logits(shape, *, seed=0, dtype=torch.bfloat16, lead=2, slab_range=None):
    return uniform(shape, seed=seed, tensor="gate", dtype=dtype, lo=-4.0, hi=4.0, lead=lead, slab_range=slab_range)


def pair_bias(shape, *, seed=0, dtype=torch.bfloat16, lead=2, slab_range=None):
    return uniform(shape, seed=seed, tensor="bias", dtype=dtype, lo=-4.0, hi=4.0, lead=lead, slab_range=slab_range)


def key_mask(shape, *, seed=0, p_zero=0.1, lead=1):
    n, inner = _slabs(shape, lead)
    out = np.empty((n,) + tuple(inner), dtype=np.uint8)
    for i in range(n):
        out[i] = (_rng(seed, "key_mask", i).random(tuple(inner)) >= p_zero).astype(np.uint8)
    return torch.from_numpy(out.reshape(shape))



def ipa_inputs(N, H=12, c=16, Pq=4, Pv=8, cz=128, seed=0, dtype=torch.bfloat16):
    """Invariant Point Attention inputs (reading G23; AF2 Alg.22 after its projections), protein-like:
    frames with uniformly random rotations (normalised random quaternions) and translations on a centred
    random walk of 3.8 A steps (C-alpha spacing); q, k, v, local points, pair bias and pair features
    U(-1, 1) (points x 4 A); per-head gamma in (0.1, 1.1).  Random numbers only -- the method's arithmetic
    lives in the kernels and the oracle.  Values are rounded to `dtype` (frames stay f32)."""
    g = torch.Generator().manual_seed(seed)
    u = lambda *s: torch.rand(*s, generator=g, dtype=torch.float64) * 2 - 1
    quat = torch.randn(N, 4, generator=g, dtype=torch.float64)
    quat = quat / quat.norm(dim=1, keepdim=True)
    a, b, cc, d = quat.unbind(1)
    R = torch.stack([
        torch.stack([a * a + b * b - cc * cc - d * d, 2 * (b * cc - a * d), 2 * (b * d + a * cc)], -1),
        torch.stack([2 * (b * cc + a * d), a * a - b * b + cc * cc - d * d, 2 * (cc * d - a * b)], -1),
        torch.stack([2 * (b * d - a * cc), 2 * (cc * d + a * b), a * a - b * b - cc * cc + d * d], -1)], 1)
    step = torch.randn(N, 3, generator=g, dtype=torch.float64)
    step = 3.8 * step / step.norm(dim=1, keepdim=True)
    t = torch.cumsum(step, 0)
    t = t - t.mean(0)
    out = dict(q=u(N, H, c), k=u(N, H, c), v=u(N, H, c), qp=4 * u(N, H, Pq, 3), kp=4 * u(N, H, Pq, 3),
               vp=4 * u(N, H, Pv, 3), bias=u(H, N, N), z=u(N, N, cz),
               gamma=0.1 + torch.rand(H, generator=g, dtype=torch.float64))
    out = {k_: v_.to(dtype) for k_, v_ in out.items()}
    out["gamma"] = out["gamma"].float()
    out["R"], out["t"] = R.float(), t.float()
    return out
