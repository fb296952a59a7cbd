#!/usr/bin/env python
"""Benchmark of the fused attention-variant forward (Flashlight, arXiv 2511.02043) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant flex|causal|...|rsa|rsa_decode]
                    [--impl ours|reference]

One "step" = one pass of the whole hot path over one batch of synthetic inputs.
Default workload (``--variant flex``) = BASELINE.json configs[1], the
FlexAttention-expressible variants at bf16 B=8 H=16 S=8192 D=128: one step runs
causal, ALiBi, sliding window 1024, softcap 20 and a 12-document mask, one
``fl_attn_fwd`` call each, on the same resident Q/K/V.  ``value`` = useful
TFLOP/s of the step (SURVEY §8(d) accounting), per-variant numbers are in
``per_call``.  Other workloads: ``diff`` (configs[2]), ``evo_row`` / ``evo_col``
(configs[3]), ``rsa`` / ``rsa_decode`` (configs[4]), and each single variant.

Under torchrun each rank runs the same per-GPU workload on its own slice of a
global batch of B*N (batch x head sharding, no collective on the data path:
weak scaling); time is max over ranks of CUDA-event time; rank 0 prints ONE JSON
line.  ``--impl reference`` times this tier's reference arm, the fp64 CPU oracle,
on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2511_02043_b200 import synth  # noqa: E402

METRIC = "attention fwd TFLOP/s per variant and % of B200 bf16 tensor peak at 1/2/4/8 GPUs"

# ------------------------------------------------------------------ workloads (BASELINE.json configs)
C2 = dict(B=8, H=16, S=8192, D=128)
VARIANTS = {
    # configs[1]: FlexAttention-expressible variants, bf16 B=8 H=16 S=8192 D=128
    "causal": dict(C2, mask="causal"),
    "alibi": dict(C2, mod="alibi"),
    "sliding": dict(C2, mask="sliding", window=1024),
    "softcap": dict(C2, mod="softcap", softcap=20.0),
    "document": dict(C2, mask="document", n_docs=12),
    "vanilla": dict(C2),
    "prefix": dict(C2, mask="prefix", prefix=256),
    "gqa": dict(C2, Hkv=2, mask="causal"),
    # the backward (dQ, dK, dV) of the configs[1] shape, not a BASELINE line
    "bwd_causal": dict(C2, mask="causal", bwd=True),
    "bwd_vanilla": dict(C2, bwd=True),
    # configs[0]: vanilla causal softmax attention fp32 B=1 H=1 S=128 D=64 (exact SIMT path, launch-latency bound)
    "c1": dict(B=1, H=1, S=128, D=64, mask="causal", dtype="f32"),
    # configs[2]: differential attention bf16 B=8 H=16 S=8192 D=64 (two maps, lambda)
    "diff": dict(B=8, H=16, S=8192, D=64, diff=True, lam=0.2),
    "bwd_diff": dict(B=8, H=16, S=8192, D=64, diff=True, lam=0.2, bwd=True),   # NEXT-3 for configs[2]
    # configs[3]: Evoformer gated self-attention with pair bias, N_seq=512 N_res=384 H=8 c=32
    "evo_row": dict(evo="row", B=1, Ns=512, Nr=384, H=8, D=32),
    "evo_col": dict(evo="col", B=1, Ns=512, Nr=384, H=8, D=32),
    # configs[4]: Rectified Sparse Attention B=4 H=32 S=32768 D=128 (blocks 128, top-16 + sink + diagonal)
    "rsa": dict(rsa="prefill", B=4, H=32, S=32768, D=128, topk=16),
    "rsa_decode": dict(rsa="decode", B=4, H=32, S=32768, D=128, topk=16),
    # SURVEY §8(f) NEXT-2 / NEXT-4 (not BASELINE lines): the whole Evoformer row-attention block (AF2 Alg.7)
    # chained from this package's kernels, and the Invariant Point Attention core (12 heads x 16)
    "evo_block": dict(special="evo_block", Ns=512, Nr=384),
    "ipa": dict(special="ipa", N=384),
}
SUITES = {"flex": ["causal", "alibi", "sliding", "softcap", "document"]}
VARIANT_KW = ("mod", "softcap", "mask", "window", "prefix", "diff", "lam")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ useful-work accounting
def kept_pairs(cfg, doc_offsets=None, key_mask=None):
    """Exact number of kept (q,k) pairs of the whole per-rank workload (per softmax map)."""
    if cfg.get("evo"):
        Nr, Ns, H = cfg["Nr"], cfg["Ns"], cfg["H"]
        km = key_mask.numpy().astype(np.int64)          # [B, Ns, Nr]
        return int(km.sum() * (Nr if cfg["evo"] == "row" else Ns) * H)
    S = cfg["S"]
    q = np.arange(S, dtype=np.int64)
    mask = cfg.get("mask", "none")
    if mask == "causal":
        per = (q + 1).sum()
    elif mask == "sliding":
        per = (np.minimum(q, cfg["window"]) + 1).sum()
    elif mask == "prefix":
        per = np.maximum(cfg["prefix"], q + 1).clip(max=S).sum()
    elif mask == "document":
        tot = 0
        for o in doc_offsets:
            ln = np.diff(o.astype(np.int64))
            tot += int((ln * ln).sum())
        return tot * cfg["H"]
    else:
        per = S * S
    return int(per) * cfg["B"] * cfg["H"]


def rsa_pairs(blk_idx, blk_cnt, Sk, Sq, blk=128):
    """Exact kept pairs of block lists (reading G10): row q keeps the keys of every listed
    block that are <= q_abs = q + Sk - Sq.  blk_idx [BH, nqb, max_sel] (-1 padded),
    blk_cnt [BH, nqb]."""
    idx = np.asarray(blk_idx).astype(np.int64)
    cnt = np.asarray(blk_cnt).astype(np.int64)
    BH, nqb, ms = idx.shape
    valid = np.arange(ms)[None, :] < cnt[:, :, None]                     # [BH, nqb, ms]
    tot = 0
    for i in range(nqb):
        rows = np.arange(i * blk, min(Sq, (i + 1) * blk), dtype=np.int64)
        qa = rows + (Sk - Sq)                                            # [R]
        j0 = idx[:, i, :] * blk                                          # [BH, ms]
        width = np.minimum(blk, Sk - j0)
        kept = np.clip(qa[None, None, :] + 1 - j0[:, :, None], 0, width[:, :, None])   # [BH, ms, R]
        tot += int((kept.sum(-1) * valid[:, i, :]).sum())
    return tot


def row_interval(cfg, q, offs_b=None):
    """Admissible keys [lo, hi) of rows q (numpy) for the interval masks (readings G4-G6, Sq = Sk)."""
    S = cfg["S"]
    mask = cfg.get("mask", "none")
    if mask == "causal":
        return np.zeros_like(q), q + 1
    if mask == "sliding":
        return np.maximum(q - cfg["window"], 0), q + 1
    if mask == "prefix":
        return np.zeros_like(q), np.minimum(np.maximum(cfg["prefix"], q + 1), S)
    if mask == "document":
        j = np.searchsorted(offs_b, q, side="right") - 1
        return offs_b[j], offs_b[j + 1]
    return np.zeros_like(q), np.full_like(q, S)


def executed_pairs(cfg, doc_offsets=None, rows_per_tile=128, blk=128):
    """(q, k) pairs of every 128 x 128 tile the kernel executes (masked pairs inside partial tiles
    included): a 128-row query tile runs the key tiles of the union of its rows' intervals."""
    S, B, H = cfg["S"], cfg["B"], cfg["H"]
    q0 = np.arange(0, S, rows_per_tile)
    q1 = np.minimum(q0 + rows_per_tile, S) - 1
    tot = 0
    for b in range(B if cfg.get("mask") == "document" else 1):
        ob = doc_offsets[b] if doc_offsets is not None else None
        lo0, hi0 = row_interval(cfg, q0, ob)
        lo1, hi1 = row_interval(cfg, q1, ob)
        lo, hi = np.minimum(lo0, lo1), np.maximum(hi0, hi1)
        tiles = np.where(hi > lo, (hi + blk - 1) // blk - lo // blk, 0)
        tot += int(tiles.sum()) * rows_per_tile * blk
    return tot * H * (1 if cfg.get("mask") == "document" else B)


def flops_per_pair(cfg):
    return 4 * cfg["D"] * (2 if cfg.get("diff") else 1)


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return False
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            out = ""
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda x: x.replace(".", "").isdigit()
        sm = [float(r[0]) for r in self.rows if num(r[0])]
        mx = [float(r[1]) for r in self.rows if num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ input construction (rank's shard)
# Strong scaling: the BASELINE config is ONE fixed problem; its independent units are split
# across the ranks by fl_shard_range (shard.py): h-major (h, b) units for the LLM configs (GQA: KV-head
# groups), MSA rows s for Evoformer rows, residue columns i for Evoformer columns.  Every rank regenerates
# exactly its slabs of the global seeded tensors (synth streams are keyed by the global slab index), so the
# gathered per-rank outputs equal the single-process output bit for bit (P10).
def dense_blocks(cfg, rank, world):
    """(g0, g1, b0, b1) rectangles of this rank's units: outer = KV-head groups (= heads for MHA and
    differential attention), inner = batch."""
    if world == 1:
        return [(0, cfg.get("Hkv", cfg["H"]), 0, cfg["B"])]
    from paper_2511_02043_b200 import shard
    return shard.unit_blocks(cfg.get("Hkv", cfg["H"]), cfg["B"], world, rank)


def dense_block_inputs(cfg, blk, seed=0):
    """Host q, k, v of one block (g0, g1, b0, b1): q [nb, maps*nh, S, D] with map m's heads at
    [m*nh, (m+1)*nh) (differential attention, G8), k [nb, maps*ng, S, D], v [nb, ng, S, D]."""
    B, H, S, D = cfg["B"], cfg["H"], cfg["S"], cfg["D"]
    Hkv = cfg.get("Hkv", H)
    grp = H // Hkv
    maps = 2 if cfg.get("diff") else 1
    g0, g1, b0, b1 = blk
    h0, h1 = g0 * grp, g1 * grp

    def gen(t, heads, lo, hi, mp):
        ids = [b * heads * mp + m * heads + h for b in range(b0, b1) for m in range(mp) for h in range(lo, hi)]
        return synth.uniform((B, heads * mp, S, D), seed=seed, tensor=t, slabs=ids,
                             dtype=torch.float32 if cfg.get("dtype") == "f32" else torch.bfloat16).reshape(
            b1 - b0, (hi - lo) * mp, S, D)
    return {"q": gen("q", H, h0, h1, maps), "k": gen("k", Hkv, g0, g1, maps), "v": gen("v", Hkv, g0, g1, 1)}


def block_cfg(cfg, blk):
    g0, g1, b0, b1 = blk
    grp = cfg["H"] // cfg.get("Hkv", cfg["H"])
    out = dict(cfg, B=b1 - b0, H=(g1 - g0) * grp)
    if "Hkv" in cfg:
        out["Hkv"] = g1 - g0
    return out


def dense_inputs(cfg, rank, world, seed=0):
    """[(block, host tensors)] of this rank's shard."""
    return [(blk, dense_block_inputs(cfg, blk, seed)) for blk in dense_blocks(cfg, rank, world)]


def doc_offsets_for(cfg, b0, b1):
    return synth.doc_offsets(cfg["B"], cfg["S"], cfg["n_docs"], seed=1)[b0:b1]


def block_variant_kw(cfg, blk):
    """Variant keywords of one block: per-head parameters are the GLOBAL heads' (ALiBi slopes of
    heads h0..h1 of H, G2), document offsets the block's batches (G6)."""
    kw = {x: cfg[x] for x in VARIANT_KW if x in cfg}
    g0, g1, b0, b1 = blk
    grp = cfg["H"] // cfg.get("Hkv", cfg["H"])
    if cfg.get("mod") == "alibi":
        kw["alibi_slopes"] = synth.alibi_slopes(cfg["H"])[g0 * grp:g1 * grp]
    offs = doc_offsets_for(cfg, b0, b1) if cfg.get("mask") == "document" else None
    if offs is not None:
        kw["doc_offsets"] = offs
    return kw, offs


def evo_range(cfg, rank, world):
    """MSA rows s (row attention) or residue columns i (column attention) of this rank."""
    n = cfg["Ns"] if cfg["evo"] == "row" else cfg["Nr"]
    if world == 1:
        return 0, n
    from paper_2511_02043_b200 import shard
    return shard.range_1d(n, world, rank)


def evo_inputs(cfg, rank, world, seed=0):
    """MSA storage [B, N_seq, N_res, H, c] of this rank's rows (row attention: Q[:, s0:s1]) or columns
    (column attention: Q[:, :, i0:i1]); the pair bias [B, H, N_res, N_res] is replicated."""
    B, Ns, Nr, H, c = cfg["B"], cfg["Ns"], cfg["Nr"], cfg["H"], cfg["D"]
    u0, u1 = evo_range(cfg, rank, world)
    if cfg["evo"] == "row":
        ids = [(b * Ns + s) * Nr + i for b in range(B) for s in range(u0, u1) for i in range(Nr)]
        shp = (B, u1 - u0, Nr, H, c)
    else:
        ids = [(b * Ns + s) * Nr + i for b in range(B) for s in range(Ns) for i in range(u0, u1)]
        shp = (B, Ns, u1 - u0, H, c)
    st = lambda t, **kw: synth.uniform((B, Ns, Nr, H, c), seed=seed, tensor=t, lead=3, slabs=ids,
                                       **kw).reshape(shp)
    host = {"Q": st("q"), "K": st("k"), "V": st("v"), "G": st("gate", lo=-4.0, hi=4.0),
            "km": torch.ones(shp[:3], dtype=torch.uint8)}      # all-ones MSA mask (tests use 10 % zeros)
    if cfg["evo"] == "row":
        host["pb"] = synth.pair_bias((B, H, Nr, Nr), seed=seed, lead=2)
    return host


def evo_views(cfg, t):
    """[B,G,H,S,D] views of MSA storage [B, N_seq, N_res, H, c] (reading G9); no copies."""
    B, H = cfg["B"], cfg["H"]
    view = (lambda x: x.permute(0, 1, 3, 2, 4)) if cfg["evo"] == "row" else (lambda x: x.permute(0, 2, 3, 1, 4))
    q, k, v = view(t["Q"]), view(t["K"]), view(t["V"])
    kw = dict(gate_mode="sigmoid", gate=view(t["G"]))
    if cfg["evo"] == "row":
        Gl, Nr = t["Q"].shape[1], t["Q"].shape[2]
        kw["bias"] = t["pb"].unsqueeze(1).expand(B, Gl, H, Nr, Nr)
        kw["key_mask"] = t["km"]
    else:
        kw["key_mask"] = t["km"].permute(0, 2, 1)
    return q, k, v, kw


# ------------------------------------------------------------------ jobs: the calls of one step
class Call:
    def __init__(self, label, fn, flops=0.0, bytes_=0.0, bound="tensor", kernel=None, alu=0.0, exec_flops=0.0):
        self.label, self.fn, self.flops, self.bytes, self.bound = label, fn, flops, bytes_, bound
        self.exec_flops = exec_flops   # flops of every executed 128 x 128 tile (masked pairs included)
        self.alu = alu            # MUFU ex2 operations per launch (bound == "alu")
        self.kernel = kernel or label
        self.ms = []


class Job:
    """What one step runs on this rank: `calls` (device-resident inputs), the useful
    flops of the step, an end-to-end closure over host buffers, and the oracle-timing
    closure for cpu_baseline."""

    def __init__(self, name, workload):
        self.name, self.workload = name, workload
        self.calls = []
        self.step_flops = 0.0
        self.e2e = None           # (fn, h2d_bytes, d2h_bytes)
        self.oracle = None        # fn(budget_s) -> (tflops, threads, sample, secs)
        self.extra = {}
        self.parity = {}          # host inputs / outputs / oracle kwargs for the full-size parity tests
        self.parity_result = {}   # per variant: GPU output vs the oracle on the cpu_baseline leg's rows
        self.units = ""           # this rank's shard, for the JSON line
        self.outputs = []         # (block, device output) of this rank's shard


def _dev_kw(kw, device):
    out = dict(kw)
    for x in ("doc_offsets", "alibi_slopes"):
        if x in out:
            out[x] = torch.as_tensor(out[x]).to(device)
    return out


def dense_job(names, rank, world, device, with_host=True):
    from paper_2511_02043_b200 import fl
    cfg0 = VARIANTS[names[0]]
    wl = names[0] if len(names) == 1 else "flexattention_variants(" + ",".join(names) + ")"
    job = Job(names[0] if len(names) == 1 else "flex",
              f"{wl}_{cfg0.get('dtype', 'bf16')}_B{cfg0['B']}_H{cfg0['H']}_S{cfg0['S']}_D{cfg0['D']}")
    maps = 2 if cfg0.get("diff") else 1
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=device)       # scheduler counter + packed key mask
    blocks = []                                                       # (blk, host, q, k, v, out)
    for blk, host in dense_inputs(cfg0, rank, world):
        q, k, v = (host[n].to(device) for n in ("q", "k", "v"))
        out = torch.empty(q.shape[0], q.shape[1] // maps, q.shape[2], v.shape[3], dtype=q.dtype, device=device)
        blocks.append((blk, host, q, k, v, out))
    job.units = "(kv-group, b) units " + ";".join(f"g[{g0},{g1})xb[{b0},{b1})" for (g0, g1, b0, b1), *_ in blocks)
    okws, pairs_by = {}, {}
    for n in names:
        cfg = VARIANTS[n]
        assert all(cfg[x] == cfg0[x] for x in ("B", "H", "S", "D")) and cfg.get("Hkv") == cfg0.get("Hkv")
        flops, eflops, nbytes, fns = 0.0, 0.0, 0, []
        for blk, host, q, k, v, out in blocks:
            kw, offs = block_variant_kw(cfg, blk)
            flops += kept_pairs(block_cfg(cfg, blk), offs) * flops_per_pair(cfg)
            if cfg.get("dtype") != "f32":                # 128 x 128 tiles of the tcgen05 kernel
                eflops += executed_pairs(block_cfg(cfg, blk), offs) * flops_per_pair(cfg)
            nbytes += sum(t.numel() * t.element_size() for t in (q, k, v, out))
            dkw = _dev_kw(kw, device)
            fns.append(lambda q=q, k=k, v=v, out=out, dkw=dkw: fl.attn_fwd(q, k, v, out=out, workspace=ws, **dkw))
            okws.setdefault(n, kw)
        f32 = cfg.get("dtype") == "f32"
        if cfg.get("bwd"):
            # backward: O, LSE and dO resident; useful flops = 2.5 x the forward's (dV, dP, dS->dQ, dK and the
            # recomputed S: the usual FlashAttention accounting); the dQ pass also recomputes S and dP
            bfns = []
            for (blk, host, q, k, v, out), f in zip(blocks, fns):
                kw_b, _ = block_variant_kw(cfg, blk)
                dkw = _dev_kw(kw_b, device)
                if cfg.get("diff"):     # the diff backward recomputes both maps' outputs and LSEs itself
                    o_b, lse_b = fl.attn_fwd(q, k, v, **dkw), None
                else:
                    o_b, lse_b = fl.attn_fwd(q, k, v, return_lse=True, **dkw)
                do_b = torch.empty_like(o_b).uniform_(-1, 1)
                g = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))
                wsb = torch.empty(fl.attn_bwd_workspace_bytes(q, k, v, o_b, lse_b, do_b, **dkw), dtype=torch.uint8,
                                  device=device)
                bfns.append(lambda q=q, k=k, v=v, o_b=o_b, lse_b=lse_b, do_b=do_b, g=g, dkw=dkw, wsb=wsb:
                            fl.attn_bwd(q, k, v, o_b, lse_b, do_b, dq=g[0], dk=g[1], dv=g[2], workspace=wsb, **dkw))
            flops *= 2.5
            job.calls.append(Call(n, (lambda fns=bfns: [f() for f in fns]), flops, nbytes, "tensor",
                                  kernel="bwd_dkdv_kernel"))
            job.step_flops += flops
            pairs_by[n] = flops / flops_per_pair(cfg)
            continue
        job.calls.append(Call(n, (lambda fns=fns: [f() for f in fns]), flops, nbytes, "latency" if f32 else "tensor",
                              kernel="attn_simt_kernel" if f32 else "attn_tc_kernel", exec_flops=eflops))
        job.step_flops += flops
        pairs_by[n] = flops / flops_per_pair(cfg)
    blk0, host0, *_, out0 = blocks[0]
    job.parity = {"host": host0, "out": out0, "oracle_kw": okws}
    job.outputs = [(blk, out) for blk, _, _, _, _, out in blocks]

    if with_host:
        runner = fl.HostRunner(device)
        legs = []
        for blk, host, q, k, v, out in blocks:
            hq, hk, hv = (host[n].pin_memory() for n in ("q", "k", "v"))
            hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
            legs.append((blk, hq, hk, hv, hout))

        def e2e_step(stream):
            for n in names:
                for blk, hq, hk, hv, hout in legs:
                    runner(hq, hk, hv, hout, stream=stream, **block_variant_kw(VARIANTS[n], blk)[0])
        h2d = sum(t.numel() * t.element_size() for _, hq, hk, hv, _ in legs for t in (hq, hk, hv))
        d2h = sum(hout.numel() * hout.element_size() for *_, hout in legs)
        job.e2e = (e2e_step, h2d * len(names), d2h * len(names))

    def oracle_fn(budget_s):
        import oracle
        bcfg = block_cfg(cfg0, blk0)
        total_rows = bcfg["B"] * bcfg["H"] * cfg0["S"]
        per_budget = budget_s / len(names)
        tot_flops, tot_s, n_rows = 0.0, 0.0, 0
        for n in names:
            cfg = VARIANTS[n]
            ok = okws[n]
            bpairs = kept_pairs(block_cfg(cfg, blk0), ok.get("doc_offsets"))
            rows = np.linspace(0, total_rows - 1, 64).astype(np.int64)
            t0 = time.perf_counter()
            oracle.attn(host0["q"], host0["k"], host0["v"], rows=rows, **ok)
            dt = time.perf_counter() - t0
            nr = int(min(total_rows, max(64, 64 * per_budget / max(dt, 1e-3))))
            rows = np.linspace(0, total_rows - 1, nr).astype(np.int64)
            t0 = time.perf_counter()
            ref, _ = oracle.attn(host0["q"], host0["k"], host0["v"], rows=rows, **ok)
            dt = time.perf_counter() - t0
            if (rank == 0 and torch.device(device).type == "cuda" and not cfg.get("bwd")
                    and out0.numel() // out0.shape[-1] == total_rows):
                # the same rows of this variant's GPU output at full size, re-run once outside the timing
                next(c for c in job.calls if c.label == n).fn()
                torch.cuda.synchronize()
                D = out0.shape[-1]
                got = out0.reshape(-1, D)[torch.as_tensor(rows, device=out0.device)].double().cpu().numpy()
                err, tol = float(np.abs(got - ref).max()), 1e-5 if cfg.get("dtype") == "f32" else 2e-2
                job.parity_result[n] = {"rows": int(nr), "max_abs": err, "max_ref": float(np.abs(ref).max()),
                                        "tol": tol, "ok": err <= tol}
            tot_flops += bpairs * flops_per_pair(cfg) * (nr / total_rows)
            tot_s += dt
            n_rows += nr
        return (tot_flops / tot_s / 1e12, oracle.num_threads(),
                f"{n_rows} evenly spaced output rows over {len(names)} variant(s) of {total_rows} rows each; "
                "useful flops scaled by row share", tot_s)
    job.oracle = oracle_fn
    return job


def evo_job(name, rank, world, device, with_host=True):
    from paper_2511_02043_b200 import fl
    cfg = VARIANTS[name]
    host = evo_inputs(cfg, rank, world)
    dev = {n: t.to(device) for n, t in host.items()}
    q, k, v, kw = evo_views(cfg, dev)
    out = torch.empty(q.shape, dtype=q.dtype, device=device)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=device)
    pairs = kept_pairs(cfg, key_mask=host["km"])
    flops = pairs * flops_per_pair(cfg)
    nbytes = sum(t.numel() * t.element_size() for t in dev.values()) + out.numel() * 2
    job = Job(name, f"evoformer_{cfg['evo']}_bf16_Nseq{cfg['Ns']}_Nres{cfg['Nr']}_H{cfg['H']}_c{cfg['D']}")
    u0, u1 = evo_range(cfg, rank, world)
    job.units = f"{'MSA rows s' if cfg['evo'] == 'row' else 'residue columns i'} [{u0},{u1})"
    # c = 32: one ex2 per kept pair against 4c = 128 MMA flops, so the MUFU (16 ex2/clk/SM), not the
    # tensor pipe, bounds the kernel (MUFU 187/250 us vs tensor 47/62 us vs HBM 77 us)
    job.calls.append(Call(name, lambda: fl.attn_fwd(q, k, v, out=out, workspace=ws, **kw), flops, nbytes, "alu",
                          kernel="attn_tc_kernel", alu=float(pairs)))
    job.step_flops = flops
    job.parity = {"host": host, "out": out}
    job.outputs = [((u0, u1), out)]

    if with_host:
        pin = {n: t.pin_memory() for n, t in host.items()}
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()

        def e2e_step(stream):
            # the user's call: pinned MSA storage -> device, fused attention on the strided views, O -> host
            with torch.cuda.stream(stream):
                for n, t in pin.items():
                    dev[n].copy_(t, non_blocking=True)
                fl.attn_fwd(q, k, v, out=out, workspace=ws, **kw)
                hout.copy_(out, non_blocking=True)
        job.e2e = (e2e_step, sum(t.numel() * t.element_size() for t in pin.values()), hout.numel() * 2)

    def oracle_fn(budget_s):
        import oracle
        hq, hk, hv, okw = evo_views(cfg, host)
        total_rows = hq.shape[0] * hq.shape[1] * hq.shape[2] * hq.shape[3]
        rows = np.linspace(0, total_rows - 1, 256).astype(np.int64)
        t0 = time.perf_counter()
        oracle.attn(hq, hk, hv, rows=rows, **okw)
        dt = time.perf_counter() - t0
        nr = int(min(total_rows, max(256, 256 * budget_s / max(dt, 1e-3))))
        rows = np.linspace(0, total_rows - 1, nr).astype(np.int64)
        t0 = time.perf_counter()
        ref, _ = oracle.attn(hq, hk, hv, rows=rows, **okw)
        dt = time.perf_counter() - t0
        if rank == 0 and torch.device(device).type == "cuda":
            job.calls[0].fn()
            torch.cuda.synchronize()
            got = out.reshape(-1, out.shape[-1])[torch.as_tensor(rows, device=out.device)].double().cpu().numpy()
            err = float(np.abs(got - ref).max())
            job.parity_result[name] = {"rows": int(nr), "max_abs": err, "max_ref": float(np.abs(ref).max()),
                                       "tol": 2e-2, "ok": err <= 2e-2}
        return (flops * nr / total_rows / dt / 1e12, oracle.num_threads(),
                f"{nr} of {total_rows} output rows (evenly spaced), useful flops scaled by row share", dt)
    job.oracle = oracle_fn
    return job


def rsa_block_inputs(cfg, blk):
    """Clustered Q/K (G10 recipe) and uniform V of one (h, b) block; decode keeps the last query."""
    B, H, S, D = cfg["B"], cfg["H"], cfg["S"], cfg["D"]
    h0, h1, b0, b1 = blk
    qh, kh = synth.clustered_qk((B, H, S, D), (B, H, S, D), seed=2, b_range=(b0, b1), kv_head_range=(h0, h1))
    ids = [b * H + h for b in range(b0, b1) for h in range(h0, h1)]
    vh = synth.uniform((B, H, S, D), seed=0, tensor="v", slabs=ids).reshape(b1 - b0, h1 - h0, S, D)
    if cfg["rsa"] == "decode":
        qh = qh[:, :, S - 1:].contiguous()
    return qh, kh, vh


def rsa_job(name, rank, world, device, with_host=True):
    """configs[4]: RSA on B=4 H=32 S=32768 D=128.  prefill step = summaries + selection +
    block-sparse attention over all 32768 queries; decode step = selection + attention for
    one query per (b,h) at position S-1 (summaries are maintained at prefill)."""
    from paper_2511_02043_b200 import fl, shard
    cfg = VARIANTS[name]
    B, H, S, D, topk = cfg["B"], cfg["H"], cfg["S"], cfg["D"], cfg["topk"]
    decode = cfg["rsa"] == "decode"
    blocks = shard.unit_blocks(H, B, world, rank)
    job = Job(name, f"rsa_{cfg['rsa']}_bf16_B{B}_H{H}_S{S}_D{D}_top{topk}")
    job.units = "(h, b) units " + ";".join(f"h[{h0},{h1})xb[{b0},{b1})" for h0, h1, b0, b1 in blocks)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=device)
    legs = []
    flops = 0.0
    listed = 0
    sum_bytes = sel_bytes = att_bytes = sel_flops = 0.0
    for blk in blocks:
        qh, kh, vh = rsa_block_inputs(cfg, blk)
        Sq = qh.shape[2]
        q, k, v = qh.to(device), kh.to(device), vh.to(device)
        out = torch.empty(q.shape[0], q.shape[1], Sq, D, dtype=q.dtype, device=device)
        nqb = (Sq + 127) // 128
        kmin, kmax = fl.rsa_build_summaries(k, 128)
        idx, cnt = fl.rsa_select(q, kmin, kmax, S, topk=topk)
        torch.cuda.synchronize()
        flops += rsa_pairs(idx.cpu().numpy(), cnt.cpu().numpy(), S, Sq) * flops_per_pair(cfg)
        nl = int(cnt.sum().item())
        listed += nl
        nbh = q.shape[0] * q.shape[1]
        sum_bytes += k.numel() * 2 + 2 * kmin.numel() * 2
        sel_flops += 2.0 * 2 * D * 128 * 128 * sum(((i * 128 + 127 + S - Sq) // 128 + 127) // 128
                                                 for i in range(nqb)) * nbh     # executed GEMM tiles
        sel_bytes += q.numel() * 2 + 2 * kmin.numel() * 2 + idx.numel() * 4 + cnt.numel() * 4
        if decode:   # each listed KV block is read once per (b,h): K + V rows
            att_bytes += q.numel() * 2 + out.numel() * 2 + nl * 128 * D * 2 * 2
        else:        # K/V read once per (b,h) (a block listed by several q-blocks is re-read from L2)
            att_bytes += (q.numel() + k.numel() + v.numel() + out.numel()) * 2
        legs.append(dict(blk=blk, host=(qh, kh, vh), q=q, k=k, v=v, out=out, kmin=kmin, kmax=kmax, idx=idx, cnt=cnt))
    nkb = (S + 127) // 128
    if not decode:
        job.calls.append(Call("rsa_summaries", lambda: [fl.rsa_build_summaries(L["k"], 128, L["kmin"], L["kmax"])
                                                        for L in legs], 0.0, sum_bytes, "hbm",
                              kernel="rsa_summaries_kernel"))
    job.calls.append(Call("rsa_select", lambda: [fl.rsa_select(L["q"], L["kmin"], L["kmax"], S, topk=topk,
                                                               blk_idx=L["idx"], blk_cnt=L["cnt"]) for L in legs],
                          sel_flops, sel_bytes, "hbm" if decode else "tensor",
                          kernel="rsa_select_small_kernel" if decode else "rsa_select_kernel"))
    job.calls.append(Call("attn_blocklist", lambda: [fl.attn_fwd(L["q"], L["k"], L["v"], out=L["out"], mask="blocklist",
                                                                 blk_idx=L["idx"], blk_cnt=L["cnt"], workspace=ws)
                                                     for L in legs], flops, att_bytes,
                          "hbm" if decode else "tensor",
                          kernel="attn_decode_split_kernel" if decode else "attn_tc_kernel"))
    job.step_flops = flops
    L0 = legs[0]
    Sq = L0["q"].shape[2]
    job.extra.update(listed_blocks=listed, rsa_decode=decode)
    job.outputs = [(L["blk"], L["out"]) for L in legs]
    job.parity = {"host": dict(zip(("q", "k", "v"), L0["host"])), "out": L0["out"], "idx": L0["idx"], "cnt": L0["cnt"],
                  "kmin": L0["kmin"], "kmax": L0["kmax"], "Sq": Sq}

    if with_host:
        pins = [(L, tuple(t.pin_memory() for t in L["host"]), torch.empty(L["out"].shape, dtype=L["out"].dtype).pin_memory())
                for L in legs]

        def e2e_step(stream):
            with torch.cuda.stream(stream):
                for L, (hq, hk, hv), hout in pins:
                    L["q"].copy_(hq, non_blocking=True)
                    L["k"].copy_(hk, non_blocking=True)
                    L["v"].copy_(hv, non_blocking=True)
                    fl.rsa_build_summaries(L["k"], 128, L["kmin"], L["kmax"], stream=stream)
                    fl.rsa_select(L["q"], L["kmin"], L["kmax"], S, topk=topk, blk_idx=L["idx"], blk_cnt=L["cnt"],
                                  stream=stream)
                    fl.attn_fwd(L["q"], L["k"], L["v"], out=L["out"], mask="blocklist", blk_idx=L["idx"],
                                blk_cnt=L["cnt"], workspace=ws, stream=stream)
                    hout.copy_(L["out"], non_blocking=True)
        h2d = sum(t.numel() * 2 for _, ts, _ in pins for t in ts)
        job.e2e = (e2e_step, h2d, sum(h.numel() * 2 for *_, h in pins))

    qh, kh, vh = L0["host"]

    def oracle_fn(budget_s):
        return rsa_oracle_rate(cfg, qh[:1, :1], kh[:1, :1], vh[:1, :1], budget_s)
    job.oracle = oracle_fn
    return job


def rsa_oracle_rate(cfg, q1, k1, v1, budget_s):
    """The oracle's selection (in full) + attention (bounded row sample) on one (b, h) head, as a rate."""
    import oracle
    S, topk = cfg["S"], cfg["topk"]
    Sq = q1.shape[2]
    t0 = time.perf_counter()
    ri, rc, _ = oracle.rsa_select(q1, k1, topk=topk)
    t_sel = time.perf_counter() - t0
    nr = min(Sq, 64)
    rows = np.linspace(0, Sq - 1, nr).astype(np.int64)
    t0 = time.perf_counter()
    oracle.attn(q1, k1, v1, rows=rows, mask="blocklist", blk_idx=ri, blk_cnt=rc)
    dt = time.perf_counter() - t0
    nr = int(min(Sq, max(nr, nr * max(budget_s - t_sel, 1.0) / max(dt, 1e-3))))
    rows = np.linspace(0, Sq - 1, nr).astype(np.int64)
    t0 = time.perf_counter()
    oracle.attn(q1, k1, v1, rows=rows, mask="blocklist", blk_idx=ri, blk_cnt=rc)
    t_att = time.perf_counter() - t0
    t_head = t_sel + t_att * Sq / nr                  # one (b,h) in full
    return (rsa_pairs(ri, rc, S, Sq) * flops_per_pair(cfg) / t_head / 1e12, oracle.num_threads(),
            f"(b=0,h=0): oracle selection in full + {nr} of {Sq} attention rows; rate of that head", t_sel + t_att)


def special_job(variant, device):
    """NEXT-2 / NEXT-4 workloads (single GPU, not sharded): one call each, flops as in tools/paper_grid.py."""
    from paper_2511_02043_b200 import fl, synth
    cfg = VARIANTS[variant]
    if variant == "evo_block":
        from paper_2511_02043_b200 import evoformer
        H, c, cm, cz, Ns, Nr = 8, 32, 256, 128, cfg["Ns"], cfg["Nr"]
        w = evoformer.synthetic_weights(c_m=cm, c_z=cz, H=H, c=c, seed=1, device=device)
        m = (synth.uniform((Ns, Nr, cm), seed=2, tensor="q", lead=2) * 2).to(torch.bfloat16).to(device)
        z = (synth.uniform((Nr, Nr, cz), seed=2, tensor="k", lead=2) * 2).to(torch.bfloat16).to(device)
        blk = evoformer.RowAttnBlock(w, Ns, Nr, device=device)
        flops = 2 * Ns * Nr * cm * 4 * H * c + 2 * Nr * Nr * cz * H + 4 * Ns * H * Nr * Nr * c + 2 * Ns * Nr * H * c * cm
        job = Job(variant, f"evoformer_row_block_bf16_Nseq{Ns}_Nres{Nr}_cm{cm}_cz{cz}_H{H}_c{c}")
        job.calls.append(Call("evo_block", lambda: blk(m, z), flops, 0, "tensor", kernel="attn_tc_kernel"))
    else:
        N = cfg["N"]
        x = {k: v.to(device) for k, v in synth.ipa_inputs(N, seed=1).items()}
        ws = torch.empty(64 << 20, dtype=torch.uint8, device=device)
        flops = 2 * 12 * N * N * (64 + 64) + 2 * 12 * N * N * (128 + 24)
        job = Job(variant, f"ipa_core_N{N}_H12_c16_Pq4_Pv8_cz128")
        job.calls.append(Call("ipa", lambda: fl.ipa_fwd(**x, workspace=ws), flops, 0, "tensor", kernel="attn_tc_kernel"))
    job.step_flops = job.calls[0].flops
    job.units = "whole problem (not sharded)"
    return job


def make_job(variant, rank, world, device, with_host=True):
    if variant in SUITES:
        return dense_job(SUITES[variant], rank, world, device, with_host)
    cfg = VARIANTS[variant]
    if cfg.get("special"):
        return special_job(variant, device)
    if cfg.get("evo"):
        return evo_job(variant, rank, world, device, with_host)
    if cfg.get("rsa"):
        return rsa_job(variant, rank, world, device, with_host)
    return dense_job([variant], rank, world, device, with_host)


# ------------------------------------------------------------------ driver
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def sum_over_ranks(vals, device, world):
    if world <= 1:
        return vals
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t]


def max_over_ranks(vals, device, world):
    if world <= 1:
        return vals
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t]


def run_reference(args, world, rank):
    """This tier's reference arm: the fp64 oracle as it stands, on the host's cores."""
    if rank != 0:
        return
    job = oracle_only_job(args.variant)
    budget = float(os.environ.get("FL_REF_BUDGET_S", max(2.0, 60.0 / (args.steps + args.warmup))))
    vals, secs, samples = [], [], ""
    for i in range(args.warmup + args.steps):
        v, cores, samples, dt = job.oracle(budget)
        if i >= args.warmup:
            vals.append(v)
            secs.append(dt)
    value = float(np.mean(vals))
    # ms_per_step: the measured wall time of one step, i.e. of the bounded sample the oracle runs per step;
    # the time a whole workload step would take at that rate is reported separately as an extrapolation
    ms_per_step = float(np.mean(secs)) * 1e3
    step_flops = getattr(job, "step_flops", None)
    full_ms = step_flops / (value * 1e12) * 1e3 if step_flops and value > 0 else None
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "full_step_ms_extrapolated": full_ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": job.workload, "variant": args.variant},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": samples},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def oracle_only_job(variant):
    """Build a job's oracle closure without touching CUDA (reference arm / CPU box)."""
    names = SUITES.get(variant, [variant])
    cfg0 = VARIANTS[names[0]]
    if cfg0.get("rsa"):
        # host-only replica of rsa_job's oracle leg (no device lists needed): head (b=0, h=0)
        q1, k1, v1 = rsa_block_inputs(cfg0, (0, 1, 0, 1))
        B, H, S, D, topk = cfg0["B"], cfg0["H"], cfg0["S"], cfg0["D"], cfg0["topk"]
        job = Job(variant, f"rsa_{cfg0['rsa']}_bf16_B{B}_H{H}_S{S}_D{D}_top{topk}")
        job.oracle = lambda budget_s: rsa_oracle_rate(cfg0, q1, k1, v1, budget_s)
        return job
    # dense / Evoformer builders never launch anything when given host tensors and no e2e leg
    if cfg0.get("evo"):
        return evo_job(variant, 0, 1, "cpu", with_host=False)
    return dense_job(names, 0, 1, "cpu", with_host=False)


EXTRA_CONFIGS = ["c1", "diff", "evo_row", "evo_col", "rsa", "rsa_decode"]   # BASELINE configs[0, 2, 3, 4]
NEXT_EXTRAS = ["bwd_causal", "bwd_diff", "evo_block", "ipa"]     # SURVEY §8(f) rows, single-GPU runs only


def time_job(job, steps, warmup, device, stream, use_graph=True, flush=None, clk=None):
    """Warm up, capture the step (and each call alone) as CUDA graphs, then time `steps` replays with CUDA
    events on the launch stream, one event pair per step; the L2 is flushed (a 256 MB write > the 126 MB
    L2) before every timed replay, outside the events.  Returns per-step and per-call mean ms."""
    from paper_2511_02043_b200 import fl
    E = lambda: torch.cuda.Event(enable_timing=True)

    def step(ev=None):
        for ci, c in enumerate(job.calls):
            if ev is not None:
                ev[ci][0].record(stream)
            c.fn()
            if ev is not None:
                ev[ci][1].record(stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = 0
    if use_graph:
        # The timed step is a CUDA graph of the step's library calls (captured once after warm-up and
        # replayed): launch overhead of the Python binding stays off the clock, which matters for the
        # microsecond-scale decode step.  Each call is also captured alone for the per-call breakdown.
        fl.launch_count(reset=True)
        g_step = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step):
            step()
        launches_per_step = fl.launch_count(reset=True)
        g_calls = []
        for c in job.calls:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                c.fn()
            g_calls.append(g)
        g_step.replay()
        for g in g_calls:
            g.replay()
        torch.cuda.synchronize()
    fl.launch_count(reset=True)
    ev_step = [(E(), E()) for _ in range(steps)]
    evs = [[(E(), E()) for _ in job.calls] for _ in range(steps)]
    if clk is not None:
        clk.__enter__()
    torch.cuda.synchronize()
    for i in range(steps):
        if flush is not None:
            flush.zero_()
        ev_step[i][0].record(stream)
        if use_graph:
            g_step.replay()
        else:
            step(evs[i])
        ev_step[i][1].record(stream)
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__(None, None, None)
    launches = launches_per_step * steps if use_graph else fl.launch_count()
    step_ms = [a.elapsed_time(b) for a, b in ev_step]
    if use_graph:
        call_ms = []
        for g in g_calls:
            tl = []
            for _ in range(steps):
                if flush is not None:
                    flush.zero_()
                c0, c1 = E(), E()
                c0.record(stream)
                g.replay()
                c1.record(stream)
                tl.append((c0, c1))
            torch.cuda.synchronize()
            call_ms.append(float(np.mean([a.elapsed_time(b) for a, b in tl])))
    else:
        call_ms = [float(np.mean([evs[i][ci][0].elapsed_time(evs[i][ci][1]) for i in range(steps)]))
                   for ci in range(len(job.calls))]
    return {"ms_per_step": float(np.mean(step_ms)), "total_ms": float(np.sum(step_ms)), "call_ms": call_ms,
            "launches": int(launches)}


def mufu_peaks(device):
    """Measured MUFU / FMA throughput on this GPU (fl_diag_pipe_rate microbenchmark: one persistent CTA per
    SM x 8 warps of independent dependency chains), in operations per second."""
    from paper_2511_02043_b200 import fl
    out = {}
    for op in ("ex2_f32", "ex2_bf16x2", "tanh_f32", "ffma2"):
        try:
            out[op] = fl.pipe_rate(op, device=device)
        except Exception as e:   # reported, never silently replaced by a derived number
            out[op] = None
            out[op + "_error"] = str(e)[:200]
    return out


def roofline_of(job, call_ms, call_flops_all, pk, pk_src, prof, mufu):
    """`roofline` object for the dominant call: algorithmic flops (bytes, ex2) per launch /
    its mean CUDA-event duration, against the measured peak of its bound unit."""
    dom_i = int(np.argmax(call_ms))
    dom = job.calls[dom_i]
    ms = call_ms[dom_i]
    prof_key = f"{dom.label if job.name == 'flex' else job.name}:{dom.kernel}"
    traffic = (prof.get(prof_key) or {}).get("dram_bytes_per_launch")
    if dom.bound == "latency":
        roof = {"bound": "latency", "achieved": ms * 1e3, "unit": "us per launch", "peak": None, "frac": None,
                "traffic": traffic, "note": "C1 (2.1 MFLOP, 128 KiB) is launch-latency bound; not a roofline case"}
    elif dom.bound == "alu":
        meas = (mufu or {}).get("ex2_f32")
        peak = meas / 1e9 if meas else 16 * 148 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
        ach = dom.alu / (ms * 1e-3) / 1e9
        roof = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Gex2/s", "frac": ach / peak,
                "traffic": traffic,
                "peak_source": "measured ex2.approx.f32 rate (fl_diag_pipe_rate, this run)" if meas
                else "derived: 16 ex2/clk/SM x 148 SMs x sm_max_mhz (measurement failed)",
                "hbm_gbs": dom.bytes / (ms * 1e-3) / 1e9, "hbm_frac": dom.bytes / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                "tensor_frac": dom.flops / (ms * 1e-3) / 1e12 / pk["bf16_tflops"]}
    elif dom.bound == "hbm":
        ach = dom.bytes / (ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"],
                "traffic": traffic, "algorithmic_bytes": dom.bytes, "peak_source": f"{pk_src} (MEASURED_PEAKS.json)"}
    else:
        ach = dom.flops / (ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": ach / pk["bf16_tflops"], "traffic": traffic, "algorithmic_flops": dom.flops,
                "frac_of_sustained": ach / pk.get("bf16_tflops_sustained", pk["bf16_tflops"]),
                "peak_source": f"{pk_src} (MEASURED_PEAKS.json burst)"}
        if dom.exec_flops:
            roof["executed_tile_flops"] = dom.exec_flops
    roof.update(kernel=dom.kernel, call=dom.label, launch_ms=ms)
    return roof


def per_call_of(job, call_ms, pk):
    per_call = {}
    for c, ms in zip(job.calls, call_ms):
        d = {"ms": ms, "share": ms / max(sum(call_ms), 1e-12)}
        if c.flops:
            d["tflops"] = c.flops / (ms * 1e-3) / 1e12
            d["frac_of_bf16_peak"] = d["tflops"] / pk["bf16_tflops"]
        if c.exec_flops:
            d["executed_tile_tflops"] = c.exec_flops / (ms * 1e-3) / 1e12
            d["useful_over_executed"] = c.flops / c.exec_flops
        if c.bytes:
            d["gbs"] = c.bytes / (ms * 1e-3) / 1e9
            d["frac_of_hbm"] = d["gbs"] / pk["hbm_gbs"]
        if c.alu:
            d["gex2_s"] = c.alu / (ms * 1e-3) / 1e9
        per_call[c.label] = d
    return per_call


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--variant", default="flex", choices=sorted(list(VARIANTS) + list(SUITES)))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the other BASELINE configs appended after the headline (default run only)")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of CUDA-graph replays of the step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            torch.distributed.barrier()
        return

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    job = make_job(args.variant, rank, world, device, with_host=not args.no_e2e)
    if world > 1:
        torch.distributed.barrier()
    clk = ClockSampler(local)
    t = time_job(job, args.steps, args.warmup, device, stream, use_graph=not args.no_graph, flush=flush, clk=clk)
    red = max_over_ranks([t["ms_per_step"]] + t["call_ms"], device, world)
    ms_per_step, call_ms = red[0], red[1:]
    # whole-job aggregate: the useful flops of ALL ranks' shards (= the fixed problem's) / max-over-ranks time
    job_flops = sum_over_ranks([job.step_flops] + [c.flops for c in job.calls], device, world)
    step_flops_all, call_flops_all = job_flops[0], job_flops[1:]
    value = step_flops_all / (ms_per_step * 1e-3) / 1e12

    e2e = None
    if job.e2e is not None:
        E = lambda: torch.cuda.Event(enable_timing=True)
        fn, h2d, d2h = job.e2e
        for _ in range(2):
            fn(stream)
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 10))
        a0, a1 = E(), E()
        a0.record(stream)
        for _ in range(n_e2e):
            fn(stream)
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks([a0.elapsed_time(a1) / n_e2e], device, world)[0]
        e2e = {"value": step_flops_all / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
               "api": "fl_attn_fwd_host / pinned host buffers (batch chunks: H2D, kernel, D2H pipelined on three streams)"}
    mufu = mufu_peaks(device) if rank == 0 else None
    pk, pk_src = peaks()
    prof = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    except Exception:
        pass

    # the other BASELINE configs, each one step of its own hot path, timed the same way (default run)
    configs = {}
    if args.variant == "flex" and not args.no_extra:
        del job.e2e
        for name in EXTRA_CONFIGS:
            xj = make_job(name, rank, world, device, with_host=False)
            xt = time_job(xj, max(3, min(args.steps, 10)), args.warmup, device, stream, flush=flush)
            xr = max_over_ranks([xt["ms_per_step"]] + xt["call_ms"], device, world)
            xf = sum_over_ranks([xj.step_flops] + [c.flops for c in xj.calls], device, world)
            if rank == 0:
                configs[name] = {"workload": xj.workload, "value": xf[0] / (xr[0] * 1e-3) / 1e12, "unit": "TFLOP/s",
                                 "ms_per_step": xr[0], "us_per_step": xr[0] * 1e3,
                                 "per_call": per_call_of(xj, xr[1:], pk),
                                 "roofline": roofline_of(xj, xr[1:], xf[1:], pk, pk_src, prof, mufu),
                                 "gpu_launches_per_step": xt["launches"] // max(1, min(args.steps, 10))}
            del xj
            torch.cuda.empty_cache()

    # the §8(f) rows (backward, Evoformer block, IPA), one GPU only: timed the same way, reported apart
    nexts = {}
    if args.variant == "flex" and not args.no_extra and world == 1:
        for name in NEXT_EXTRAS:
            xj = make_job(name, rank, world, device, with_host=False)
            xt = time_job(xj, 3, args.warmup, device, stream, flush=flush)
            nexts[name] = {"workload": xj.workload, "value": xj.step_flops / (xt["ms_per_step"] * 1e-3) / 1e12,
                           "unit": "TFLOP/s", "ms_per_step": xt["ms_per_step"],
                           "gpu_launches_per_step": xt["launches"] // 3}
            del xj
            torch.cuda.empty_cache()

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
        return
    roof = roofline_of(job, call_ms, call_flops_all, pk, pk_src, prof, mufu)
    cfg0 = VARIANTS[SUITES.get(args.variant, [args.variant])[0]]
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded Philox, DESIGN.md §4)",
            "config": {"workload": job.workload, "variant": args.variant,
                       "global_batch": cfg0.get("B", 1), "seq_len": cfg0.get("S", cfg0.get("Nr")),
                       "parallelism": f"fixed problem split over {world} GPU(s) by fl_shard_range, "
                                      f"rank 0: {job.units}; no collective on the data path",
                       "useful_tflop_per_step": step_flops_all / 1e12,
                       "l2": "256 MB L2 flush before every timed step (outside the CUDA events)"},
            "per_call": per_call_of(job, call_ms, pk), "roofline": roof, "gpu_launches": t["launches"],
            "clocks": clk.summary(), "mufu_measured": mufu,
            "timing": "CUDA-graph replay of the step, one event pair per step (per call: graph of that call alone)"
                      if not args.no_graph else "eager launches, CUDA events around each call"}
    for key, val in job.extra.items():
        line["config"][key] = val
    if e2e:
        line["e2e"] = e2e
    if configs:
        line["configs"] = configs
    if nexts:
        line["next"] = nexts
    if not args.no_cpu_baseline and job.oracle is not None:
        v_cpu, cores, sample, _ = job.oracle(15.0)
        line["cpu_baseline"] = {"value": v_cpu, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample}
        if job.parity_result:
            line["parity"] = {"vs": "fp64 oracle on the cpu_baseline rows (block 0 of the step, full size)",
                              "variants": job.parity_result}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
