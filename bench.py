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
    # configs[2]: differential attention bf16 B=8 H=16 S=8192 D=64 (two maps, lambda)
    "diff": dict(B=8, H=16, S=8192, D=64, diff=True, lam=0.2),
    # configs[3]: Evoformer gated self-attention with pair bias, N_seq=512 N_res=384 H=8 c=32
    "evo_row": dict(evo="row", B=1, Ns=512, Nr=384, H=8, D=32),
    "evo_col": dict(evo="col", B=1, Ns=512, Nr=384, H=8, D=32),
    # configs[4]: Rectified Sparse Attention B=4 H=32 S=32768 D=128 (blocks 128, top-16 + sink + diagonal)
    "rsa": dict(rsa="prefill", B=4, H=32, S=32768, D=128, topk=16),
    "rsa_decode": dict(rsa="decode", B=4, H=32, S=32768, D=128, topk=16),
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


# ------------------------------------------------------------------ input construction (rank's slice)
def dense_inputs(cfg, rank, world, seed=0):
    """Host tensors of rank `rank`'s slice of the global problem (global batch = B * world)."""
    B, H, S, D = cfg["B"], cfg["H"], cfg["S"], cfg["D"]
    Hkv = cfg.get("Hkv", H)
    maps = 2 if cfg.get("diff") else 1
    gB = B * world

    def gen(t, heads):
        return synth.uniform((gB, heads, S, D), seed=seed, tensor=t, lead=2,
                             slab_range=(rank * B * heads, (rank + 1) * B * heads)).reshape(B, heads, S, D)
    host = {"q": gen("q", H * maps), "k": gen("k", Hkv * maps), "v": gen("v", Hkv)}
    return host


def doc_offsets_for(cfg, rank, world):
    return synth.doc_offsets(cfg["B"] * world, cfg["S"], cfg["n_docs"], seed=1)[rank * cfg["B"]:(rank + 1) * cfg["B"]]


def evo_inputs(cfg, rank, world, seed=0):
    B, Ns, Nr, H, c = cfg["B"], cfg["Ns"], cfg["Nr"], cfg["H"], cfg["D"]
    gb = rank * B
    rng = (gb * Ns * Nr, (gb + B) * Ns * Nr)
    st = lambda t, **kw: synth.uniform((B * world, Ns, Nr, H, c), seed=seed, tensor=t, lead=3, slab_range=rng,
                                       **kw).reshape(B, Ns, Nr, H, c)
    host = {"Q": st("q"), "K": st("k"), "V": st("v"), "G": st("gate", lo=-4.0, hi=4.0),
            "km": torch.ones(B, Ns, Nr, dtype=torch.uint8)}      # all-ones MSA mask (tests use 10 % zeros)
    if cfg["evo"] == "row":
        host["pb"] = synth.pair_bias((B * world, H, Nr, Nr), seed=seed, lead=2,
                                     slab_range=(gb * H, (gb + B) * H)).reshape(B, H, Nr, Nr)
    return host


def evo_views(cfg, t):
    """[B,G,H,S,D] views of MSA storage [B, N_seq, N_res, H, c] (reading G9); no copies."""
    B, Ns, Nr, H = cfg["B"], cfg["Ns"], cfg["Nr"], cfg["H"]
    view = (lambda x: x.permute(0, 1, 3, 2, 4)) if cfg["evo"] == "row" else (lambda x: x.permute(0, 2, 3, 1, 4))
    q, k, v = view(t["Q"]), view(t["K"]), view(t["V"])
    kw = dict(gate_mode="sigmoid", gate=view(t["G"]))
    if cfg["evo"] == "row":
        kw["bias"] = t["pb"].unsqueeze(1).expand(B, Ns, H, Nr, Nr)
        kw["key_mask"] = t["km"]
    else:
        kw["key_mask"] = t["km"].permute(0, 2, 1)
    return q, k, v, kw


# ------------------------------------------------------------------ jobs: the calls of one step
class Call:
    def __init__(self, label, fn, flops=0.0, bytes_=0.0, bound="tensor", kernel=None, alu=0.0):
        self.label, self.fn, self.flops, self.bytes, self.bound = label, fn, flops, bytes_, bound
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


def dense_job(names, rank, world, device, with_host=True):
    from paper_2511_02043_b200 import fl
    cfg0 = VARIANTS[names[0]]
    host = dense_inputs(cfg0, rank, world)
    q, k, v = (host[n].to(device) for n in ("q", "k", "v"))
    maps = 2 if cfg0.get("diff") else 1
    out = torch.empty(q.shape[0], q.shape[1] // maps, q.shape[2], v.shape[3], dtype=q.dtype, device=device)
    wl = names[0] if len(names) == 1 else "flexattention_variants(" + ",".join(names) + ")"
    job = Job(names[0] if len(names) == 1 else "flex",
              f"{wl}_bf16_B{cfg0['B']}_H{cfg0['H']}_S{cfg0['S']}_D{cfg0['D']}")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=device)       # scheduler counter + packed key mask
    kws, pairs_by = {}, {}
    for n in names:
        cfg = VARIANTS[n]
        assert all(cfg[x] == cfg0[x] for x in ("B", "H", "S", "D")) and cfg.get("Hkv") == cfg0.get("Hkv")
        kw = {x: cfg[x] for x in VARIANT_KW if x in cfg}
        offs = None
        if cfg.get("mask") == "document":
            offs = doc_offsets_for(cfg, rank, world)
            kw["doc_offsets"] = torch.from_numpy(offs).to(device)
        pairs = kept_pairs(cfg, offs)
        flops = pairs * flops_per_pair(cfg)
        nbytes = sum(t.numel() * t.element_size() for t in (q, k, v, out))
        job.calls.append(Call(n, (lambda kw=kw: fl.attn_fwd(q, k, v, out=out, workspace=ws, **kw)), flops, nbytes,
                              "tensor",
                              kernel="attn_tc_kernel"))
        job.step_flops += flops
        kws[n] = (kw, offs)
        pairs_by[n] = pairs
    job.parity = {"host": host, "out": out,
                  "oracle_kw": {n: dict({x: VARIANTS[n][x] for x in VARIANT_KW if x in VARIANTS[n]},
                                        **({"doc_offsets": kws[n][1]} if kws[n][1] is not None else {}))
                                for n in names}}

    if with_host:
        runner = fl.HostRunner(device)
        hq, hk, hv = (host[n].pin_memory() for n in ("q", "k", "v"))
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        hkws = {}
        for n in names:
            kw, offs = kws[n]
            hkw = dict(kw)
            if offs is not None:
                hkw["doc_offsets"] = torch.from_numpy(offs)
            hkws[n] = hkw

        def e2e_step(stream):
            for n in names:
                runner(hq, hk, hv, hout, stream=stream, **hkws[n])
        per = sum(t.numel() * t.element_size() for t in (hq, hk, hv))
        job.e2e = (e2e_step, per * len(names), hout.numel() * hout.element_size() * len(names))

    def oracle_fn(budget_s):
        import oracle
        B, H, S = cfg0["B"], cfg0["H"], cfg0["S"]
        total_rows = B * H * S
        per_budget = budget_s / len(names)
        tot_flops, tot_s, n_rows = 0.0, 0.0, 0
        for n in names:
            cfg = VARIANTS[n]
            kw, offs = kws[n]
            ok = {x: cfg[x] for x in VARIANT_KW if x in cfg}
            if offs is not None:
                ok["doc_offsets"] = offs
            rows = np.linspace(0, total_rows - 1, 64).astype(np.int64)
            t0 = time.perf_counter()
            oracle.attn(host["q"], host["k"], host["v"], rows=rows, **ok)
            dt = time.perf_counter() - t0
            nr = int(min(total_rows, max(64, 64 * per_budget / max(dt, 1e-3))))
            rows = np.linspace(0, total_rows - 1, nr).astype(np.int64)
            t0 = time.perf_counter()
            oracle.attn(host["q"], host["k"], host["v"], rows=rows, **ok)
            dt = time.perf_counter() - t0
            tot_flops += pairs_by[n] * flops_per_pair(cfg) * (nr / total_rows)
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
    # c = 32: one ex2 per kept pair against 4c = 128 MMA flops, so the MUFU (16 ex2/clk/SM), not the
    # tensor pipe, bounds the kernel (MUFU 187/250 us vs tensor 47/62 us vs HBM 77 us)
    job.calls.append(Call(name, lambda: fl.attn_fwd(q, k, v, out=out, workspace=ws, **kw), flops, nbytes, "alu",
                          kernel="attn_tc_kernel", alu=float(pairs)))
    job.step_flops = flops
    job.parity = {"host": host, "out": out}

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
        oracle.attn(hq, hk, hv, rows=rows, **okw)
        dt = time.perf_counter() - t0
        return (flops * nr / total_rows / dt / 1e12, oracle.num_threads(),
                f"{nr} of {total_rows} output rows (evenly spaced), useful flops scaled by row share", dt)
    job.oracle = oracle_fn
    return job


def rsa_job(name, rank, world, device, with_host=True):
    """configs[4]: RSA on B=4 H=32 S=32768 D=128.  prefill step = summaries + selection +
    block-sparse attention over all 32768 queries; decode step = selection + attention for
    one query per (b,h) at position S-1 (summaries are maintained at prefill)."""
    from paper_2511_02043_b200 import fl
    cfg = VARIANTS[name]
    B, H, S, D, topk = cfg["B"], cfg["H"], cfg["S"], cfg["D"], cfg["topk"]
    decode = cfg["rsa"] == "decode"
    qh, kh = synth.clustered_qk((B * world, H, S, D), (B * world, H, S, D), seed=2,
                                b_range=(rank * B, (rank + 1) * B))
    vh = synth.uniform((B * world, H, S, D), seed=0, tensor="v", slab_range=(rank * B * H, (rank + 1) * B * H)
                       ).reshape(B, H, S, D)
    if decode:
        qh = qh[:, :, S - 1:].contiguous()
    Sq = qh.shape[2]
    q, k, v = qh.to(device), kh.to(device), vh.to(device)
    out = torch.empty(B, H, Sq, D, dtype=q.dtype, device=device)
    nqb, nkb = (Sq + 127) // 128, (S + 127) // 128
    kmin, kmax = fl.rsa_build_summaries(k, 128)
    idx, cnt = fl.rsa_select(q, kmin, kmax, S, topk=topk)
    torch.cuda.synchronize()
    pairs = rsa_pairs(idx.cpu().numpy(), cnt.cpu().numpy(), S, Sq)
    flops = pairs * flops_per_pair(cfg)
    listed = int(cnt.sum().item())
    job = Job(name, f"rsa_{cfg['rsa']}_bf16_B{B}_H{H}_S{S}_D{D}_top{topk}")
    sum_bytes = k.numel() * 2 + 2 * kmin.numel() * 2
    if not decode:
        job.calls.append(Call("rsa_summaries", lambda: fl.rsa_build_summaries(k, 128, kmin, kmax), 0.0, sum_bytes,
                              "hbm", kernel="rsa_summaries_kernel"))
    sel_flops = 2.0 * 2 * D * 128 * 128 * sum(((i * 128 + 127 + S - Sq) // 128 + 127) // 128
                                            for i in range(nqb)) * B * H   # executed GEMM tiles
    sel_bytes = q.numel() * 2 + 2 * kmin.numel() * 2 + idx.numel() * 4 + cnt.numel() * 4
    job.calls.append(Call("rsa_select", lambda: fl.rsa_select(q, kmin, kmax, S, topk=topk, blk_idx=idx, blk_cnt=cnt),
                          sel_flops, sel_bytes, "hbm" if decode else "tensor",
                          kernel="rsa_select_small_kernel" if decode else "rsa_select_kernel"))
    if decode:   # each listed KV block is read once per (b,h): K + V rows
        att_bytes = q.numel() * 2 + out.numel() * 2 + listed * 128 * D * 2 * 2
    else:        # K/V read once per (b,h) (a block listed by several q-blocks is re-read from L2)
        att_bytes = (q.numel() + k.numel() + v.numel() + out.numel()) * 2
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=device)
    job.calls.append(Call("attn_blocklist", lambda: fl.attn_fwd(q, k, v, out=out, mask="blocklist", blk_idx=idx,
                                                                blk_cnt=cnt, workspace=ws), flops, att_bytes,
                          "hbm" if decode else "tensor",
                          kernel="attn_decode_split_kernel" if decode else "attn_tc_kernel"))
    job.step_flops = flops
    job.extra.update(listed_blocks=listed, kv_blocks=nkb * B * H * nqb, rsa_decode=decode)
    job.parity = {"host": {"q": qh, "k": kh, "v": vh}, "out": out, "idx": idx, "cnt": cnt, "kmin": kmin,
                  "kmax": kmax, "Sq": Sq}

    if with_host:
        hq, hk, hv = qh.pin_memory(), kh.pin_memory(), vh.pin_memory()
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()

        def e2e_step(stream):
            with torch.cuda.stream(stream):
                q.copy_(hq, non_blocking=True)
                k.copy_(hk, non_blocking=True)
                v.copy_(hv, non_blocking=True)
                fl.rsa_build_summaries(k, 128, kmin, kmax, stream=stream)
                fl.rsa_select(q, kmin, kmax, S, topk=topk, blk_idx=idx, blk_cnt=cnt, stream=stream)
                fl.attn_fwd(q, k, v, out=out, mask="blocklist", blk_idx=idx, blk_cnt=cnt, workspace=ws, stream=stream)
                hout.copy_(out, non_blocking=True)
        h2d = (hq.numel() + hk.numel() + hv.numel()) * 2
        job.e2e = (e2e_step, h2d, hout.numel() * 2)

    def oracle_fn(budget_s):
        import oracle
        # selection + attention of the oracle on (b=0, h=0), its own list; extrapolated by row share
        q1, k1, v1 = qh[:1, :1], kh[:1, :1], vh[:1, :1]
        t0 = time.perf_counter()
        ri, rc, _ = oracle.rsa_select(q1, k1, topk=topk)
        t_sel = time.perf_counter() - t0
        rows_total = Sq
        nr = 64
        rows = np.linspace(0, rows_total - 1, nr).astype(np.int64)
        t0 = time.perf_counter()
        oracle.attn(q1, k1, v1, rows=rows, mask="blocklist", blk_idx=ri, blk_cnt=rc)
        dt = time.perf_counter() - t0
        nr = int(min(rows_total, max(64, 64 * max(budget_s - t_sel, 1.0) / max(dt, 1e-3))))
        rows = np.linspace(0, rows_total - 1, nr).astype(np.int64)
        t0 = time.perf_counter()
        oracle.attn(q1, k1, v1, rows=rows, mask="blocklist", blk_idx=ri, blk_cnt=rc)
        t_att = time.perf_counter() - t0
        head_pairs = rsa_pairs(ri, rc, S, Sq)
        t_head = t_sel + t_att * rows_total / nr                  # one (b,h) in full
        return (head_pairs * flops_per_pair(cfg) / t_head / 1e12, oracle.num_threads(),
                f"(b=0,h=0): oracle selection in full + {nr} of {rows_total} attention rows; rate of that head", t_sel + t_att)
    job.oracle = oracle_fn
    return job


def make_job(variant, rank, world, device, with_host=True):
    if variant in SUITES:
        return dense_job(SUITES[variant], rank, world, device, with_host)
    cfg = VARIANTS[variant]
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
    vals, samples = [], ""
    for i in range(args.warmup + args.steps):
        v, cores, samples, _ = job.oracle(budget)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    # one full-workload step at the sampled rate (the oracle runs a bounded sample of it per step)
    step_flops = getattr(job, "step_flops", None)
    ms_per_step = step_flops / (value * 1e12) * 1e3 if step_flops and value > 0 else None
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
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
        # host-only replica of rsa_job's oracle leg (no device lists needed)
        B, H, S, D, topk = cfg0["B"], cfg0["H"], cfg0["S"], cfg0["D"], cfg0["topk"]
        qh, kh = synth.clustered_qk((B, 1, S, D), (B, 1, S, D), seed=2, b_range=(0, 1))
        vh = synth.uniform((B, H, S, D), seed=0, tensor="v", slab_range=(0, 1)).reshape(1, 1, S, D)
        if cfg0["rsa"] == "decode":
            qh = qh[:, :, S - 1:].contiguous()
        job = Job(variant, f"rsa_{cfg0['rsa']}_bf16_B{B}_H{H}_S{S}_D{D}_top{topk}")
        Sq = qh.shape[2]

        def oracle_fn(budget_s):
            import oracle
            t0 = time.perf_counter()
            ri, rc, _ = oracle.rsa_select(qh, kh, topk=topk)
            t_sel = time.perf_counter() - t0
            nr = min(Sq, 64)
            rows = np.linspace(0, Sq - 1, nr).astype(np.int64)
            t0 = time.perf_counter()
            oracle.attn(qh, kh, vh, rows=rows, mask="blocklist", blk_idx=ri, blk_cnt=rc)
            dt = time.perf_counter() - t0
            nr = int(min(Sq, max(nr, nr * max(budget_s - t_sel, 1.0) / max(dt, 1e-3))))
            rows = np.linspace(0, Sq - 1, nr).astype(np.int64)
            t0 = time.perf_counter()
            oracle.attn(qh, kh, vh, rows=rows, mask="blocklist", blk_idx=ri, blk_cnt=rc)
            t_att = time.perf_counter() - t0
            t_head = t_sel + t_att * Sq / nr
            return (rsa_pairs(ri, rc, S, Sq) * flops_per_pair(cfg0) / t_head / 1e12, oracle.num_threads(),
                    f"(b=0,h=0): oracle selection in full + {nr} of {Sq} attention rows; rate of that head",
                    t_sel + t_att)
        job.oracle = oracle_fn
        return job
    # dense / Evoformer builders never launch anything when given host tensors and no e2e leg
    if cfg0.get("evo"):
        return evo_job(variant, 0, 1, "cpu", with_host=False)
    return dense_job(names, 0, 1, "cpu", with_host=False)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--variant", default="flex", choices=sorted(list(VARIANTS) + list(SUITES)))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
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

    from paper_2511_02043_b200 import fl
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    job = make_job(args.variant, rank, world, device, with_host=not args.no_e2e)
    stream = torch.cuda.current_stream(device)

    def step(ev=None):
        for ci, c in enumerate(job.calls):
            if ev is not None:
                ev[ci][0].record(stream)
            c.fn()
            if ev is not None:
                ev[ci][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    E = lambda: torch.cuda.Event(enable_timing=True)
    # The timed step is a CUDA graph of the step's library calls (captured once after warm-up and
    # replayed): launch overhead of the Python binding stays off the clock, which matters for the
    # microsecond-scale decode step.  Each call is also captured alone for the per-call breakdown.
    use_graph = not args.no_graph
    launches_per_step = 0
    if use_graph:
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
    if world > 1:
        torch.distributed.barrier()
    evs = [[(E(), E()) for _ in job.calls] for _ in range(args.steps)]
    fl.launch_count(reset=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0, t1 = E(), E()
        t0.record(stream)
        for i in range(args.steps):
            if use_graph:
                g_step.replay()
            else:
                step(evs[i])
        t1.record(stream)
        torch.cuda.synchronize()
    launches = launches_per_step * args.steps if use_graph else fl.launch_count()
    total_ms = t0.elapsed_time(t1)
    if use_graph:
        call_ms = []
        for g in g_calls:
            c0, c1 = E(), E()
            c0.record(stream)
            for _ in range(args.steps):
                g.replay()
            c1.record(stream)
            torch.cuda.synchronize()
            call_ms.append(c0.elapsed_time(c1) / args.steps)
    else:
        call_ms = [float(np.mean([evs[i][ci][0].elapsed_time(evs[i][ci][1]) for i in range(args.steps)]))
                   for ci in range(len(job.calls))]
    red = max_over_ranks([total_ms] + call_ms, device, world)
    total_ms, call_ms = red[0], red[1:]
    ms_per_step = total_ms / args.steps
    value = job.step_flops * world / (ms_per_step * 1e-3) / 1e12          # whole-job aggregate

    e2e = None
    if job.e2e is not None:
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
        e2e = {"value": job.step_flops * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms}

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
        return
    pk, pk_src = peaks()
    prof = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    except Exception:
        pass
    per_call = {}
    for c, ms in zip(job.calls, call_ms):
        d = {"ms": ms, "share": ms / max(sum(call_ms), 1e-12)}
        if c.flops:
            d["tflops"] = c.flops / (ms * 1e-3) / 1e12
            d["frac_of_bf16_peak"] = d["tflops"] / pk["bf16_tflops"]
        if c.bytes:
            d["gbs"] = c.bytes / (ms * 1e-3) / 1e9
        per_call[c.label] = d
    dom_i = int(np.argmax(call_ms))
    dom = job.calls[dom_i]
    # ncu --set full summary of this kernel on this workload (profiles/ncu_summary.json, key "<variant>:<kernel>")
    prof_key = f"{dom.label if job.name == 'flex' else job.name}:{dom.kernel}"
    traffic = (prof.get(prof_key) or {}).get("dram_bytes_per_launch")
    if dom.bound == "alu":
        # MUFU ex2 roofline: 16 ex2/clk/SM (B200; the 2x SFU rate is sm_103a-only) x 148 SMs x max SM clock
        mufu_peak = 16 * 148 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
        ach = dom.alu / (call_ms[dom_i] * 1e-3) / 1e9
        roof = {"bound": "alu", "achieved": ach, "peak": mufu_peak, "unit": "Gex2/s", "frac": ach / mufu_peak,
                "traffic": traffic, "peak_derivation": "16 ex2/clk/SM x 148 SMs x sm_max_mhz (DESIGN.md)",
                "hbm_gbs": dom.bytes / (call_ms[dom_i] * 1e-3) / 1e9, "hbm_frac": dom.bytes / (call_ms[dom_i] * 1e-3) / 1e9 / pk["hbm_gbs"],
                "tensor_frac": dom.flops / (call_ms[dom_i] * 1e-3) / 1e12 / pk["bf16_tflops"]}
    elif dom.bound == "hbm":
        ach = dom.bytes / (call_ms[dom_i] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"],
                "traffic": traffic, "algorithmic_bytes": dom.bytes}
    else:
        ach = dom.flops / (call_ms[dom_i] * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": ach / pk["bf16_tflops"], "traffic": traffic, "algorithmic_flops": dom.flops,
                "frac_of_sustained": ach / pk.get("bf16_tflops_sustained", pk["bf16_tflops"])}
    roof.update(kernel=dom.kernel, call=dom.label, launch_ms=call_ms[dom_i],
                peak_source="derived (DESIGN.md §6)" if dom.bound == "alu"
                else f"{pk_src} (MEASURED_PEAKS.json burst)")
    cfg0 = VARIANTS[SUITES.get(args.variant, [args.variant])[0]]
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded Philox, DESIGN.md §4)",
            "config": {"workload": job.workload, "variant": args.variant,
                       "global_batch": cfg0.get("B", 1) * world, "seq_len": cfg0.get("S", cfg0.get("Nr")),
                       "parallelism": f"batch-x-head shards over {world} GPU(s), no collective",
                       "useful_tflop_per_step_per_gpu": job.step_flops / 1e12,
                       "l2": "inputs larger than L2 (per-GPU working set > 126 MB); no flush"},
            "per_call": per_call, "roofline": roof, "gpu_launches": int(launches), "clocks": clk.summary(),
            "timing": "CUDA-graph replay of the step (per call: graph of that call alone)" if use_graph
                      else "eager launches, CUDA events around each call"}
    for key, val in job.extra.items():
        if key != "dev":
            line["config"][key] = val
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and job.oracle is not None:
        v_cpu, cores, sample, _ = job.oracle(15.0)
        line["cpu_baseline"] = {"value": v_cpu, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
