#!/usr/bin/env python
"""Benchmark of the fused attention-variant forward (Flashlight, arXiv 2511.02043) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant causal|alibi|...] [--impl ours|reference]

One "step" = one pass of the whole hot path over one batch of synthetic inputs
= one fl_attn_fwd call (C ABI) on the workload of BASELINE.json configs[1]
(bf16, B=8 H=16 S=8192 D=128; causal is the headline variant).  Under torchrun
each rank runs the same per-GPU workload on its own slice of a global batch of
8*N sequences (batch x head sharding, no collective on the data path: weak
scaling); timing is max over ranks of CUDA-event time.  Rank 0 prints ONE JSON
line.  ``--impl reference`` times the fp64 CPU oracle (the reference arm of
this tier) on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
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
VARIANTS = {
    # configs[1]: FlexAttention-expressible variants, bf16 B=8 H=16 S=8192 D=128
    "causal": dict(B=8, H=16, S=8192, D=128, mask="causal"),
    "vanilla": dict(B=8, H=16, S=8192, D=128),
    "alibi": dict(B=8, H=16, S=8192, D=128, mod="alibi"),
    "sliding": dict(B=8, H=16, S=8192, D=128, mask="sliding", window=1024),
    "softcap": dict(B=8, H=16, S=8192, D=128, mod="softcap", softcap=20.0),
    "document": dict(B=8, H=16, S=8192, D=128, mask="document", n_docs=12),
    "prefix": dict(B=8, H=16, S=8192, D=128, mask="prefix", prefix=256),
    "gqa": dict(B=8, H=16, Hkv=2, S=8192, D=128, mask="causal"),
    # configs[2]: differential attention bf16 B=8 H=16 S=8192 D=64 (two maps, lambda)
    "diff": dict(B=8, H=16, S=8192, D=64, diff=True, lam=0.2),
    # configs[3]: Evoformer gated self-attention with pair bias, N_seq=512 N_res=384 H=8 c=32
    "evo_row": dict(evo="row", B=1, Ns=512, Nr=384, H=8, D=32),
    "evo_col": dict(evo="col", B=1, Ns=512, Nr=384, H=8, D=32),
}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def kept_pairs(cfg, doc_offsets=None, key_mask=None):
    """Exact number of kept (q,k) pairs of the whole workload (per map), from the
    mask definitions (SURVEY §8(d) accounting: masked pairs are not useful work)."""
    S = cfg.get("S")
    if cfg.get("evo"):
        Ns, Nr, B, H = cfg["Ns"], cfg["Nr"], cfg["B"], cfg["H"]
        km = key_mask.numpy().astype(np.int64)          # [B, Ns, Nr]
        if cfg["evo"] == "row":                          # per (b,s,h): Nr queries x kept keys of row s
            return int(km.sum() * Nr * H)
        return int(km.sum() * Ns * H)                    # per (b,i,h): Ns queries x kept keys of column i
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


def flops_per_pair(cfg):
    D = cfg["D"]
    return (2 * D + 2 * D) * (2 if cfg.get("diff") else 1)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None

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
        self.rows = []
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
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ input construction
def make_inputs(cfg, rank, world, device, seed=0):
    """Rank `rank`'s slice of the global problem (global batch = B * world)."""
    dt = torch.bfloat16
    kw = {}
    if cfg.get("evo"):
        B, Ns, Nr, H, c = cfg["B"], cfg["Ns"], cfg["Nr"], cfg["H"], cfg["D"]
        gb = rank * B  # this rank's MSA stacks are global batch indices [rank*B, rank*B+B)
        st = lambda t: synth.uniform((B * world, Ns, Nr, H, c), seed=seed, tensor=t, lead=3,
                                     slab_range=(gb * Ns * Nr, (gb + B) * Ns * Nr)).reshape(B, Ns, Nr, H, c)
        Q, K, V = st("q"), st("k"), st("v")
        Gt = synth.uniform((B * world, Ns, Nr, H, c), seed=seed, tensor="gate", lo=-4, hi=4, lead=3,
                           slab_range=(gb * Ns * Nr, (gb + B) * Ns * Nr)).reshape(B, Ns, Nr, H, c)
        km = torch.ones(B, Ns, Nr, dtype=torch.uint8)     # all-ones MSA mask (bench); tests use 10% zeros
        host = {"Q": Q, "K": K, "V": V, "G": Gt, "km": km}
        if cfg["evo"] == "row":
            view = lambda t: t.permute(0, 1, 3, 2, 4)
            pb = synth.pair_bias((B * world, H, Nr, Nr), seed=seed, lead=2,
                                 slab_range=(gb * H, (gb + B) * H)).reshape(B, H, Nr, Nr)
            host["pb"] = pb
        else:
            view = lambda t: t.permute(0, 2, 3, 1, 4)
        dev = {n: t.to(device) for n, t in host.items()}
        q, k, v = view(dev["Q"]), view(dev["K"]), view(dev["V"])
        kw = dict(gate_mode="sigmoid", gate=view(dev["G"]))
        if cfg["evo"] == "row":
            kw["bias"] = dev["pb"].unsqueeze(1).expand(B, Ns, H, Nr, Nr)
            kw["key_mask"] = dev["km"]
        else:
            kw["key_mask"] = dev["km"].permute(0, 2, 1)
        out = torch.empty(q.shape, dtype=dt, device=device)
        return (q, k, v, out, kw, host)
    B, H, S, D = cfg["B"], cfg["H"], cfg["S"], cfg["D"]
    Hkv = cfg.get("Hkv", H)
    maps = 2 if cfg.get("diff") else 1
    gB = B * world
    lead = 2
    def gen(t, heads):
        return synth.uniform((gB, heads, S, D), seed=seed, tensor=t, lead=lead,
                             slab_range=(rank * B * heads, (rank + 1) * B * heads)).reshape(B, heads, S, D)
    host = {"q": gen("q", H * maps), "k": gen("k", Hkv * maps), "v": gen("v", Hkv)}
    for key in ("mod", "softcap", "mask", "window", "prefix", "diff", "lam"):
        if key in cfg:
            kw[key] = cfg[key]
    if cfg.get("mask") == "document":
        offs = synth.doc_offsets(gB, S, cfg["n_docs"], seed=1)[rank * B:(rank + 1) * B]
        kw["doc_offsets"] = torch.from_numpy(offs)
        host["doc_offsets"] = offs
    q, k, v = (host[n].to(device) for n in ("q", "k", "v"))
    if "doc_offsets" in kw:
        kw["doc_offsets"] = kw["doc_offsets"].to(device)
    out = torch.empty(B, H, S, D, dtype=dt, device=device)
    return (q, k, v, out, kw, host)


def oracle_kwargs(cfg, kw, host):
    import oracle  # noqa: F401  (cpu_baseline / reference legs only)
    ok = {k: v for k, v in kw.items() if k in ("mod", "softcap", "mask", "window", "prefix", "diff", "lam")}
    if "doc_offsets" in host:
        ok["doc_offsets"] = host["doc_offsets"]
    return ok


def time_oracle(cfg, host, kw, budget_s=15.0):
    """Time the fp64 oracle (as it stands) on a bounded row sample; returns
    (useful TFLOP/s, threads, description)."""
    import oracle
    if cfg.get("evo"):
        B, Ns, Nr, H = cfg["B"], cfg["Ns"], cfg["Nr"], cfg["H"]
        view = (lambda t: t.permute(0, 1, 3, 2, 4)) if cfg["evo"] == "row" else (lambda t: t.permute(0, 2, 3, 1, 4))
        q, k, v = view(host["Q"]), view(host["K"]), view(host["V"])
        ok = dict(gate_mode="sigmoid", gate=view(host["G"]))
        if cfg["evo"] == "row":
            ok["bias"] = host["pb"].unsqueeze(1).expand(B, Ns, H, Nr, Nr)
            ok["key_mask"] = host["km"]
        else:
            ok["key_mask"] = host["km"].permute(0, 2, 1)
        total_rows = B * q.shape[1] * H * q.shape[3]
        Sq = q.shape[3]
    else:
        q, k, v = host["q"], host["k"], host["v"]
        ok = oracle_kwargs(cfg, kw, host)
        Sq = cfg["S"]
        total_rows = cfg["B"] * cfg["H"] * Sq
    # sample rows evenly over the flat (b,g,h,q) space so masked work is represented
    n = 256
    pairs_total = kept_pairs(cfg, host.get("doc_offsets"), host.get("km"))
    rows = np.linspace(0, total_rows - 1, n).astype(np.int64)
    t0 = time.perf_counter()
    oracle.attn(q, k, v, rows=rows, **ok)
    dt = time.perf_counter() - t0
    # scale the sample so one measurement is ~budget_s of CPU work (bounded)
    n2 = int(min(total_rows, max(n, n * budget_s / max(dt, 1e-3))))
    n2 = min(n2, 65536)
    rows = np.linspace(0, total_rows - 1, n2).astype(np.int64)
    t0 = time.perf_counter()
    oracle.attn(q, k, v, rows=rows, **ok)
    dt = time.perf_counter() - t0
    flops = pairs_total * flops_per_pair(cfg) * (n2 / total_rows)
    return flops / dt / 1e12, oracle.num_threads(), f"{n2} of {total_rows} output rows (evenly spaced), full workload rate extrapolated by row share", dt


def dist_setup(args):
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


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    _, _, _, _, kw, host = make_inputs(cfg, 0, 1, "cpu")
    vals = []
    for i in range(args.warmup + args.steps):
        v, cores, sample, dt = time_oracle(cfg, host, kw, budget_s=max(2.0, 60.0 / (args.steps + args.warmup)))
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(cfg, args.variant), "variant": args.variant},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_name(cfg, variant):
    if cfg.get("evo"):
        return f"evoformer_{cfg['evo']}_bf16_Nseq{cfg['Ns']}_Nres{cfg['Nr']}_H{cfg['H']}_c{cfg['D']}"
    return f"{variant}_bf16_B{cfg['B']}_H{cfg['H']}_S{cfg['S']}_D{cfg['D']}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--variant", default="causal", choices=sorted(VARIANTS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(VARIANTS[args.variant])
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    from paper_2511_02043_b200 import fl
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    q, k, v, out, kw, host = make_inputs(cfg, rank, world, device)
    stream = torch.cuda.current_stream(device)
    pairs = kept_pairs(cfg, host.get("doc_offsets"), host.get("km"))
    flops = pairs * flops_per_pair(cfg)                    # useful FLOPs per step on this rank
    workspace = torch.empty(1 << 20, dtype=torch.uint8, device=device)

    def step():
        fl.attn_fwd(q, k, v, out=out, workspace=workspace, **kw)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    fl.launch_count(reset=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    launches = fl.launch_count()
    total_ms = t0.elapsed_time(t1)
    per_launch_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([total_ms, per_launch_ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, per_launch_ms = float(tt[0]), float(tt[1])
    ms_per_step = total_ms / args.steps
    value = flops * world / (ms_per_step * 1e-3) / 1e12     # whole-job aggregate

    # ---- end-to-end through the host-buffer C-ABI entry (H2D + kernel + D2H per step)
    e2e = None
    if not args.no_e2e and not cfg.get("evo"):
        runner = fl.HostRunner(device)
        hq, hk, hv = (host[n].pin_memory() for n in ("q", "k", "v"))
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        hkw = dict(kw)
        if "doc_offsets" in hkw:
            hkw["doc_offsets"] = torch.from_numpy(host["doc_offsets"])
        for _ in range(2):
            runner(hq, hk, hv, hout, stream=stream, **hkw)
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 10))
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(n_e2e):
            runner(hq, hk, hv, hout, stream=stream, **hkw)
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(a1) / n_e2e
        if world > 1:
            tt = torch.tensor([e2e_ms], device=device)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(tt[0])
        h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv))
        e2e = {"value": flops * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(hout.numel() * hout.element_size()),
               "ms_per_step": e2e_ms}

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
        return
    pk, pk_src = peaks()
    achieved = flops / (per_launch_ms * 1e-3) / 1e12
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get(args.variant, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": achieved / pk["bf16_tflops"], "traffic": traffic, "peak_source": pk_src,
            "frac_of_sustained": achieved / pk.get("bf16_tflops_sustained", pk["bf16_tflops"])}
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_name(cfg, args.variant), "variant": args.variant,
                       "global_batch": cfg.get("B", 1) * world, "seq_len": cfg.get("S", cfg.get("Nr")),
                       "parallelism": f"batch-x-head shards dp{world}, no collective",
                       "useful_tflop_per_step_per_gpu": flops / 1e12,
                       "l2": "inputs larger than L2 (per-GPU working set > 126 MB)"},
            "roofline": roof, "gpu_launches": int(launches), "clocks": clk.summary()}
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        v_cpu, cores, sample, _ = time_oracle(cfg, host, kw)
        line["cpu_baseline"] = {"value": v_cpu, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
