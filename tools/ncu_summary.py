#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run HERE, no GPU needed).

    python tools/ncu_summary.py full <name> <report.ncu-rep|raw.csv> [variant]   # one --set full capture
    python tools/ncu_summary.py launches <name> <launches.csv>           # gpu__time_duration launch list

`full` updates profiles/ncu_summary.json[variant] (bench.py reads
dram_bytes_per_launch from it for roofline.traffic) and writes
profiles/<name>.txt with the metrics that justify the design choices.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.per_cycle_active", "smsp__sass_inst_executed_op_tmem_ldt.sum",
    "smsp__sass_inst_executed_op_tmem_stt.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3,
        "us": 1e-6, "ns": 1e-9, "nsecond": 1e-9, "second": 1.0, "Ghz": 1e9, "Mhz": 1e6}


def _val(vals, key, default=None):
    v = vals.get(key)
    return v[0] * UNIT.get(v[1], 1.0) if v else default


def full(name, rep, variant):
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    raw = raw[raw.index('"ID"'):] if '"ID"' in raw else raw
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out_lines, summ = [f"ncu --set full capture {os.path.basename(rep)} (clock-control none)"], {}
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        kname = rec.get("Kernel Name", "?")
        vals = {}
        for k in KEYS:
            if k in rec and rec[k] not in ("", "n/a"):
                try:
                    vals[k] = (float(rec[k].replace(",", "")), units[hdr.index(k)])
                except ValueError:
                    pass
        out_lines.append(f"kernel: {kname}")
        for k, (v, u) in vals.items():
            out_lines.append(f"  {k:78s} {v:>16.4f} {u}")
        dr, dw = _val(vals, "dram__bytes_read.sum"), _val(vals, "dram__bytes_write.sum")
        if dr is not None and dw is not None:
            short = kname.split("(")[0].replace("void ", "").split("<")[0].strip()
            summ[short] = {"kernel": kname, "dram_bytes_per_launch": dr + dw,
                    "ncu_duration_s": _val(vals, "gpu__time_duration.sum"),
                    "tensor_pipe_pct": _val(vals, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                    "xu_pipe_pct": _val(vals, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                    "fma_pipe_pct": _val(vals, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                    "sm_clock_hz": _val(vals, "sm__cycles_elapsed.avg.per_second"),
                    "source": os.path.basename(rep)}
    os.makedirs(PROF, exist_ok=True)
    open(os.path.join(PROF, f"{name}.txt"), "w").write("\n".join(out_lines) + "\n")
    jp = os.path.join(PROF, "ncu_summary.json")
    allj = json.load(open(jp)) if os.path.exists(jp) else {}
    if len(summ) == 1:
        allj[variant] = next(iter(summ.values()))
    for short, rec in summ.items():
        allj[f"{variant}:{short}"] = rec
    json.dump(allj, open(jp, "w"), indent=1, sort_keys=True)
    print("\n".join(out_lines))


def launches(name, path):
    lines = [l for l in open(path).read().splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    agg = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1e-9))
    tot = sum(sum(v) for v in agg.values())
    out = [f"launch list {os.path.basename(path)}: {sum(len(v) for v in agg.values())} launches, "
           f"{tot * 1e3:.3f} ms total (cold-cache, serialised: compare shares, not absolutes)"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"  {100 * sum(v) / tot:6.2f}%  n={len(v):4d}  mean {1e6 * sum(v) / len(v):10.1f} us  {k}")
    os.makedirs(PROF, exist_ok=True)
    open(os.path.join(PROF, f"{name}.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "causal")
    else:
        launches(sys.argv[2], sys.argv[3])
