#!/usr/bin/env python
"""Per-phase cycle breakdown of the bf16 kernel's softmax warpgroups (needs a -DFL_TIMING build:
FL_TIMING=1 python -c 'from paper_2511_02043_b200 import build; build.build()').

    python tools/timing_probe.py [variant ...]      (variants of bench.py, one launch each)
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_02043_b200 import _lib, fl  # noqa: E402

NAMES = ["bookkeeping", "S wait", "S tmem.ld", "score+mask+max", "O rescale", "ping-pong wait", "exp loop",
         "P store+arrive", "tail", "bias wait", "epilogue", "unit id wait", "unit setup"]


def main():
    variants = sys.argv[1:] or ["causal"]
    dev = torch.device("cuda", 0)
    buf = (C.c_uint64 * 48)()
    for v in variants:
        job = bench.make_job(v, 0, 1, dev, with_host=False)
        call = job.calls[-1]
        call.fn()
        torch.cuda.synchronize()
        _lib.check(_lib.lib().fl_debug_timing(buf, 1))          # reset
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call.fn()
        e1.record()
        torch.cuda.synchronize()
        _lib.check(_lib.lib().fl_debug_timing(buf, 0))
        ms = e0.elapsed_time(e1)
        print(f"== {v}: {ms:.3f} ms (timing build), {call.flops / ms / 1e9:.1f} TFLOP/s")
        for wg in range(2):
            tiles = buf[wg * 16 + 15]
            tot = sum(buf[wg * 16 + i] for i in range(13))
            print(f"  WG{wg}: {tiles} tiles (thread 0 of each CTA, summed), {tot / max(tiles, 1):.0f} cycles/tile")
            for i, n in enumerate(NAMES):
                c = buf[wg * 16 + i]
                print(f"    {n:16s} {c / max(tiles, 1):8.0f} cyc/tile  {100 * c / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main()
