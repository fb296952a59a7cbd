"""Build libfl_attn.so (the C-ABI library of include/fl_attn.h) in-tree with nvcc.

sm_100a SASS only (-gencode arch=compute_100a,code=sm_100a), -lineinfo for ncu's
source page, static cudart (no dependency on torch's runtime version).  Objects
are compiled in parallel and relinked only when a source is newer than the .so.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "..", "build")
SO = os.path.join(HERE, "libfl_attn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-diag-suppress", "177"]


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(HERE, "..", "include", "fl_attn.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src, extra):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not _stale(obj, [src] + _deps()) and not extra:
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False, extra=None) -> str:
    extra = list(extra or [])
    if os.environ.get("FL_DEBUG_HANG"):
        extra.append("-DFL_DEBUG_HANG")
    if os.environ.get("FL_TIMING"):
        extra.append("-DFL_TIMING")
    extra += os.environ.get("FL_EXTRA", "").split()   # experiment flags, e.g. "-DFL_EMU_MASK=0"
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(lambda s: _compile(s, extra), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(f"== {os.path.basename(o)}\n{log}", file=sys.stderr)
    if _stale(SO, objs) or extra:
        # --no-undefined: a symbol missing from the objects fails the link here, not the dlopen on the GPU box
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-Xlinker", "--no-undefined", "-o", SO, *objs]
        subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
