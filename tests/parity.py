"""Parity checker shared by the GPU tests and bench (compares CUDA output with the
oracle).  The metric follows SURVEY §8(c) "Parity procedure": max-abs error on
the final output, no NaN/Inf, and -- for peaked (needle) and constant-V inputs --
max|ref| >= 0.1 so that a near-zero output cannot pass.  Tolerances are the
north_star's: 2e-2 (bf16 inputs, fp32 accumulate) and 1e-5 (fp32 path)."""
from __future__ import annotations

import numpy as np

TOL = {"bf16": 2e-2, "f32": 1e-5}


def compare(got, ref) -> dict:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    finite = bool(np.isfinite(got).all())
    err = np.abs(got - ref)
    mref = float(np.abs(ref).max()) if ref.size else 0.0
    return {"max_abs": float(err.max()) if err.size else 0.0,
            "rms": float(np.sqrt((err ** 2).mean())) if err.size else 0.0,
            "max_ref": mref,
            "rel": float(err.max() / max(mref, 1e-30)) if err.size else 0.0,
            "finite": finite}


def check(got, ref, tol: float, min_ref: float = 0.0, what: str = "") -> dict:
    r = compare(got, ref)
    assert r["finite"], f"{what}: NaN/Inf in output"
    assert r["max_abs"] <= tol, f"{what}: max-abs {r['max_abs']:.3e} > {tol:g} ({r})"
    assert r["max_ref"] >= min_ref, f"{what}: max|ref| {r['max_ref']:.3e} < {min_ref} -- check too weak"
    return r
