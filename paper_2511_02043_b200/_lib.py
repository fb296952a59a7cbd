"""ctypes mirror of include/fl_attn.h (argument marshalling only).

Loading is lazy; if libfl_attn.so is missing the first call raises -- there is
no CPU or library fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libfl_attn.so")

FL_BF16, FL_F32, FL_U8, FL_I32 = 0, 1, 2, 3
ABI_VERSION = 4

EXPORTS = ["fl_attn_fwd", "fl_attn_workspace_size", "fl_attn_host_scratch_size", "fl_attn_fwd_host",
           "fl_rsa_build_summaries", "fl_rsa_update_summaries", "fl_rsa_select", "fl_shard_range", "fl_diag_umma_gemm",
           "fl_diag_pipe_rate", "fl_debug_schedule", "fl_attn_args_size", "fl_attn_bwd_args_size", "fl_attn_bwd",
           "fl_attn_bwd_workspace_size", "fl_status_string", "fl_last_error", "fl_abi_version", "fl_launch_count", "fl_debug_timing",
           "fl_linear", "fl_ipa_fwd", "fl_ipa_workspace_size"]


class Tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("rank", C.c_int32),
                ("size", C.c_int64 * 5), ("stride", C.c_int64 * 5)]


class Variant(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("scale", C.c_float), ("mod", C.c_int32), ("softcap", C.c_float),
        ("alibi_slopes", Tensor), ("mask", C.c_int32), ("window", C.c_int32), ("prefix_len", C.c_int32),
        ("doc_offsets", Tensor), ("doc_causal", C.c_int32), ("causal_align", C.c_int32),
        ("bias", Tensor), ("key_mask", Tensor), ("gate_mode", C.c_int32), ("gate", Tensor),
        ("diff", C.c_int32), ("lambda_", C.c_float), ("lambda_h", Tensor),
        ("blk_idx", Tensor), ("blk_cnt", Tensor), ("blk_q", C.c_int32), ("blk_k", C.c_int32),
        ("kv_page_table", Tensor), ("kv_len", C.c_int32),
        ("lambda_qk", Tensor), ("lambda_init", C.c_float), ("diff_norm", C.c_int32), ("diff_norm_eps", C.c_float),
        ("diff_norm_w", Tensor),
    ]


class AttnArgs(C.Structure):
    _fields_ = [("q", Tensor), ("k", Tensor), ("v", Tensor), ("o", Tensor), ("lse", Tensor),
                ("var", Variant), ("stream", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t)]


class BwdArgs(C.Structure):
    _fields_ = [("q", Tensor), ("k", Tensor), ("v", Tensor), ("o", Tensor), ("lse", Tensor), ("dout", Tensor),
                ("dq", Tensor), ("dk", Tensor), ("dv", Tensor), ("var", Variant), ("stream", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t), ("dgate", Tensor),
                ("dbias", Tensor), ("dlambda", Tensor)]


class LinearArgs(C.Structure):
    _fields_ = [("x", Tensor), ("w", Tensor), ("bias", Tensor), ("ln_gamma", Tensor), ("ln_beta", Tensor),
                ("y", Tensor), ("ln_eps", C.c_float), ("stream", C.c_void_p)]


class IpaArgs(C.Structure):
    _fields_ = [(n, Tensor) for n in ("q", "k", "v", "qp", "kp", "vp", "R", "t", "bias", "z", "gamma", "o", "op",
                                      "opair")] + [("stream", C.c_void_p), ("workspace", C.c_void_p),
                                                   ("workspace_bytes", C.c_size_t)]


class FlError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{status_string(status)}: {detail}")
        self.status = status
        self.detail = detail


_lib = None


def lib():
    """Load libfl_attn.so (raises if it was never built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise FileNotFoundError(
                f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(SO_PATH)
        L.fl_attn_fwd.argtypes = [C.POINTER(AttnArgs)]
        L.fl_attn_workspace_size.argtypes = [C.POINTER(AttnArgs), C.POINTER(C.c_size_t)]
        L.fl_attn_host_scratch_size.argtypes = [C.POINTER(AttnArgs), C.POINTER(C.c_size_t)]
        L.fl_attn_fwd_host.argtypes = [C.POINTER(AttnArgs), C.c_void_p, C.c_size_t]
        L.fl_rsa_build_summaries.argtypes = [C.POINTER(Tensor), C.POINTER(Tensor), C.POINTER(Tensor), C.c_int32,
                                             C.c_void_p]
        L.fl_rsa_update_summaries.argtypes = [C.POINTER(Tensor), C.POINTER(Tensor), C.POINTER(Tensor), C.c_int32,
                                              C.c_int64, C.c_void_p]
        L.fl_rsa_select.argtypes = [C.POINTER(Tensor), C.POINTER(Tensor), C.POINTER(Tensor), C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_int32, C.POINTER(Tensor), C.POINTER(Tensor),
                                    C.c_void_p]
        L.fl_shard_range.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.fl_shard_range.restype = None
        L.fl_diag_umma_gemm.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_void_p]
        L.fl_diag_pipe_rate.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
        L.fl_diag_pipe_rate.restype = C.c_int
        L.fl_debug_schedule.argtypes = [C.POINTER(AttnArgs), C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int32)]
        L.fl_debug_schedule.restype = C.c_int
        L.fl_ipa_fwd.argtypes = [C.POINTER(IpaArgs)]
        L.fl_ipa_fwd.restype = C.c_int
        L.fl_ipa_workspace_size.argtypes = [C.POINTER(IpaArgs), C.POINTER(C.c_size_t)]
        L.fl_ipa_workspace_size.restype = C.c_int
        L.fl_linear.argtypes = [C.POINTER(LinearArgs)]
        L.fl_linear.restype = C.c_int
        L.fl_attn_bwd.argtypes = [C.POINTER(BwdArgs)]
        L.fl_attn_bwd.restype = C.c_int
        L.fl_attn_bwd_workspace_size.argtypes = [C.POINTER(BwdArgs), C.POINTER(C.c_size_t)]
        L.fl_attn_bwd_workspace_size.restype = C.c_int
        L.fl_status_string.argtypes = [C.c_int]
        L.fl_status_string.restype = C.c_char_p
        L.fl_last_error.restype = C.c_char_p
        L.fl_abi_version.restype = C.c_int32
        L.fl_debug_timing.argtypes = [C.POINTER(C.c_uint64), C.c_int32]
        L.fl_debug_timing.restype = C.c_int
        L.fl_launch_count.argtypes = [C.c_int32]
        L.fl_launch_count.restype = C.c_int64
        for name in ("fl_attn_fwd", "fl_attn_workspace_size", "fl_attn_host_scratch_size", "fl_attn_fwd_host",
                     "fl_rsa_build_summaries", "fl_rsa_update_summaries", "fl_rsa_select", "fl_diag_umma_gemm"):
            getattr(L, name).restype = C.c_int
        if L.fl_abi_version() != ABI_VERSION:
            raise RuntimeError("libfl_attn.so ABI version mismatch")
        L.fl_attn_args_size.restype = C.c_size_t
        if L.fl_attn_args_size() != C.sizeof(AttnArgs):
            raise RuntimeError(f"libfl_attn.so was built for a different fl_attn_args layout "
                               f"({L.fl_attn_args_size()} vs {C.sizeof(AttnArgs)} bytes): rebuild it")
        L.fl_attn_bwd_args_size.restype = C.c_size_t
        if L.fl_attn_bwd_args_size() != C.sizeof(BwdArgs):
            raise RuntimeError(f"libfl_attn.so was built for a different fl_attn_bwd_args layout "
                               f"({L.fl_attn_bwd_args_size()} vs {C.sizeof(BwdArgs)} bytes): rebuild it")
        _lib = L
    return _lib


def status_string(s: int) -> str:
    try:
        return lib().fl_status_string(s).decode()
    except Exception:  # pragma: no cover
        return f"status {s}"


def check(status: int) -> None:
    if status != 0:
        raise FlError(status, lib().fl_last_error().decode())
