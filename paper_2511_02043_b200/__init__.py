"""B200-native (sm_100a) fused attention-variant forward -- the hot path of
Flashlight (arXiv 2511.02043), behind the C-ABI in include/fl_attn.h.

Importing the package is cheap; the CUDA library is loaded on first use by
``paper_2511_02043_b200.fl`` (see ``_lib.py``), and every entry point raises if
it is missing: there is no CPU fallback.
"""
__all__ = ["fl", "synth"]
