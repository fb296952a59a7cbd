"""Per-rank shards of a fixed problem: the attention forward partitions into
independent units with no exchange step -- Flashlight's p-dims are "data-independent ...
embarrassingly parallel" (§3.1) and the outer dims of the logical grid (§3.6)
are what is split across GPUs.  Units are linearised outer-major (h-major (h, b) for the LLM configs,
so every rank gets whole heads across all batches and per-batch document offsets balance out; MSA
rows s or residue columns i for the Evoformer configs) and each rank takes the contiguous range
``fl_shard_range`` (include/fl_attn.h) gives it.  A range is returned as at most three rectangles of
the (outer, inner) grid, each one ``fl_attn_fwd`` call on strided views.  No collective.
"""
from __future__ import annotations

from typing import List, Tuple

from . import fl


def unit_blocks(n_outer: int, n_inner: int, world: int, rank: int) -> List[Tuple[int, int, int, int]]:
    """Rank ``rank``'s units of the grid u = o * n_inner + i as rectangles (o0, o1, i0, i1)."""
    u0, u1 = fl.shard_range(n_outer * n_inner, world, rank)
    blocks = []
    u = u0
    while u < u1:
        o, i = divmod(u, n_inner)
        if i == 0 and u1 - u >= n_inner:
            n = (u1 - u) // n_inner
            blocks.append((o, o + n, 0, n_inner))
            u += n * n_inner
        else:
            e = min(u1, (o + 1) * n_inner)
            blocks.append((o, o + 1, i, e - o * n_inner))
            u = e
    return blocks


def range_1d(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank ``rank``'s contiguous range of n units (MSA rows / residue columns)."""
    return fl.shard_range(n, world, rank)
