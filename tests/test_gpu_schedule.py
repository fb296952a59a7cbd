"""T2 scheduler / tile-classifier test (-m gpu): the persistent kernel's
work decomposition and KV-tile classes, dumped on the device by the kernel's own decode_work / needs /
tile_inside (fl_debug_schedule), against brute-force enumeration of the oracle's kept-key predicate
(oracle.keep_rows, definition step 2).  Checks, for every variant and shape:
  * the linearised unit ids invert onto the (b, g, h, q) rows exactly once (a1, §3.6),
  * every tile holding a kept key of a row is run by that row's warpgroup (no dropped work),
  * a tile run mask-free by a warp has all 128 keys kept for all 32 of its rows (no missing mask),
  * no run tile is empty for every row of its warpgroup (a2: skipped tiles are skipped)."""
import numpy as np
import pytest
import torch

import oracle
from tests import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl as _fl
    return _fl


SCHED_CASES = [
    dict(name="causal", B=2, Hq=2, S=1000, D=128, mask="causal"),
    dict(name="vanilla_ragged", S=333, D=64),
    dict(name="sliding", S=1500, D=128, mask="sliding", window=300),
    dict(name="sliding_w0", S=400, D=64, mask="sliding", window=0),
    dict(name="prefix", S=900, D=64, mask="prefix", prefix=200),
    dict(name="document", B=2, S=1700, D=128, mask="document", n_docs=7),
    dict(name="document_causal", B=2, S=1200, D=64, mask="document", n_docs=5, doc_causal=True),
    dict(name="sq_lt_sk_bottom_right", Sq=300, Sk=1000, D=128, mask="causal"),
    dict(name="sq_lt_sk_top_left", Sq=300, Sk=1000, D=128, mask="causal", causal_align=1),
    dict(name="diff_causal", Hq=2, S=700, D=64, diff=True, lam=0.3, mask="causal"),
    dict(name="gqa", Hq=4, Hkv=2, S=600, D=128, mask="causal"),
]


def _check(rec, keep_of, B, G, H, Sq, Sk, maps=1):
    mt = rec.shape[1] - 8
    seen = np.zeros((B, G, H, Sq), dtype=np.int32)
    waste = 0
    for r in rec:
        u, wg, b, g, h, q0, lo, hi = (int(x) for x in r[:8])
        codes = r[8:]
        if g >= G:                                     # PAIR: the idle half of the last row pair
            assert (codes == -1).all()
            continue
        rows = np.arange(q0, min(q0 + 128, Sq))
        if rows.size == 0:
            assert (codes == -1).all()
            continue
        seen[b, g, h, rows] += 1
        keep = keep_of(b, g, h, rows)                  # [len(rows), Sk] bool
        for j in range(mt):
            kt = keep[:, j * 128:(j + 1) * 128]
            if codes[j] < 0:
                assert not kt.any(), f"unit {u} wg {wg}: tile {j} holds kept keys but is not run"
                continue
            if not kt.any():
                waste += 1
            for w in range(4):
                if not (codes[j] >> w) & 1:            # mask-free for warp w: every key of its rows kept
                    sub = kt[w * 32:(w + 1) * 32]
                    assert sub.shape[1] == 128 and sub.all(), f"unit {u} wg {wg} tile {j} warp {w} skips a needed mask"
    # differential attention: warpgroup i computes map i of the same rows (G8) -> every row twice
    assert (seen == maps).all(), "unit decomposition does not cover every row exactly once per map"
    return waste


@pytest.mark.parametrize("case", SCHED_CASES, ids=[c["name"] for c in SCHED_CASES])
def test_schedule_dump_matches_keep_predicate(fl, case):
    ins, gk, ok = cases.build(dict(case, dtype="bf16"))
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    rec = fl.debug_schedule(q, k, v, **kw)
    B, Hq = q.shape[0], q.shape[1] // (2 if case.get("diff") else 1)
    Sq, Sk = q.shape[2], k.shape[2]

    def keep_of(b, g, h, rows):
        ids = ((b * 1 + g) * Hq + h) * Sq + rows
        return oracle.keep_rows(ins["q"], ins["k"], ins["v"], ids, **ok).astype(bool)
    waste = _check(rec, keep_of, B, 1, Hq, Sq, Sk, maps=2 if case.get("diff") else 1)
    assert waste == 0, f"{waste} run tiles hold no kept key"


@pytest.mark.parametrize("Ns,Nr,kind", [(5, 130, "row"), (4, 384, "row"), (7, 300, "row"), (3, 200, "col")])
def test_schedule_dump_evoformer_views(fl, Ns, Nr, kind):
    """Rank-5 strided views and the paired-G units (PAIR: two MSA rows per unit when S_q % 256 <= 128)."""
    ins, gk, ok = cases.evoformer(dict(kind=kind, B=1, Ns=Ns, Nr=Nr, H=2, c=32, p_zero=0.0))
    q, k, v = (ins[n].cuda() for n in ("q", "k", "v"))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    rec = fl.debug_schedule(q, k, v, **kw)
    B, G, H, Sq, _ = q.shape
    Sk = k.shape[3]

    def keep_of(b, g, h, rows):
        ids = ((b * G + g) * H + h) * Sq + rows
        return oracle.keep_rows(ins["q"], ins["k"], ins["v"], ids, **ok).astype(bool)
    _check(rec, keep_of, B, G, H, Sq, Sk)
