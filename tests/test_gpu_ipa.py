"""NEXT-4 parity (-m gpu): the Invariant Point Attention core (fl_ipa_fwd: augmented 64-column tensor-core
contraction for the point-distance logits + the fused attention kernel + the pair / point output kernel)
against the fp64 oracle (oracle.ipa, reading G23, pinned in tests/test_oracle_pins.py) on protein-like
inputs (12 heads x 16; AF2's 4 query and 8 value points, c_z = 128).
Bars: o and the pair output 2e-2 max-abs (G20; |v|, |z| <= 1) with max|ref| >= 0.1; the point output,
whose values are global coordinates of up to |t| + 4 sqrt(3) A, within 2^-7 of that scale -- the logits
carry bf16 rounding of order 2^-8 (relative weight error <= 2^-8, twice that on a convex combination)."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2511_02043_b200 import synth
from tests.parity import check

pytestmark = pytest.mark.gpu


IPA_CASES = [dict(N=100), dict(N=300),
             # ragged row block (77 % 16), one head group of 5, 4 value points, c_z = 64 (half the feature lanes)
             dict(N=77, H=5, Pv=4, cz=64),
             # three key chunks (520 = 2 x 256 + 8), head groups 6 + 1, c_z = 192 (two feature passes)
             dict(N=520, H=7, cz=192)]


@pytest.mark.parametrize("case", IPA_CASES, ids=lambda c: "_".join(f"{k}{v}" for k, v in c.items()))
def test_ipa_vs_oracle(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl
    N = case["N"]
    x = synth.ipa_inputs(seed=N, **case)
    dev = {k: v.cuda() for k, v in x.items()}
    o, op, opair = fl.ipa_fwd(**dev)
    torch.cuda.synchronize()
    ro, rop, ropair = oracle.ipa(**x)
    check(o.cpu().double().numpy(), ro, 2e-2, min_ref=0.1, what=f"ipa o N{N}")
    check(opair.cpu().double().numpy(), ropair, 2e-2, min_ref=0.1, what=f"ipa opair N{N}")
    scale = float(x["t"].abs().max()) + 4 * math.sqrt(3)
    r = check(op.cpu().double().numpy(), rop, 2 ** -7 * scale, min_ref=1.0, what=f"ipa op N{N}")
    assert np.isfinite(r["max_abs"])


def test_ipa_global_motion_invariance_on_gpu():
    """The GPU outputs (not only the oracle's) are invariant under a global rigid motion of the frames, up to
    the same rounding bound -- the property the hi/lo split of the global coordinates protects."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl
    x = synth.ipa_inputs(200, seed=7)
    G = torch.tensor([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    y = dict(x, R=(G @ x["R"]).contiguous(), t=(x["t"] @ G.T + torch.tensor([30.0, -20.0, 10.0])).contiguous())
    a = fl.ipa_fwd(**{k: v.cuda() for k, v in x.items()})
    b = fl.ipa_fwd(**{k: v.cuda() for k, v in y.items()})
    torch.cuda.synchronize()
    assert (a[0].float() - b[0].float()).abs().max().item() < 2e-2
    assert (a[2].float() - b[2].float()).abs().max().item() < 2e-2
    assert (a[1] - b[1]).abs().max().item() < 2 ** -7 * (float(y["t"].abs().max()) + 7)


def test_ipa_unsupported_is_loud():
    """P_v outside {0, 4, 8} (the float4 point sums) is refused with FL_ERR_UNSUPPORTED, not computed wrongly."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl
    x = synth.ipa_inputs(40, Pv=3, seed=1)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.ipa_fwd(**{k: v.cuda() for k, v in x.items()})
