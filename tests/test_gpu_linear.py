"""NEXT-2 parity (-m gpu): fl_linear (fused LayerNorm-prologue tcgen05 linear, AF2 Alg.7 lines 1-4 and 7)
against the fp64 oracle (oracle.linear_ln, pinned in tests/test_oracle_pins.py).  Inputs are bf16 (what
both sides read); the bound is derived from the kernel's arithmetic: xhat is rounded to bf16 before the
product (|dxhat| <= 2^-9 |xhat|, so <= 2^-9 sum_k |xhat||w| on y) and y to bf16 (<= 2^-9 |y|); fp32 LN
statistics and accumulation add ~1e-6 relative.  Checked with 2x slack: |y - ref| <= 2^-8 (yabs + |ref|)
+ 1e-4, element by element."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_02043_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import fl as _fl
    return _fl


def _inputs(M, K, N, seed, ln=True, bias=True):
    x = synth.uniform((M, K), seed=seed, tensor="q", dtype=torch.bfloat16) * 3
    x = x.to(torch.bfloat16)
    w = (synth.uniform((N, K), seed=seed, tensor="k", dtype=torch.float32) / np.sqrt(K)).to(torch.bfloat16)
    g = torch.Generator().manual_seed(seed)
    gam = (torch.rand(K, generator=g) + 0.5) if ln else None
    bet = (torch.rand(K, generator=g) - 0.5) if ln else None
    b = (torch.rand(N, generator=g) - 0.5) if bias else None
    return x, w, gam, bet, b


def _check(got, x, w, gam, bet, b, eps, what):
    ref, ya = oracle.linear_ln(x, w, bias=b, ln_gamma=gam, ln_beta=bet, eps=eps, with_abs=True)
    got = got.double().cpu().numpy()
    bound = 2.0 ** -8 * (ya + np.abs(ref)) + 1e-4
    err = np.abs(got - ref)
    assert np.abs(ref).max() > 0.5, what
    assert (err <= bound).all(), f"{what}: max err {err.max():.3e}, worst ratio {(err / bound).max():.2f}"


CASES = [
    dict(M=300, K=256, N=1024, ln=True, bias=True),     # Evoformer q|k|v|g projection (c_m = 256, 4 H c)
    dict(M=1000, K=256, N=256, ln=False, bias=True),    # output projection (H c = 256 -> c_m)
    dict(M=129, K=128, N=48, ln=True, bias=False),      # ragged M, N < 256, not a multiple of 32
    dict(M=64, K=64, N=16, ln=True, bias=True),         # one partial row tile, smallest N tile
    dict(M=517, K=192, N=300, ln=False, bias=False),    # K = 192, two N tiles (256 + ragged 44)
]


@pytest.mark.parametrize("c", CASES, ids=lambda c: "M{M}-K{K}-N{N}-ln{ln}-b{bias}".format(**c))
def test_linear_vs_oracle(fl, c):
    x, w, gam, bet, b = _inputs(c["M"], c["K"], c["N"], seed=c["M"], ln=c["ln"], bias=c["bias"])
    cu = lambda t: None if t is None else t.cuda()
    y = fl.linear(x.cuda(), w.cuda(), bias=cu(b), ln_gamma=cu(gam), ln_beta=cu(bet), eps=1e-5)
    torch.cuda.synchronize()
    _check(y, x, w, gam, bet, b, 1e-5, str(c))


def test_linear_strided_output(fl):
    """Pair-bias layout (AF2 Alg.7 line 3): rows (i, j) of LN(z) [N_r^2, c_z] projected to H = 8 heads and
    written head-major [H, i, j] through a transposed output view (y strides (1, N_r^2))."""
    Nr, cz, H = 40, 128, 8
    x, w, gam, bet, _ = _inputs(Nr * Nr, cz, H, seed=5, bias=False)
    out = torch.empty(H, Nr * Nr, device="cuda", dtype=torch.bfloat16)
    fl.linear(x.cuda(), w.cuda(), ln_gamma=gam.cuda(), ln_beta=bet.cuda(), out=out.t())
    torch.cuda.synchronize()
    _check(out.t(), x, w, gam, bet, None, 1e-5, "strided pair bias")


def test_linear_errors_are_loud(fl):
    x = torch.zeros(4, 96, device="cuda", dtype=torch.bfloat16)
    w = torch.zeros(8, 96, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(fl.FlError, match="UNSUPPORTED"):
        fl.linear(x, w)                                 # K = 96 not in {64, 128, 192, 256}
    x = torch.zeros(4, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(fl.FlError, match="SHAPE"):
        fl.linear(x, torch.zeros(8, 128, device="cuda", dtype=torch.bfloat16))
