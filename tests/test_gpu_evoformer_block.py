"""NEXT-2 / NEXT-4 (-m gpu): the Evoformer MSA row-attention block (AF2 Alg.7) chained from this
package's kernels (paper_2511_02043_b200/evoformer.py: LN+projection fl_linear, pair-bias fl_linear,
fl_attn_fwd, output fl_linear) against the same chain of fp64 oracle steps (oracle.linear_ln, oracle.attn),
with the block's bf16 activations (projections, pair bias, attention output) rounded to bf16 between the
oracle's steps as the data format.  Bar: the north_star's 2e-2 max-abs on the block output (G20), with
max|ref| >= 0.1 so the comparison is not vacuous."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_02043_b200 import synth
from tests.parity import check

pytestmark = pytest.mark.gpu


def _bf(t):
    return torch.as_tensor(t).to(torch.bfloat16)


@pytest.mark.parametrize("Ns,Nr,masked", [(6, 100, False), (5, 300, True)])
def test_row_attention_block_vs_oracle(Ns, Nr, masked):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02043_b200 import evoformer
    H, c, cm, cz = 8, 32, 256, 128
    w = evoformer.synthetic_weights(c_m=cm, c_z=cz, H=H, c=c, seed=1)
    m = synth.uniform((Ns, Nr, cm), seed=2, tensor="q", lead=2) * 2
    z = synth.uniform((Nr, Nr, cz), seed=2, tensor="k", lead=2) * 2
    m, z = _bf(m), _bf(z)
    km = synth.key_mask((1, Ns, Nr), seed=3, p_zero=0.1, lead=2) if masked else None
    blk = evoformer.RowAttnBlock(w, Ns, Nr)
    out = blk(m.cuda(), z.cuda(), None if km is None else km.cuda())
    torch.cuda.synchronize()

    cpu = lambda t: t.detach().cpu()
    proj = _bf(oracle.linear_ln(m, cpu(w.w_qkvg), bias=cpu(w.b_qkvg), ln_gamma=cpu(w.ln_m_g),
                                ln_beta=cpu(w.ln_m_b), eps=1e-5))                       # [Ns, Nr, 4 H c]
    pb = _bf(oracle.linear_ln(z, cpu(w.w_b), ln_gamma=cpu(w.ln_z_g), ln_beta=cpu(w.ln_z_b), eps=1e-5))
    bias = pb.permute(2, 0, 1).contiguous()                                            # [H, i, j]
    blk5 = lambda i: proj[:, :, i * H * c:(i + 1) * H * c].reshape(1, Ns, Nr, H, c).permute(0, 1, 3, 2, 4)
    okw = dict(gate_mode="sigmoid", gate=blk5(3), bias=bias.unsqueeze(0).unsqueeze(0).expand(1, Ns, H, Nr, Nr))
    if km is not None:
        okw["key_mask"] = km
    o, _ = oracle.attn(blk5(0), blk5(1), blk5(2), **okw)                                # [1, Ns, H, Nr, c]
    o = _bf(torch.from_numpy(np.asarray(o)).reshape(1, Ns, H, Nr, c).permute(0, 1, 3, 2, 4).reshape(Ns * Nr, H * c))
    ref = oracle.linear_ln(o, cpu(w.w_o), bias=cpu(w.b_o)).reshape(Ns, Nr, cm)
    check(out.cpu().double().numpy(), ref, 2e-2, min_ref=0.1, what=f"evoformer row block Ns{Ns} Nr{Nr}")
