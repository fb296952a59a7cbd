"""Evoformer MSA row attention with pair bias (AlphaFold2 Alg.7; the paper's second workload)
as a chain of this package's kernels -- argument marshalling only, every step runs in libfl_attn.so:

  1-4  m <- LayerNorm(m); q | k | v | g = m W_qkvg^T (+ b_g)     one fl_linear (LN prologue, N = 4 H c)
  3    b = LayerNorm(z) W_b^T, written head-major [H, i, j]      one fl_linear (strided epilogue)
  5-6  o = sigmoid(g) * softmax(q k^T / sqrt(c) + b) v           fl_attn_fwd (row attention, reading G9)
  7    m~ = o W_o^T + b_o                                        one fl_linear

The attention reads q, k, v, g in place as strided [B, G = s, H, S = i, c] views of the projection output
(rows (s, i), columns h c), and writes o into a [B, N_seq, N_res, H, c] buffer that the output
projection reads as [N_seq N_res, H c] rows.  SURVEY §8(f) NEXT-2 (prologue / epilogue passes) and NEXT-4
(a synthetic-weights Evoformer block)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

from . import fl


@dataclass
class RowAttnWeights:
    """AF2 Alg.7 parameters (bf16 weights in the PyTorch Linear [out, in] layout, f32 vectors)."""
    ln_m_g: torch.Tensor      # [c_m]
    ln_m_b: torch.Tensor      # [c_m]
    w_qkvg: torch.Tensor      # [4 H c, c_m]: rows q | k | v | g, head-major within each block
    b_qkvg: torch.Tensor      # [4 H c]: zero for q, k, v (LinearNoBias), the gate bias for g
    ln_z_g: torch.Tensor      # [c_z]
    ln_z_b: torch.Tensor      # [c_z]
    w_b: torch.Tensor         # [H, c_z]
    w_o: torch.Tensor         # [c_m, H c]
    b_o: torch.Tensor         # [c_m]
    H: int
    c: int


def synthetic_weights(c_m=256, c_z=128, H=8, c=32, seed=0, device="cuda") -> RowAttnWeights:
    """Random-init weights of the block's shapes (no trained checkpoint exists here): Linear weights
    U(-1, 1)/sqrt(fan_in) (bf16), LayerNorm gamma ~ 1 + U(-0.1, 0.1), beta ~ U(-0.1, 0.1), biases ~ U(-0.5, 0.5)."""
    g = torch.Generator().manual_seed(seed)
    u = lambda *s: torch.rand(*s, generator=g) * 2 - 1
    hc = H * c
    b = torch.zeros(4 * hc)
    b[3 * hc:] = 0.5 * u(hc)
    return RowAttnWeights(
        ln_m_g=(1 + 0.1 * u(c_m)).to(device), ln_m_b=(0.1 * u(c_m)).to(device),
        w_qkvg=(u(4 * hc, c_m) / c_m ** 0.5).to(torch.bfloat16).to(device), b_qkvg=b.to(device),
        ln_z_g=(1 + 0.1 * u(c_z)).to(device), ln_z_b=(0.1 * u(c_z)).to(device),
        w_b=(u(H, c_z) / c_z ** 0.5).to(torch.bfloat16).to(device),
        w_o=(u(c_m, hc) / hc ** 0.5).to(torch.bfloat16).to(device), b_o=(0.5 * u(c_m)).to(device), H=H, c=c)


class RowAttnBlock:
    """Buffers for one (N_seq, N_res) shape, reused across calls (so a CUDA graph can capture __call__)."""

    def __init__(self, w: RowAttnWeights, n_seq: int, n_res: int, device="cuda", eps: float = 1e-5):
        self.w, self.eps = w, eps
        self.Ns, self.Nr = n_seq, n_res
        hc = w.H * w.c
        self.proj = torch.empty(n_seq, n_res, 4 * hc, device=device, dtype=torch.bfloat16)
        self.bias = torch.empty(w.H, n_res, n_res, device=device, dtype=torch.bfloat16)
        self.o = torch.empty(1, n_seq, n_res, w.H, w.c, device=device, dtype=torch.bfloat16)
        self.out = torch.empty(n_seq, n_res, w.ln_m_g.numel(), device=device, dtype=torch.bfloat16)
        self.ws = None

    def views(self):
        """[B=1, G=s, H, S=i, c] views of the projection's q | k | v | g column blocks (no copies)."""
        H, c, Ns, Nr = self.w.H, self.w.c, self.Ns, self.Nr
        blk = lambda i: self.proj[:, :, i * H * c:(i + 1) * H * c].reshape(1, Ns, Nr, H, c).permute(0, 1, 3, 2, 4)
        return blk(0), blk(1), blk(2), blk(3)

    def __call__(self, m: torch.Tensor, z: torch.Tensor, msa_mask: Optional[torch.Tensor] = None) -> torch.Tensor:
        """m: bf16 [N_seq, N_res, c_m]; z: bf16 [N_res, N_res, c_z]; msa_mask: u8 [1, N_seq, N_res] or None."""
        w, Ns, Nr = self.w, self.Ns, self.Nr
        fl.linear(m, w.w_qkvg, bias=w.b_qkvg, ln_gamma=w.ln_m_g, ln_beta=w.ln_m_b, eps=self.eps, out=self.proj)
        fl.linear(z, w.w_b, ln_gamma=w.ln_z_g, ln_beta=w.ln_z_b, eps=self.eps,
                  out=self.bias.view(w.H, Nr * Nr).t())
        q, k, v, g = self.views()
        kw = dict(gate_mode="sigmoid", gate=g, bias=self.bias.unsqueeze(0).unsqueeze(0).expand(1, Ns, w.H, Nr, Nr))
        if msa_mask is not None:
            kw["key_mask"] = msa_mask
        fl.attn_fwd(q, k, v, out=self.o.permute(0, 1, 3, 2, 4), **kw)
        fl.linear(self.o.view(Ns * Nr, w.H * w.c), w.w_o, bias=w.b_o, out=self.out.view(Ns * Nr, -1))
        return self.out
