#!/usr/bin/env python
"""CONTEXT ONLY (SURVEY §8(d) 'optional context'; not a bench line, not on the product path):
on-box PyTorch FlexAttention (torch.compile'd flex_attention, Triton) and SDPA (cuDNN / flash backends)
on the BASELINE configs[1] shapes, timed like bench.py (CUDA events, warm-up, 20 launches), TFLOP/s
of the same useful-pair accounting.  Prints one line per variant.

    python tools/context_flex.py
"""
import sys

import torch
import torch.nn.functional as F

B, H, S, D = 8, 16, 8192, 128
W, CAP, NDOC = 1024, 20.0, 12


def timeit(fn, n=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    from torch.nn.attention.flex_attention import create_block_mask, flex_attention
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.rand(B, H, S, D, device=dev, generator=g, dtype=torch.float32).mul_(2).sub_(1).bfloat16()
               for _ in range(3))
    fa = torch.compile(flex_attention)
    pairs_causal = B * H * S * (S + 1) / 2
    pairs_full = B * H * S * S
    pairs_sw = B * H * sum(min(i, W) + 1 for i in range(S))
    cuts = torch.sort(torch.randint(1, S - 1, (B, NDOC - 1), generator=torch.Generator().manual_seed(1)), 1)[0]
    offs = torch.cat([torch.zeros(B, 1, dtype=torch.long), cuts, torch.full((B, 1), S, dtype=torch.long)], 1)
    doc_id = torch.zeros(B, S, dtype=torch.long)
    for b in range(B):
        for j in range(NDOC):
            doc_id[b, offs[b, j]:offs[b, j + 1]] = j
    pairs_doc = H * sum(int(((offs[b, 1:] - offs[b, :-1]) ** 2).sum()) for b in range(B))
    doc_id = doc_id.to(dev)
    slopes = torch.tensor([2 ** (-8 * (h + 1) / H) for h in range(H)], device=dev)

    def causal(b, h, qi, ki):
        return qi >= ki

    def sliding(b, h, qi, ki):
        return (qi >= ki) & (qi - ki <= W)

    def document(b, h, qi, ki):
        return doc_id[b, qi] == doc_id[b, ki]

    def alibi(score, b, h, qi, ki):
        return score + slopes[h] * (ki - qi)

    def softcap(score, b, h, qi, ki):
        return CAP * torch.tanh(score / CAP)

    fl = 4 * D   # flops per kept pair: 2*D (QK) + 2*D (PV)
    cases = [
        ("causal", dict(block_mask=create_block_mask(causal, None, None, S, S)), pairs_causal),
        ("alibi", dict(score_mod=alibi), pairs_full),
        ("sliding", dict(block_mask=create_block_mask(sliding, None, None, S, S)), pairs_sw),
        ("softcap", dict(score_mod=softcap), pairs_full),
        ("document", dict(block_mask=create_block_mask(document, B, None, S, S)), pairs_doc),
    ]
    print(f"torch {torch.__version__}, {torch.cuda.get_device_name()}, B{B} H{H} S{S} D{D} bf16 (context only)")
    for name, kw, pairs in cases:
        try:
            ms = timeit(lambda: fa(q, k, v, **kw))
            print(f"flex_attention {name:9s} {ms:8.3f} ms  {pairs * fl / ms / 1e9:8.1f} TFLOP/s")
        except Exception as e:  # pragma: no cover
            print(f"flex_attention {name:9s} failed: {str(e).splitlines()[0][:100]}")
        sys.stdout.flush()
    for be in ("CUDNN_ATTENTION", "FLASH_ATTENTION", "EFFICIENT_ATTENTION"):
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel
            with sdpa_kernel(getattr(SDPBackend, be)):
                ms = timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True))
            print(f"sdpa[{be}] causal {ms:8.3f} ms  {pairs_causal * fl / ms / 1e9:8.1f} TFLOP/s")
        except Exception as e:  # pragma: no cover
            print(f"sdpa[{be}] causal failed: {str(e).splitlines()[0][:100]}")


if __name__ == "__main__":
    main()
