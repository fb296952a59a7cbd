"""Debug: resident pair-bias path -- determinism, guard, oracle parity on small row cases."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, numpy as np
from tests import cases
from tests.test_gpu_guard import _nan_guard, _canary_out
from paper_2511_02043_b200 import fl

for (Ns, Nr, pz) in [(5, 384, 0.1), (5, 384, 0.0), (4, 384, 0.0), (2, 100, 0.0), (3, 300, 0.1)]:
    ins, gk, ok = cases.evoformer(dict(kind="row", B=1, Ns=Ns, Nr=Nr, H=2, c=32, p_zero=pz))
    Q, K, V = (t.cuda() for t in ins["storage"])
    view = lambda t: t.permute(0, 1, 3, 2, 4)
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    a = fl.attn_fwd(view(Q), view(K), view(V), **kw); torch.cuda.synchronize()
    b = fl.attn_fwd(view(Q), view(K), view(V), **kw); torch.cuda.synchronize()
    ref, _ = cases.run_oracle(ins, ok)
    err = np.abs(a.cpu().double().numpy().reshape(ref.shape) - ref)
    gQ, gK, gV = (_nan_guard(t) for t in (Q, K, V))
    gkw = dict(kw)
    pb = _nan_guard(kw["bias"][:, 0].contiguous())
    gkw["bias"] = pb.unsqueeze(1).expand(kw["bias"].shape)
    c = fl.attn_fwd(view(gQ), view(gK), view(gV), **gkw); torch.cuda.synchronize()
    gkw2 = dict(kw); gkw2["gate"] = view(_nan_guard(view(gk["gate"]).contiguous()))
    d = fl.attn_fwd(view(Q), view(K), view(V), **gkw2); torch.cuda.synchronize()
    diff_c = (c.float() - a.float()).abs()
    print(f"Ns{Ns} Nr{Nr} pz{pz}: det {torch.equal(a, b)} oracle max {err.max():.3e} (argmax {np.unravel_index(err.argmax(), err.shape)}) "
          f"guard-bias/qkv eq {torch.equal(a, c)} maxdiff {diff_c.max().item():.3e} nan {torch.isnan(c).any().item()} "
          f"guard-gate eq {torch.equal(a, d)}")
    if not torch.equal(a, c):
        idx = (diff_c > 0).nonzero()
        print("   differing idx (first 10):", idx[:10].tolist(), "count", idx.shape[0])
