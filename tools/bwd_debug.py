import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02043_b200 import fl
torch.manual_seed(0)
D = int(sys.argv[1]) if len(sys.argv) > 1 else 128
S = int(sys.argv[2]) if len(sys.argv) > 2 else 300
q, k, v = (torch.rand(1, 1, S, D, device="cuda").bfloat16() for _ in range(3))
o, lse = fl.attn_fwd(q, k, v, return_lse=True)
torch.cuda.synchronize()
print("fwd ok", flush=True)
do = torch.rand_like(o)
dq, dk, dv = fl.attn_bwd(q, k, v, o, lse, do)
torch.cuda.synchronize()
print("bwd ok", dq.abs().max().item(), dk.abs().max().item(), dv.abs().max().item(), flush=True)
