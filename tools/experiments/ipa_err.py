import sys, math; sys.path.insert(0, '.')
import torch, numpy as np, oracle
from paper_2511_02043_b200 import synth, fl
for N in (100, 300):
    x = synth.ipa_inputs(N, seed=N)
    o, op, opair = fl.ipa_fwd(**{k: v.cuda() for k, v in x.items()}); torch.cuda.synchronize()
    ro, rop, rpair = oracle.ipa(**x)
    print(N, "o", np.abs(o.cpu().double().numpy()-ro).max(), np.abs(ro).max(), "opair", np.abs(opair.cpu().double().numpy()-rpair).max(), np.abs(rpair).max(),
          "op", np.abs(op.cpu().double().numpy()-rop).max(), np.abs(rop).max(), "|t|max", float(x["t"].abs().max()))
