"""T7 (-m gpu): compute-sanitizer over one small call of every kernel family --
tcgen05 attention (interval mask, block list, Evoformer small head with key mask / bias / gate,
differential attention), split-KV decode, fp32 SIMT, RSA summaries / selection, paged KV.  memcheck
(out-of-bounds and misaligned global / shared accesses) must report 0 errors; synccheck (barrier
misuse) likewise."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, torch
sys.path.insert(0, %r)
from tests import cases
from paper_2511_02043_b200 import fl
def run(case):
    ins, gk, ok = cases.build(dict(case, dtype=case.get("dtype", "bf16")))
    kw = {x: cases.to_dev(y, "cuda") for x, y in gk.items()}
    fl.attn_fwd(*(ins[n].cuda() for n in ("q", "k", "v")), **kw)
run(dict(S=300, D=128, mask="causal"))
run(dict(S=300, D=64, Hq=2, diff=True, lam=0.3))
run(dict(S=200, D=32, bias="bf16", key_mask=True, gate_mode="sigmoid"))
run(dict(S=700, D=128, mask="blocklist", topk=2))
run(dict(Sq=1, Sk=2000, D=128, mask="causal"))
run(dict(S=100, D=64, mask="sliding", window=20, dtype="f32"))
ins, gk, ok = cases.evoformer(dict(kind="row", B=1, Ns=3, Nr=130, H=2, c=32, p_zero=0.1))
fl.attn_fwd(*(ins[n].cuda() for n in ("q", "k", "v")), **{x: cases.to_dev(y, "cuda") for x, y in gk.items()})
k = torch.randn(1, 2, 1000, 128, device="cuda").to(torch.bfloat16)
q = torch.randn(1, 2, 1000, 128, device="cuda").to(torch.bfloat16)
kmin, kmax = fl.rsa_build_summaries(k, 128)
fl.rsa_select(q, kmin, kmax, 1000, topk=2)
fl.rsa_select(q[:, :, -1:], kmin, kmax, 1000, topk=2)
kp, vp, t = fl.paged_kv(k, k, seed=1)
fl.attn_fwd(q, kp, vp, kv_page_table=t.cuda(), kv_len=1000, mask="causal")
torch.cuda.synchronize()
print("SANITIZED_RUN_OK")
''' % ROOT


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    cs = _sanitizer()
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "17", sys.executable, "-c", SCRIPT],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "SANITIZED_RUN_OK" in out, out[-3000:]
    assert r.returncode == 0 and "ERROR SUMMARY: 0 errors" in out, out[-3000:]
