"""Gradient / output errors vs the oracle for a few cases (optionally against another library build):
python scripts/grad_errors.py [LIB]"""
import os, sys
if len(sys.argv) > 1:
    os.environ["ENTMAX_ATTN_LIB"] = os.path.abspath(sys.argv[1])
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from tests.parity import make_case, run_gpu, check_head
rep = []
for (N, gen, causal, alpha) in [(2, "gaussian", True, 1.5), (300, "gaussian", True, 1.5), (1024, "planted", False, 1.5),
                                 (1024, "gaussian", False, 1.5), (1024, "gaussian", True, 2.0), (1024, "gaussian", False, 1.25)]:
    spec = synth.HeadSpec(gen, rho=0.25) if gen == "planted" else synth.HeadSpec(gen)
    dev, ref = make_case(1, 2, N, 64, torch.bfloat16, seed=N * 7 + 64, spec=spec)
    fw, grads = run_gpu(dev, alpha, causal, 3)
    errs = []
    for bh in range(2):
        try:
            out = check_head(fw, ref, bh, alpha, causal, 3, torch.bfloat16, grads=grads)
        except AssertionError as e:
            out = {"fail": str(e)[:60]}
        errs.append({k: (round(v, 5) if isinstance(v, float) else v) for k, v in out.items() if k in ("O", "dQ", "dK", "dV", "fail")})
    print(N, gen, causal, alpha, errs)
