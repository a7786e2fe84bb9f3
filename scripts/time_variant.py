"""Per-kernel times (library event timing) of one library build on config 2:
python scripts/time_variant.py LIB gen rho   (LIB = path of a libentmax*.so)"""
import os, sys
os.environ["ENTMAX_ATTN_LIB"] = os.path.abspath(sys.argv[1])
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2502_12082_b200 as P
gen = sys.argv[2] if len(sys.argv) > 2 else "gaussian"
rho = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in synth.make_inputs(4, 12, 8192, 64, 7, synth.HeadSpec(gen, rho=rho))]
for _ in range(3):
    fw = P.entmax_attn_fwd(q, k, v, 1.5, False, 3)
torch.cuda.synchronize()
P.profile_reset(); P.profile_enable(True)
for _ in range(10):
    P.entmax_attn_fwd(q, k, v, 1.5, False, 3, out=fw)
P.profile_enable(False)
pr = P.profile_collect()
print(os.path.basename(sys.argv[1]), gen, rho, {k: round(v[1] / v[0], 4) for k, v in pr.items()},
      "density", round(fw.mask.float().mean().item(), 4))
