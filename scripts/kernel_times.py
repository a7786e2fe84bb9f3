"""Per-kernel times (library event timing) of fwd+bwd on one config:
python scripts/kernel_times.py B H N d alpha causal [gen rho]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2502_12082_b200 as P
B, H, N, d = map(int, sys.argv[1:5]); alpha = float(sys.argv[5]); causal = sys.argv[6] == "1"
gen = sys.argv[7] if len(sys.argv) > 7 else "gaussian"; rho = float(sys.argv[8]) if len(sys.argv) > 8 else 1.0
q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in synth.make_inputs(B, H, N, d, 7, synth.HeadSpec(gen, rho=rho))]
fw = P.entmax_attn_fwd(q, k, v, alpha, causal, 3)
g = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))
def step():
    P.entmax_attn_fwd(q, k, v, alpha, causal, 3, out=fw)
    P.entmax_attn_bwd(q, k, v, do, fw, alpha, causal, grads=g)
for _ in range(3): step()
torch.cuda.synchronize()
P.profile_reset(); P.profile_enable(True)
for _ in range(10): step()
P.profile_enable(False)
pr = P.profile_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): step()
e1.record(); torch.cuda.synchronize()
print(sys.argv[1:], "step ms", round(e0.elapsed_time(e1) / 10, 4), {k: round(v[1] / v[0], 4) for k, v in pr.items()})
