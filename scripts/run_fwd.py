"""Run the forward (and optionally backward) once for profiling: python scripts/run_fwd.py gen rho [bwd]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2502_12082_b200 as P
gen = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
rho = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
bwd = len(sys.argv) > 3 and sys.argv[3] == "bwd"
B, H, N, d = map(int, os.environ.get("SHAPE", "4 12 8192 64").split())
causal = os.environ.get("CAUSAL", "0") == "1"
q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in synth.make_inputs(B, H, N, d, 7, synth.HeadSpec(gen, rho=rho))]
for _ in range(2):
    fw = P.entmax_attn_fwd(q, k, v, 1.5, causal, 3)
    if bwd:
        P.entmax_attn_bwd(q, k, v, do, fw, 1.5, causal)
torch.cuda.synchronize()
print("density", fw.mask.float().mean().item(), "cand rows", fw.row_cnt.float().mean().item())
