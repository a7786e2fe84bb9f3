"""One row-wise solver call (8192 x 8192, alpha=1.5, T=3) for ncu: python scripts/run_rowwise.py [f32|bf16] [bwd]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2502_12082_b200 as P
dt = torch.bfloat16 if len(sys.argv) > 1 and sys.argv[1] == "bf16" else torch.float32
s, dp = synth.rowwise_scores(8192, 8192, seed=0)
x = torch.from_numpy(s).to(dt).cuda()
g = torch.from_numpy(dp).to(dt).cuda()
for _ in range(2):
    p, _ = P.entmax_rowwise_fwd(x, 1.5, 3)
    if len(sys.argv) > 2 and sys.argv[2] == "bwd":
        P.entmax_rowwise_bwd(p, g, 1.5)
torch.cuda.synchronize()
