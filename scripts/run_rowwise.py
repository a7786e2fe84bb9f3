"""One row-wise solver call (8192 x 8192 fp32, alpha=1.5, T=3) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2502_12082_b200 as P
s, _ = synth.rowwise_scores(8192, 8192, seed=0)
x = torch.from_numpy(s).cuda()
for _ in range(2):
    P.entmax_rowwise_fwd(x, 1.5, 3)
torch.cuda.synchronize()
