"""Small fwd+bwd cases for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_12082_b200 as P
from tests.parity import make_case
for (B, H, N, d, dt, causal) in [(1, 2, 300, 64, torch.bfloat16, True), (1, 1, 384, 128, torch.bfloat16, False),
                                 (1, 2, 300, 128, torch.bfloat16, True),
                                 (1, 1, 200, 64, torch.float32, True)]:
    dev, _ = make_case(B, H, N, d, dt, seed=3)
    q, k, v, do = dev
    for masked in (True, False):
        fw = P.entmax_attn_fwd(q, k, v, 1.5, causal, 3, masked=masked)
        P.entmax_attn_bwd(q, k, v, do, fw, 1.5, causal)
P.pack_mask(torch.randint(0, 2, (2, 3, 37), dtype=torch.uint8, device="cuda"))
for N in (600, 1100):   # long rows (fp32 U) next to the short-row consistent-U kernels above
    dev, _ = make_case(1, 1, N, 64, torch.bfloat16, seed=5)
    q, k, v, do = dev
    fw = P.entmax_attn_fwd(q, k, v, 1.75, True, 3)
    P.entmax_attn_bwd(q, k, v, do, fw, 1.75, True)
p, t = P.entmax_rowwise_fwd(torch.randn(8, 1000, device="cuda"), 1.5, 3)
P.entmax_rowwise_bwd(p, torch.randn_like(p), 1.5)
p, t = P.entmax_rowwise_fwd(torch.randn(4, 20000, device="cuda"), 1.5, 23, halley=False)
# more rows than resident CTAs: every register-kernel CTA bulk-prefetches a later row into L2
for dt in (torch.bfloat16, torch.float32):
    p, t = P.entmax_rowwise_fwd(torch.randn(1500, 4096, device="cuda", dtype=dt), 1.5, 3)
    P.entmax_rowwise_bwd(p, torch.randn_like(p), 1.5)
torch.cuda.synchronize()
print("sanitize case ok")
