import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2502_12082_b200 as P
from tests.parity import make_case
for zero in (True, False):
    dev, ref = make_case(1, 1, 1, 64, torch.bfloat16, seed=65)
    q, k, v, do = dev
    fw = P.entmax_attn_fwd(q, k, v, 1.5, True, 3)
    n = P.workspace_bytes(q, True)[1]
    ws = torch.zeros(n, dtype=torch.uint8, device='cuda') if zero else torch.full((n,), 0xff, dtype=torch.uint8, device='cuda')
    dq, dk, dv = P.entmax_attn_bwd(q, k, v, do, fw, 1.5, True, workspace=ws)
    torch.cuda.synchronize()
    print("zero ws" if zero else "0xff ws", "delta", ws[:4].view(torch.float32).item(), "dq", dq.abs().max().item(),
          "dk", dk.abs().max().item(), "dv", dv.abs().max().item(), "tau", fw.tau.item(), "o2", fw.o2.abs().max().item(),
          "mask", fw.mask.tolist(), fw.row_cnt.tolist())
