"""Locate τ mismatches vs the oracle for one head: python scripts/debug_tau.py alpha causal N [gen]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, synth
import oracle as O
from parity import make_case, run_gpu
alpha, causal, N = float(sys.argv[1]), sys.argv[2] == "1", int(sys.argv[3])
gen = sys.argv[4] if len(sys.argv) > 4 else "gaussian"
dev, ref = make_case(8, 12, N, 64, torch.bfloat16, seed=int(alpha * 100), spec=synth.HeadSpec(gen))
fw, _ = run_gpu(dev, alpha, causal, 3, training=False)
for bh in (0, 95):
    q, k = ref[0].reshape(-1, N, 64)[bh], ref[1].reshape(-1, N, 64)[bh]
    t_ref = O.solve_tau(q, k, alpha, causal, 3)
    t_g = fw.tau.reshape(-1, N)[bh].double().cpu().numpy()
    err = np.abs(t_g - t_ref) / np.maximum(1, np.abs(t_ref))
    bad = np.nonzero(err > 1e-3)[0]
    print("bh", bh, "bad rows", len(bad), "blocks", sorted(set((bad // 128).tolist())), "max err", err.max())
    if len(bad):
        r = bad[0]
        S = (q[r] @ k[: (r + 1 if causal else N)].T) / 8
        z = (alpha - 1) * S
        print("  row", r, "tau gpu", t_g[r], "ref", t_ref[r], "zmax", z.max(), "ncand(z>m-1)", (z > z.max() - 1).sum())
        for rr in bad[:8]:
            S = (q[rr] @ k[: (rr + 1 if causal else N)].T) / 8; z = (alpha - 1) * S
            print("   ", rr, t_g[rr], t_ref[rr], "ncand", (z > z.max() - 1).sum())
