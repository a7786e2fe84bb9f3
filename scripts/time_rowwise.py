"""Row-wise solver timing (NEXT-1 line of bench.py, standalone): python scripts/time_rowwise.py [rows n]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, bench
import paper_2502_12082_b200 as P
rows, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8192, 8192)
r = bench.run_rowwise(P, synth, torch, torch.device("cuda", 0), bench.load_peaks(), rows, n)
for k in ("f32", "bf16"):
    print(k, {a: (round(b, 4) if isinstance(b, float) else b) for a, b in r[k].items() if a != "roofline"},
          "HBM frac", round(r[k]["roofline"]["frac"], 3))
