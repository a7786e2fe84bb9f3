"""Run tests/probe/ubench_tma.cu: TMA streaming rate with the attention access pattern (64 CTAs per head
stream the same tiles in the same order), unicast vs 2-CTA multicast, with and without an MMA consumer.
Diagnostic only."""
import ctypes, json, os, sys
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench_tma.so"))
L.tma_rate_run.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_void_p]
heads, nblk = 48, 64
out = {}
for boxes in (1, 2):
    K = torch.randn(boxes * heads * nblk * 128, 64, device="cuda").to(torch.bfloat16)
    for mc in (1, 2, 3):
        for mma in (0, 1):
            grid = heads * 64
            cyc = torch.zeros(grid, dtype=torch.int64, device="cuda")
            ms = ctypes.c_float()
            rc = L.tma_rate_run(boxes, mc, mma, K.data_ptr(), heads, nblk, nblk, cyc.data_ptr(), ctypes.byref(ms))
            c = cyc[cyc > 0].float().mean().item() / nblk
            byt = grid * nblk * boxes * (8192 if mc == 3 else 16384)
            name = f"boxes={boxes} mc={mc} mma={mma}"
            print(f"{name}: rc={rc} cycles/tile={c:7.1f} B/cyc/SM(CTA)={boxes * (8192 if mc == 3 else 16384) / c:6.1f} "
                  f"ms={ms.value:.3f} chip TB/s (SM ingress)={byt / ms.value / 1e9:.2f}", flush=True)
            out[name] = dict(cycles_per_tile=c, ms=ms.value, ingress_tbs=byt / ms.value / 1e9, rc=rc)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
