"""Run tests/probe/ubench_mma.cu (tcgen05 issue-rate modes) on the GPU and print cycles per tile
against the per-SM dense bf16 floor (8192 flop/cycle/SM).  Diagnostic only."""
import ctypes
import json
import os
import sys

import torch

L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench_mma.so"))
L.mma_rate_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
# mode: (name, per-SM flops per tile)
MODES = {0: ("c1 SS 128x128x64", 2 * 128 * 128 * 64), 1: ("c1 SS 128x256x64", 2 * 128 * 256 * 64),
         2: ("c1 TS 128x64x128", 2 * 128 * 64 * 128), 3: ("c1 SS 128x64x128", 2 * 128 * 64 * 128),
         4: ("c2 SS 256x128x64", 2 * 128 * 128 * 64), 5: ("c2 SS 256x256x64", 2 * 128 * 256 * 64),
         6: ("c2 TS 256x128x128", 2 * 128 * 128 * 128), 7: ("c1 TS 128x128x128", 2 * 128 * 128 * 128),
         9: ("c2 TS 256x64x128 SW64", 2 * 128 * 64 * 128), 10: ("c2 SS 256x64x128 SW64", 2 * 128 * 64 * 128)}
out = {}
for mode, (name, fl) in MODES.items():
    if len(sys.argv) > 2 and str(mode) not in sys.argv[2].split(','):
        continue
    for grid in (2, 148):
        cyc = torch.zeros(grid, dtype=torch.int64, device="cuda")
        ms = ctypes.c_float()
        ntile = 4096
        rc = L.mma_rate_run(mode, grid, ntile, cyc.data_ptr(), ctypes.byref(ms))
        c = cyc[cyc > 0].float().mean().item() / ntile
        floor = fl / 8192
        tf = grid * fl * ntile / (ms.value * 1e-3) / 1e12
        print(f"{name:20s} grid={grid:3d} rc={rc} cycles/tile={c:7.1f} floor={floor:6.1f} eff={floor / c:5.2f} "
              f"chip TF/s={tf:7.1f}", flush=True)
        out[f"{name} grid{grid}"] = dict(cycles=c, floor=floor, eff=floor / c, tflops=tf, rc=rc)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
