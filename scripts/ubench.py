"""Run the tcgen05/TMA microbenchmarks of tests/probe/ubench.cu on the GPU (diagnostic)."""
import ctypes
import os

import torch

L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.ubench_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
nrows = 8192 * 48
for kdim in (64, 128):
    K = torch.randn(nrows, kdim, device="cuda").to(torch.bfloat16)
    for mode, name in ((0, "mma_ss"), (3, "mma_ts"), (1, "tma"), (2, "tma+ss"), (4, "tma+ts")):
        for nst in (2, 4, 8):
            if mode in (0, 3) and nst != 2:
                continue
            if kdim == 128 and nst == 8:
                continue
            for grid in (1, 148):
                cyc = torch.zeros(grid, dtype=torch.int64, device="cuda")
                ms = ctypes.c_float()
                ntile = 512
                rc = L.ubench_run(mode, nst, grid, ntile, kdim, K.data_ptr(), nrows, cyc.data_ptr(), ctypes.byref(ms))
                c = cyc.float().mean().item()
                print(f"d={kdim} {name:8s} nst={nst} grid={grid:3d} rc={rc} cycles/tile={c / ntile:7.1f} "
                      f"ms={ms.value:.3f} GB/s={grid * ntile * 128 * kdim * 2 / ms.value / 1e6:.0f}", flush=True)
