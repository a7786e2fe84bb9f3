import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.ubench_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
nrows = 8192 * 48
K = torch.randn(nrows, 64, device="cuda").to(torch.bfloat16)
for mode in (1, 0, 3, 30, 31):
    for grid in (1, 148):
        cyc = torch.zeros(2 * grid, dtype=torch.int64, device="cuda"); ms = ctypes.c_float()
        rc = L.ubench_run(mode, 4, grid, 512, 64, K.data_ptr(), nrows, cyc.data_ptr(), ctypes.byref(ms))
        c = cyc.float().view(2, grid).mean(1) / 512
        print(f"mode={mode:2d} grid={grid:3d} rc={rc} tma/tile={c[0].item():6.1f} mma/tile={c[1].item():6.1f}", flush=True)
