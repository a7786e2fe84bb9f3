import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.ubench_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
nrows = 8192 * 48
K = torch.randn(nrows, 64, device="cuda").to(torch.bfloat16)
for mode in (11, 20):
    for nst in (2, 4, 8):
        for grid in (1, 148):
            cyc = torch.zeros(grid, dtype=torch.int64, device="cuda"); ms = ctypes.c_float()
            rc = L.ubench_run(mode, nst, grid, 512, 64, K.data_ptr(), nrows, cyc.data_ptr(), ctypes.byref(ms))
            c = cyc.float().mean().item() / 512
            print(f"mode={mode} nst={nst} grid={grid:3d} rc={rc} cycles/16KB={c:6.1f} B/cyc/SM={16384/c:5.1f}", flush=True)
