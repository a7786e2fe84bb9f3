import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.ubench_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
nrows = 8192 * 48
K = torch.randn(nrows, 64, device="cuda").to(torch.bfloat16)
for mode, per in ((1, 1), (40, 2), (41, 4)):
    for nst in (2, 4):
        if mode == 41 and nst == 4: continue
        cyc = torch.zeros(2 * 148, dtype=torch.int64, device="cuda"); ms = ctypes.c_float()
        rc = L.ubench_run(mode, nst, 148, 256, 64, K.data_ptr(), nrows, cyc.data_ptr(), ctypes.byref(ms))
        c = cyc[:148].float().mean().item() / (256 * per)
        print(f"mode={mode} nst={nst} rc={rc} cycles/16KB={c:6.1f} B/cyc/SM={16384/c:5.1f}", flush=True)
