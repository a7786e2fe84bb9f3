import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.ubench_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
nrows = 8192 * 48
K = torch.randn(nrows, 64, device="cuda").to(torch.bfloat16)
for mode in (0, 6, 7, 2):
    cyc = torch.zeros(2 * 148, dtype=torch.int64, device="cuda"); ms = ctypes.c_float()
    rc = L.ubench_run(mode, 4, 148, 512, 64, K.data_ptr(), nrows, cyc.data_ptr(), ctypes.byref(ms))
    c = cyc[:148].float().mean().item() / 512
    print(f"mode={mode} rc={rc} cycles per tile (4 MMAs 128x128x16)={c:6.1f}", flush=True)
