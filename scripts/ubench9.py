import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.ubench_mc_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
L.ubench_run.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
nrows = 8192 * 48
K = torch.randn(nrows, 64, device="cuda").to(torch.bfloat16)
cyc = torch.zeros(2 * 148, dtype=torch.int64, device="cuda"); ms = ctypes.c_float()
rc = L.ubench_run(2, 4, 148, 512, 64, K.data_ptr(), nrows, cyc.data_ptr(), ctypes.byref(ms))
print("unicast tma+ss  rc", rc, "cycles/tile", cyc[:148].float().mean().item() / 512, flush=True)
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
rc = L.ubench_mc_run(148, 512, K.data_ptr(), nrows, cyc.data_ptr())
print("multicast x2    rc", rc, "cycles/tile", cyc.float().mean().item() / 512, flush=True)
