import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "probe", "libubench.so"))
L.tmem_rd_run.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_void_p]
for x in (16, 32):
    for nw in (4, 8, 16):
        cyc = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
        sink = torch.zeros(148 * 512, dtype=torch.int32, device="cuda")
        iters = 2000
        rc = L.tmem_rd_run(x, nw, iters, cyc.data_ptr(), sink.data_ptr())
        c = cyc.view(148, 16)[:, :nw].float().max(1).values.mean().item()
        bytes_ = nw * 32 * x * 4 * iters
        print(f"x={x} warps={nw} rc={rc} cycles={c:.0f} B/cycle/SM={bytes_ / c:.1f} cycles/ld={c/iters:.1f}", flush=True)
