"""Per-tile timeline of one dK/dV CTA (kernel id 2) from the -DENTMAX_TRACE build (make trace):
MMA-warp issue times vs math-warp phases.  usage: python scripts/trace_fb.py [cta_x] [kid]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["ENTMAX_ATTN_LIB"] = os.path.join(ROOT, "tests", "probe", "libentmax_trace.so")
sys.path.insert(0, ROOT)
import torch, synth
import paper_2502_12082_b200 as P
L = P._lib.lib()
L.entmax_trace_reset.argtypes = [ctypes.c_int]; L.entmax_trace_read.argtypes = [ctypes.c_void_p]
L.entmax_trace_kernel.argtypes = [ctypes.c_int]
bx = int(sys.argv[1]) if len(sys.argv) > 1 else 30
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B, H, N, d = map(int, os.environ.get("SHAPE", "4 12 8192 64").split())
q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in synth.make_inputs(B, H, N, d, 7)]
fw = P.entmax_attn_fwd(q, k, v, 1.5, False, 3); g = P.entmax_attn_bwd(q, k, v, do, fw, 1.5, False)
torch.cuda.synchronize()
L.entmax_trace_kernel(kid); L.entmax_trace_reset(bx)
fw = P.entmax_attn_fwd(q, k, v, 1.5, False, 3); g = P.entmax_attn_bwd(q, k, v, do, fw, 1.5, False)
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64); L.entmax_trace_read(buf.ctypes.data)
L.entmax_trace_kernel(-1)
ev = buf.astype(np.int64)
t0 = ev[8002] if ev[8002] else ev[ev > 0].min()
b = np.where(ev > 0, ev - t0, -1)
n = int((b[0:8 * 200:8] >= 0).sum()) + 1
names = {2: ["SdP(k+1) issued", "p_full(k) seen", "-", "math s_full(k)", "math loads+compute", "math p_empty ok",
             "math p_full arrived", "prod load(k)"],
         3: ["SdP(k+1) issued", "ds_full(k) seen", "-", "math s_full(k)", "math compute", "math ds_empty ok",
             "math ds_full arrived", "prod load(k)"],
         1: ["S(k) issued", "p_full(k) seen", "-", "math s_full(k)", "math compute", "-", "math p_full arrived",
             "prod load(k)"]}[kid]
print("k   " + " | ".join(f"{x:>18s}" for x in names))
for kk in list(range(0, 6)) + list(range(n // 2, n // 2 + 3)) + list(range(max(0, n - 3), n)):
    print(f"{kk:3d} " + " | ".join(f"{b[8 * kk + e]:18d}" for e in range(8)))
math_start = b[3:8 * n:8]; math_ld = b[4:8 * n:8]; math_pe = b[5:8 * n:8]; math_end = b[6:8 * n:8]
mma_p = b[1:8 * n:8]
ok = (math_start >= 0) & (math_end >= 0)
print("tiles", n, "CTA span", b[8003], "per tile", b[8003] / max(1, n))
print("median: math s_full->compute done", np.median((math_ld - math_start)[ok]),
      " compute->p_empty", np.median((math_pe - math_ld)[ok]), " p_empty->arrive", np.median((math_end - math_pe)[ok]),
      " arrive->next s_full", np.median(math_start[1:][ok[1:]] - math_end[:-1][ok[1:]]))
print("median MMA: p_full seen after math arrive", np.median((mma_p - math_end)[ok & (mma_p >= 0)]))
print("tile period (math_end diff)", np.median(np.diff(math_end[ok])))
if kid == 2:
    qf = b[4096:4096 + n]; se = b[4160:4160 + n]; pt = b[4224:4224 + n]
    wa = b[4288:4288 + 8 * n].reshape(n, 8)
    print("k  prod_tma  mma_qdfull  mma_sempty  sdp_issued | warp s_empty arrivals (min..max)")
    for kk in list(range(0, 5)) + list(range(30, 35)) + list(range(n - 4, n - 1)):
        print(f"{kk:3d} {pt[kk]:9d} {qf[kk]:10d} {se[kk]:10d} {b[8 * kk]:10d} | {wa[kk].min():9d} .. {wa[kk].max():9d}")
    ok = slice(2, n - 2)
    print("median: prod TMA issue -> qd_full seen", np.median(qf[ok] - pt[ok]),
          " qd_full -> s_empty passed", np.median(se[ok] - qf[ok]),
          " warp arrive spread", np.median(wa[ok].max(1) - wa[ok].min(1)))
