"""Timeline of one τ-kernel CTA + fallback-tier counts from the -DENTMAX_TRACE build (make trace).
usage: python scripts/trace_tau.py [gen] [cta] [rho]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["ENTMAX_ATTN_LIB"] = os.path.join(ROOT, "tests", "probe", os.environ.get("TRACE_LIB", "libentmax_trace.so"))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2502_12082_b200 as P
L = P._lib.lib()
L.entmax_trace_reset.argtypes = [ctypes.c_int]; L.entmax_trace_read.argtypes = [ctypes.c_void_p]
gen = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
rho = float(sys.argv[3]) if len(sys.argv) > 3 else 1 / 64
B, H, N, d = map(int, os.environ.get("SHAPE", "4 12 8192 64").split())
alpha = float(os.environ.get("ALPHA", "1.5")); causal = os.environ.get("CAUSAL", "0") == "1"
q, k, v, do = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in synth.make_inputs(B, H, N, d, 7, synth.HeadSpec(gen, rho=rho))]
P.entmax_attn_fwd(q, k, v, alpha, causal, 3); torch.cuda.synchronize()
L.entmax_trace_reset(int(sys.argv[2]) if len(sys.argv) > 2 else 30)
P.entmax_attn_fwd(q, k, v, alpha, causal, 3); torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64); L.entmax_trace_read(buf.ctypes.data)
t0 = 0
print(f"CTAs {buf[8102]}  tier-1 rebuilds {buf[8100]}  tier-2 streaming after tier 1 {buf[8101]}, directly {buf[8103]}")
t0 = int(buf[:8100][buf[:8100] > 0].min())
t = lambda i: int(buf[i]) - int(t0) if buf[i] else -1
print("phases (cycles from first event): start", t(8000), "math ready", t(8003), "stream done", t(8004),
      "lists ready", t(8005), "pre-cluster-sync", t(8006), "end", t(8007))
print("tail: iterations done", t(8008), "mask loop done", t(8009), "barrier", t(8010), "compacted", t(8011))
ev = buf[:8100]
t0 = ev[ev > 0].min(); b = ev.astype(np.int64) - int(t0); b[ev == 0] = -1
n = int((b[0:1024:4] >= 0).sum())
mma_k = b[0:4 * n:4]; mma_kf = b[1:4 * n:4]; mma_se = b[2:4 * n:4]
m_pre = b[3072:3072 + 3 * n:3]; m_full = b[3073:3073 + 3 * n:3]; m_rel = b[3074:3074 + 3 * n:3]
prod = b[6144:6144 + n]
print("step  prod_ready  mma_start kfull_ok sempty_ok | math_wait s_full_ok released")
for s in sorted(set(list(range(0, 8)) + list(range(n // 2, n // 2 + 6)) + list(range(n - 6, n)))):
    print(f"{s:4d} {prod[s]:10d} {mma_k[s]:10d} {mma_kf[s]:8d} {mma_se[s]:9d} | {m_pre[s]:9d} {m_full[s]:9d} {m_rel[s]:8d}")
d = np.diff(mma_se[:n]); print("tiles", n, "MMA issue interval: median", np.median(d), "mean", d.mean())
print("MMA waits: k_full", np.median(mma_kf[:n] - mma_k[:n]), "s_empty", np.median(mma_se[:n] - mma_kf[:n]))
print("math: wait for S", np.median(m_full[:n] - m_pre[:n]), " hold", np.median(m_rel[:n] - m_full[:n]),
      " between tiles", np.median(m_pre[1:n] - m_rel[:n - 1]))
print("latency MMA issue -> math sees S:", np.median(m_full[:n] - mma_se[:n]))
print("CTA span (first..last event):", b[b >= 0].max(), "cycles;", b[b >= 0].max() / n, "per tile")
