"""GPU-vs-oracle parity harness (used by tests/test_gpu_*.py and __graft_entry__.smoke()).

Inputs come from ``synth`` (float32), are rounded ONCE to the kernel dtype by torch (RN),
and the same rounded values feed the CUDA path and the float64 oracle.  Tolerances are the
ones BASELINE.json's north_star states:
  τ   : |τ_gpu − τ_ref| <= 1e-3 · max(1, |τ_ref|)            (τ_ref = Alg. 1 mirror, same T)
  O   : max |O_gpu − O_ref| <= 2e-2 (bf16 inputs), 1e-4 (fp32 inputs); same bar for O⁽²⁾
  grad: ‖g_gpu − g_ref‖₂ / ‖g_ref‖₂ <= 3e-2 (bf16); 1e-3 (fp32)
  M   : bit-exact vs the oracle's mask from its own τ (requires block margin > 1e-4).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
import synth

TOL = {torch.bfloat16: dict(o=2e-2, g=3e-2), torch.float32: dict(o=1e-4, g=1e-3)}
TAU_RTOL = 1e-3
MARGIN_MIN = 1e-4


def make_case(B, H, N, d, dtype, seed=0, spec=None, device="cuda"):
    q, k, v, do = synth.make_inputs(B, H, N, d, seed, spec)
    ts = [torch.from_numpy(x).to(dtype) for x in (q, k, v, do)]
    dev = [t.to(device) for t in ts]
    ref = [t.double().numpy() for t in ts]        # the rounded values, exactly
    return dev, ref


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def check_head(res, ref_inputs, bh, alpha, causal, n_iter, dtype, with_bwd=True, grads=None, report=None):
    """Full (all rows) comparison of one head (index bh into the flattened B·H)."""
    q, k, v, do = [x.reshape((-1,) + x.shape[-2:])[bh] for x in ref_inputs]
    N = q.shape[0]
    tol = TOL[dtype]
    fw = O.attn_fwd(q, k, v, alpha, causal, n_iter)
    tau_g = res.tau.reshape(-1, N)[bh].double().cpu().numpy()
    err_tau = np.max(np.abs(tau_g - fw["tau"]) / np.maximum(1.0, np.abs(fw["tau"])))
    assert err_tau <= TAU_RTOL, ("tau", bh, err_tau)
    d = q.shape[1]
    o_g = res.o.reshape(-1, N, d)[bh].double().cpu().numpy()
    err_o = np.abs(o_g - fw["O"]).max()
    assert err_o <= tol["o"], ("O", bh, err_o)
    if res.o2 is not None:
        o2_g = res.o2.reshape(-1, N, d)[bh].double().cpu().numpy()
        err_o2 = np.abs(o2_g - fw["O2"]).max()
        assert err_o2 <= tol["o"], ("O2", bh, err_o2)
    M_ref, margin = O.block_mask(q, k, fw["tau"], alpha, causal)
    assert margin > MARGIN_MIN, ("block margin too small for a bit-exact mask check", margin)
    Tr, Tc = M_ref.shape
    M_g = res.mask.reshape(-1, Tr, Tc)[bh].cpu().numpy()
    assert np.array_equal(M_g, M_ref), ("mask", bh, np.argwhere(M_g != M_ref)[:10])
    Qt, _ = O.lookup_tables(M_ref)
    cnt = res.row_cnt.reshape(-1, Tr)[bh].cpu().numpy()
    idx = res.row_idx.reshape(-1, Tr, Tc)[bh].cpu().numpy()
    for i in range(Tr):
        assert cnt[i] == len(Qt[i]) and np.array_equal(idx[i, :cnt[i]], Qt[i]), ("row table", bh, i)
    out = dict(tau=err_tau, O=err_o, margin=margin, density=float(M_ref.mean()))
    if with_bwd and grads is not None:
        bw = O.attn_bwd(q, k, v, do, fw["tau"], alpha, causal)
        for name, g_gpu, g_ref in zip(("dQ", "dK", "dV"), grads, (bw["dQ"], bw["dK"], bw["dV"])):
            gg = g_gpu.reshape(-1, N, d)[bh].double().cpu().numpy()
            e = rel_l2(gg, g_ref)
            assert e <= tol["g"], (name, bh, e)
            out[name] = e
    if report is not None:
        report.append(out)
    return out


def run_gpu(dev_inputs, alpha, causal, n_iter, training=True):
    import paper_2502_12082_b200 as P
    q, k, v, do = dev_inputs
    fw = P.entmax_attn_fwd(q, k, v, alpha, causal, n_iter, training=training)
    grads = P.entmax_attn_bwd(q, k, v, do, fw, alpha, causal) if training else None
    torch.cuda.synchronize()
    return fw, grads
