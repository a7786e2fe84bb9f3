"""GPU parity of the standalone row-wise α-entmax solver (include/entmax_rowwise.h, SURVEY §8f
NEXT-1) against the float64 oracle (oracle/rowwise.py), through the C ABI.

Inputs: synth.rowwise_scores — the paper's solver benchmark rows, s ~ N(0, 1) — rounded
once to the kernel dtype; the same rounded values feed both sides.
Bars: τ |Δ| <= 1e-3·max(1, |τ_ref|) against the T-step mirror (Alg. 1, or Eq. 4
bisection); p max-abs <= 1e-4 (fp32) / 4e-3 (bf16: p is stored in bf16, 2^-8 of p <= 1);
ds relative-L2 <= 1e-3 (fp32) / 3e-2 (bf16), against oracle.entmax_vjp on the GPU's own p.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

P_TOL = {torch.float32: 1e-4, torch.bfloat16: 4e-3}
G_TOL = {torch.float32: 1e-3, torch.bfloat16: 3e-2}


def _case(rows, n, dtype, seed, sigma=1.0):
    s, dp = synth.rowwise_scores(rows, n, seed, sigma)
    st, dpt = torch.from_numpy(s).to(dtype), torch.from_numpy(dp).to(dtype)
    return st.cuda(), dpt.cuda(), st.double().numpy(), dpt.double().numpy()


def _check_fwd(p, tau, s_ref, alpha, T, halley, dtype):
    z = (alpha - 1.0) * s_ref
    tau_ref = O.halley_bisection(z, alpha, T, halley=halley)
    tg = tau.double().cpu().numpy()
    err_tau = np.max(np.abs(tg - tau_ref) / np.maximum(1.0, np.abs(tau_ref)))
    assert err_tau <= 1e-3, ("tau", err_tau)
    p_ref = O.entmax_probs(z, tau_ref, alpha)
    err_p = np.abs(p.double().cpu().numpy() - p_ref).max()
    assert err_p <= P_TOL[dtype], ("p", err_p)
    return err_tau, err_p


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("n", [1, 7, 256, 1000, 4096, 8192, 12345, 20000])
@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0, 1.7])
def test_rowwise_halley_parity(dtype, n, alpha):
    import paper_2502_12082_b200 as P
    rows = 48 if n <= 8192 else 12
    s, dp, s_ref, dp_ref = _case(rows, n, dtype, seed=n + int(alpha * 100))
    p, tau = P.entmax_rowwise_fwd(s, alpha, 3)
    _check_fwd(p, tau, s_ref, alpha, 3, True, dtype)
    ds = P.entmax_rowwise_bwd(p, dp, alpha)
    g_ref = O.entmax_vjp(p.double().cpu().numpy(), dp_ref, alpha)
    gg = ds.double().cpu().numpy()
    e = np.linalg.norm(gg - g_ref) / max(np.linalg.norm(g_ref), 1e-30)
    assert e <= G_TOL[dtype], ("ds", e)


@pytest.mark.parametrize("T", [1, 2, 8, 23])
def test_rowwise_bisection_mode(T):
    """halley = 0: Eq. 4 bisection, τ = midpoint after the T-th bracket update."""
    import paper_2502_12082_b200 as P
    s, _, s_ref, _ = _case(32, 8192, torch.float32, seed=5 + T)
    p, tau = P.entmax_rowwise_fwd(s, 1.5, T, halley=False)
    _check_fwd(p, tau, s_ref, 1.5, T, False, torch.float32)


def test_rowwise_converges_to_exact_tau():
    """Halley-bisection reaches the exact τ* in 3 iterations (to fp32 precision here)."""
    import paper_2502_12082_b200 as P
    s, _, s_ref, _ = _case(64, 8192, torch.float32, seed=3)
    for alpha in (1.5, 2.0):
        _, tau = P.entmax_rowwise_fwd(s, alpha, 3 if alpha == 1.5 else 6)
        tau_star = O.tau_exact((alpha - 1.0) * s_ref, alpha)
        assert np.max(np.abs(tau.double().cpu().numpy() - tau_star)) < 1e-5


def test_rowwise_strided_inplace_and_batched_shapes():
    import paper_2502_12082_b200 as P
    s, _, s_ref, _ = _case(40, 300, torch.float32, seed=9)
    # [2, 4, 5, 300] view, ragged n (300 % 4 == 0 but not a multiple of 8 for bf16)
    p4, tau4 = P.entmax_rowwise_fwd(s.view(2, 4, 5, 300), 1.5, 3)
    assert p4.shape == (2, 4, 5, 300) and tau4.shape == (2, 4, 5)
    _check_fwd(p4.reshape(40, 300), tau4.reshape(40), s_ref, 1.5, 3, True, torch.float32)
    # strided rows (ld > n), in-place through the raw ABI
    import ctypes
    from paper_2502_12082_b200 import _lib
    big = torch.zeros(40, 320, device="cuda")
    big[:, :300] = s
    rc = _lib.lib().entmax_rowwise_fwd(ctypes.c_void_p(big.data_ptr()), 40, 300, 320, 1, 1.5, 3, 1,
                                       ctypes.c_void_p(big.data_ptr()), None, None)
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(big[:, :300], p4.reshape(40, 300))
    assert torch.count_nonzero(big[:, 300:]) == 0


def test_rowwise_autograd_and_determinism():
    import paper_2502_12082_b200 as P
    s, dp, s_ref, dp_ref = _case(16, 2048, torch.float32, seed=21)
    x = s.clone().requires_grad_(True)
    y = P.entmax(x, 1.5, 3)
    y.backward(dp)
    g_ref = O.entmax_vjp(y.detach().double().cpu().numpy(), dp_ref, 1.5)
    e = np.linalg.norm(x.grad.double().cpu().numpy() - g_ref) / np.linalg.norm(g_ref)
    assert e <= 1e-3
    p1, t1 = P.entmax_rowwise_fwd(s, 1.5, 3)
    p2, t2 = P.entmax_rowwise_fwd(s, 1.5, 3)
    assert torch.equal(p1, p2) and torch.equal(t1, t2)


def test_rowwise_paper_benchmark_size():
    """The paper's solver benchmark shape (8192 × 8192 fp32, T = 3), sampled rows vs the oracle."""
    import paper_2502_12082_b200 as P
    s, _, s_ref, _ = _case(8192, 8192, torch.float32, seed=1)
    p, tau = P.entmax_rowwise_fwd(s, 1.5, 3)
    rows = np.random.default_rng(0).choice(8192, 64, replace=False)
    _check_fwd(p[rows], tau[rows], s_ref[rows], 1.5, 3, True, torch.float32)
    # every row is on the simplex up to the T = 3 residual (reading c12: |Σp − 1| is the mirror's own
    # f(τ_T), not a kernel error): the worst rows match the mirror's residual
    res = (p.double().sum(-1) - 1).abs().cpu().numpy()
    assert res.max() < 1e-2
    worst = np.argsort(res)[-4:]
    z = 0.5 * s_ref[worst]
    r_ref = np.abs(O.entmax_probs(z, O.halley_bisection(z, 1.5, 3), 1.5).sum(-1) - 1)
    assert np.all(np.abs(res[worst] - r_ref) < 1e-5), (res[worst], r_ref)
