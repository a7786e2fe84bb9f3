"""Pins for oracle/attention.py (forward, mask, tables, backward).  CPU only."""
import numpy as np
import pytest

import oracle as O
from synth import planted_head


def _qkv(n, d, seed, sq=6.0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, d)) * np.sqrt(sq), rng.standard_normal((n, d)),
            rng.standard_normal((n, d)))


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
@pytest.mark.parametrize("causal", [False, True])
def test_v_identity_gives_p(alpha, causal):
    """with V = I (n = d) the output row is the probability row."""
    n = 24
    q, k, _ = _qkv(n, n, 1)
    fw = O.attn_fwd(q, k, np.eye(n), alpha, causal, exact=True)
    z = (alpha - 1) * O.scores(q, k, O.default_scale(n), causal)
    p = O.entmax(z / (alpha - 1), alpha)
    np.testing.assert_allclose(fw["O"], p, atol=1e-12)
    np.testing.assert_allclose(fw["O"].sum(1), 1.0, atol=1e-10)     # rows on the simplex


def test_single_row_and_causal_pair():
    q, k, v = _qkv(1, 8, 2)
    np.testing.assert_allclose(O.attn_fwd(q, k, v, 1.5, False, 3)["O"], v, atol=1e-14)
    q, k, v = _qkv(2, 8, 3)
    fw = O.attn_fwd(q, k, v, 1.5, True, 3)
    np.testing.assert_allclose(fw["O"][0], v[0], atol=1e-14)
    np.testing.assert_allclose(fw["O2"][0], v[0], atol=1e-14)


def test_alpha2_one_hot_rows():
    """α=2 with one-hot attention rows: O = O⁽²⁾ = V_argmax."""
    n, d = 16, 16
    rng = np.random.default_rng(4)
    perm = rng.permutation(n)
    q = 40.0 * np.eye(n)[perm] * np.sqrt(d)
    k = np.eye(n)
    v = rng.standard_normal((n, d))
    fw = O.attn_fwd(q, k, v, 2.0, False, exact=True)
    np.testing.assert_allclose(fw["O"], v[perm], atol=1e-12)
    np.testing.assert_allclose(fw["O2"], v[perm], atol=1e-12)


def test_alpha_to_one_attention_is_softmax_attention():
    q, k, v = _qkv(32, 8, 5, sq=1.0)
    ref = O.softmax_attention(q, k, v)
    gaps = [np.abs(O.attn_fwd(q, k, v, a, exact=True)["O"] - ref).max() for a in (1.1, 1.01, 1.001)]
    assert gaps[0] > gaps[1] > gaps[2] and gaps[2] < 5e-3
    assert 5 < gaps[0] / gaps[1] < 20 and 5 < gaps[1] / gaps[2] < 20   # linear in α−1


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_mirror_converges_to_exact(alpha):
    q, k, v = _qkv(200, 16, 6)
    a = O.attn_fwd(q, k, v, alpha, True, n_iter=40)
    b = O.attn_fwd(q, k, v, alpha, True, exact=True)
    np.testing.assert_allclose(a["tau"], b["tau"], atol=1e-12)
    np.testing.assert_allclose(a["O"], b["O"], atol=1e-10)


def test_row_subset_equals_full():
    q, k, v = _qkv(300, 16, 7)
    full = O.attn_fwd(q, k, v, 1.5, True, 3)
    rows = np.array([0, 5, 127, 128, 299])
    sub = O.attn_fwd(q, k, v, 1.5, True, 3, rows=rows)
    np.testing.assert_array_equal(sub["tau"], full["tau"][rows])
    np.testing.assert_allclose(sub["O"], full["O"][rows], atol=1e-14)


def _fd_grads(q, k, v, W, alpha, causal, h=1e-6):
    def loss(qq, kk, vv):
        return float((O.attn_fwd(qq, kk, vv, alpha, causal, exact=True)["O"] * W).sum())
    out = []
    for which in range(3):
        base = [q.copy(), k.copy(), v.copy()]
        g = np.zeros_like(base[which])
        for idx in np.ndindex(*g.shape):
            plus = [x.copy() for x in base]
            minus = [x.copy() for x in base]
            plus[which][idx] += h
            minus[which][idx] -= h
            g[idx] = (loss(*plus) - loss(*minus)) / (2 * h)
        out.append(g)
    return out


def _far_from_boundary(q, k, alpha, causal, eps=1e-4):
    z = (alpha - 1) * O.scores(q, k, O.default_scale(q.shape[1]), causal)
    tau = O.tau_exact(z, alpha)
    x = z - tau[:, None]
    return np.all(np.abs(x[np.isfinite(x)]) > eps)


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
@pytest.mark.parametrize("causal", [False, True])
def test_backward_matches_finite_differences(alpha, causal):
    """analytic dQ, dK, dV vs central differences of L = Σ O ⊙ W."""
    seed = 10
    while True:
        q, k, v = _qkv(12, 4, seed, sq=4.0)
        if _far_from_boundary(q, k, alpha, causal):
            break
        seed += 1
    W = np.random.default_rng(seed + 100).standard_normal((12, 4))
    tau = O.solve_tau(q, k, alpha, causal)
    g = O.attn_bwd(q, k, v, W, tau, alpha, causal)
    fd = _fd_grads(q, k, v, W, alpha, causal)
    for name, a, f in zip(("dQ", "dK", "dV"), (g["dQ"], g["dK"], g["dV"]), fd):
        err = np.abs(a - f).max() / max(1.0, np.abs(f).max())
        assert err < 1e-6, (name, err)


def test_mutation_without_delta_fails_fd():
    """dropping δ must break the FD agreement (validates the harness)."""
    seed = 20
    while True:
        q, k, v = _qkv(12, 4, seed, sq=1.0)
        if _far_from_boundary(q, k, 1.5, False):
            break
        seed += 1
    W = np.random.default_rng(1).standard_normal((12, 4))
    tau = O.solve_tau(q, k, 1.5, False)
    g = O.attn_bwd(q, k, v, W, tau, 1.5, False, use_delta=False)
    fd = _fd_grads(q, k, v, W, 1.5, False)
    assert np.abs(g["dQ"] - fd[0]).max() > 1e-3


def test_zero_upstream_gives_zero_grads():
    q, k, v = _qkv(40, 8, 8)
    tau = O.solve_tau(q, k, 1.5, True, 3)
    g = O.attn_bwd(q, k, v, np.zeros_like(v), tau, 1.5, True)
    for key in ("dQ", "dK", "dV"):
        assert np.all(g[key] == 0)


def test_dv_of_sum_is_column_sums_of_p():
    """d(Σ O)/dV = Pᵀ 1 (every column of dV equals P's column sums)."""
    q, k, v = _qkv(30, 6, 9)
    tau = O.solve_tau(q, k, 1.5, False, 3)
    g = O.attn_bwd(q, k, v, np.ones_like(v), tau, 1.5, False)
    p = O.probs(q, k, tau, 1.5, False, O.default_scale(6), np.arange(30))
    np.testing.assert_allclose(g["dV"], np.repeat(p.sum(0)[:, None], 6, 1), atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("Br,Bc", [(16, 16), (32, 8), (128, 128)])
def test_block_mask_equals_bruteforce(causal, Br, Bc):
    q, k, _ = _qkv(150, 8, 11)
    tau = O.solve_tau(q, k, 1.5, causal, 3)
    p = O.probs(q, k, tau, 1.5, causal, O.default_scale(8), np.arange(150))
    M, margin = O.block_mask(q, k, tau, 1.5, causal, None, Br, Bc)
    assert np.array_equal(M, O.mask_from_p(p, Br, Bc))
    assert margin > 0
    # mask soundness: every non-zero P lies in an active block
    rows, cols = np.nonzero(p)
    assert np.all(M[rows // Br, cols // Bc] == 1)


def test_lookup_tables_spec_example_and_roundtrip():
    Qt, Kt = O.lookup_tables(np.array([[1, 0], [1, 1]]))
    assert [list(x) for x in Qt] == [[0], [0, 1]]
    assert [list(x) for x in Kt] == [[0, 1], [1]]
    rng = np.random.default_rng(12)
    M = (rng.random((7, 9)) < 0.3).astype(np.uint8)
    Qt, Kt = O.lookup_tables(M)
    R1 = np.zeros_like(M)
    R2 = np.zeros_like(M)
    for i, js in enumerate(Qt):
        R1[i, js] = 1
    for j, is_ in enumerate(Kt):
        R2[is_, j] = 1
    assert np.array_equal(R1, M) and np.array_equal(R2, M)
    assert all(len(O.lookup_tables(np.zeros((3, 3)))[0][i]) == 0 for i in range(3))


def test_planted_generator_realises_target_density():
    """The planted recipe gives the requested block density under
    the oracle's mask, with a comfortable block margin."""
    for rho in (1.0, 0.25, 1 / 16):
        q, k, v, do, owned = planted_head(1024, 64, rho, seed=3, b=0, h=0)
        q64, k64 = q.astype(np.float64), k.astype(np.float64)
        tau = O.solve_tau(q64, k64, 1.5, False, 3)
        M, margin = O.block_mask(q64, k64, tau, 1.5, False)
        expect = max(1, round(rho * 8)) / 8
        assert abs(M.mean() - expect) < 1e-12, (rho, M.mean())
        for i in range(M.shape[0]):
            assert np.array_equal(np.nonzero(M[i])[0], owned[i])
        assert margin > 1e-2


def test_near_tie_outcomes_cover_every_float32_divergence():
    """Reading r10: the oracle's near-tie fork (halley_bisection_outcomes) must contain every
    result a float32 run of Alg. 1 (with the r5 slack) reaches when it branches away from the
    float64 mirror.  Swept over small causal heads at T = 1..3 where divergences occur; the main
    run is bitwise the mirror."""
    import synth
    div = 0
    for seed in range(60):
        for N in (2, 3, 5, 9, 17, 40):
            for alpha in (1.25, 1.5, 2.0, 1.33):
                for T in (1, 2, 3):
                    q, k, _, _ = synth.gaussian_head(N, 16, seed=seed)
                    z = (alpha - 1) * O.scores(q.astype(np.float64), k.astype(np.float64), 0.25, True)
                    t64, alts = O.halley_bisection_outcomes(z, alpha, T)
                    assert np.array_equal(t64, O.halley_bisection(z, alpha, T))
                    t32 = O.halley_bisection(z, alpha, T, dtype=np.float32, slack_ulps=8)
                    d = np.abs(t32 - t64) > 1e-3 * np.maximum(1.0, np.abs(t64))
                    if d.any():
                        div += int(d.sum())
                        assert alts.size, (seed, N, alpha, T)
                        near = np.abs(alts[:, d] - t32[d]) <= 1e-3 * np.maximum(1.0, np.abs(t32[d]))
                        assert near.any(0).all(), (seed, N, alpha, T)
    assert div >= 5, "no float32/float64 branch divergence found to exercise the fork"


def test_near_tie_fork_flags_an_exact_tie_and_spares_converged_rows():
    """A row whose Eq. 4 decision is an exact tie gets an alternative outcome; rows of the paper's
    Gaussian benchmark at T >= 3 (converged) get almost none; mirror_tau holds every unflagged row
    to the float64 mirror whatever value the GPU reports."""
    from tests.parity import mirror_tau
    # α = 2, z = [0, −1/2] (n = 2): bracket [−1, −1/2], τ0 = −3/4, f(τ0) = 3/4 + 1/4 − 1 = 0 exactly —
    # an exact tie of Eq. 4 at the root: both branches give τ = −3/4 (immaterial), no alternative
    z = np.array([[0.0, -0.5]])
    lo, hi, tau0 = O.bracket_init(z, 2.0)
    assert tau0[0] == -0.75 and O.root_f(z, tau0, 2.0)[0][0] == 0.0
    t, alts = O.halley_bisection_outcomes(z, 2.0, 1)
    assert t[0] == -0.75 and (alts.size == 0 or not np.isfinite(alts).any())
    # Gaussian benchmark rows, T = 3: few flagged rows
    import synth
    q, k, _, _ = synth.gaussian_head(512, 64, seed=3)
    q, k = q.astype(np.float64), k.astype(np.float64)
    for alpha in (1.25, 1.5):
        t64, alts = O.solve_tau_outcomes(q, k, alpha, False, 3)
        flagged = np.isfinite(alts).any(0) if alts.size else np.zeros(512, bool)
        assert flagged.mean() <= 0.02, (alpha, flagged.mean())
        junk = t64 + 0.37                                   # a wrong "GPU" τ
        got = mirror_tau(q, k, alpha, False, 3, junk)
        assert np.array_equal(got[~flagged], t64[~flagged])


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0, 1.7])
@pytest.mark.parametrize("causal", [False, True])
def test_o2_matches_the_delta_identity(alpha, causal):
    """P:L786-796 (Eq. getting_di): δ_i = U_iᵀ dP_i / ‖U_i‖₁ = dO_iᵀ O⁽²⁾_i.  attn_fwd's O⁽²⁾ must give
    the δ of the first line computed densely (U = P^{2−α}, dP = dO Vᵀ), and the δ attn_bwd uses —
    which the finite-difference gradient tests pin (dropping it breaks them)."""
    rng = np.random.default_rng(31)
    q, k, v = _qkv(96, 16, 30)
    dO = rng.standard_normal(v.shape)
    fw = O.attn_fwd(q, k, v, alpha, causal, exact=True)
    delta_o2 = np.sum(dO * fw["O2"], 1)
    p = O.probs(q, k, fw["tau"], alpha, causal, O.default_scale(16), np.arange(96))
    u = np.where(p > 0, np.power(np.where(p > 0, p, 1.0), 2.0 - alpha), 0.0)
    dP = dO @ v.T
    delta_first = (u * dP).sum(1) / u.sum(1)
    np.testing.assert_allclose(delta_o2, delta_first, atol=1e-10, rtol=0)
    bw = O.attn_bwd(q, k, v, dO, fw["tau"], alpha, causal)
    np.testing.assert_allclose(delta_o2, bw["delta"], atol=1e-10, rtol=0)
    assert np.abs(u.sum(1) - 1.0).max() > 1e-2 or alpha == 2.0   # ‖U‖₁ ≠ 1: normalisation matters


def test_o2_hand_example_three_keys():
    """One query, three keys, α = 1.5, c = 1, V = I.  Scaled scores z = (α−1)s = [0.5, 0, −2].
    On the support {1, 2}: a = z1 − τ, b = a − 1/2, a² + b² = 1 (Eq. 3, e = 2) ⇒ 2a² − a − 3/4 = 0,
    a = (1 + √7)/4, b = (√7 − 1)/4, τ = 1/2 − a; z3 − τ = −2 − τ < 0 (off the support).
    P = [a², b², 0] (Eq. 2); U = P^{1/2} = [a, b, 0], ‖U‖₁ = √7/2 ≠ 1:
    O = P, O⁽²⁾ = [a, b, 0]/(√7/2)."""
    a = (1 + np.sqrt(7)) / 4
    b = (np.sqrt(7) - 1) / 4
    q = np.array([[1.0]])
    k = np.array([[1.0], [0.0], [-4.0]])
    fw = O.attn_fwd(q, k, np.eye(3), 1.5, False, exact=True, scale=1.0)
    np.testing.assert_allclose(fw["tau"], [0.5 - a], atol=1e-14)
    np.testing.assert_allclose(fw["O"][0], [a * a, b * b, 0.0], atol=1e-14)
    np.testing.assert_allclose(fw["O2"][0], [a / (np.sqrt(7) / 2), b / (np.sqrt(7) / 2), 0.0], atol=1e-14)
    np.testing.assert_allclose(fw["usum"], [np.sqrt(7) / 2], atol=1e-14)
