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


def test_parity_mirror_selection_prefers_the_matching_precision():
    """tests/parity.mirror_tau (reading r10) returns the float64 mirror when the GPU τ agrees with
    it, and, row by row, the float32 twin when the GPU τ sits on that twin's branch."""
    from tests.parity import mirror_tau
    import synth
    found = False
    for seed, N, alpha, T in ((13, 2, 1.5, 2), (20, 5, 1.5, 2), (23, 3, 2.0, 1)):   # known divergences
        q, k, _, _ = synth.gaussian_head(N, 16, seed=seed)
        q, k = q.astype(np.float64), k.astype(np.float64)
        if True:
            t64 = O.solve_tau(q, k, alpha, True, T)
            t32 = O.solve_tau(q, k, alpha, True, T, dtype=np.float32)
            assert np.array_equal(mirror_tau(q, k, alpha, True, T, t64.copy()), t64)
            diff = np.abs(t32 - t64) > 1e-6
            if diff.any():
                got = mirror_tau(q, k, alpha, True, T, t32.copy())
                assert np.array_equal(got[diff], t32[diff])
                found = True
    assert found, "no float32/float64 branch divergence found to exercise the selection"
