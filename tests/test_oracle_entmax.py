"""Pins for oracle/rowwise.py (row-wise α-entmax).  CPU only.

Each test ties the oracle to something other than itself: worked examples
(tests/golden/spec_examples.txt, cited), brute-force enumeration of supports,
closed forms, limits, invariants and the paper's convergence claims.
"""
import itertools
import os

import numpy as np
import pytest

from oracle import rowwise as E

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def _golden():
    rows = []
    with open(GOLDEN) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            name, alpha, s, tau, p = [t.strip() for t in line.split("|")]
            rows.append((name, float(alpha), np.array([float(x) for x in s.split(",")]),
                         float(tau), np.array([float(x) for x in p.split(",")])))
    return rows


@pytest.mark.parametrize("name,alpha,s,tau,p", _golden())
def test_golden_examples(name, alpha, s, tau, p):
    z = (alpha - 1.0) * s[None, :]
    t_exact = E.tau_exact(z, alpha)[0]
    assert abs(t_exact - tau) <= 1e-12, name
    np.testing.assert_allclose(E.entmax_probs(z, np.array([t_exact]), alpha)[0], p, atol=1e-12)
    # Alg. 1 mirror converges to the same example (T = 30 >> needed)
    t_mirror = E.halley_bisection(z, alpha, 30)[0]
    assert abs(t_mirror - tau) <= 1e-12, name


def test_root_f_spec_values():
    # s=[0,0] (scaled), α=2, τ=−0.5 → f=0, f'=−2, f''=0
    f, f1, f2 = E.root_f(np.array([[0.0, 0.0]]), np.array([-0.5]), 2.0)
    assert (f[0], f1[0], f2[0]) == (0.0, -2.0, 0.0)
    # [1,0], α=2, τ=0 → f = 0
    assert E.root_f(np.array([[1.0, 0.0]]), np.array([0.0]), 2.0)[0][0] == 0.0
    # [0.5,0.2], α=2, τ=−0.15 → f=0, f'=−2
    f, f1, _ = E.root_f(np.array([[0.5, 0.2]]), np.array([-0.15]), 2.0)
    assert abs(f[0]) < 1e-15 and f1[0] == -2.0


def test_halley_step_spec():
    # root is a fixed point; α=2 (f''=0): f=0.5, f'=−2, τ=1 → Newton 1.25
    th, ok = E.halley_update(np.array([0.5]), np.array([-2.0]), np.array([0.0]), np.array([1.0]))
    assert ok[0] and th[0] == 1.25
    th, ok = E.halley_update(np.array([0.0]), np.array([-3.0]), np.array([1.0]), np.array([0.7]))
    assert ok[0] and th[0] == 0.7
    # zero denominator is flagged so the caller bisects
    _, ok = E.halley_update(np.array([0.0]), np.array([0.0]), np.array([0.0]), np.array([0.0]))
    assert not ok[0]


def _brute_tau(z, alpha):
    """Enumerate every support set S; solve Σ_{i∈S}(z_i−τ)^e = 1 on S with a
    polynomial root finder and keep the unique consistent S (z_i > τ on S,
    z_j <= τ off S).  Independent of sorting and of bisection."""
    e = int(round(1.0 / (alpha - 1.0)))
    n = len(z)
    found = []
    for r in range(1, n + 1):
        for S in itertools.combinations(range(n), r):
            zs = z[list(S)]
            # Σ (z_i − τ)^e − 1 as a polynomial in τ
            poly = np.zeros(e + 1)
            for zi in zs:
                poly = np.polyadd(poly, np.poly1d([-1.0, zi]) ** e)
            poly = np.polysub(poly, [1.0])
            roots = np.roots(np.atleast_1d(poly))
            for t in roots:
                if abs(t.imag) > 1e-9:
                    continue
                t = t.real
                inside = np.all(zs > t + 1e-12)
                outside = np.all(np.delete(z, list(S)) <= t + 1e-12)
                if inside and outside:
                    found.append(t)
    found = np.unique(np.round(found, 10))
    assert len(found) == 1, found
    return found[0]


@pytest.mark.parametrize("alpha", [2.0, 1.5, 1.25])
def test_exact_tau_vs_bruteforce(alpha):
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = rng.integers(1, 7)
        z = rng.standard_normal(n) * rng.choice([0.1, 1.0, 3.0])
        t_b = _brute_tau(z, alpha)
        t = E.tau_exact(z[None, :], alpha)[0]
        assert abs(t - t_b) < 1e-8, (trial, z, t, t_b)


@pytest.mark.parametrize("alpha", [2.0, 1.5])
def test_sort_forms_match_long_bisection(alpha):
    rng = np.random.default_rng(1)
    for n in (2, 3, 17, 256, 8192):
        z = (alpha - 1) * rng.standard_normal((8, n))
        np.testing.assert_allclose(E.tau_exact(z, alpha), E.tau_bisect_exact(z, alpha), atol=1e-12, rtol=0)


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_simplex_sparsity_rule_and_equivariances(alpha):
    rng = np.random.default_rng(3)
    s = rng.standard_normal((32, 64)) * 2
    p = E.entmax(s, alpha)
    np.testing.assert_allclose(p.sum(1), 1.0, atol=1e-10)
    assert (p >= 0).all()
    z = (alpha - 1) * s
    tau = E.tau_exact(z, alpha)
    assert np.array_equal(p == 0, z <= tau[:, None])          # P:L126 zero rule
    np.testing.assert_allclose(E.entmax(s + 3.7, alpha), p, atol=1e-10)   # shift invariance
    perm = rng.permutation(64)
    np.testing.assert_allclose(E.entmax(s[:, perm], alpha), p[:, perm], atol=1e-12)


def test_alpha2_is_simplex_projection():
    """α=2 is sparsemax = argmin_p ||p − s||² on the simplex; check the
    KKT conditions of that QP directly."""
    rng = np.random.default_rng(11)
    s = rng.standard_normal((50, 20))
    p = E.entmax(s, 2.0)
    for i in range(50):
        sup = p[i] > 0
        lam = (s[i] - p[i])[sup]                         # s − p = λ on the support
        assert np.ptp(lam) < 1e-12
        assert np.all(s[i][~sup] - p[i][~sup] <= lam[0] + 1e-12)


def test_alpha_to_one_recovers_softmax():
    """α → 1 recovers softmax; the gap shrinks ~linearly in α−1."""
    rng = np.random.default_rng(5)
    s = rng.standard_normal((16, 32))
    sm = np.exp(s - s.max(1, keepdims=True))
    sm /= sm.sum(1, keepdims=True)
    gaps = [np.abs(E.entmax(s, a) - sm).max() for a in (1.1, 1.01, 1.001)]
    assert gaps[0] > gaps[1] > gaps[2]
    assert gaps[2] < 2e-3
    assert 5 < gaps[0] / gaps[1] < 20 and 5 < gaps[1] / gaps[2] < 20


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_alg1_bracket_invariants(alpha):
    rng = np.random.default_rng(2)
    z = (alpha - 1) * rng.standard_normal((64, 300)) * 2
    tau0_lo, tau0_hi, _ = E.bracket_init(z, alpha)
    f_lo = E.root_f(z, tau0_lo, alpha)[0]
    f_hi = E.root_f(z, tau0_hi, alpha)[0]
    assert (f_lo >= 0).all() and (f_hi <= 0).all()          # Alg. 1 bracket is sound
    _, _, _, hist = E.halley_bisection(z, alpha, 12, return_state=True)
    width = tau0_hi - tau0_lo
    for tau, lo, hi in hist:
        assert (lo <= tau).all() and (tau <= hi).all()
        assert (E.root_f(z, lo, alpha)[0] >= 0).all()
        assert (E.root_f(z, hi, alpha)[0] <= 0).all()
        assert (hi - lo <= width + 1e-15).all()
        width = hi - lo


def test_bisection_halving_identity():
    """bracket width after T pure-bisection steps = initial width / 2^T."""
    rng = np.random.default_rng(4)
    z = 0.5 * rng.standard_normal((5, 100))
    lo0, hi0, _ = E.bracket_init(z, 1.5)
    _, lo, hi, _ = E.halley_bisection(z, 1.5, 10, return_state=True, halley=False)
    np.testing.assert_allclose(hi - lo, (hi0 - lo0) / 1024, rtol=1e-12)


def test_convergence_claim_p250():
    """P:L250 (Fig. 2): with α=1.5 on n=8192 N(0,1) logits Halley-bisection needs
    3 iterations to reach machine precision; plain bisection needs 23."""
    rng = np.random.default_rng(0)
    s = rng.standard_normal((32, 8192))
    z = 0.5 * s
    p_star = E.entmax_probs(z, E.tau_entmax15(z), 1.5)
    def mae(T, halley):
        t = E.halley_bisection(z, 1.5, T, halley=halley)
        return np.abs(E.entmax_probs(z, t, 1.5) - p_star).mean()
    halley = [mae(T, True) for T in range(1, 5)]
    assert halley[2] <= 1e-6                      # "only 3 iterations"
    assert halley[3] <= 1e-15
    # bisection: first T reaching the error Halley reaches at T=3
    target = max(halley[2], 1e-16)
    T_bis = next(T for T in range(1, 60) if mae(T, False) <= target)
    assert T_bis >= 15, T_bis                     # "takes 23 iterations" (same order)
    # Halley dominates bisection at every iteration count
    assert all(h <= mae(T + 1, False) for T, h in enumerate(halley))


def test_degenerate_rows():
    # n = 1 → p = 1; causal-style row with one visible entry
    z = np.array([[3.0, -np.inf, -np.inf]])
    for a in (1.25, 1.5, 2.0):
        t = E.halley_bisection(z, a, 3)
        np.testing.assert_allclose(E.entmax_probs(z, t, a), [[1.0, 0, 0]], atol=1e-15)


def test_vjp_null_space_and_fd():
    rng = np.random.default_rng(9)
    for alpha in (1.5, 2.0):
        s = rng.standard_normal((4, 16))
        p = E.entmax(s, alpha)
        np.testing.assert_allclose(E.entmax_vjp(p, np.ones_like(p) * 2.5, alpha), 0, atol=1e-12)
        dp = rng.standard_normal(p.shape)
        g = E.entmax_vjp(p, dp, alpha)
        h = 1e-6
        fd = np.zeros_like(s)
        for j in range(s.shape[1]):
            sp, sm_ = s.copy(), s.copy()
            sp[:, j] += h
            sm_[:, j] -= h
            fd[:, j] = ((E.entmax(sp, alpha) - E.entmax(sm_, alpha)) * dp).sum(1) / (2 * h)
        np.testing.assert_allclose(g, fd, atol=1e-6)


def test_float32_mirror_is_the_same_algorithm():
    """The float32-precision twin of the Alg. 1 mirror (reading r10) follows the same steps: it
    agrees with the float64 mirror to float32 rounding once the iteration has converged, keeps the
    bracket invariants, and reproduces the SPEC worked examples."""
    import synth
    s, _ = synth.rowwise_scores(64, 2048, 5)
    for alpha in (1.25, 1.5, 2.0, 1.7):
        z = (alpha - 1.0) * s.astype(np.float64)
        T = 6
        t64 = E.halley_bisection(z, alpha, T)
        t32 = E.halley_bisection(z, alpha, T, dtype=np.float32)
        assert np.all(np.abs(t32 - t64) <= 4e-6 * np.maximum(1.0, np.abs(t64))), alpha
        m = z.max(-1)
        assert np.all(t32 >= m - 1.0 - 1e-6) and np.all(t32 <= m + 1e-6)
    for zz, tau in (([0.5, 0.2], -0.15), ([0.0, 0.0], -0.5)):   # α = 2
        t = E.halley_bisection(np.array([zz]), 2.0, 8, dtype=np.float32)[0]
        assert abs(t - tau) < 1e-6
    # bisection-only mode: the same midpoint sequence
    z = 0.5 * s[:8].astype(np.float64)
    assert np.allclose(E.halley_bisection(z, 1.5, 10, halley=False),
                       E.halley_bisection(z, 1.5, 10, halley=False, dtype=np.float32), atol=1e-5)


@pytest.mark.parametrize("alpha", [1.25, 1.5, 1.7, 1.33, 2.0])
def test_root_f_derivatives_by_central_differences(alpha):
    """Eqs. 6-7: f′ and f″ returned by root_f are the derivatives of Eq. 3's f in τ.
    Central differences of f (for f′) and of f′ (for f″) at τ values whose x = z − τ keep a distance
    of at least 1e-3 from 0 (f is smooth there), for integer and non-integer 1/(α−1).  A dropped or
    mis-scaled coefficient of Eq. 6 or 7 (e.g. (2−α)/(α−1) instead of (2−α)/(α−1)²) fails."""
    rng = np.random.default_rng(17)
    z = (alpha - 1.0) * rng.standard_normal((200, 64)) * 2
    m = z.max(1)
    tau = m - rng.uniform(0.05, 1.0, 200)
    x = z - tau[:, None]
    keep = np.min(np.abs(x), 1) > 1e-3
    z, tau = z[keep], tau[keep]
    assert len(tau) > 100
    h = 1e-6
    f, f1, f2 = E.root_f(z, tau, alpha)
    fp, f1p, _ = E.root_f(z, tau + h, alpha)
    fm, f1m, _ = E.root_f(z, tau - h, alpha)
    np.testing.assert_allclose(f1, (fp - fm) / (2 * h), rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(f2, (f1p - f1m) / (2 * h), rtol=1e-5, atol=1e-6)
    if alpha != 2.0:
        assert np.abs(f2).max() > 1e-2                      # the check is not vacuous


def test_halley_convergence_alpha_125_p250_protocol():
    """P:L246-250 protocol (n = 8192 N(0,1) rows) at α = 1.25 (e = 4): Halley-bisection converges
    in a few iterations (cubic near the root: each iteration at least squares the error once in the
    basin), far faster than bisection; with f″ replaced by 0 (a Newton-bisection, i.e. a wrong Eq. 7)
    it is measurably slower — so the convergence claim depends on the f″ the oracle computes."""
    rng = np.random.default_rng(2)
    z = 0.25 * rng.standard_normal((32, 8192))
    t_star = E.tau_bisect_exact(z, 1.25)
    p_star = E.entmax_probs(z, t_star, 1.25)
    errs = [np.abs(E.entmax_probs(z, E.halley_bisection(z, 1.25, T), 1.25) - p_star).mean() for T in range(1, 6)]
    assert errs[2] <= 1e-8 and errs[4] <= 1e-15, errs
    bis = np.abs(E.entmax_probs(z, E.halley_bisection(z, 1.25, 3, halley=False), 1.25) - p_star).mean()
    assert bis > 1e3 * errs[2]
    # Newton variant: same Alg. 1 loop with f″ := 0
    lo, hi, tau = E.bracket_init(z, 1.25)
    for _ in range(3):
        f, f1, _ = E.root_f(z, tau, 1.25)
        lo, hi = E.bisection_update(f, tau, lo, hi)
        th, ok = E.halley_update(f, f1, np.zeros_like(f), tau)
        ok &= (th >= lo) & (th <= hi)
        tau = np.where(ok, th, 0.5 * (lo + hi))
    newton = np.abs(E.entmax_probs(z, tau, 1.25) - p_star).mean()
    assert newton > 10 * errs[2], (newton, errs[2])
