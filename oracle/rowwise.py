"""Row-wise α-entmax in float64 — TEST INFRASTRUCTURE (see oracle/__init__.py).

Every function follows PAPER.md (/root/reference/PAPER.md, cited as P:L<n>) in
the paper's order and notation.  Inputs ``z`` are rows of *pre-scaled* scores
z = (α−1)·s (Alg. 1 line 3).  Entries equal to −inf are "not visible"
(causal mask / padding) and contribute nothing; ``n`` in Alg. 1 line 5 is the
count of visible entries per row (reading c8).
"""
from __future__ import annotations

import numpy as np


def relu_pow(x: np.ndarray, p: float) -> np.ndarray:
    """[x]_+^p with the strict-indicator convention [x]_+^p := 0 for x <= 0 for
    every p (reading c7; Eqs. 6-7 P:L226-227 raise [·]_+ to powers that
    may be 0 or negative)."""
    out = np.zeros_like(x, dtype=np.float64)
    m = x > 0
    out[m] = np.power(x[m], p)
    return out


def root_f(z: np.ndarray, tau: np.ndarray, alpha: float):
    """f(τ), f'(τ), f''(τ) of Eq. 3 and Eqs. 6-7, on
    pre-scaled rows z (shape (..., n)) and per-row τ (shape (...))."""
    e = 1.0 / (alpha - 1.0)
    x = z - tau[..., None]
    f = relu_pow(x, e).sum(-1) - 1.0                                   # Eq. 3
    f1 = -(1.0 / (alpha - 1.0)) * relu_pow(x, e - 1.0).sum(-1)         # Eq. 6
    f2 = ((2.0 - alpha) / (alpha - 1.0) ** 2) * relu_pow(x, e - 2.0).sum(-1)  # Eq. 7
    return f, f1, f2


def bracket_init(z: np.ndarray, alpha: float):
    """Alg. 1 lines 4-6: τ_lo = max − 1, τ_hi = max − n^{1−α},
    τ = midpoint; n = visible entries per row."""
    m = z.max(-1)
    n = np.isfinite(z).sum(-1).astype(np.float64)
    tau_lo = m - 1.0
    tau_hi = m - n ** (1.0 - alpha)
    return tau_lo, tau_hi, 0.5 * (tau_lo + tau_hi)


def bisection_update(f, tau, tau_lo, tau_hi):
    """Eq. 4: (τ_lo, τ) if f(τ) < 0 else (τ, τ_hi).  A tie f = 0
    takes the 'otherwise' branch (reading c5)."""
    neg = f < 0
    return np.where(neg, tau_lo, tau), np.where(neg, tau, tau_hi)


def halley_update(f, f1, f2, tau):
    """Eq. 5: H_f(τ) = τ − 2 f f' / (2 f'^2 − f f'').  Returns
    (τ_H, ok) with ok False where the denominator is 0 or non-finite (reading c6)."""
    den = 2.0 * f1 * f1 - f * f2
    with np.errstate(divide="ignore", invalid="ignore"):
        tau_h = tau - 2.0 * f * f1 / den
    ok = np.isfinite(tau_h) & (den != 0)
    return tau_h, ok


def halley_bisection(z: np.ndarray, alpha: float, T: int, return_state: bool = False,
                     halley: bool = True, dtype=np.float64, slack_ulps: int = 0):
    """Alg. 1 run for exactly T iterations, row-wise (the "T-step
    mirror" the GPU is compared against).  Each iteration: evaluate f, f', f'' at
    the current τ; bracket update (line 8); Halley candidate (line 9); accept it iff
    inside the *updated* bracket [τ_lo, τ_hi] (inclusive, line 10), else take the
    midpoint (line 13).  The returned τ is the one after the T-th update (reading
    c4).  ``halley=False`` gives the pure-bisection scheme of Eq. 4 whose answer is
    the midpoint after the last bracket update.

    ``dtype=np.float32`` runs the same steps in float32 arithmetic: Alg. 1's discrete
    decisions (the sign of f in Eq. 4, the Halley acceptance test) then fall where a float32
    implementation's can, which a parity check needs when T is too small for the iteration to
    have converged (a near-tie decided differently in float64 sends the float64 mirror down
    another branch).  The float64 mirror is the reference; this is its float32-precision twin
    (reading r10).  ``slack_ulps`` (low precision only): accept a Halley candidate up to
    that many ulps outside the bracket and clamp it in (reading r5, the GPU's finite-precision
    form of line 10's inclusive test)."""
    if T < 1:
        raise ValueError("T >= 1 required (S:L54)")
    if dtype is not np.float64:
        with np.errstate(all="ignore"):
            return _halley_bisection_lowp(np.asarray(z, dtype=dtype), alpha, T, halley, dtype, slack_ulps)
    z = np.asarray(z, dtype=np.float64)
    tau_lo, tau_hi, tau = bracket_init(z, alpha)
    history = []
    for _ in range(T):
        f, f1, f2 = root_f(z, tau, alpha)
        tau_lo, tau_hi = bisection_update(f, tau, tau_lo, tau_hi)
        mid = 0.5 * (tau_lo + tau_hi)
        if halley:
            tau_h, ok = halley_update(f, f1, f2, tau)
            ok &= (tau_h >= tau_lo) & (tau_h <= tau_hi)
            tau = np.where(ok, tau_h, mid)
        else:
            tau = mid
        if return_state:
            history.append((tau.copy(), tau_lo.copy(), tau_hi.copy()))
    if return_state:
        return tau, tau_lo, tau_hi, history
    return tau


def _alg1_step(z, alpha, tau, tau_lo, tau_hi, halley, flip_sign=None, flip_accept=None):
    """One Alg. 1 iteration (lines 7-14) with optional forced flips of its two discrete decisions
    (the Eq. 4 sign of f, the line-10 acceptance of the Halley candidate), rows where the flip mask
    is True taking the other branch.  Returns (τ, τ_lo, τ_hi) and the decisions' relative margins."""
    e = 1.0 / (alpha - 1.0)
    f, f1, f2 = root_f(z, tau, alpha)
    scale_t = np.maximum(1.0, np.abs(tau))
    ssum = relu_pow(z - tau[..., None], e).sum(-1)
    m_sign = np.abs(f) / (ssum + np.abs(f1) * scale_t)
    if flip_sign is not None:
        # the other side of a near-tie of Eq. 4: f of the opposite sign, same magnitude (a finite-
        # precision run that sees the other sign computes its Halley candidate from that f too)
        f = np.where(flip_sign, -f, f)
    neg = f < 0
    lo = np.where(neg, tau_lo, tau)
    hi = np.where(neg, tau, tau_hi)
    mid = 0.5 * (lo + hi)
    if not halley:
        return mid, lo, hi, m_sign, np.full_like(m_sign, np.inf)
    tau_h, ok = halley_update(f, f1, f2, tau)
    den = 2.0 * f1 * f1 - f * f2
    with np.errstate(divide="ignore", invalid="ignore"):
        m_den = np.where(ok, np.abs(den) / (2.0 * f1 * f1 + np.abs(f * f2)), np.inf)
        th = np.where(ok, tau_h, 0.0)
        # The updated bracket has τ itself at one end; the Halley step moves away from τ in the
        # direction the sign of f gives (f >= 0 → τ = τ_lo and τ_H >= τ for den > 0), the same sign
        # that moved the bracket, so a candidate is never in doubt at that end (a finite-precision
        # run sees both with one sign) unless den is near 0.  The decision can only tie at the FAR
        # end: relative distance of τ_H to it, inside or outside.
        far = np.where(neg, lo, hi)
        m_far = np.where(ok, np.abs(th - far) / scale_t, np.inf)
    acc = ok & (th >= lo) & (th <= hi)
    m_acc = np.minimum(m_far, m_den)
    # A candidate ON the far end to within float64 rounding (Newton/Halley landing exactly on
    # τ_lo = m − 1, e.g. a one-element support) is accepted by the inclusive test of exact
    # arithmetic (reading c6) and by any finite-precision form of it with a rounding slack (r5):
    # not a near-tie when accepted (a float64 rejection 1 ulp outside still is one).
    m_acc = np.where(acc & (m_far <= 4.0 * np.finfo(np.float64).eps), m_den, m_acc)
    if flip_accept is not None:
        acc = np.where(flip_accept & ok, ~acc, acc)
    return np.where(acc, th, mid), lo, hi, m_sign, m_acc


def halley_bisection_outcomes(z: np.ndarray, alpha: float, T: int, halley: bool = True,
                              margin: float = 3e-5, material: float = 1e-4):
    """Alg. 1 for T iterations in float64, plus every *other* valid outcome a
    finite-precision run could reach through a near-tie (reading r10).

    Each iteration takes two discrete decisions: the sign of f(τ) in Eq. 4 and the
    acceptance of the Halley candidate in line 10 (inside the updated bracket, finite, non-zero
    denominator).  A float32 implementation rounds z, τ and the sums at ~1e-7 relative, so where a
    decision's relative margin (``_alg1_step``) is below ``margin`` it may go the other way.  For
    every such decision the run is forked with that one decision flipped and continued to T
    iterations; forks whose final τ differs from the main run by more than ``material``·max(1, |τ|)
    are alternative outcomes.  Returns (τ_T, alts) with alts of shape (n_alt, rows) (NaN where a
    row has no material near-tie).  Decided from the float64 trajectory alone — never from a value
    under test."""
    z = np.asarray(z, dtype=np.float64)
    lo, hi, tau = bracket_init(z, alpha)
    states = []
    for _ in range(T):
        states.append((tau, lo, hi))
        tau, lo, hi, _, _ = _alg1_step(z, alpha, tau, lo, hi, halley)
    main = tau
    alts = []
    for t, (tau0, lo0, hi0) in enumerate(states):
        _, _, _, m_sign, m_acc = _alg1_step(z, alpha, tau0, lo0, hi0, halley)
        for kind, m in (("sign", m_sign), ("accept", m_acc)):
            near = m < margin
            if not near.any():
                continue
            fs = near if kind == "sign" else None
            fa = near if kind == "accept" else None
            tt, ll, hh, _, _ = _alg1_step(z, alpha, tau0, lo0, hi0, halley, flip_sign=fs, flip_accept=fa)
            for _ in range(t + 1, T):
                tt, ll, hh, _, _ = _alg1_step(z, alpha, tt, ll, hh, halley)
            differs = near & (np.abs(tt - main) > material * np.maximum(1.0, np.abs(main)))
            if differs.any():
                alts.append(np.where(differs, tt, np.nan))
    return main, (np.stack(alts) if alts else np.empty((0,) + main.shape))


def _halley_bisection_lowp(z, alpha, T, halley, dt, slack_ulps=0):
    """Alg. 1 exactly as above, every operation in ``dt`` (see halley_bisection)."""
    a = dt(alpha)
    one, two, half = dt(1.0), dt(2.0), dt(0.5)
    e = one / (a - one)
    m = z.max(-1)
    n = np.isfinite(z).sum(-1).astype(dt)
    lo = m - one
    hi = m - np.power(n, one - a)
    tau = half * (lo + hi)
    for _ in range(T):
        x = z - tau[..., None]
        pos = x > 0
        xp = np.where(pos, x, dt(1.0))
        f = np.where(pos, np.power(xp, e), dt(0)).sum(-1, dtype=dt) - one
        f1 = -e * np.where(pos, np.power(xp, e - one), dt(0)).sum(-1, dtype=dt)
        f2 = ((two - a) / ((a - one) * (a - one))) * np.where(pos, np.power(xp, e - two), dt(0)).sum(-1, dtype=dt)
        neg = f < 0
        lo, hi = np.where(neg, lo, tau), np.where(neg, tau, hi)
        mid = half * (lo + hi)
        if halley:
            den = two * f1 * f1 - f * f2
            th = tau - two * f * f1 / den
            sl = dt(slack_ulps) * np.finfo(dt).eps * np.maximum(np.abs(lo), np.abs(hi))
            ok = np.isfinite(th) & (den != 0) & (th >= lo - sl) & (th <= hi + sl)
            tau = np.where(ok, np.minimum(np.maximum(th, lo), hi), mid)
        else:
            tau = mid
    return tau.astype(np.float64)


# ---------------------------------------------------------------------------
# Exact thresholds (the definition the iteration converges to)
# ---------------------------------------------------------------------------

def tau_sparsemax(z: np.ndarray) -> np.ndarray:
    """Exact τ for α = 2 (Euclidean projection onto the simplex),
    sort-and-scan: k* = max{k : 1 + k z_(k) > Σ_{r<=k} z_(r)},
    τ = (Σ_{r<=k*} z_(r) − 1)/k*.  Rows of pre-scaled z (α−1 = 1)."""
    z = np.asarray(z, dtype=np.float64)
    zs = -np.sort(-z, axis=-1)
    zs_f = np.where(np.isfinite(zs), zs, 0.0)
    cs = np.cumsum(zs_f, axis=-1)
    k = np.arange(1, z.shape[-1] + 1, dtype=np.float64)
    cond = (1.0 + k * zs_f > cs) & np.isfinite(zs)
    kstar = cond.shape[-1] - np.argmax(cond[..., ::-1], axis=-1)   # last True (1-based)
    csk = np.take_along_axis(cs, (kstar - 1)[..., None], -1)[..., 0]
    return (csk - 1.0) / kstar


def tau_entmax15(z: np.ndarray) -> np.ndarray:
    """Exact τ for α = 1.5 by the sort-based method of Peters et al.,
    derived from Eq. 3 with exponent 1/(α−1) = 2 on a fixed top-k support:
    Σ_{r<=k} (z_(r) − τ)^2 = 1  ⇒  τ_k = μ_k − sqrt((1 − k·σ²_k)/k)
    (μ_k mean, σ²_k = mean of squares − μ_k² of the top k), and
    k* = max{k : τ_k <= z_(k)}.  Rows of pre-scaled z."""
    z = np.asarray(z, dtype=np.float64)
    zs = -np.sort(-z, axis=-1)
    fin = np.isfinite(zs)
    zs_f = np.where(fin, zs, 0.0)
    k = np.arange(1, z.shape[-1] + 1, dtype=np.float64)
    mu = np.cumsum(zs_f, axis=-1) / k
    ms = np.cumsum(zs_f * zs_f, axis=-1) / k
    var = ms - mu * mu
    disc = (1.0 - k * var) / k
    with np.errstate(invalid="ignore"):
        tau_k = mu - np.sqrt(disc)
    cond = (disc >= 0) & (tau_k <= zs_f) & fin
    kstar = cond.shape[-1] - np.argmax(cond[..., ::-1], axis=-1)
    return np.take_along_axis(tau_k, (kstar - 1)[..., None], -1)[..., 0]


def tau_bisect_exact(z: np.ndarray, alpha: float, iters: int = 200) -> np.ndarray:
    """Exact τ for general α: Eq. 4 bisection from the Alg. 1 bracket, run until
    the float64 bracket collapses (200 halvings of a width <= 1)."""
    return halley_bisection(z, alpha, iters, halley=False)


def tau_exact(z: np.ndarray, alpha: float) -> np.ndarray:
    if alpha == 2.0:
        return tau_sparsemax(z)
    if alpha == 1.5:
        return tau_entmax15(z)
    return tau_bisect_exact(z, alpha)


def entmax_probs(z: np.ndarray, tau: np.ndarray, alpha: float) -> np.ndarray:
    """Eq. 2 on pre-scaled z: p = [z − τ]_+^{1/(α−1)}."""
    return relu_pow(z - tau[..., None], 1.0 / (alpha - 1.0))


def entmax(s: np.ndarray, alpha: float, T: int | None = None) -> np.ndarray:
    """α-entmax of raw scores s (Eq. 2): exact τ if T is None, else the T-step
    Halley-bisection mirror (Alg. 1)."""
    z = (alpha - 1.0) * np.asarray(s, dtype=np.float64)
    tau = tau_exact(z, alpha) if T is None else halley_bisection(z, alpha, T)
    return entmax_probs(z, tau, alpha)


def entmax_vjp(p: np.ndarray, dp: np.ndarray, alpha: float) -> np.ndarray:
    """Sparse Jacobian-vector product:
    J = Diag(u) − u uᵀ/‖u‖₁ with u_j = p_j^{2−α} (0 off support)."""
    u = np.where(p > 0, np.power(np.where(p > 0, p, 1.0), 2.0 - alpha), 0.0)
    return u * dp - (np.sum(u * dp, -1, keepdims=True) / np.sum(u, -1, keepdims=True)) * u
