"""α-entmax attention forward/backward in float64 — TEST INFRASTRUCTURE
(see oracle/__init__.py).  One head at a time: Q, K, V, dO are (n, d) arrays.

Forward  = App. A.1 with τ from Alg. 1 (T-step mirror) or exact;
Mask     = Eq. 9 read as "block (i, j) is active iff some entry of
           P in it is non-zero" (readings c1, c2, c3);
Tables   = 𝒬_i, 𝒦_j;
Backward = App. A.2 with the 1/√d factor on dQ, dK that Eq. 1
            implies (reading c9).

Memory: rows are processed in chunks so that no more than ``_CHUNK_ELEMS``
score entries are alive at once; a chunk is a plain slice of the dense
definition (the sums over rows in dK/dV are accumulated chunk by chunk).
"""
from __future__ import annotations

import numpy as np

from .rowwise import entmax_probs, halley_bisection, halley_bisection_outcomes, tau_exact

_CHUNK_ELEMS = 1 << 24


def default_scale(d: int) -> float:
    """c = 1/√d (Eq. 1)."""
    return 1.0 / np.sqrt(d)


def scores(q, k, scale, causal, rows=None):
    """S = c·Q Kᵀ (Eq. 1) for the given query rows, −inf where key j > query i
    under causal masking (reading c13)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    rows = np.arange(q.shape[0]) if rows is None else np.asarray(rows)
    s = scale * (q[rows] @ k.T)
    if causal:
        s[np.arange(k.shape[0])[None, :] > rows[:, None]] = -np.inf
    return s


def _row_chunks(rows, n_keys):
    step = max(1, _CHUNK_ELEMS // max(1, n_keys))
    for a in range(0, len(rows), step):
        yield rows[a:a + step]


def solve_tau(q, k, alpha, causal, n_iter=None, scale=None, rows=None, dtype=np.float64):
    """τ per query row: Alg. 1 mirror for ``n_iter`` iterations, or the exact
    threshold when ``n_iter`` is None.  Pre-scaled convention z = (α−1)·S (Alg. 1
    line 3), i.e. the τ of Eq. 2.  ``dtype``: precision of the mirror's iteration
    (halley_bisection); the scores are float64 either way."""
    n, d = np.asarray(q).shape
    scale = default_scale(d) if scale is None else scale
    rows = np.arange(n) if rows is None else np.asarray(rows)
    out = np.empty(len(rows))
    pos = 0
    for rc in _row_chunks(rows, k.shape[0]):
        z = (alpha - 1.0) * scores(q, k, scale, causal, rc)
        out[pos:pos + len(rc)] = (tau_exact(z, alpha) if n_iter is None
                                  else halley_bisection(z, alpha, n_iter, dtype=dtype))
        pos += len(rc)
    return out


def solve_tau_outcomes(q, k, alpha, causal, n_iter, scale=None, rows=None):
    """The T-step Alg. 1 mirror per query row plus its alternative valid outcomes through
    near-ties (``halley_bisection_outcomes``, reading r10): returns (τ_T, alts) with alts of shape
    (n_alt, len(rows)), NaN where a row has none."""
    n, d = np.asarray(q).shape
    scale = default_scale(d) if scale is None else scale
    rows = np.arange(n) if rows is None else np.asarray(rows)
    main = np.empty(len(rows))
    alt_parts = []
    pos = 0
    for rc in _row_chunks(rows, k.shape[0]):
        z = (alpha - 1.0) * scores(q, k, scale, causal, rc)
        t, a = halley_bisection_outcomes(z, alpha, n_iter)
        main[pos:pos + len(rc)] = t
        alt_parts.append((pos, a))
        pos += len(rc)
    n_alt = max((a.shape[0] for _, a in alt_parts), default=0)
    alts = np.full((n_alt, len(rows)), np.nan)
    for p0, a in alt_parts:
        alts[:a.shape[0], p0:p0 + a.shape[1]] = a
    return main, alts


def probs(q, k, tau_rows, alpha, causal, scale, rows):
    """P rows (Eq. 2 / Alg. 2 line 13) for given rows and their τ."""
    z = (alpha - 1.0) * scores(q, k, scale, causal, rows)
    return entmax_probs(z, tau_rows, alpha)


def u_of_p(p, alpha):
    """U = P^{2−α}, 0 where P = 0."""
    return np.where(p > 0, np.power(np.where(p > 0, p, 1.0), 2.0 - alpha), 0.0)


def attn_fwd(q, k, v, alpha, causal=False, n_iter=3, scale=None, Br=128, Bc=128,
             exact=False, rows=None, tau=None):
    """Forward pass of App. A.1: τ (Alg. 1), then O_i = Σ_j P_ij V_j
    (Eq. getting-oi) and O⁽²⁾_i = Σ_j U_ij V_j / ‖U_i‖₁.

    ``rows`` restricts the computation to those query rows (row-sampled checks at
    full size); ``tau`` supplies precomputed per-row thresholds for those rows.
    Returns dict(tau, O, O2, usum, rows)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n, d = q.shape
    scale = default_scale(d) if scale is None else scale
    rows = np.arange(n) if rows is None else np.asarray(rows)
    if tau is None:
        tau = solve_tau(q, k, alpha, causal, None if exact else n_iter, scale, rows)
    O = np.empty((len(rows), v.shape[1]))
    O2 = np.empty_like(O)
    usum = np.empty(len(rows))
    pos = 0
    for rc in _row_chunks(rows, k.shape[0]):
        t = tau[pos:pos + len(rc)]
        p = probs(q, k, t, alpha, causal, scale, rc)
        u = u_of_p(p, alpha)
        O[pos:pos + len(rc)] = p @ v
        us = u.sum(1)
        O2[pos:pos + len(rc)] = (u @ v) / us[:, None]
        usum[pos:pos + len(rc)] = us
        pos += len(rc)
    return dict(tau=tau, O=O, O2=O2, usum=usum, rows=rows)


def block_mask(q, k, tau, alpha, causal=False, scale=None, Br=128, Bc=128, row_blocks=None):
    """Eq. 9 with readings c1/c2: M_ij = 1 iff some P entry of block
    (i, j) is non-zero, i.e. ∃ i′ ∈ block i, j′ ∈ block j with (α−1)S_{i′j′} − τ_{i′} > 0.
    ``tau`` holds τ for ALL rows.  ``row_blocks`` restricts to those block rows.
    Also returns the block margin min_ij |max_{(i′,j′) ∈ block} (z − τ)| that
    decides how robust the mask is to rounding."""
    q = np.asarray(q, dtype=np.float64)
    n, d = q.shape
    scale = default_scale(d) if scale is None else scale
    Tr, Tc = -(-n // Br), -(-k.shape[0] // Bc)
    row_blocks = range(Tr) if row_blocks is None else row_blocks
    M = np.zeros((len(row_blocks), Tc), dtype=np.uint8)
    margin = np.inf
    for a, i in enumerate(row_blocks):
        rows = np.arange(i * Br, min(n, (i + 1) * Br))
        x = (alpha - 1.0) * scores(q, k, scale, causal, rows) - tau[rows][:, None]
        for j in range(Tc):
            xb = x[:, j * Bc:min(k.shape[0], (j + 1) * Bc)]
            mx = xb.max()
            if np.isfinite(mx):
                M[a, j] = 1 if mx > 0 else 0
                margin = min(margin, abs(mx))
    return M, margin


def mask_from_p(P, Br=128, Bc=128):
    """Brute-force mask: block-OR of P > 0 over a dense P (pin for block_mask)."""
    n, m = P.shape
    Tr, Tc = -(-n // Br), -(-m // Bc)
    M = np.zeros((Tr, Tc), dtype=np.uint8)
    for i in range(Tr):
        for j in range(Tc):
            M[i, j] = np.any(P[i * Br:(i + 1) * Br, j * Bc:(j + 1) * Bc] > 0)
    return M


def lookup_tables(M):
    """Pointer-increment lookup tables:
    𝒬_i = {j | M_ij = 1} per query block, 𝒦_j = {i | M_ij = 1} per key block."""
    M = np.asarray(M)
    Q = [np.nonzero(M[i])[0] for i in range(M.shape[0])]
    K = [np.nonzero(M[:, j])[0] for j in range(M.shape[1])]
    return Q, K


def attn_bwd(q, k, v, dO, tau, alpha, causal=False, scale=None, key_cols=None, use_delta=True, rows=None):
    """Backward pass of App. A.2, dense over rows (chunked):
      δ_i  = dO_iᵀ O⁽²⁾_i
      dP   = dO Vᵀ
      dS   = U ⊙ (dP − δ)
      dV   = Pᵀ dO
      dQ   = c · dS K ,  dK = c · dSᵀ Q             (× c from Eq. 1)
    ``tau`` is τ for ALL rows (the forward's τ).  ``key_cols`` restricts
    dK/dV to those key rows (row-sampled checks); dQ is then not returned.
    ``use_delta=False`` drops δ (mutation test only).  ``rows`` restricts the query rows whose
    contributions are summed (dK/dV become partial sums; bench.py's bounded CPU sample only)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    dO = np.asarray(dO, dtype=np.float64)
    n, d = q.shape
    scale = default_scale(d) if scale is None else scale
    cols = np.arange(k.shape[0]) if key_cols is None else np.asarray(key_cols)
    dQ = np.zeros_like(q) if key_cols is None else None
    dK = np.zeros((len(cols), d))
    dV = np.zeros((len(cols), v.shape[1]))
    delta = np.zeros(n)
    for rc in _row_chunks(np.arange(n) if rows is None else np.asarray(rows), k.shape[0]):
        p = probs(q, k, tau[rc], alpha, causal, scale, rc)
        u = u_of_p(p, alpha)
        o2 = (u @ v) / u.sum(1)[:, None]
        dl = np.sum(dO[rc] * o2, axis=1) if use_delta else np.zeros(len(rc))
        delta[rc] = dl
        dp = dO[rc] @ v.T
        ds = u * (dp - dl[:, None])
        if dQ is not None:
            dQ[rc] = scale * (ds @ k)
        dK += scale * (ds[:, cols].T @ q[rc])
        dV += p[:, cols].T @ dO[rc]
    return dict(dQ=dQ, dK=dK, dV=dV, delta=delta)


def softmax_attention(q, k, v, causal=False, scale=None):
    """Eq. 1 with π = softmax: the α → 1 limit of Eq. 2."""
    q = np.asarray(q, dtype=np.float64)
    scale = default_scale(q.shape[1]) if scale is None else scale
    s = scores(q, k, scale, causal)
    s = s - s.max(1, keepdims=True)
    e = np.exp(s)
    return (e / e.sum(1, keepdims=True)) @ np.asarray(v, dtype=np.float64)
