"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NO arithmetic of the method (no scores, no entmax, no τ):
it only draws random tensors with the shapes and structure of the paper's
workloads, so that the oracle (``oracle/``) and the CUDA path
(``paper_2502_12082_b200``) can be fed bit-identical inputs without sharing
any code.  Recipes (DESIGN.md §"Input recipe"):

* ``gaussian``  — the paper's efficiency-benchmark generator: Q ~ N(0, σ²=6),
  K, V, dO ~ N(0, 1) ("σ² = 6 of query vectors").
* ``planted``   — planted block sparsity for the Fig. 1 "runtime vs input
  sparsity" sweep (modified).  Each query block
  is assigned a cluster direction u_c; each cluster owns m = max(1, round(ρ·T_c))
  key blocks (C <= 8 clusters).  Q rows are a·u_c + ε_q with ε_q ~ N(0, σ_q²=6)
  projected orthogonally to every cluster direction; owned K rows are a·u_c + N(0,1); dead K rows are N(0,1).
  With a = sqrt(gap·sqrt(d)) the scores of a query against its owned keys are
  gap + N(0, ≈7.4) after the 1/√d scale, against dead keys N(0, ≈7.4): inside
  the owned blocks the rows look like the paper's Gaussian benchmark (a few
  support keys per row, spread over all owned blocks), the dead blocks sit far
  below τ, so the realised block density is the target ρ with large margins.
  Keys keep a Gaussian spread around their cluster direction (a near-constant
  key set would make dQ = Σ dS·K a near-total cancellation).

* ``planted_tight`` — SURVEY App. P3's original recipe, kept as a stress case: the same planted block
  structure with near-duplicate keys and queries, Q = a·u_c + 0.02·N(0,1), owned K = a·u_c + 0.02·N(0,1)
  (dead K = N(0,1)).  Rows see hundreds of nearly equal scores and dQ = c·Σ_j dS_ij K_j is an almost
  total cancellation (real attention sees repeated tokens; reading r12).

* ``step``      — Gaussian with the first half of the keys scaled by 0.2 (structure test for the
  τ kernel's list-overflow tiers; no paper workload).

Every head (b, h) is drawn from its own stream seeded by (seed, b, h), so a rank
that owns a slice of heads regenerates exactly its slice.
Arrays are float32 numpy; callers round to the kernel dtype (bf16 RN via torch)
and hand the SAME rounded values to both sides.
"""
from __future__ import annotations

import numpy as np

__all__ = ["head_rng", "gaussian_head", "planted_head", "planted_tight_head", "step_head", "make_inputs", "HeadSpec", "rowwise_scores"]


def head_rng(seed: int, b: int, h: int, stream: int = 0) -> np.random.Generator:
    """Counter-style independent stream per (seed, b, h, stream)."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(b), int(h), int(stream)])))


def gaussian_head(N: int, d: int, seed: int, b: int = 0, h: int = 0, sigma2_q: float = 6.0):
    """Q ~ N(0, sigma2_q), K, V, dO ~ N(0, 1); each (N, d) float32."""
    rng = head_rng(seed, b, h)
    q = rng.standard_normal((N, d), dtype=np.float32) * np.float32(np.sqrt(sigma2_q))
    k = rng.standard_normal((N, d), dtype=np.float32)
    v = rng.standard_normal((N, d), dtype=np.float32)
    do = rng.standard_normal((N, d), dtype=np.float32)
    return q, k, v, do


def planted_head(N: int, d: int, rho: float, seed: int, b: int = 0, h: int = 0,
                 Br: int = 128, Bc: int = 128, gap: float = 12.0, sigma2_q: float = 6.0):
    """Planted block-sparse head.  Returns (q, k, v, do, owned) where
    ``owned[i_block]`` is the sorted array of key blocks planted for query block i.
    Only generator structure lives here; which blocks are *active* is decided by the
    method (oracle or kernel), never read from ``owned``."""
    rng = head_rng(seed, b, h)
    Tr = (N + Br - 1) // Br
    Tc = (N + Bc - 1) // Bc
    m = max(1, int(round(rho * Tc)))
    m = min(m, Tc)
    C = max(1, min(8, d // 4, Tc // m, Tr))          # few clusters: noise keeps d − C free dims
    # orthonormal cluster directions (columns of a random orthogonal matrix)
    g = rng.standard_normal((d, d))
    qmat, _ = np.linalg.qr(g)
    u = qmat[:, :C].T.astype(np.float64)          # (C, d)
    a = np.sqrt(gap * np.sqrt(d))
    perm = rng.permutation(Tc)
    cluster_blocks = [np.sort(perm[c * m:(c + 1) * m]) for c in range(C)]
    qc = rng.integers(0, C, size=Tr)               # cluster of each query block
    q = np.empty((N, d), dtype=np.float64)
    for i in range(Tr):
        r0, r1 = i * Br, min(N, (i + 1) * Br)
        eps = np.sqrt(sigma2_q) * rng.standard_normal((r1 - r0, d))
        eps -= (eps @ u.T) @ u                     # keep the query noise off every cluster axis
        q[r0:r1] = a * u[qc[i]] + eps
    k = rng.standard_normal((N, d))
    owner = np.full(Tc, -1)
    for c in range(C):
        owner[cluster_blocks[c]] = c
    for j in range(Tc):
        if owner[j] >= 0:
            c0, c1 = j * Bc, min(N, (j + 1) * Bc)
            k[c0:c1] += a * u[owner[j]]
    v = rng.standard_normal((N, d))
    do = rng.standard_normal((N, d))
    owned = [cluster_blocks[qc[i]] for i in range(Tr)]
    f32 = lambda x: x.astype(np.float32)
    return f32(q), f32(k), f32(v), f32(do), owned


def planted_tight_head(N: int, d: int, rho: float, seed: int, b: int = 0, h: int = 0,
                       Br: int = 128, Bc: int = 128, gap: float = 12.0, noise: float = 0.02):
    """SURVEY App. P3 planted head with near-duplicate keys/queries (see module doc).  Same cluster
    bookkeeping as planted_head; returns (q, k, v, do, owned)."""
    rng = head_rng(seed, b, h, stream=3)
    Tr = (N + Br - 1) // Br
    Tc = (N + Bc - 1) // Bc
    m = min(max(1, int(round(rho * Tc))), Tc)
    C = max(1, min(8, d // 4, Tc // m, Tr))
    qmat, _ = np.linalg.qr(rng.standard_normal((d, d)))
    u = qmat[:, :C].T.astype(np.float64)
    a = np.sqrt(gap * np.sqrt(d))
    perm = rng.permutation(Tc)
    cluster_blocks = [np.sort(perm[c * m:(c + 1) * m]) for c in range(C)]
    qc = rng.integers(0, C, size=Tr)
    q = np.empty((N, d), dtype=np.float64)
    for i in range(Tr):
        r0, r1 = i * Br, min(N, (i + 1) * Br)
        q[r0:r1] = a * u[qc[i]] + noise * rng.standard_normal((r1 - r0, d))
    k = rng.standard_normal((N, d))
    for c in range(C):
        for j in cluster_blocks[c]:
            c0, c1 = j * Bc, min(N, (j + 1) * Bc)
            k[c0:c1] = a * u[c] + noise * rng.standard_normal((c1 - c0, d))
    v = rng.standard_normal((N, d))
    do = rng.standard_normal((N, d))
    owned = [cluster_blocks[qc[i]] for i in range(Tr)]
    f32 = lambda x: x.astype(np.float32)
    return f32(q), f32(k), f32(v), f32(do), owned


def step_head(N: int, d: int, seed: int, b: int = 0, h: int = 0, sigma2_q: float = 6.0, low: float = 0.2):
    """Gaussian head whose first ⌊N/2⌋ keys are scaled by ``low``: their scores are bunched far below
    the row maxima, which all sit in the second half.  A structure test for streaming τ solvers
    that filter against a running maximum (the early keys all pass the early thresholds)."""
    q, k, v, do = gaussian_head(N, d, seed, b, h, sigma2_q)
    k[: N // 2] *= np.float32(low)
    return q, k, v, do


class HeadSpec:
    """Plain description of one generated workload."""

    def __init__(self, kind: str = "gaussian", sigma2_q: float = 6.0, rho: float = 1.0,
                 Br: int = 128, Bc: int = 128):
        self.kind, self.sigma2_q, self.rho, self.Br, self.Bc = kind, sigma2_q, rho, Br, Bc

    def head(self, N, d, seed, b, h):
        if self.kind == "gaussian":
            return gaussian_head(N, d, seed, b, h, self.sigma2_q)
        if self.kind == "planted":
            return planted_head(N, d, self.rho, seed, b, h, self.Br, self.Bc)[:4]
        if self.kind == "planted_tight":
            return planted_tight_head(N, d, self.rho, seed, b, h, self.Br, self.Bc)[:4]
        if self.kind == "step":
            return step_head(N, d, seed, b, h, self.sigma2_q)
        raise ValueError(f"unknown generator kind {self.kind!r}")


def make_inputs(B: int, H: int, N: int, d: int, seed: int, spec: HeadSpec | None = None,
                heads: range | None = None):
    """Stack heads into [B, H, N, d] float32 arrays (q, k, v, do).

    ``heads`` (flattened b*H+h indices) restricts generation to a contiguous
    slice; the returned arrays then have shape [len(heads), N, d]."""
    spec = spec or HeadSpec()
    if heads is None:
        out = [np.empty((B, H, N, d), dtype=np.float32) for _ in range(4)]
        for b in range(B):
            for h in range(H):
                for t, x in zip(out, spec.head(N, d, seed, b, h)):
                    t[b, h] = x
        return tuple(out)
    out = [np.empty((len(heads), N, d), dtype=np.float32) for _ in range(4)]
    for n_, bh in enumerate(heads):
        b, h = divmod(bh, H)
        for t, x in zip(out, spec.head(N, d, seed, b, h)):
            t[n_] = x
    return tuple(out)


def rowwise_scores(rows: int, n: int, seed: int, sigma: float = 1.0, with_grad: bool = True):
    """Inputs of the standalone row-wise solver benchmark ("random tensors from a standard
    Gaussian distribution (μ = 0, σ² = 1) with a fixed sequence length of n = 8192"): s ~ N(0, σ²)
    of shape (rows, n) float32, and an upstream gradient dp ~ N(0, 1) of the same shape."""
    rng = head_rng(seed, 0, 0, stream=7)
    s = rng.standard_normal((rows, n), dtype=np.float32) * np.float32(sigma)
    dp = rng.standard_normal((rows, n), dtype=np.float32) if with_grad else None
    return s, dp
