"""Float64 CPU oracle for AdaSplash α-entmax attention (arXiv 2502.12082).

*** TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH. ***
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg / ``--impl reference`` arm may import or call anything in this package.
The CUDA path (``paper_2502_12082_b200``) never imports it, and it never imports
the CUDA path; the two share no code.  Inputs come from ``synth`` (generators
only, no method arithmetic).

Plain, slow, obviously-correct numpy float64.  Every function cites the
PAPER.md passage it follows (P:L<n> = /root/reference/PAPER.md line n).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  * tau_sparsemax / tau_entmax15 — brute force over all supports on tiny rows,
    SPEC worked examples in tests/golden/, agreement with long bisection,
    closed forms ([10,0] → τ=4; all-equal → uniform).
  * halley_bisection (Alg. 1 mirror) — bracket soundness/monotone width,
    convergence claims of P:L250 (3 vs 23 iterations), fixed point at the root.
  * attn_fwd — V = I gives P, n = 1 gives V, causal n = 2, α → 1 tends to softmax
    (P:L127), α = 2 one-hot rows, rows of P on the simplex.
  * attn_bwd — central finite differences of the forward (exact τ), J·1 = 0,
    dO = 0 ⇒ 0, and a mutation test (dropping δ breaks the FD agreement).
  * block_mask / lookup_tables — brute-force block-OR of P > 0, transpose
    round trip, SPEC table example.
No function is "parity unpinned".
"""
from .rowwise import (relu_pow, root_f, bracket_init, bisection_update, halley_update,
                     halley_bisection, halley_bisection_outcomes, tau_sparsemax, tau_entmax15, tau_bisect_exact,
                     tau_exact, entmax_probs, entmax, entmax_vjp)
from .attention import (default_scale, scores, solve_tau, solve_tau_outcomes, probs, u_of_p, attn_fwd,
                        block_mask, mask_from_p, lookup_tables, attn_bwd,
                        softmax_attention)
