"""Randomised GPU-vs-oracle sweep: shapes, α, causal, generators, T, modes and dtypes drawn from a
fixed seed (ENTMAX_RANDOM_SEED / ENTMAX_RANDOM_CASES override it), each case checked element by
element against the float64 oracle (tests/parity.py bars; τ against the T-step mirror, reading r10)."""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_head, make_case

pytestmark = pytest.mark.gpu

import os
_rng = np.random.default_rng(int(os.environ.get("ENTMAX_RANDOM_SEED", "2502")))
CASES = []
for _ in range(int(os.environ.get("ENTMAX_RANDOM_CASES", "24"))):
    N = int(_rng.choice([1, 2, 17, 128, 129, 255, 256, 300, 511, 640, 700]))
    d = int(_rng.choice([64, 64, 128]))
    alpha = float(_rng.choice([1.25, 1.5, 2.0, round(float(_rng.uniform(1.15, 1.95)), 3)]))
    causal = bool(_rng.integers(2))
    gen = str(_rng.choice(["gaussian", "gaussian", "planted", "step"]))
    masked = bool(_rng.integers(4))   # 1 in 4 unmasked
    T = int(_rng.choice([1, 2, 3, 5]))
    dt = "fp32" if _rng.integers(6) == 0 else "bf16"   # 1 in 6 on the SIMT fp32 path
    if dt == "fp32":
        # the fp32 bars (O 1e-4, grads 1e-3) assume a converged iteration (T >= 3, the paper's
        # default) and a well-conditioned U = x^{e-1}: at α = 2 it is the step 1[x > 0] (float32 and
        # float64 may pick different subgradients for an element at x ≈ 0), and for α > 1.5 its
        # slope e-1 < 1 is unbounded at x -> 0+, so O⁽²⁾ near the support boundary amplifies the
        # float32 rounding of τ past 1e-4.  fp32 therefore draws α ∈ {1.25, 1.5} (config 1 is
        # α = 1.5 fp32); generic α is swept in bf16, where these effects sit far below the bars.
        T, N = max(T, 3), max(N, 17)
        alpha = 1.25 if alpha < 1.4 else 1.5
    CASES.append((N, d, alpha, causal, gen, masked, T, dt))


@pytest.mark.parametrize("N,d,alpha,causal,gen,masked,T,dt", CASES)
def test_random_case(N, d, alpha, causal, gen, masked, T, dt):
    import paper_2502_12082_b200 as P
    spec = synth.HeadSpec(gen, rho=0.25) if gen == "planted" else synth.HeadSpec(gen)
    if gen == "planted" and N < 256:
        spec = synth.HeadSpec("gaussian")
    dtype = torch.float32 if dt == "fp32" else torch.bfloat16
    dev, ref = make_case(1, 2, N, d, dtype, seed=N * 7 + d, spec=spec)
    q, k, v, do = dev
    fw = P.entmax_attn_fwd(q, k, v, alpha, causal, T, masked=masked)
    grads = P.entmax_attn_bwd(q, k, v, do, fw, alpha, causal)
    torch.cuda.synchronize()
    if not masked:   # compare the tables of a masked run against the oracle; results are identical bits
        fm = P.entmax_attn_fwd(q, k, v, alpha, causal, T)
        torch.cuda.synchronize()
        assert torch.equal(fm.o, fw.o) and torch.equal(fm.tau, fw.tau)
        fw = fm
    for bh in range(2):
        check_head(fw, ref, bh, alpha, causal, T, dtype, grads=grads)
