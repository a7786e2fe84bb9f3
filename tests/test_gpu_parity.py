"""GPU parity: CUDA path (through the C ABI) vs the float64 oracle, element by element.

Sizes span several 128×128 tiles and ragged tails; the oracle finishes each in seconds.
"""
import numpy as np
import pytest
import torch

import synth
from tests.parity import check_head, make_case, run_gpu

pytestmark = pytest.mark.gpu


def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")


CASES = [
    # (B, H, N, d, dtype, alpha, causal, n_iter)
    (1, 1, 256, 64, torch.float32, 1.5, False, 3),      # BASELINE config 1 (fp32)
    (1, 1, 256, 64, torch.float32, 1.5, False, 8),
    (1, 2, 512, 64, torch.bfloat16, 1.5, False, 3),
    (1, 2, 512, 64, torch.bfloat16, 1.5, True, 3),
    (1, 2, 512, 64, torch.bfloat16, 1.25, True, 3),
    (1, 2, 512, 64, torch.bfloat16, 2.0, True, 5),
    (1, 2, 512, 64, torch.bfloat16, 2.0, False, 5),
    (2, 1, 300, 64, torch.bfloat16, 1.5, True, 3),      # ragged tail (T_r = 3, 44-row last block)
    (1, 1, 129, 64, torch.bfloat16, 1.5, False, 3),     # one-row tail
    (1, 1, 1, 64, torch.bfloat16, 1.5, True, 3),        # N = 1 (degenerate)
    (1, 2, 384, 128, torch.bfloat16, 1.5, True, 3),     # d = 128
    (1, 1, 640, 128, torch.bfloat16, 1.75, False, 4),   # generic α (non-integer exponent)
    (1, 1, 200, 32, torch.float32, 1.5, True, 3),       # SIMT-only head dim
    (1, 1, 256, 64, torch.float32, 2.0, False, 5),      # fp32 bar at α = 2 (sparsemax; O2 reading r11)
    (1, 2, 300, 64, torch.float32, 1.33, True, 4),      # fp32 bar at a generic α (non-integer 1/(α−1))
]


@pytest.mark.parametrize("B,H,N,d,dtype,alpha,causal,n_iter", CASES)
def test_parity_gaussian(B, H, N, d, dtype, alpha, causal, n_iter):
    _require_gpu()
    dev, ref = make_case(B, H, N, d, dtype, seed=N + d)
    import paper_2502_12082_b200 as P
    expect = 1 if (dtype == torch.bfloat16 and d in (64, 128)) else 0
    assert P.impl_for(dev[0]) == expect        # the tcgen05 kernels must be the ones under test
    fw, grads = run_gpu(dev, alpha, causal, n_iter)
    for bh in range(B * H):
        check_head(fw, ref, bh, alpha, causal, n_iter, dtype, grads=grads)


@pytest.mark.parametrize("rho", [0.25, 1 / 16])
@pytest.mark.parametrize("causal", [False, True])
def test_parity_planted_block_sparse(rho, causal):
    """Planted block sparsity (Fig. 1 sweep generator): the mask has real zeros and the
    skipped blocks must not change any result."""
    _require_gpu()
    spec = synth.HeadSpec("planted", rho=rho)
    dev, ref = make_case(1, 2, 1024, 64, torch.bfloat16, seed=5, spec=spec)
    fw, grads = run_gpu(dev, 1.5, causal, 3)
    for bh in range(2):
        out = check_head(fw, ref, bh, 1.5, causal, 3, torch.bfloat16, grads=grads)
        if not causal:
            assert out["density"] < 1.0


def test_inference_mode_skips_o2():
    _require_gpu()
    dev, ref = make_case(1, 1, 256, 64, torch.bfloat16, seed=1)
    fw, _ = run_gpu(dev, 1.5, False, 3, training=False)
    assert fw.o2 is None
    check_head(fw, ref, 0, 1.5, False, 3, torch.bfloat16, with_bwd=False)


def test_autograd_function_matches_explicit_calls():
    _require_gpu()
    import paper_2502_12082_b200 as P
    dev, _ = make_case(1, 2, 256, 64, torch.bfloat16, seed=2)
    q, k, v, do = [t.clone().requires_grad_(i < 3) for i, t in enumerate(dev)]
    o = P.entmax_attention(q, k, v, 1.5, True, 3)
    o.backward(do)
    fw, grads = run_gpu(dev, 1.5, True, 3)
    assert torch.equal(o.detach(), fw.o)
    for a, b in zip((q.grad, k.grad, v.grad), grads):
        assert torch.equal(a, b)


def test_deterministic_and_head_sharding_bitwise():
    """Heads are independent: running head slices separately (as ranks do) gives the same
    bits as one call over all heads (SURVEY §4c fake multi-GPU)."""
    _require_gpu()
    dev, _ = make_case(2, 2, 384, 64, torch.bfloat16, seed=3)
    fw, grads = run_gpu(dev, 1.5, True, 3)
    q, k, v, do = dev
    for sl in (slice(0, 1), slice(1, 2)):
        part = [t[sl].contiguous() for t in (q, k, v, do)]
        fw2, g2 = run_gpu(part, 1.5, True, 3)
        assert torch.equal(fw2.o, fw.o[sl]) and torch.equal(fw2.tau, fw.tau[sl])
        assert torch.equal(fw2.mask, fw.mask[sl])
        for a, b in zip(g2, grads):
            assert torch.equal(a, b[sl])


@pytest.mark.parametrize("N,alpha,sigma2,causal", [
    (512, 1.5, 0.05, False),    # near-uniform rows: every key is a τ candidate → list overflow path
    (640, 1.5, 0.05, True),
    (4096, 1.25, 6.0, False),   # small α: wide candidate set
])
def test_parity_candidate_overflow_fallback(N, alpha, sigma2, causal):
    """Rows whose candidate list (z > τ_lo) overflows shared memory even at the exact threshold
    take the streaming Alg. 3 passes (tier 2) inside the τ kernel; results must be identical in
    quality."""
    _require_gpu()
    spec = synth.HeadSpec("gaussian", sigma2_q=sigma2)
    dev, ref = make_case(1, 2, N, 64, torch.bfloat16, seed=9, spec=spec)
    fw, grads = run_gpu(dev, alpha, causal, 3)
    for bh in range(2):
        check_head(fw, ref, bh, alpha, causal, 3, torch.bfloat16, grads=grads)


@pytest.mark.parametrize("N,causal", [(2048, False), (2304, True)])
def test_parity_transient_overflow_rebuild(N, causal):
    """`step` heads: every early key passes the running threshold, so the one-pass lists overflow;
    the exact-threshold rebuild pass (tier 1) holds the final candidates."""
    _require_gpu()
    dev, ref = make_case(1, 2, N, 64, torch.bfloat16, seed=13, spec=synth.HeadSpec("step"))
    fw, grads = run_gpu(dev, 1.5, causal, 3)
    for bh in range(2):
        check_head(fw, ref, bh, 1.5, causal, 3, torch.bfloat16, grads=grads)


@pytest.mark.parametrize("alpha,causal,d", [(1.1, False, 64), (1.33, True, 64), (1.9, False, 64), (1.6, True, 128),
                                             (1.01, False, 64), (1.01, True, 128)])
def test_parity_generic_alpha(alpha, causal, d):
    """Non-integer 1/(α−1): P, U via lg2/ex2 in the tcgen05 kernels, the τ sums
    via the generic accumulation.  α = 1.1 gives e = 10 (steep powers), α = 1.9 e ≈ 1.11; α = 1.01
    (e = 100) is the start of the paper's α annealing."""
    _require_gpu()
    dev, ref = make_case(1, 2, 640, d, torch.bfloat16, seed=int(alpha * 100) + d)
    fw, grads = run_gpu(dev, alpha, causal, 4)
    for bh in range(2):
        check_head(fw, ref, bh, alpha, causal, 4, torch.bfloat16, grads=grads)


def test_cuda_graph_capture_replays_bitwise():
    """The C ABI is stream-ordered with no host synchronisation or allocation inside, so a whole
    fwd+bwd step can be captured in a CUDA graph (launch-bound small configs) and replayed."""
    _require_gpu()
    import paper_2502_12082_b200 as P
    dev, _ = make_case(2, 3, 1024, 64, torch.bfloat16, seed=21)
    q, k, v, do = dev
    fw = P.entmax_attn_fwd(q, k, v, 1.5, True, 3)
    ws_f = torch.empty(P.workspace_bytes(q, True)[0], dtype=torch.uint8, device=q.device)
    ws_b = torch.empty(P.workspace_bytes(q, True)[1], dtype=torch.uint8, device=q.device)
    grads = tuple(torch.empty_like(t) for t in (q, k, v))

    def step():
        P.entmax_attn_fwd(q, k, v, 1.5, True, 3, out=fw, workspace=ws_f)
        P.entmax_attn_bwd(q, k, v, do, fw, 1.5, True, grads=grads, workspace=ws_b)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref_o, ref_g = fw.o.clone(), [g.clone() for g in grads]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for t in (fw.o, *grads):
        t.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(fw.o, ref_o)
    for a, b in zip(grads, ref_g):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype,d", [(torch.bfloat16, 64), (torch.bfloat16, 128), (torch.float32, 64)])
@pytest.mark.parametrize("causal", [False, True])
def test_unmasked_mode_matches_masked_bitwise(dtype, d, causal):
    """Unmasked mode (every visible block, no mask/tables): the skipped blocks of
    the masked mode hold P = U = dS = 0 exactly, so both modes give the same bits; and the unmasked
    mode matches the oracle on its own."""
    _require_gpu()
    import paper_2502_12082_b200 as P
    spec = synth.HeadSpec("planted", rho=0.25)
    dev, ref = make_case(1, 2, 1024, d, dtype, seed=31 + d, spec=spec)
    q, k, v, do = dev
    fm = P.entmax_attn_fwd(q, k, v, 1.5, causal, 3)
    gm = P.entmax_attn_bwd(q, k, v, do, fm, 1.5, causal)
    fu = P.entmax_attn_fwd(q, k, v, 1.5, causal, 3, masked=False)
    gu = P.entmax_attn_bwd(q, k, v, do, fu, 1.5, causal)
    torch.cuda.synchronize()
    assert fu.mask is None and fu.row_idx is None
    if not causal:
        assert fm.mask.float().mean().item() < 0.5          # the masked run really skipped blocks
    assert torch.equal(fu.tau, fm.tau) and torch.equal(fu.o, fm.o) and torch.equal(fu.o2, fm.o2)
    for a, b in zip(gu, gm):
        assert torch.equal(a, b)
    o = P.entmax_attention(q.clone().requires_grad_(), k, v, 1.5, causal, 3, masked=False)
    assert torch.equal(o.detach(), fu.o)
    check_head(fm, ref, 0, 1.5, causal, 3, dtype, grads=gu)   # (the oracle's mask vs the masked run)


def test_unmasked_mode_rejects_partial_null_tables():
    _require_gpu()
    import ctypes
    import paper_2502_12082_b200 as P
    from paper_2502_12082_b200 import _lib
    dev, _ = make_case(1, 1, 256, 64, torch.bfloat16, seed=1)
    q = dev[0]
    fw = P.entmax_attn_fwd(q, q, q, 1.5, False, 3)
    s = P._shape(q)
    ws = torch.empty(P.workspace_bytes(q, False)[0], dtype=torch.uint8, device=q.device)
    rc = _lib.lib().entmax_attn_fwd(P._ptr(q), P._ptr(q), P._ptr(q), ctypes.byref(s), 0, 1.5, 0, 3, 0.0,
                                    P._ptr(fw.o), P._ptr(fw.o2), P._ptr(fw.tau), P._ptr(fw.mask), None, None,
                                    P._ptr(ws), ws.numel(), None)
    assert rc == 1


@pytest.mark.parametrize("gen,N,alpha,causal", [("gaussian", 2048, 1.5, False), ("step", 2048, 1.5, True),
                                                ("gaussian", 1024, 1.25, True), ("gaussian", 1024, 1.75, False)])
def test_repeated_runs_bitwise_identical(gen, N, alpha, causal):
    """The τ kernel's candidate lists depend on a racy running max and may take a fallback tier or not
    from run to run; the fixed-point iteration sums make τ — and so every output — bitwise identical
    whichever path ran."""
    _require_gpu()
    import paper_2502_12082_b200 as P
    dev, _ = make_case(2, 4, N, 64, torch.bfloat16, seed=17, spec=synth.HeadSpec(gen))
    q, k, v, do = dev
    ref = None
    for _ in range(6):
        fw = P.entmax_attn_fwd(q, k, v, alpha, causal, 3)
        g = P.entmax_attn_bwd(q, k, v, do, fw, alpha, causal)
        torch.cuda.synchronize()
        cur = [fw.tau.clone(), fw.o.clone(), fw.mask.clone()] + [t.clone() for t in g]
        if ref is None:
            ref = cur
        else:
            for a, b in zip(cur, ref):
                assert torch.equal(a, b)


def test_pack_mask_bits():
    """Bit-packed M (NEXT-2): bit b of word w of row r equals M[r, 32w + b]; padding bits zero."""
    _require_gpu()
    import paper_2502_12082_b200 as P
    g = torch.Generator().manual_seed(0)
    for Tc in (1, 31, 32, 33, 64, 100):
        m = (torch.rand(3, 5, 7, Tc, generator=g) < 0.4).to(torch.uint8)
        pk = P.pack_mask(m.cuda()).cpu().numpy().astype(np.uint32)
        mm = m.numpy()
        for w in range(pk.shape[-1]):
            for b in range(32):
                col = 32 * w + b
                want = mm[..., col] if col < Tc else np.zeros(mm.shape[:-1], np.uint8)
                assert np.array_equal((pk[..., w] >> b) & 1, want.astype(np.uint32))


@pytest.mark.parametrize("causal", [False, True])
def test_padded_layout_qkv_split(causal):
    """q, k, v as views of one [B, H, N, 3d] buffer (row stride 3d, the fused-QKV layout the ABI's
    strides allow): outputs and gradients are written with q's strides, stay inside their own
    allocations, and match the oracle like contiguous inputs do."""
    _require_gpu()
    import paper_2502_12082_b200 as P
    B, H, N, d = 1, 2, 384, 64
    dev, ref = make_case(B, H, N, d, torch.bfloat16, seed=77)
    qkv = torch.empty((B, H, N, 3 * d), dtype=torch.bfloat16, device="cuda")
    for c in range(3):
        qkv[..., c * d:(c + 1) * d] = dev[c]
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    guard = qkv.clone()
    fw = P.entmax_attn_fwd(q, k, v, 1.5, causal, 3)
    grads = P.entmax_attn_bwd(q, k, v, dev[3], fw, 1.5, causal)
    torch.cuda.synchronize()
    assert fw.o.stride() == q.stride() and all(g.stride() == q.stride() for g in grads)
    assert torch.equal(qkv, guard)                          # inputs untouched
    for bh in range(B * H):
        check_head(fw, ref, bh, 1.5, causal, 3, torch.bfloat16, grads=grads)
    fc, gc = run_gpu(dev, 1.5, causal, 3)                   # same bits as the contiguous layout
    assert torch.equal(fc.o, fw.o) and all(torch.equal(a, b) for a, b in zip(gc, grads))


@pytest.mark.parametrize("N,causal,d", [(1024, False, 64), (1024, True, 64), (768, False, 128)])
def test_parity_near_duplicate_keys(N, causal, d):
    """SURVEY App. P3's original planted recipe (synth 'planted_tight': queries and owned keys
    a·u_c + 0.02·N(0,1)): rows see hundreds of near-equal scores and dQ = c·Σ_j dS_ij K_j cancels to
    ~2 % of its terms, so the bf16 rounding leak of dS must be removed (reading r12: ρ_i·K̄ correction)
    for dQ to meet the 3e-2 bar.  Everything else is checked at the usual bars."""
    _require_gpu()
    spec = synth.HeadSpec("planted_tight", rho=0.25)
    dev, ref = make_case(1, 2, N, d, torch.bfloat16, seed=41 + d, spec=spec)
    fw, grads = run_gpu(dev, 1.5, causal, 3)
    for bh in range(2):
        out = check_head(fw, ref, bh, 1.5, causal, 3, torch.bfloat16, grads=grads)
        assert out["dQ"] <= 1e-2, out


@pytest.mark.parametrize("N,causal,rho", [(1152, False, 0.25), (1152, True, 0.25), (1408, True, 0.25)])
def test_parity_pair_output_pass_d128(N, causal, rho):
    """d = 128 runs the output pass on CTA pairs with 2-SM MMAs (sm100_fb2.cuh): the two query blocks of
    a pair visit the union of their candidate lists.  Planted block sparsity gives adjacent query blocks
    different lists (a block in one list only must contribute exact zeros to the other CTA's rows, and
    each CTA's mask / 𝒬 table must stay its own), and an odd T_r leaves the last pair with a CTA past
    the end; O, O⁽²⁾, τ, the mask, the tables and the gradients are checked against the oracle."""
    _require_gpu()
    spec = synth.HeadSpec("planted", rho=rho)
    dev, ref = make_case(1, 2, N, 128, torch.bfloat16, seed=int(N * 10 + 100 * rho) + causal, spec=spec)
    fw, grads = run_gpu(dev, 1.5, causal, 3)
    half = fw.mask.shape[2] // 2   # the two query blocks of some pair must have different block sets
    assert bool((fw.mask[:, :, 0:2 * half:2] != fw.mask[:, :, 1:2 * half:2]).any())
    for bh in range(2):
        check_head(fw, ref, bh, 1.5, causal, 3, torch.bfloat16, grads=grads)
