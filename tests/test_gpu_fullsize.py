"""Parity at BASELINE.json's full sizes, through the same entry points and launch configuration
bench.py times, checked on sampled query blocks / key blocks the oracle computes one by one, plus
size-independent identities of the backward."""
import pytest
import torch

import synth
from tests.parity import check_grad_identities, check_head, check_head_sampled, make_case, run_gpu

pytestmark = pytest.mark.gpu


def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")


@pytest.mark.parametrize("gen", ["gaussian", "planted"])
def test_config2_sparsity_sweep_shape(gen):
    """configs[1]: B=4 H=12 N=8192 d=64 α=1.5 non-causal bf16 (the bench workload; planted ρ=0.05)."""
    _gpu()
    spec = synth.HeadSpec(gen, rho=0.05)
    dev, ref = make_case(4, 12, 8192, 64, torch.bfloat16, seed=1234, spec=spec)
    fw, grads = run_gpu(dev, 1.5, False, 3)
    check_head_sampled(fw, ref, 0, 1.5, False, 3, torch.bfloat16, row_blocks=(0, 37, 63), key_blocks=(5, 63),
                       grads=grads)
    check_head_sampled(fw, ref, 47, 1.5, False, 3, torch.bfloat16, row_blocks=(11, 62), grads=grads)
    check_grad_identities(grads, ref, 20, torch.bfloat16)


@pytest.mark.parametrize("N", [512, 8192])
def test_config3_encoder(N):
    """configs[2]: RoBERTa/ModernBERT-shaped B=8 H=12 d=64, N ∈ {512, 8192}, α=1.5."""
    _gpu()
    dev, ref = make_case(8, 12, N, 64, torch.bfloat16, seed=N)
    fw, grads = run_gpu(dev, 1.5, False, 3)
    if N == 512:
        for bh in (0, 50, 95):
            check_head(fw, ref, bh, 1.5, False, 3, torch.bfloat16, grads=grads)
    else:
        check_head_sampled(fw, ref, 95, 1.5, False, 3, torch.bfloat16, row_blocks=(0, 63), key_blocks=(31,),
                           grads=grads)


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_config4_gpt2_causal(alpha):
    """configs[3]: GPT-2-shaped causal B=8 H=12 d=64 N=1024, α ∈ {1.25, 1.5, 2.0}, fwd+bwd."""
    _gpu()
    n_iter = 3 if alpha != 2.0 else 5   # α=2 needs T=5 to stay near the mirror at N=1024
    dev, ref = make_case(8, 12, 1024, 64, torch.bfloat16, seed=int(alpha * 100))
    fw, grads = run_gpu(dev, alpha, True, n_iter)
    for bh in (0, 95):
        check_head(fw, ref, bh, alpha, True, n_iter, torch.bfloat16, grads=grads)


@pytest.mark.parametrize("N", [32768, 65536])
def test_config5_long_context_causal(N):
    """configs[4]: long-context causal B=1 H=16 d=128, α=1.5; sampled blocks + the last key block."""
    _gpu()
    dev, ref = make_case(1, 16, N, 128, torch.bfloat16, seed=N + 1)
    fw, grads = run_gpu(dev, 1.5, True, 3)
    Tr = N // 128
    check_head_sampled(fw, ref, 3, 1.5, True, 3, torch.bfloat16, row_blocks=(0, Tr // 2, Tr - 1),
                       key_blocks=(Tr - 1,), grads=grads)
    check_grad_identities(grads, ref, 15, torch.bfloat16)
