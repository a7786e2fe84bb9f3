"""the GPT-2-124M training step with the attention swapped (Table 4).

Timing-only workload (quality needs the dataset), so the test checks that one optimizer step runs through
the library's autograd op in all 12 layers: a finite loss, non-zero finite gradients reaching the first
block's QKV projection (they pass through `entmax_attn_bwd`), and a short timing run of the bench's
`next4_gpt2` line.
"""
import math
import os
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

pytestmark = pytest.mark.gpu


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def test_gpt2_step_gradients_flow_through_entmax():
    _gpu()
    import gpt2_step
    import paper_2502_12082_b200 as P
    torch.manual_seed(0)
    model = gpt2_step.GPT2(lambda q, k, v: P.entmax_attention(q, k, v, alpha=1.5, causal=True, n_iter=3),
                           layers=2).cuda()
    toks = torch.randint(0, 50257, (2, 1025), device="cuda")
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(toks[:, :-1])
        loss = torch.nn.functional.cross_entropy(logits.float().view(-1, logits.shape[-1]), toks[:, 1:].reshape(-1))
    loss.backward()
    assert math.isfinite(loss.item())
    g = model.blocks[0].qkv.weight.grad
    assert g is not None and torch.isfinite(g).all() and g.abs().max() > 0
    # the Q/K rows of the projection only get gradient through the attention's dQ/dK
    assert g[:2 * 768].abs().max() > 0


def test_gpt2_step_timing_line():
    _gpu()
    import gpt2_step
    out = gpt2_step.run(batch=2, steps=2, warmup=1, alphas=(1.5,))
    for key in ("softmax_sdpa", "entmax_alpha_1.5"):
        assert out[key]["ms_per_step"] > 0 and math.isfinite(out[key]["loss"])
