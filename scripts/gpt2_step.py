"""GPT-2-124M training-step timing with the attention swapped (timing only).

The paper trains GPT-2 with α-entmax attention (Table 4); quality needs the
dataset and stays out of scope.  This times one optimizer step of a randomly initialised GPT-2-124M
(12 layers, 12 heads, d = 64, 768 wide, context 1024) on synthetic tokens, bf16 autocast, with the
attention of every layer either `paper_2502_12082_b200.entmax_attention` (causal, α, T = 3) or the
same-box softmax SDPA, so the attention's share of a real step is visible.  Plain PyTorch for
everything but the attention (cuBLAS GEMMs, fused AdamW) — this is a harness, not product code.

python scripts/gpt2_step.py [--batch 8] [--steps 10] [--alphas 1.25,1.5,2.0]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import torch
import torch.nn as nn
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class Block(nn.Module):
    def __init__(self, width, heads, attn):
        super().__init__()
        self.ln1, self.ln2 = nn.LayerNorm(width), nn.LayerNorm(width)
        self.qkv, self.proj = nn.Linear(width, 3 * width), nn.Linear(width, width)
        self.fc, self.out = nn.Linear(width, 4 * width), nn.Linear(4 * width, width)
        self.heads, self.attn = heads, attn

    def forward(self, x):
        B, N, W = x.shape
        q, k, v = self.qkv(self.ln1(x)).view(B, N, 3, self.heads, W // self.heads).permute(2, 0, 3, 1, 4)
        a = self.attn(q.contiguous(), k.contiguous(), v.contiguous())
        x = x + self.proj(a.transpose(1, 2).reshape(B, N, W))
        return x + self.out(F.gelu(self.fc(self.ln2(x)), approximate="tanh"))


class GPT2(nn.Module):
    def __init__(self, attn, vocab=50257, ctx=1024, width=768, layers=12, heads=12):
        super().__init__()
        self.wte, self.wpe = nn.Embedding(vocab, width), nn.Embedding(ctx, width)
        self.blocks = nn.ModuleList(Block(width, heads, attn) for _ in range(layers))
        self.ln = nn.LayerNorm(width)
        self.apply(lambda m: nn.init.normal_(m.weight, std=0.02) if isinstance(m, (nn.Linear, nn.Embedding)) else None)

    def forward(self, idx):
        x = self.wte(idx) + self.wpe(torch.arange(idx.shape[1], device=idx.device))
        for b in self.blocks:
            x = b(x)
        return self.ln(x) @ self.wte.weight.t()     # tied LM head


def time_step(attn, batch, steps, warmup, seed=0):
    torch.manual_seed(seed)
    dev = torch.device("cuda")
    model = GPT2(attn).to(dev)
    opt = torch.optim.AdamW(model.parameters(), lr=6e-4, fused=True)
    g = torch.Generator(device=dev).manual_seed(seed)
    toks = torch.randint(0, 50257, (batch, 1025), device=dev, generator=g)

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = model(toks[:, :-1])
            loss = F.cross_entropy(logits.float().view(-1, logits.shape[-1]), toks[:, 1:].reshape(-1))
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        return loss

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    assert math.isfinite(loss.item())
    return ms, loss.item()


def run(batch=8, steps=10, warmup=3, alphas=(1.25, 1.5, 2.0)):
    import paper_2502_12082_b200 as P
    out = {"workload": f"GPT-2-124M random init, synthetic tokens, batch {batch} x 1024, bf16 autocast, AdamW",
           "tokens_per_step": batch * 1024}
    ms, loss = time_step(lambda q, k, v: F.scaled_dot_product_attention(q, k, v, is_causal=True), batch, steps, warmup)
    out["softmax_sdpa"] = {"ms_per_step": ms, "tokens_per_s": batch * 1024 / ms * 1e3, "loss": loss}
    for a in alphas:
        ms, loss = time_step(lambda q, k, v, a=a: P.entmax_attention(q, k, v, alpha=a, causal=True, n_iter=3),
                             batch, steps, warmup)
        out[f"entmax_alpha_{a}"] = {"ms_per_step": ms, "tokens_per_s": batch * 1024 / ms * 1e3, "loss": loss}
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--alphas", default="1.25,1.5,2.0")
    a = ap.parse_args()
    print(json.dumps(run(a.batch, a.steps, 3, tuple(float(x) for x in a.alphas.split(",")))))
