"""A LLaMA-style decoder stack for the real-module integration.

Test infrastructure, not product: RMSNorm -> causal self-attention (q/k/v/o
projections, rotary-free) -> RMSNorm -> SwiGLU MLP per block, token
embedding and an untied LM head — the tensor list of a LLaMA checkpoint at a
chosen width.  Parameters are bf16; the optimizer binds them to its flat
buffer with ``DistributedOptimizer.attach``.
"""

import torch
import torch.nn.functional as F
from torch import nn


class RMSNorm(nn.Module):
    def __init__(self, dim, eps=1e-5):
        super().__init__()
        self.weight = nn.Parameter(torch.ones(dim))
        self.eps = eps

    def forward(self, x):
        h = x.float()
        h = h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + self.eps)
        return (h * self.weight.float()).to(x.dtype)


class Block(nn.Module):
    def __init__(self, dim, heads, ffn):
        super().__init__()
        self.heads = heads
        self.attn_norm = RMSNorm(dim)
        self.q = nn.Linear(dim, dim, bias=False)
        self.k = nn.Linear(dim, dim, bias=False)
        self.v = nn.Linear(dim, dim, bias=False)
        self.o = nn.Linear(dim, dim, bias=False)
        self.mlp_norm = RMSNorm(dim)
        self.gate = nn.Linear(dim, ffn, bias=False)
        self.up = nn.Linear(dim, ffn, bias=False)
        self.down = nn.Linear(ffn, dim, bias=False)

    def forward(self, x):
        b, t, c = x.shape
        h = self.attn_norm(x)
        q, k, v = (m(h).view(b, t, self.heads, c // self.heads).transpose(1, 2) for m in (self.q, self.k, self.v))
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + self.o(a.transpose(1, 2).reshape(b, t, c))
        h = self.mlp_norm(x)
        return x + self.down(F.silu(self.gate(h)) * self.up(h))


class LlamaStack(nn.Module):
    def __init__(self, vocab=1000, dim=256, layers=3, heads=4, ffn=688):
        super().__init__()
        self.embed = nn.Embedding(vocab, dim)
        self.blocks = nn.ModuleList(Block(dim, heads, ffn) for _ in range(layers))
        self.norm = RMSNorm(dim)
        self.head = nn.Linear(dim, vocab, bias=False)

    def forward(self, tokens):
        x = self.embed(tokens)
        for blk in self.blocks:
            x = blk(x)
        return self.head(self.norm(x))


def build(device, seed=0, **kw):
    torch.manual_seed(seed)
    m = LlamaStack(**kw)
    for name, p in m.named_parameters():
        if p.dim() > 1:
            nn.init.normal_(p, std=0.02)
    return m.to(device=device, dtype=torch.bfloat16)


def batch(vocab, tokens, seq, step, rank, device):
    g = torch.Generator(device=device).manual_seed(7000 + 100 * step + rank)
    x = torch.randint(0, vocab, (tokens // seq, seq + 1), generator=g, device=device)
    return x[:, :-1], x[:, 1:]


def loss_fn(model, inp, tgt):
    logits = model(inp)
    return F.cross_entropy(logits.float().reshape(-1, logits.shape[-1]), tgt.reshape(-1))
