"""Seeded synthetic contents of the precomputed KV pools (SURVEY.md §8(d) "Pool contents").

Synthetic stand-ins for offline artifacts: the hot path is defined
for any pool bytes, so parity tests draw them here; the oracle materialises real pools
itself where an invariant needs them (exact-cache tests). No method arithmetic: values
are drawn directly in their stored formats.

Registration layout (include/rc.h, rc_pool_register_blocks): [n_tok][L][2][H_kv][d_h].
  * item blocks: bf16 ~ N(0,1), canonical start position P.
  * history prototype rows: int8 codes ~ clamp(round(40 N(0,1)), -127, 127) and fp32
    scales 0.025 * (0.5 + U[0,1)) per (row, layer, K/V, kv-head) (SURVEY R15 format).
  * prefix block: bf16 ~ N(0,1) at positions 0..P-1 (tests that need the exact prefix
    KV materialise it with the oracle instead).
Each block has its own generator seed, so any subset regenerates alone.
"""
import torch

from .shapes import ModelShape
from .weights import subseed


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def item_kv(shape: ModelShape, item_len: int, items, seed: int = 1, device="cpu"):
    L, Hk, dh = shape.n_layers, shape.n_kv_heads, shape.head_dim
    out = torch.empty((len(items), item_len, L, 2, Hk, dh), dtype=torch.bfloat16, device=device)
    for j, it in enumerate(items):
        g = _gen(subseed(seed, 7, int(it)), device)
        out[j] = torch.randn((item_len, L, 2, Hk, dh), generator=g, device=device).to(torch.bfloat16)
    return out


def hist_kv(shape: ModelShape, protos, seed: int = 2, device="cpu"):
    L, Hk, dh = shape.n_layers, shape.n_kv_heads, shape.head_dim
    q = torch.empty((len(protos), L, 2, Hk, dh), dtype=torch.int8, device=device)
    sc = torch.empty((len(protos), L, 2, Hk), dtype=torch.float32, device=device)
    for j, pi in enumerate(protos):
        g = _gen(subseed(seed, 9, int(pi)), device)
        z = torch.randn((L, 2, Hk, dh), generator=g, device=device)
        q[j] = torch.clamp(torch.round(z * 40.0), -127, 127).to(torch.int8)
        sc[j] = 0.025 * (0.5 + torch.rand((L, 2, Hk), generator=g, device=device))
    return q, sc


def prefix_kv(shape: ModelShape, prefix_len: int, seed: int = 3, device="cpu"):
    L, Hk, dh = shape.n_layers, shape.n_kv_heads, shape.head_dim
    g = _gen(subseed(seed, 11), device)
    return torch.randn((prefix_len, L, 2, Hk, dh), generator=g, device=device).to(torch.bfloat16)
