"""Seeded random-init weights, in HF tensor naming.

Each tensor is drawn from its own torch.Generator seeded by splitmix64(seed, tensor index),
so any subset (e.g. one layer) can be regenerated alone. Values are drawn in fp32 and
rounded to bf16 by torch (round-to-nearest-even). Distribution (builder choice, R26 with
non-unit norms so that a swapped or dropped norm weight is visible to the tests):
  embedding ~ N(0, 1); matrices ~ N(0, 1/fan_in); RMSNorm gains ~ 1 + N(0, 0.1^2);
  QKV biases (Qwen2 shape) ~ N(0, 0.1^2).
Generation on a CUDA device uses the CUDA generator (different values than CPU for the
same seed) -- used only for bench-scale weights; every parity test uses CPU weights, or
host copies of the device tensors as oracle inputs.
"""
import torch

from .shapes import ModelShape

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def subseed(seed: int, *idx: int) -> int:
    s = splitmix64(seed)
    for i in idx:
        s = splitmix64(s ^ (i & MASK64))
    return s & ((1 << 63) - 1)


def layer_tensor_names(shape: ModelShape):
    names = ["ln1", "wq", "wk", "wv"]
    if shape.qkv_bias:
        names += ["bq", "bk", "bv"]
    names += ["wo", "ln2", "wg", "wu", "wd"]
    return names


def tensor_spec(shape: ModelShape, name: str):
    """(dims, kind, fan_in) of a per-layer tensor or a global one."""
    d, F = shape.d_model, shape.d_ff
    table = {
        "embed": ((shape.vocab, d), "embed", None),
        "norm": ((d,), "norm", None),
        "lm_head": ((shape.vocab, d), "mat", d),
        "ln1": ((d,), "norm", None),
        "ln2": ((d,), "norm", None),
        "wq": ((shape.q_dim, d), "mat", d),
        "wk": ((shape.kv_dim, d), "mat", d),
        "wv": ((shape.kv_dim, d), "mat", d),
        "bq": ((shape.q_dim,), "bias", None),
        "bk": ((shape.kv_dim,), "bias", None),
        "bv": ((shape.kv_dim,), "bias", None),
        "wo": ((d, shape.q_dim), "mat", shape.q_dim),
        "wg": ((F, d), "mat", d),
        "wu": ((F, d), "mat", d),
        "wd": ((d, F), "mat", F),
    }
    return table[name]


def _draw(dims, kind, fan_in, seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(dims, generator=g, dtype=torch.float32, device=device)
    if kind == "mat":
        x.mul_(fan_in ** -0.5)
    elif kind == "norm":
        x.mul_(0.1).add_(1.0)
    elif kind == "bias":
        x.mul_(0.1)
    return x.to(torch.bfloat16)


def gen_tensor(shape: ModelShape, name: str, layer: int = -1, seed: int = 0, device="cpu"):
    dims, kind, fan_in = tensor_spec(shape, name)
    gidx = {"embed": 0, "norm": 1, "lm_head": 2}
    if layer < 0:
        tid = gidx[name]
    else:
        tid = 16 + layer * 32 + layer_tensor_names(shape).index(name)
    return _draw(dims, kind, fan_in, subseed(seed, tid), device)


def gen_weights(shape: ModelShape, seed: int = 0, device="cpu", n_layers=None):
    """dict: 'embed','norm','lm_head' and 'layers': list of dicts of bf16 tensors."""
    L = shape.n_layers if n_layers is None else n_layers
    w = {k: gen_tensor(shape, k, -1, seed, device) for k in ("embed", "norm", "lm_head")}
    w["layers"] = [
        {k: gen_tensor(shape, k, l, seed, device) for k in layer_tensor_names(shape)}
        for l in range(L)
    ]
    return w
