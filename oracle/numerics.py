"""Exact numeric definitions shared by the oracle's modules (test infrastructure only).

bf16: round-to-nearest-even of an fp32 value (the stored form of every KV byte).
RoPE: HF rotate-half pairs (i, i + d_h/2) with theta_i = base^(-2i/d_h) (
      "positional adjustment (e.g., RoPE rotation)"). cos/sin are computed in
      fp64 with the C library (Python math module) and rounded once to fp32, indexed by the
      signed offset Delta. The fp32 rotation is y0 = x0*c - x1*s, y1 = x1*c + x0*s with every
      product rounded to fp32 before the add/sub (numpy float32 elementwise ops, no FMA).
int8: dequant = fp32(q) * scale, one fp32 rounding.
Deviation: SURVEY R4 fixed point; per term y = fp32(|a - b|), t = floor(min(y, 2^16-2^-24)
      * 2^24) as uint64, D = sum t (Eq. 3 divergence term).
"""
import math

import numpy as np

F32 = np.float32


def bf16_bits(x) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round to nearest even (NaN kept quiet)."""
    u = np.ascontiguousarray(np.asarray(x, dtype=F32)).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
    r = np.where(nan, ((u >> 16) | 0x40) & 0xFFFF, r)
    return r.astype(np.uint16)


def bf16_to_f32(bits) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (b.astype(np.uint32) << 16).view(F32)


def round_bf16(x) -> np.ndarray:
    """Value of x rounded to bf16 (via fp32), returned as float64."""
    return bf16_to_f32(bf16_bits(np.asarray(x, dtype=np.float64).astype(F32))).astype(np.float64)


def inv_freq(theta: float, head_dim: int):
    return [math.pow(theta, -2.0 * i / head_dim) for i in range(head_dim // 2)]


def rope_cos_sin(theta: float, head_dim: int, deltas):
    """fp32 cos/sin tables [len(deltas)][head_dim/2] for integer offsets (may be negative)."""
    f = inv_freq(theta, head_dim)
    deltas = [int(d) for d in np.asarray(deltas).ravel()]
    c = np.array([[math.cos(float(d) * fi) for fi in f] for d in deltas], dtype=F32)
    s = np.array([[math.sin(float(d) * fi) for fi in f] for d in deltas], dtype=F32)
    return c, s


class RopeTable:
    """Memoised fp32 tables, row lookup by signed Delta."""

    def __init__(self, theta: float, head_dim: int):
        self.theta, self.head_dim = theta, head_dim
        self._c, self._s = {}, {}

    def get(self, deltas):
        deltas = np.asarray(deltas, dtype=np.int64).ravel()
        miss = [int(d) for d in np.unique(deltas) if int(d) not in self._c]
        if miss:
            c, s = rope_cos_sin(self.theta, self.head_dim, miss)
            for j, d in enumerate(miss):
                self._c[d], self._s[d] = c[j], s[j]
        c = np.stack([self._c[int(d)] for d in deltas]) if len(deltas) else np.zeros((0, self.head_dim // 2), F32)
        s = np.stack([self._s[int(d)] for d in deltas]) if len(deltas) else np.zeros((0, self.head_dim // 2), F32)
        return c, s


def rope_rotate_f32(x, c, s):
    """R13 fp32 rotation. x float32 [..., d_h]; c, s float32 broadcastable to [..., d_h/2]."""
    x = np.asarray(x, dtype=F32)
    h = x.shape[-1] // 2
    x0, x1 = x[..., :h], x[..., h:]
    y0 = (x0 * c).astype(F32) - (x1 * s).astype(F32)
    y1 = (x1 * c).astype(F32) + (x0 * s).astype(F32)
    return np.concatenate([y0.astype(F32), y1.astype(F32)], axis=-1)


def rope_rotate_f64(x, c, s):
    """Model RoPE in the fp64 oracle (same fp32 tables, widened)."""
    x = np.asarray(x, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    h = x.shape[-1] // 2
    x0, x1 = x[..., :h], x[..., h:]
    return np.concatenate([x0 * c - x1 * s, x1 * c + x0 * s], axis=-1)


def dequant_int8(q, scale):
    """fp32(q) * scale, scale broadcast over the trailing d_h axis."""
    return (np.asarray(q).astype(F32) * np.asarray(scale, dtype=F32)[..., None]).astype(F32)


DEV_CLAMP = 2.0 ** 16 - 2.0 ** -24


def deviation_terms(a, b) -> np.ndarray:
    """Per-element fixed-point terms of |a - b| (a, b exactly representable in fp32)."""
    y = np.abs(np.asarray(a, dtype=F32) - np.asarray(b, dtype=F32)).astype(np.float64)
    return np.floor(np.minimum(y, DEV_CLAMP) * 2.0 ** 24).astype(np.uint64)


def deviation_fixed(a, b) -> np.ndarray:
    """D over the trailing axis."""
    return deviation_terms(a, b).sum(axis=-1, dtype=np.uint64)
