"""Pins of oracle/numerics.py against definitions independent of it (not gpu)."""
import math
from fractions import Fraction

import numpy as np
import torch

from oracle.numerics import (bf16_bits, bf16_to_f32, rope_cos_sin, rope_rotate_f32, rope_rotate_f64,
                             dequant_int8, deviation_fixed, deviation_terms, RopeTable)


def test_bf16_rne_matches_torch():
    # library routine: torch's fp32 -> bf16 cast is round-to-nearest-even
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 100000),
                        np.array([0.0, -0.0, 1.0, -1.0, 65504.0, 1e-40, -1e-40, np.inf, -np.inf], np.float32)])
    # exact ties: low 16 bits == 0x8000 with both parities of bit 16
    ties = (np.arange(1000, dtype=np.uint32) << 17 | 0x3F800000 | 0x8000).view(np.float32)
    ties2 = ((np.arange(1000, dtype=np.uint32) << 17) | 0x3F810000 | 0x8000).view(np.float32)
    x = np.concatenate([x, ties, ties2]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bf16_bits(x), ref)
    assert np.array_equal(bf16_to_f32(ref), torch.from_numpy(ref.view(np.int16)).view(torch.bfloat16).float().numpy())


def test_rope_tables_closed_form():
    # tables = fp32(cos/sin(delta * theta^(-2i/d))) computed in fp64 (R13)
    c, s = rope_cos_sin(5e5, 128, [-4095, -1, 0, 1, 7, 4095])
    for r, d in enumerate([-4095, -1, 0, 1, 7, 4095]):
        for i in (0, 1, 31, 63):
            ang = d * 5e5 ** (-2.0 * i / 128)
            assert c[r, i] == np.float32(math.cos(ang)) and s[r, i] == np.float32(math.sin(ang))
    assert np.all(c[2] == 1.0) and np.all(s[2] == 0.0)


def test_rope_matches_complex_rotation():
    # closed form: pair (x_i, x_{i+d/2}) as a complex number times e^{i delta theta_i}
    rng = np.random.default_rng(1)
    d, theta = 128, 5e5
    x = rng.standard_normal((1000, d))
    deltas = rng.integers(-4096, 4096, 1000)
    c, s = rope_cos_sin(theta, d, deltas)
    y = rope_rotate_f64(x, c, s)
    i = np.arange(d // 2)
    z = (x[:, :d // 2] + 1j * x[:, d // 2:]) * np.exp(1j * deltas[:, None] * theta ** (-2.0 * i / d))
    ref = np.concatenate([z.real, z.imag], axis=1)
    assert np.max(np.abs(y - ref)) < 1e-5 * np.max(np.abs(x))  # fp32 table rounding only
    # norm preservation (isometry)
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-6)


def test_rope_fp32_identity_additivity_encode_at_target():
    rng = np.random.default_rng(2)
    d, theta = 128, 5e5
    tab = RopeTable(theta, d)
    x = rng.standard_normal((1000, d)).astype(np.float32)
    c0, s0 = tab.get(np.zeros(1000, int))
    assert np.array_equal(rope_rotate_f32(x, c0, s0), x)          # identity at delta = 0, bit-exact
    o = rng.integers(0, 4096, 1000)
    p = rng.integers(0, 4096, 1000)
    co, so = tab.get(o)
    cd, sd = tab.get(p - o)
    cp, sp = tab.get(p)
    enc_o = rope_rotate_f32(x, co, so)                                 # K computed at o
    re = rope_rotate_f32(enc_o, cd, sd)                               # re-aligned to p
    direct = rope_rotate_f32(x, cp, sp)                               # K computed at p
    rel = np.linalg.norm(re - direct, axis=1) / np.linalg.norm(direct, axis=1)
    assert rel.max() < 2e-6                                            # SURVEY 8(c) pin, fp32


def test_rope_rotation_op_order_is_per_product_rounding():
    # y0 = fp32(x0 c) - fp32(x1 s), no fused multiply-add (R13): check against Fractions
    rng = np.random.default_rng(3)
    x = rng.standard_normal((64, 16)).astype(np.float32)
    c, s = rope_cos_sin(1e4, 16, np.arange(64) - 32)
    y = rope_rotate_f32(x, c, s)
    for r in range(64):
        for i in range(8):
            a = np.float32(Fraction(float(x[r, i])) * Fraction(float(c[r, i])))
            b = np.float32(Fraction(float(x[r, i + 8])) * Fraction(float(s[r, i])))
            assert y[r, i] == np.float32(a - b)
            a2 = np.float32(Fraction(float(x[r, i + 8])) * Fraction(float(c[r, i])))
            b2 = np.float32(Fraction(float(x[r, i])) * Fraction(float(s[r, i])))
            assert y[r, i + 8] == np.float32(a2 + b2)


def test_dequant_brute_force_and_roundtrip():
    rng = np.random.default_rng(4)
    q = rng.integers(-127, 128, (50, 8, 16)).astype(np.int8)
    sc = (rng.random((50, 8)) * 0.1).astype(np.float32)
    y = dequant_int8(q, sc)
    for a in range(50):
        for h in range(8):
            for j in range(16):
                assert y[a, h, j] == np.float32(Fraction(int(q[a, h, j])) * Fraction(float(sc[a, h])))
    # quantise (R15: scale = absmax/127, q = rint) then dequantise: error <= scale/2
    x = rng.standard_normal((100, 128)).astype(np.float32)
    s = (np.abs(x).max(axis=1) / 127).astype(np.float32)
    qq = np.clip(np.rint(x / s[:, None]), -127, 127).astype(np.int8)
    assert np.all(np.abs(dequant_int8(qq, s) - x) <= s[:, None] / 2 * (1 + 1e-6))


def test_deviation_fixed_point_brute_force():
    rng = np.random.default_rng(5)
    a = bf16_to_f32(bf16_bits(rng.standard_normal((20, 256)).astype(np.float32) * 3))
    b = bf16_to_f32(bf16_bits(rng.standard_normal((20, 256)).astype(np.float32) * 3))
    D = deviation_fixed(a, b)
    for r in range(20):
        tot = 0
        for j in range(256):
            y = np.float32(abs(np.float32(a[r, j]) - np.float32(b[r, j])))
            yq = min(Fraction(float(y)), Fraction(2 ** 16) - Fraction(1, 2 ** 24))
            tot += math.floor(yq * 2 ** 24)
        assert int(D[r]) == tot
    assert np.all(deviation_fixed(a, a) == 0)                          # identical cache -> 0
    big = deviation_terms(np.float32([1e9, 70000.0, 65535.99609375]), np.float32([0, 0, 0]))
    assert list(big) == [2 ** 40 - 1, 2 ** 40 - 1, int(65535.99609375 * 2 ** 24)]
