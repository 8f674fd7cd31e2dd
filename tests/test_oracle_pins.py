"""Pins of the oracle parts the round-1 review found unpinned (not gpu).

* classify_tokens ("cache misses are computed on-the-fly"): the tokens
  of a non-resident item become FORCED; resident items and every other class are untouched.
* O-ASM HIST-K branch (PAPER.md:549 prototypes, :566 "positional adjustment (e.g., RoPE
  rotation)"): every element of both rotate-half halves of every history key
  equals bf16_RNE(fp32 rotation of fp32(q)*scale_K by Delta = p - o_pi), evaluated here with
  exact rational arithmetic and an explicit round-to-nearest-even of each intermediate (no
  numpy rounding), and -- independently of any table -- the re-aligned history key of a
  prototype materialised at o_pi equals the key computed at p to within the int8 + bf16 error,
  while the opposite Delta sign does not.
"""
import math
from fractions import Fraction

import numpy as np
import torch

import rcgen
from oracle.assemble import assemble
from oracle.layout import FORCED, HIST, ITEM, PREFIX, classify_tokens
from oracle.model import OracleModel, full_prefill
from oracle.numerics import bf16_to_f32
from tests.helpers import layouts, make_case, oracle_pools, rel_l2


def _round_rne(x: Fraction, mant_bits: int, emin: int) -> Fraction:
    """Exact round-to-nearest-even of a rational to a binary format with `mant_bits` explicit
    significand bits (fp32: 23, bf16: 7) and minimum normal exponent `emin` (-126 for both)."""
    if x == 0:
        return Fraction(0)
    sgn = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    e = max(e, emin)
    scale = Fraction(2) ** (mant_bits - e)
    m = a * scale
    q, r = divmod(m.numerator, m.denominator)
    if 2 * r > m.denominator or (2 * r == m.denominator and q % 2 == 1):
        q += 1
    return sgn * Fraction(q) / scale


def f32(x: Fraction) -> Fraction:
    return _round_rne(x, 23, -126)


def bf16(x: Fraction) -> Fraction:
    return _round_rne(x, 7, -126)


def test_round_rne_helper_against_known_values():
    # independent sanity of the helper: exact powers, ties to even, the fp32 / bf16 spacing
    assert f32(Fraction(1)) == 1 and bf16(Fraction(3, 2)) == Fraction(3, 2)
    assert bf16(Fraction(1) + Fraction(1, 256)) == 1                  # tie -> even (1.0)
    assert bf16(Fraction(1) + Fraction(3, 256)) == Fraction(1) + Fraction(1, 64)  # tie -> even (1+2/128)
    assert f32(Fraction(1) + Fraction(1, 2 ** 24)) == 1               # tie -> even
    assert f32(Fraction(1) + Fraction(3, 2 ** 25)) == Fraction(1) + Fraction(1, 2 ** 23)
    assert f32(Fraction(1, 10)) == Fraction(float(np.float32(0.1)))
    assert bf16(Fraction(-1, 3)) == -Fraction(171, 512)              # -0.333984375


def test_classify_tokens_misses_become_forced():
    case = make_case(rcgen.CFG1)
    lay = layouts(case)[0]
    items = sorted({int(i) for i in lay.src_id[lay.cls == ITEM]})
    assert len(items) == 4
    resident = set(items[::2])                       # items 0 and 2 of the request stay resident
    out = classify_tokens(lay, resident)
    for p in range(lay.n):
        c0, c1 = int(lay.cls[p]), int(out.cls[p])
        if c0 == ITEM and int(lay.src_id[p]) not in resident:
            assert c1 == FORCED, p                   # a miss is recomputed (R18)
        else:
            assert c1 == c0, p                       # residents and PREFIX/HIST/FORCED untouched
    # everything but the class array is unchanged, and the input layout is not mutated
    assert np.array_equal(out.tokens, lay.tokens) and np.array_equal(out.src_id, lay.src_id)
    assert np.array_equal(out.src_off, lay.src_off) and out.seg_start == lay.seg_start
    assert int((lay.cls == FORCED).sum()) == rcgen.CFG1.tail_len
    n_miss = sum(1 for p in range(lay.n) if lay.cls[p] == ITEM and int(lay.src_id[p]) not in resident)
    assert n_miss == 2 * rcgen.CFG1.item_len
    assert int((out.cls == FORCED).sum()) == rcgen.CFG1.tail_len + n_miss
    # no residency information -> the layout as decomposed; everything resident -> no change
    assert classify_tokens(lay, None) is lay
    assert np.array_equal(classify_tokens(lay, set(items)).cls, lay.cls)
    assert np.array_equal(classify_tokens(lay, set()).cls == FORCED, np.isin(lay.cls, [ITEM, FORCED]))


def test_assemble_hist_k_every_element_fraction_exact():
    wl = rcgen.CFG1
    case = make_case(wl)
    pools = oracle_pools(case)
    lay = layouts(case)[0]
    s = case["shape"]
    gf = 1
    K, V, dfn = assemble(s, lay, pools["items"], pools["hist"], pools["prefix"], gather_from=gf)
    h2 = s.head_dim // 2
    inv = [math.pow(s.rope_theta, -2.0 * i / s.head_dim) for i in range(h2)]
    hist_pos = np.nonzero(lay.cls == HIST)[0]
    assert len(hist_pos) == wl.hist_len
    deltas = set()
    for p in hist_pos:
        q, sc, o = pools["hist"][int(lay.src_id[p])]
        d = int(p) - int(o)
        deltas.add(d)
        cs = [Fraction(float(np.float32(math.cos(d * f)))) for f in inv]
        sn = [Fraction(float(np.float32(math.sin(d * f)))) for f in inv]
        for l in range(gf, s.n_layers):
            assert dfn[l, p]
            got = bf16_to_f32(K[l, p])
            for h in range(s.n_kv_heads):
                skey = Fraction(float(sc[l, 0, h]))              # the K scale: [l][K=0][h]
                x = [f32(Fraction(int(q[l, 0, h, j])) * skey) for j in range(s.head_dim)]
                for i in range(h2):
                    y0 = f32(f32(x[i] * cs[i]) - f32(x[i + h2] * sn[i]))
                    y1 = f32(f32(x[i + h2] * cs[i]) + f32(x[i] * sn[i]))
                    assert Fraction(float(got[h, i])) == bf16(y0), (p, l, h, i)
                    assert Fraction(float(got[h, i + h2])) == bf16(y1), (p, l, h, i + h2)
        for l in range(gf):
            assert not dfn[l, p]                         # layers < gather_from are recomputed
    # the workload really exercises signed offsets (history prototypes live at other positions)
    assert any(d < 0 for d in deltas) and any(d > 0 for d in deltas)


def _quant_r15(x):
    """SURVEY R15, written out for the test: per (layer, K/V, head) absmax/127 scale, RNE codes."""
    x = np.asarray(x, np.float32)
    amax = np.abs(x).max(axis=-1)
    scale = (amax / np.float32(127.0)).astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(scale[..., None] > 0, np.rint(x / scale[..., None]), 0)
    return np.clip(q, -127, 127).astype(np.int8), scale


def test_assemble_hist_k_realigned_prototype_equals_key_at_target():
    # A prototype is materialised at its canonical position o (R17: K post-RoPE at o, int8 per
    # R15). Placed at prompt position p, assemble() must give the key computed at p (the token's
    # layer-0 K is context-free, so O-FULL of the token at p is the ground truth), up to the int8
    # and bf16 rounding -- and the opposite Delta sign must be far off.
    wl = rcgen.CFG1
    case = make_case(wl)
    s = case["shape"]
    m = OracleModel(s, case["W"])
    lay = layouts(case)[0]
    hist_pos = [int(p) for p in np.nonzero(lay.cls == HIST)[0]]
    n = lay.n
    toks = lay.tokens.tolist()
    # ground truth at the true positions: layer-0 K of every prompt token
    full = full_prefill(m, toks)
    errs, wrong = [], []
    for p in hist_pos[::3]:
        o = int(case["protos"].canon_pos[int(lay.src_id[p])])
        # materialise the prototype: the same token sitting at position o
        seq = [toks[p]] * (o + 1)
        k_at_o = full_prefill(m, seq)["K"][0][o]                    # [Hk][dh], RoPE at o
        q, sc = _quant_r15(np.stack([k_at_o, k_at_o]))
        qq = np.zeros((s.n_layers, 2, s.n_kv_heads, s.head_dim), np.int8)
        ss = np.ones((s.n_layers, 2, s.n_kv_heads), np.float32)
        qq[0] = q
        ss[0] = sc
        hist = {int(lay.src_id[p]): (qq, ss, o)}
        one = type(lay)(lay.tokens, np.where(np.arange(n) == p, HIST, FORCED).astype(np.uint8),
                        lay.src_id, lay.src_off, lay.seg_start, lay.cand_idtok)
        K, _, _ = assemble(s, one, {}, hist, None, gather_from=0)
        got = bf16_to_f32(K[0, p]).astype(np.float64)
        errs.append(rel_l2(got, full["K"][0][p]))
        # the opposite sign of Delta (rotate to o - (p - o)) is a different key
        seq2 = [toks[p]] * (2 * o - p + 1) if 2 * o - p >= 0 else None
        if seq2 is not None and p != o:
            wrong.append(rel_l2(got, full_prefill(m, seq2)["K"][0][2 * o - p]))
    assert max(errs) < 1.5e-2, errs
    assert wrong and min(wrong) > 0.1, wrong
