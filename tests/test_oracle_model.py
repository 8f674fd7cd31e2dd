"""Pins of O-FULL / O-ASM / O-SEL against library routines and invariants (not gpu).

* O-FULL vs HF transformers LlamaForCausalLM / Qwen2ForCausalLM in fp32 (library routine).
* r = 0, c = 0, FORCED = tail  ==  HF forward of the tail over past_key_values = stitched KV.
* r = 100%  ==  O-FULL (exact prefix KV).
* exact cache (pools = O-FULL KV of this prompt, Delta = 0)  ==  O-FULL for every r, c.
* O-ASM: brute-force element checks and the encode-at-target property of Delta-RoPE.
"""
import numpy as np
import pytest
import torch

import rcgen
from oracle.model import OracleModel, forward, full_prefill
from oracle.assemble import assemble
from oracle.selective import selective_prefill
from oracle.layout import FORCED, HIST, ITEM, PREFIX, layout_from_request
from oracle.numerics import bf16_bits, bf16_to_f32, round_bf16, RopeTable, rope_rotate_f32, dequant_int8
from tests.helpers import make_case, oracle_pools, layouts, hf_model, rel_l2


def _hf_logits_and_kv(model, tokens):
    with torch.no_grad():
        out = model(torch.tensor([tokens]), use_cache=True)
    kv = out.past_key_values
    return out.logits[0].double().numpy(), kv


@pytest.mark.parametrize("shape", [rcgen.TINY, rcgen.TINY_Q7])
def test_full_prefill_matches_hf(shape):
    W = rcgen.gen_weights(shape)
    toks = np.random.default_rng(0).integers(0, shape.vocab, 144).tolist()
    m = OracleModel(shape, W)
    o = full_prefill(m, toks)
    hf = hf_model(shape, W)
    logits, kv = _hf_logits_and_kv(hf, toks)
    assert rel_l2(o["logits_fn"](), logits) < 2e-5
    for l in range(shape.n_layers):
        k_hf = kv.layers[l].keys[0].permute(1, 0, 2).double().numpy()
        v_hf = kv.layers[l].values[0].permute(1, 0, 2).double().numpy()
        assert rel_l2(o["K"][l], k_hf) < 2e-5 and rel_l2(o["V"][l], v_hf) < 2e-5


def test_full_prefill_matches_hf_8b_width():
    # 2 layers of the Llama-3-8B shape (real widths, GQA 4, theta 5e5) with a small vocabulary
    import dataclasses
    shape = dataclasses.replace(rcgen.LLAMA3_8B, n_layers=2, vocab=1024, name="llama-w2")
    W = rcgen.gen_weights(shape)
    toks = np.random.default_rng(1).integers(0, shape.vocab, 48).tolist()
    o = full_prefill(OracleModel(shape, W), toks)
    logits, _ = _hf_logits_and_kv(hf_model(shape, W), toks)
    assert rel_l2(o["logits_fn"](), logits) < 1e-4


def _tiny_setup(wl, exact_prefix=True):
    case = make_case(wl)
    m = OracleModel(case["shape"], case["W"])
    pkv = None
    if exact_prefix:   # materialise the exact prefix KV with O-FULL of the system prompt (R8)
        f = full_prefill(m, case["sys"].tolist())
        kv = np.stack([np.stack([f["K"][l], f["V"][l]], 1) for l in range(case["shape"].n_layers)], 1)
        pkv = torch.from_numpy(kv.astype(np.float32)).to(torch.bfloat16)
    pools = oracle_pools(case, prefix_kv=pkv)
    lay = layouts(case)[0]
    return case, m, pools, lay


def test_assemble_elements_brute_force():
    case, m, pools, lay = _tiny_setup(rcgen.CFG1, exact_prefix=False)
    s = case["shape"]
    K, V, dfn = assemble(s, lay, pools["items"], pools["hist"], pools["prefix"], gather_from=1)
    tab = RopeTable(s.rope_theta, s.head_dim)
    pre = pools["prefix"].view(torch.int16).numpy().view(np.uint16)
    for p in range(lay.n):
        c = lay.cls[p]
        assert dfn[0, p] == (c == PREFIX) and dfn[1, p] == (c != FORCED)
        if c == PREFIX:
            assert np.array_equal(K[:, p], pre[p, :, 0]) and np.array_equal(V[:, p], pre[p, :, 1])
        if c == ITEM:
            it, j = int(lay.src_id[p]), int(lay.src_off[p])
            kv = pools["items"][it][0].view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(V[1, p], kv[j, 1, 1])
            cs, sn = tab.get([p - (rcgen.CFG1.prefix_len + j)])
            k32 = bf16_to_f32(kv[j, 1, 0])
            for h in range(s.n_kv_heads):
                for i in range(s.head_dim // 2):
                    y0 = np.float32(np.float32(k32[h, i] * cs[0, i]) - np.float32(k32[h, i + 8] * sn[0, i]))
                    assert K[1, p, h, i] == bf16_bits(np.float32([y0]))[0]
        if c == HIST:
            q, sc, o = pools["hist"][int(lay.src_id[p])]
            assert np.array_equal(V[1, p], bf16_bits(q[1, 1].astype(np.float32) * sc[1, 1][:, None]))


def test_assemble_realign_equals_encode_at_target():
    # an item materialised at canonical start s and re-aligned to b equals K computed at b
    s = rcgen.TINY
    W = rcgen.gen_weights(s)
    m = OracleModel(s, W)
    toks = np.random.default_rng(5).integers(0, s.vocab, 20).tolist()
    f = full_prefill(m, toks)
    # K at positions 0..19 has RoPE at p; re-rotating K[p] by delta must equal RoPE at p + delta
    tab = RopeTable(s.rope_theta, s.head_dim)
    k32 = f["K"][1].astype(np.float32)
    for delta in (-7, 0, 13, 100):
        c, sn = tab.get(np.full(20, delta))
        re = rope_rotate_f32(k32, c[:, None], sn[:, None])
        _, k_at, _ = m.qkv(1, None if False else _x_at_layer(m, toks, 1), np.arange(20) + delta)
        assert rel_l2(re, k_at) < 2e-6


def _x_at_layer(m, toks, l):
    x = m.embed(toks)
    pos = np.arange(len(toks))
    for j in range(l):
        q, k, v = m.qkv(j, x, pos)
        x = m.post(j, x, m.attend(q, pos, k, v))
    return x


@pytest.mark.parametrize("wl", [rcgen.CFG1, rcgen.CFG1_Q7])
def test_selective_r100_equals_full(wl):
    case, m, pools, lay = _tiny_setup(wl)
    K, V, _ = assemble(case["shape"], lay, pools["items"], pools["hist"], pools["prefix"], gather_from=1)
    sel = selective_prefill(m, lay, K, V, 10000, 10000, check_layer=1)
    full = full_prefill(m, lay.tokens.tolist())
    # the prefix KV is bf16-stored, so compare with O-FULL over that same prefix cache
    P = wl.prefix_len
    pK = [bf16_to_f32(K[l][:P]).astype(np.float64) for l in range(case["shape"].n_layers)]
    pV = [bf16_to_f32(V[l][:P]).astype(np.float64) for l in range(case["shape"].n_layers)]
    ref = forward(m, lay.tokens[P:].tolist(), P, pK, pV)
    assert len(sel["sel"]) == lay.n - P
    assert rel_l2(sel["logits"], ref["logits_last"]) < 1e-10
    assert rel_l2(sel["x_sel"], ref["x"]) < 1e-10
    assert rel_l2(sel["logits"], full["logits_last"]) < 2e-2      # bf16 prefix cache only


@pytest.mark.parametrize("c", [0, 1])
def test_selective_r0_equals_hf_tail_over_stitched_cache(c):
    # r = 0: Sel is exactly the FORCED tail. c = 0: the tail attends over the stitched KV at
    # every layer. c = 1: layer 0 is recomputed for all of U (R12), so the tail's layer-0 context
    # is the prefix cache + the fresh layer-0 K/V of U -- which depend only on (token, position),
    # so HF's own full forward supplies them -- and layers >= 1 are the stitched KV.
    wl = rcgen.CFG1
    case, m, pools, lay = _tiny_setup(wl, exact_prefix=False)
    s = case["shape"]
    K, V, _ = assemble(s, lay, pools["items"], pools["hist"], pools["prefix"], gather_from=c)
    sel = selective_prefill(m, lay, K, V, 0, 0, check_layer=c)
    T = wl.tail_len
    n = lay.n
    P = wl.prefix_len
    assert list(sel["sel"]) == list(range(n - T, n))
    # library routine: HF forward of the tail with past_key_values = that context
    from transformers import DynamicCache
    hf = hf_model(s, case["W"])
    _, kv_full = _hf_logits_and_kv(hf, lay.tokens.tolist())
    cache = DynamicCache(config=hf.config)
    for l in range(s.n_layers):
        k = torch.from_numpy(bf16_to_f32(K[l][:n - T])).permute(1, 0, 2)[None]
        v = torch.from_numpy(bf16_to_f32(V[l][:n - T])).permute(1, 0, 2)[None]
        if l < c:   # fresh layer-0 K/V of U from HF's own forward of the whole prompt
            k[:, :, P:] = kv_full.layers[l].keys[:, :, P:n - T]
            v[:, :, P:] = kv_full.layers[l].values[:, :, P:n - T]
        cache.update(k, v, l)
    with torch.no_grad():
        out = hf(torch.tensor([lay.tokens[n - T:].tolist()]), past_key_values=cache,
                 position_ids=torch.arange(n - T, n)[None], use_cache=True)
    assert rel_l2(sel["logits"], out.logits[0, -1].double().numpy()) < 2e-5
    # non-forced positions keep their stitched bytes at every layer >= c; layers < c hold the
    # fresh K of U (HF's values, to fp32 rounding)
    for l in range(s.n_layers):
        if l >= c:
            assert np.array_equal(bf16_bits(sel["K"][l][:n - T].astype(np.float32)), K[l][:n - T])
        else:
            k_hf = kv_full.layers[l].keys[0].permute(1, 0, 2).double().numpy()
            assert rel_l2(sel["K"][l][P:n], k_hf[P:n]) < 2e-5


@pytest.mark.parametrize("r_bp,c,lam", [(0, 1, 1.0), (1500, 1, 1.0), (1500, 0, 1.0), (5000, 1, 1.0),
                                        (1500, 0, 0.5), (3000, 1, 0.0)])
def test_exact_cache_selective_equals_full(r_bp, c, lam):
    # pools holding the O-FULL KV of this very prompt at the same positions (Delta = 0),
    # kept lossless (fp32 test mode): the stitched cache IS the full-prefill cache
    case, m, pools, lay = _tiny_setup(rcgen.CFG1)
    s = case["shape"]
    full = full_prefill(m, lay.tokens.tolist())
    Kx = [full["K"][l].copy() for l in range(s.n_layers)]
    Vx = [full["V"][l].copy() for l in range(s.n_layers)]
    sel = selective_prefill(m, lay, Kx, Vx, r_bp, r_bp, check_layer=c, exact_kv=True, lam=lam)
    assert rel_l2(sel["logits"], full["logits_last"]) < 1e-10
    for l in range(s.n_layers):
        assert rel_l2(sel["K"][l], full["K"][l]) < 1e-10
    # deviation: K_new equals the cached K up to bf16 rounding of one side -> D <= 1 ulp terms
    assert int(sel["D"].max()) <= 2 * s.n_kv_heads * s.head_dim * 2 ** 24 // 64


def test_selective_lambda_one_is_deviation_only_and_lambda_orders_by_mass():
    case, m, pools, lay = _tiny_setup(rcgen.CFG1)
    K, V, _ = assemble(case["shape"], lay, pools["items"], pools["hist"], pools["prefix"], gather_from=1)
    a = selective_prefill(m, lay, K, V, 1500, 1500, lam=1.0)
    assert a["A"] is None and np.array_equal(a["S"], a["D"])
    b = selective_prefill(m, lay, K, V, 1500, 1500, lam=0.0)
    # lambda = 0: S = A on HIST/ITEM rows, and the budgets pick the largest column masses per class
    reuse = np.isin(lay.cls, [HIST, ITEM])
    assert np.array_equal(b["S"][reuse], b["A"][reuse])
    assert len(b["sel"]) == len(a["sel"])
    for cl in (HIST, ITEM):
        members = np.nonzero(lay.cls == cl)[0]
        chosen = [p for p in b["sel"] if lay.cls[p] == cl]
        rest = [p for p in members if p not in set(chosen)]
        if chosen and rest:
            assert min(int(b["A"][p]) for p in chosen) >= max(int(b["A"][p]) for p in rest)


def test_selective_deterministic_and_sel_shape():
    case, m, pools, lay = _tiny_setup(rcgen.CFG1)
    K, V, _ = assemble(case["shape"], lay, pools["items"], pools["hist"], pools["prefix"], gather_from=1)
    a = selective_prefill(m, lay, K, V, 1500, 1500)
    b = selective_prefill(m, lay, K, V, 1500, 1500, forced_sel=a["sel"])
    assert np.array_equal(a["logits"], b["logits"])
    assert len(a["sel"]) == 8 + 10 + 10          # 10 + 10 + 8 = 28
    assert sorted(a["rank"].tolist()) == list(range(4))
