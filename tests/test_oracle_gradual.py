"""Pins of the gradual-filtering variant of O-SEL (reading R-GF, NEXT-1; not gpu).

* r_start = r: every step keeps its whole previous Sel, so the result is the one-shot O-SEL.
* exact cache (pools = the O-FULL KV of this prompt): any Sel at any step gives O-FULL, so a
  misindexed row compaction (queries, residuals, positions) fails here.
* structure: Sel_i is nested in Sel_{i-1} with the step budget ceil(r_i |class|); its class
  members are the top by (D_l desc, position asc) among Sel_{i-1}; D_l is the R4 divergence of
  layer l's fresh K/V (as stored in the returned cache) from the stitched input cache.
"""
import dataclasses

import numpy as np
import pytest

import rcgen
from oracle.assemble import assemble
from oracle.layout import FORCED, HIST, ITEM, budget
from oracle.model import OracleModel, full_prefill
from oracle.numerics import bf16_to_f32, round_bf16, deviation_fixed
from oracle.select import gradual_ratio_bp, sel_count, select_sel
from oracle.selective import selective_prefill
from tests.helpers import make_case, oracle_pools, layouts, rel_l2

WL4 = dataclasses.replace(rcgen.CFG1, shape=dataclasses.replace(rcgen.CFG1.shape, n_layers=4, name="tiny4"),
                          name="cfg1-tiny4")


def _setup(wl=WL4):
    case = make_case(wl)
    m = OracleModel(case["shape"], case["W"])
    pools = oracle_pools(case)
    lay = layouts(case)[0]
    K, V, _ = assemble(case["shape"], lay, pools["items"], pools["hist"], pools["prefix"], gather_from=0)
    return case, m, lay, K, V


def test_gradual_ratio_schedule():
    assert [gradual_ratio_bp(10000, 1500, i, 2) for i in range(3)] == [10000, 5750, 1500]
    assert [gradual_ratio_bp(3000, 1500, i, 4) for i in range(5)] == [3000, 2625, 2250, 1875, 1500]
    assert [gradual_ratio_bp(1000, 999, i, 3) for i in range(4)] == [1000, 1000, 1000, 999]   # truncation
    assert gradual_ratio_bp(4000, 1500, 0, 0) == 1500                                         # g = 0: one shot
    cls = np.array([0] * 3 + [HIST] * 10 + [ITEM] * 7 + [FORCED] * 2)
    D = np.arange(len(cls))[::-1].astype(np.uint64)
    prev = select_sel(cls, D, 6000, 6000)
    sel = select_sel(cls, D, 3000, 3000, among=prev)
    assert set(sel) <= set(prev) and len(sel) == sel_count(cls, 3000, 3000)
    with pytest.raises(AssertionError):   # a step may not grow a class beyond the previous Sel
        select_sel(cls, D, 9000, 9000, among=prev)


@pytest.mark.parametrize("c,g", [(0, 2), (1, 2), (0, 3)])
def test_gradual_without_shrink_is_one_shot(c, g):
    case, m, lay, K, V = _setup()
    a = selective_prefill(m, lay, K, V, 1500, 1500, check_layer=c)
    b = selective_prefill(m, lay, K, V, 1500, 1500, check_layer=c, gradual=g, r_start_rev_bp=1500, r_start_item_bp=1500)
    assert np.array_equal(a["sel"], b["sel"]) and all(np.array_equal(s, a["sel"]) for s in b["sel_steps"])
    assert np.array_equal(a["logits"], b["logits"])
    for l in range(case["shape"].n_layers):
        assert np.array_equal(a["K"][l], b["K"][l]) and np.array_equal(a["V"][l], b["V"][l])


@pytest.mark.parametrize("c,g,r0,r", [(0, 3, 10000, 1500), (1, 2, 8000, 0), (1, 1, 5000, 2000)])
def test_gradual_exact_cache_equals_full(c, g, r0, r):
    case, m, lay, _, _ = _setup()
    s = case["shape"]
    full = full_prefill(m, lay.tokens.tolist())
    Kx = [full["K"][l].copy() for l in range(s.n_layers)]
    Vx = [full["V"][l].copy() for l in range(s.n_layers)]
    out = selective_prefill(m, lay, Kx, Vx, r, r, check_layer=c, exact_kv=True, gradual=g,
                            r_start_rev_bp=r0, r_start_item_bp=r0)
    sizes = [len(x) for x in out["sel_steps"]]
    assert sizes == sorted(sizes, reverse=True) and sizes[0] > sizes[-1]   # the set really shrinks
    assert rel_l2(out["logits"], full["logits_last"]) < 1e-10
    for l in range(s.n_layers):
        assert rel_l2(out["K"][l], full["K"][l]) < 1e-10 and rel_l2(out["V"][l], full["V"][l]) < 1e-10


@pytest.mark.parametrize("c,g,r0,r,window", [(0, 3, 9000, 1500, 0), (1, 2, 6000, 1000, 5)])
def test_gradual_steps_nested_topk_and_deviation_of_the_stored_kv(c, g, r0, r, window):
    case, m, lay, K, V = _setup()
    s = case["shape"]
    out = selective_prefill(m, lay, K, V, r, r, check_layer=c, window=window, gradual=g,
                            r_start_rev_bp=r0, r_start_item_bp=r0)
    steps, Ds = out["sel_steps"], out["D_steps"]
    assert len(steps) == g + 1 and np.array_equal(steps[-1], out["sel"])
    n = lay.n
    win = set(range(n - window, n)) if window else set()
    nh = sum(1 for p in range(n) if lay.cls[p] == HIST and p not in win)
    ni = sum(1 for p in range(n) if lay.cls[p] == ITEM and p not in win)
    forced = {p for p in range(n) if lay.cls[p] == FORCED} | win
    for i in range(g + 1):
        rh = gradual_ratio_bp(r0, r, i, g)
        sel = set(int(p) for p in steps[i])
        assert forced <= sel
        assert len(sel) == len(forced) + budget(rh, nh) + budget(rh, ni) == sel_count(lay.cls, rh, rh, window)
        if i == 0:
            continue
        prev = set(int(p) for p in steps[i - 1])
        assert sel <= prev
        l = c + i
        Dl = Ds[i]
        for cl in (HIST, ITEM):
            cand = [p for p in prev if lay.cls[p] == cl and p not in win]
            kept = [p for p in cand if p in sel]
            gone = [p for p in cand if p not in sel]
            if kept and gone:   # R6 order: (D desc, position asc)
                assert min((int(Dl[p]), -p) for p in kept) > max((int(Dl[p]), -p) for p in gone)
            # D_l is the divergence of the fresh layer-l K/V (what the returned cache holds at the rows
            # of Sel_{i-1}) from the stitched input cache at layer l
            for p in cand:
                kf = round_bf16(out["K"][l][p]).reshape(1, -1)
                vf = round_bf16(out["V"][l][p]).reshape(1, -1)
                ks = bf16_to_f32(K[l][p]).reshape(1, -1)
                vs = bf16_to_f32(V[l][p]).reshape(1, -1)
                assert int(Dl[p]) == int(deviation_fixed(kf, ks)[0] + deviation_fixed(vf, vs)[0]) > 0
        # rows outside Sel_{i-1} keep their stitched bytes at layer l; rows inside are fresh
        stitched = [p for p in range(n) if p not in prev]
        assert np.array_equal(out["K"][l][stitched], bf16_to_f32(K[l][stitched]).astype(np.float64))


def test_gradual_forced_steps_reproduce_the_free_run():
    case, m, lay, K, V = _setup()
    a = selective_prefill(m, lay, K, V, 1000, 1000, check_layer=1, gradual=2, r_start_rev_bp=7000,
                          r_start_item_bp=4000)
    b = selective_prefill(m, lay, K, V, 1000, 1000, check_layer=1, gradual=2, r_start_rev_bp=7000,
                          r_start_item_bp=4000, forced_steps=a["sel_steps"])
    assert np.array_equal(a["logits"], b["logits"])
    # a different (valid, nested) trajectory gives different logits: the steps are really used
    alt = [a["sel_steps"][0], a["sel_steps"][0], a["sel_steps"][0]]
    c_ = selective_prefill(m, lay, K, V, 1000, 1000, check_layer=1, gradual=2, r_start_rev_bp=7000,
                           r_start_item_bp=4000, forced_steps=alt)
    assert not np.array_equal(a["logits"], c_["logits"])
