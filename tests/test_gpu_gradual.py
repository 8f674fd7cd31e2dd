"""Gradual filtering (NEXT-1 variant, reading R-GF) through the C-ABI vs the oracle.

Several selections are correct where deviations nearly tie (R21), so the oracle is driven along
the GPU's own trajectory Sel_0 .. Sel_g (`sel_trace`) and the test checks (1) that every GPU step
is a valid per-class top-k of the oracle's layer-l divergence among the previous step, up to near
ties, (2) Sel_0 against the oracle's own one-shot choice, and (3) logits and hidden states of the
final Sel within the R20 tolerance. Without shrinking (r_start = r) the gradual path must equal the
one-shot path bit for bit in deterministic mode.
"""
import dataclasses

import numpy as np
import pytest
import torch

import rcgen
from oracle.assemble import assemble
from oracle.layout import HIST, ITEM, FORCED
from oracle.model import OracleModel
from oracle.selective import selective_prefill
from tests.helpers import make_case, oracle_pools, layouts, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-2
WL4 = dataclasses.replace(rcgen.CFG1, shape=dataclasses.replace(rcgen.CFG1.shape, n_layers=4, name="tiny4"),
                          name="cfg1-tiny4")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07443_b200.build import build
    build()


def _run(case, pools, c, g, r0, r, deterministic=False, window=0):
    from tests import gpu_helpers as G
    n_tok = sum(l.n for l in layouts(case))
    ctx, _ = G.make_ctx(case, pools, n_tok)
    lays = G.gpu_layouts(ctx, case)
    seqs = ctx.assemble(lays, prefix_id=G.PREFIX_ID, gather_from=c)
    n_cand = sum(len(l["cand_idtok"]) for l in lays)
    out = ctx.selective_prefill(seqs, r, r, check_layer=c, window=window, hidden=True, n_cand=n_cand, gradual=g,
                                r_start_rev_bp=r0, r_start_item_bp=r0, sel_trace=g > 0, deterministic=deterministic)
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}
    ctx.release(seqs)
    ctx.close()
    return res


def _topk_valid(sel, prev, D, lay, window):
    """sel keeps, per class, the largest D among prev, except for near ties (within 2 %)."""
    n = lay.n
    win = set(range(n - window, n)) if window else set()
    for cl in (HIST, ITEM):
        cand = [p for p in prev if lay.cls[p] == cl and p not in win]
        kept = [p for p in cand if p in sel]
        gone = [p for p in cand if p not in sel]
        if not kept or not gone:
            continue
        lo = min(int(D[p]) for p in kept)
        hi = max(int(D[p]) for p in gone)
        if hi > lo and hi - lo > 0.02 * hi:
            return False
    return True


@pytest.mark.parametrize("wl,n_req,c,g,r0,r,window", [
    (rcgen.MINI_L, 1, 1, 1, 6000, 1500, 0),
    (rcgen.MINI_L, 2, 0, 2, 10000, 1500, 0),
    (rcgen.MINI_Q, 1, 1, 1, 5000, 1000, 0),
    (WL4, 2, 1, 2, 8000, 1000, 12),
    (WL4, 1, 0, 3, 10000, 0, 0),
])
def test_gradual_matches_oracle_along_the_gpu_trajectory(wl, n_req, c, g, r0, r, window):
    case = make_case(wl, n_req=n_req)
    pools = oracle_pools(case)
    res = _run(case, pools, c, g, r0, r, window=window)
    m = OracleModel(case["shape"], case["W"])
    off, trace, sel_off = res["trace_off"], res["sel_trace"], res["sel_off"]
    for k, lay in enumerate(layouts(case)):
        steps = [trace[off[i * n_req + k]:off[i * n_req + k + 1]] for i in range(g + 1)]
        sizes = [len(s) for s in steps]
        assert sizes == sorted(sizes, reverse=True) and sizes[0] > sizes[-1]
        final = res["sel_pos"][sel_off[k]:sel_off[k + 1]]
        assert np.array_equal(steps[-1], final)
        assert set(np.nonzero(lay.cls == FORCED)[0]) <= set(final.tolist())
        K, V, _ = assemble(case["shape"], lay, pools["items"], pools["hist"], pools["prefix"], gather_from=c)
        kw = dict(check_layer=c, window=window, gradual=g, r_start_rev_bp=r0, r_start_item_bp=r0)
        forced = selective_prefill(m, lay, K, V, r, r, forced_steps=steps, **kw)
        own = selective_prefill(m, lay, K, V, r, r, **kw)
        # step 0 is the one-shot selection at r_start: Jaccard against the oracle's own choice
        a, b = set(steps[0].tolist()), set(own["sel_steps"][0].tolist())
        assert len(a) == len(b) and len(a & b) / len(a | b) >= 0.95
        for i in range(1, g + 1):
            prev, cur = set(steps[i - 1].tolist()), set(steps[i].tolist())
            assert cur <= prev
            assert _topk_valid(cur, prev, forced["D_steps"][i], lay, window), i
        assert rel_l2(res["logits"][k], forced["logits"]) < TOL
        assert rel_l2(res["hidden"][sel_off[k]:sel_off[k + 1]], forced["x_sel"]) < TOL


def test_gradual_without_shrink_is_bitwise_the_one_shot_path():
    wl = rcgen.MINI_L
    case = make_case(wl, n_req=2)
    pools = oracle_pools(case)
    a = _run(case, pools, 1, 0, 1500, 1500, deterministic=True)
    b = _run(case, pools, 1, 1, 1500, 1500, deterministic=True)
    assert np.array_equal(a["sel_pos"], b["sel_pos"])
    assert np.array_equal(a["logits"], b["logits"]) and np.array_equal(a["hidden"], b["hidden"])
    steps = b["sel_trace"]
    assert np.array_equal(steps[:len(steps) // 2], steps[len(steps) // 2:])


def test_gradual_argument_checks():
    from paper_2605_07443_b200 import _lib as R
    from tests import gpu_helpers as G
    wl = rcgen.MINI_L
    case = make_case(wl)
    pools = oracle_pools(case)
    ctx, _ = G.make_ctx(case, pools, wl.n)
    lays = G.gpu_layouts(ctx, case)
    seqs = ctx.assemble(lays, prefix_id=G.PREFIX_ID, gather_from=1)
    n_cand = len(lays[0]["cand_idtok"])
    bad = [dict(gradual=2, r_start_rev_bp=5000, r_start_item_bp=5000),     # c + g beyond the last layer
           dict(gradual=1, r_start_rev_bp=1000, r_start_item_bp=5000),     # start below the final ratio
           dict(gradual=R.RC_MAX_GRADUAL + 1 if hasattr(R, "RC_MAX_GRADUAL") else 17)]
    for kw in bad:
        with pytest.raises(R.RcError) as e:
            ctx.selective_prefill(seqs, 1500, 1500, check_layer=1, n_cand=n_cand, **kw)
        assert e.value.code == R.RC_E_INVALID
    sel = ctx.selective_prefill(seqs, 1500, 1500, check_layer=1, n_cand=n_cand)["sel_pos"].cpu().numpy()
    with pytest.raises(R.RcError) as e:
        ctx.selective_prefill(seqs, 1500, 1500, check_layer=1, n_cand=n_cand, forced_sel=[sel], gradual=1,
                              r_start_rev_bp=3000, r_start_item_bp=3000)
    assert e.value.code == R.RC_E_UNSUPPORTED
    ctx.release(seqs)
    ctx.close()
