"""Pools materialised by the model itself (SURVEY §8(d) "Pool contents", R16/R17)
and the exact-cache invariant on the GPU (SURVEY §8(c) O-SEL pin (3)).

* librc's dense path materialises the prefix, item and prototype pools (rc_seq_export_kv); the oracle
  re-materialises the prefix, one item and one prototype itself as a spot check.
* selective prefill on those pools against O-SEL (forced to the GPU's selection) and the selection
  against the oracle's own on the same pool bytes -- deviations now measure real drift.
* exact cache: pools = the GPU's own full-prefill KV of this very prompt at Delta = 0 (items bf16 at
  their prompt offsets, history tokens int8 per R15 at their own positions) => selective == full
  within the R20 tolerance for r in {0, 15%, 100%}, and the item deviations are ~0.
"""
import numpy as np
import pytest
import torch

import rcgen
from oracle.assemble import assemble
from oracle.layout import FORCED, HIST, ITEM, PREFIX
from oracle.model import OracleModel, full_prefill
from oracle.numerics import bf16_to_f32
from oracle.selective import selective_prefill
from tests.helpers import make_case, layouts, rel_l2, rms_err, assert_top10_ranking

pytestmark = pytest.mark.gpu

TOL = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07443_b200.build import build
    build()


def _G():
    from tests import gpu_helpers
    return gpu_helpers


def selection_agrees(sel_gpu, own, lay, min_jac=0.95):
    """R21 end to end: Jaccard >= min_jac, or (small Sel) at most one swapped pair per class that is a
    near-tie of the oracle's own scores (within 2 %). Returns the Jaccard."""
    a, b = set(int(x) for x in sel_gpu), set(int(x) for x in own["sel"])
    jac = len(a & b) / len(a | b)
    if jac >= min_jac:
        return jac
    S = own["S"].astype(np.float64)
    for cl in (HIST, ITEM):
        gin = [p for p in a - b if lay.cls[p] == cl]
        gout = [p for p in b - a if lay.cls[p] == cl]
        assert len(gin) == len(gout) <= 1, (cl, gin, gout, jac)
        for p, q in zip(gin, gout):
            assert abs(S[p] - S[q]) <= 0.02 * max(S[p], S[q]), (p, q, S[p], S[q])
    return jac


@pytest.mark.parametrize("wl", [rcgen.MINI_L, rcgen.MINI_Q])
def test_materialized_pools_spot_check(wl):
    """The oracle re-materialises the prefix, one item (R16) and one prototype (R17 + R15) itself."""
    G = _G()
    case = make_case(wl)
    ctx, pools, _ = G.make_ctx_materialized(case, wl.n)
    ctx.close()
    s = case["shape"]
    m = OracleModel(s, case["W"])
    sys_tok = case["sys"].tolist()
    P = wl.prefix_len
    f = full_prefill(m, sys_tok)
    pre = pools["prefix"].float().numpy()
    for l in range(s.n_layers):
        assert rel_l2(pre[:, l, 0], f["K"][l]) < TOL and rel_l2(pre[:, l, 1], f["V"][l]) < TOL
    it = pools["item_ids"][len(pools["item_ids"]) // 2]
    fi = full_prefill(m, sys_tok + case["cat"].tokens[it].tolist())
    kv = pools["items"][it][0].float().numpy()
    for l in range(s.n_layers):
        assert rel_l2(kv[:, l, 0], fi["K"][l][P:]) < TOL and rel_l2(kv[:, l, 1], fi["V"][l][P:]) < TOL
    corpus, seq_of, off_of = pools["corpus"]
    for j in (0, len(pools["proto_ids"]) - 1):
        pid = pools["proto_ids"][j]
        fp = full_prefill(m, sys_tok + corpus[seq_of[j]].tolist())
        q, sc, o = pools["hist"][pid]
        assert o == P + off_of[j] and corpus[seq_of[j], off_of[j]] == case["protos"].token[pid]
        deq = q.astype(np.float64) * sc[..., None].astype(np.float64)   # [L][2][Hk][dh]
        for l in range(s.n_layers):
            # int8 (R15, absmax/127 per row) + the bf16 KV it was quantised from
            assert rel_l2(deq[l, 0], fp["K"][l][o]) < 2 * TOL and rel_l2(deq[l, 1], fp["V"][l][o]) < 2 * TOL
            assert np.abs(q[l]).max() == 127                                # absmax row code


@pytest.mark.parametrize("wl,r_bp,c", [(rcgen.MINI_L, 1500, 1), (rcgen.MINI_Q, 1500, 1), (rcgen.MINI_L, 3000, 2)])
def test_selective_parity_on_materialized_pools(wl, r_bp, c):
    G = _G()
    case = make_case(wl, n_req=2)
    olays = layouts(case)
    n_tok = sum(l.n for l in olays)
    ctx, pools, _ = G.make_ctx_materialized(case, n_tok)
    lays = G.gpu_layouts(ctx, case)
    seqs = ctx.assemble(lays, prefix_id=G.PREFIX_ID, gather_from=c)
    n_cand = sum(len(l["cand_idtok"]) for l in lays)
    out = ctx.selective_prefill(seqs, r_bp, r_bp, check_layer=c, hidden=True, n_cand=n_cand)
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}
    ctx.release(seqs)
    ctx.close()
    m = OracleModel(case["shape"], case["W"])
    co = 0
    for r, lay in enumerate(olays):
        sel = res["sel_pos"][res["sel_off"][r]:res["sel_off"][r + 1]]
        K, V, _ = assemble(case["shape"], lay, pools["items"], pools["hist"], pools["prefix"], gather_from=c)
        own = selective_prefill(m, lay, K, V, r_bp, r_bp, check_layer=c)
        forced = selective_prefill(m, lay, K, V, r_bp, r_bp, check_layer=c, forced_sel=sel)
        assert len(own["sel"]) == len(sel)
        jac = selection_agrees(sel, own, lay)
        print(f"materialised pools {wl.name} r={r_bp} c={c} request {r}: Jaccard {jac:.4f}")
        assert rel_l2(res["logits"][r], forced["logits"]) < TOL
        assert rel_l2(res["hidden"][res["sel_off"][r]:res["sel_off"][r + 1]], forced["x_sel"]) < TOL
        nc = len(lay.cand_idtok)
        cg = res["cand_scores"][co:co + nc]
        assert np.array_equal(cg, res["logits"][r][lay.cand_idtok])          # readout is exact
        assert np.max(np.abs(cg - forced["cand_scores"])) <= 5 * TOL * np.sqrt(np.mean(forced["logits"] ** 2))
        co += nc
        # real drift: item tokens carry a nonzero deviation (context differs from materialisation)
        assert own["D"][lay.cls == ITEM].min() > 0


def _exact_cache_ctx(case, lay_g, r_full):
    """Pools holding the GPU's own full-prefill KV of the prompt at Delta = 0."""
    from paper_2605_07443_b200 import _lib as R
    from paper_2605_07443_b200.api import RcContext
    G = _G()
    wl, shape = case["wl"], case["shape"]
    n = len(lay_g["tokens"])
    P = wl.prefix_len
    kv_full = r_full["kv"]                                   # bf16 [n][L][2][Hk][dh]
    Wd = r_full["Wd"]
    hist_pos = np.nonzero(lay_g["cls"] == HIST)[0]
    items = list(dict.fromkeys(int(i) for i in lay_g["src_id"][lay_g["cls"] == ITEM]))
    ctx = RcContext(shape, Wd, item_rows=n, hist_rows=len(hist_pos), prefix_rows=P, arena_rows=2 * n,
                    max_seq_len=max(n, 256), max_batch_tokens=2 * n)
    ctx.pool_register_blocks(R.RC_POOL_PREFIX_BF16, [G.PREFIX_ID], [P], [0], kv_full[:P].contiguous())
    starts, lens = [], []
    for it in items:
        pos = np.nonzero((lay_g["cls"] == ITEM) & (lay_g["src_id"] == it))[0]
        starts.append(int(pos[0]))
        lens.append(len(pos))
    blk = torch.cat([kv_full[s:s + ln] for s, ln in zip(starts, lens)]).contiguous()
    ctx.pool_register_blocks(R.RC_POOL_ITEM_BF16, items, lens, starts, blk)   # canonical start = prompt offset
    # history: one prototype per history position, int8 (R15) of the full-prefill KV at that position
    q, sc = r_full["hist_q"], r_full["hist_s"]
    pids = [10_000_000 + int(p) for p in hist_pos]
    ctx.pool_register_blocks(R.RC_POOL_HIST_INT8, pids, [1] * len(pids), [int(p) for p in hist_pos], q, sc)
    lay = dict(lay_g)
    lay["src_id"] = lay_g["src_id"].copy()
    lay["src_id"][hist_pos] = pids
    torch.cuda.synchronize()
    return ctx, lay


@pytest.mark.parametrize("wl", [rcgen.MINI_L, rcgen.MINI_Q])
def test_exact_cache_selective_equals_full_on_gpu(wl):
    G = _G()
    case = make_case(wl)
    pools_unused = None
    shape = case["shape"]
    from tests.helpers import oracle_pools
    pools = oracle_pools(case)
    ctx, Wd = G.make_ctx(case, pools, wl.n)
    lay_g = G.gpu_layouts(ctx, case)[0]
    n = len(lay_g["tokens"])
    # the GPU's own full prefill (every position recomputed, no prefix reuse)
    full_lay = dict(lay_g, cls=np.full(n, FORCED, np.uint8))
    seqs = ctx.assemble([full_lay], prefix_id=G.PREFIX_ID, gather_from=0)
    out_f = ctx.selective_prefill(seqs, 10000, 10000, check_layer=0, n_cand=len(lay_g["cand_idtok"]))
    kv = ctx.export_kv(seqs[0], 0, n)
    hist_pos = np.nonzero(lay_g["cls"] == HIST)[0]
    q_all, s_all = ctx.export_kv(seqs[0], 0, n, int8=True)
    torch.cuda.synchronize()
    logits_full = out_f["logits"][0].cpu().numpy()
    ctx.release(seqs)
    ctx.close()
    hp = torch.as_tensor(hist_pos, device=q_all.device)
    r_full = dict(kv=kv, Wd=Wd, hist_q=q_all[hp].contiguous(), hist_s=s_all[hp].contiguous())
    ref = full_prefill(OracleModel(shape, case["W"]), lay_g["tokens"].tolist())["logits_last"]
    assert rel_l2(logits_full, ref) < TOL
    for r_bp in (0, 1500, 10000):
        ctx2, lay = _exact_cache_ctx(case, lay_g, r_full)
        seqs = ctx2.assemble([lay], prefix_id=G.PREFIX_ID, gather_from=1)
        U = int((lay["cls"] != PREFIX).sum())
        score = torch.zeros(U, dtype=torch.int64, device="cuda")
        out = ctx2.selective_prefill(seqs, r_bp, r_bp, check_layer=1, n_cand=len(lay["cand_idtok"]), score_out=score)
        torch.cuda.synchronize()
        lg = out["logits"][0].cpu().numpy()
        D = score.cpu().numpy().view(np.uint64)
        ctx2.release(seqs)
        ctx2.close()
        e_gpu, e_ref = rel_l2(lg, logits_full), rel_l2(lg, ref)
        print(f"exact cache {wl.name} r={r_bp}: rel-L2 vs GPU full {e_gpu:.2e}, vs oracle full {e_ref:.2e}")
        assert e_gpu < TOL and e_ref < TOL
        # items hold the exact bf16 full-prefill KV at Delta = 0: the check layer's K_new/V_new recompute
        # them from the same inputs, so their deviation is only the rounding of the U-only layer 0
        ucls = lay["cls"][wl.prefix_len:]
        d_item = D[ucls == ITEM].astype(np.float64)
        d_scale = 2 * shape.n_kv_heads * shape.head_dim * 2.0 ** 24  # one unit of |new - cached| per element
        assert d_item.mean() < 0.02 * d_scale, d_item.mean() / d_scale
