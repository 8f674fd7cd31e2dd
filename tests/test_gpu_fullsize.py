"""Full-size parity: BASELINE.json configs[1] (cfg3: Llama-3-8B shape, n = 4096, batch 32, r = 15%,
c = 1) in the launch configuration bench.py times (same generators, same batch, the same pools
materialised by the model, RC_ATTN_AUTO, so the paired-tile attention and the large-grid GEMM
schedules run), checked on sampled outputs the oracle computes one request at a time:
  * requests 0 and 31 end to end against O-SEL forced to the GPU's selection (last-token logits,
    x_L[Sel], K/V of the last layer at Sel: rel-L2 <= 1e-2; candidate scores);
  * the GPU's selection against the oracle's own (Jaccard; bf16 noise in layer 0 may flip near-ties).
    The oracle's selection is taken from a 2-layer truncation: Sel is fixed at the check layer c = 1
    (Eq. 3), so layers > c cannot change it;
  * non-selected reused positions keep the gathered bytes at the last layer (bit-exact vs O-ASM).
The oracle consumes the registered pool bytes: the model-materialised ones for batch 32 and the cfg3 batch-1
materialised test, the generator's seeded stand-ins for the other checks (SURVEY §8(d) "Pool contents").
"""
import dataclasses
import json
import os

import numpy as np
import pytest
import torch

import rcgen
from oracle.assemble import assemble
from oracle.layout import layout_from_request
from oracle.model import OracleModel
from oracle.numerics import bf16_to_f32
from oracle.selective import selective_prefill
from tests.helpers import rel_l2, assert_top10_ranking, rms_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 1e-2
R_BP = 1500
C = 1
LOGITS_TOL_PER_REQUEST = 1e-2   # north_star: rel-L2 <= 1e-2 on logits, per request
_LOGITS = {}
CHECK_REQS = tuple(int(x) for x in os.environ.get("RC_FULLSIZE_REQS", "0,31").split(","))


def _setup(wl, batch, check_reqs, materialize=False, gkw=None):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07443_b200.build import build
    from paper_2605_07443_b200.api import RcContext
    from paper_2605_07443_b200 import _lib as R
    build()
    shape = wl.shape
    dev = torch.device("cuda", 0)
    W = rcgen.gen_weights(shape, seed=0, device=dev)
    cat, protos, sys_tok = rcgen.gen_catalog(wl), rcgen.gen_protos(wl), rcgen.gen_system_prompt(wl)
    reqs = rcgen.gen_requests(wl, cat, protos, batch, start=0)  # bench.py's first batch at N=1
    items = sorted({int(i) for r in reqs for i in r.cand_items})
    pids = sorted({int(p) for r in reqs for p in r.hist_protos})
    n = wl.n
    ctx = RcContext(shape, W, item_rows=len(items) * wl.item_len, hist_rows=len(pids), prefix_rows=wl.prefix_len,
                    arena_rows=batch * n, max_seq_len=n, max_batch_tokens=batch * n)
    item_kv = None
    if materialize:  # SURVEY §8(d) "Pool contents": the model's own KV (R16/R17, int8 prototypes per R15)
        from paper_2605_07443_b200 import materialize as MZ
        pkv = MZ.register_prefix(ctx, sys_tok, 1)
        item_kv = {i: v.cpu() for i, v in MZ.register_items(ctx, sys_tok, 1, items, [cat.tokens[i] for i in items],
                                                            keep=True).items()}
        corpus, seq_of, off_of = rcgen.proto_corpus(wl, protos, pids)
        hq, hs = MZ.register_protos(ctx, sys_tok, 1, pids, [int(protos.canon_pos[p]) for p in pids], corpus, seq_of,
                                    off_of)
    else:
        for i0 in range(0, len(items), 128):
            ids = items[i0:i0 + 128]
            kv = rcgen.pools.item_kv(shape, wl.item_len, ids, device=dev)
            ctx.pool_register_blocks(R.RC_POOL_ITEM_BF16, ids, [wl.item_len] * len(ids), [wl.prefix_len] * len(ids),
                                     kv.reshape(len(ids) * wl.item_len, *kv.shape[2:]))
        hq, hs = rcgen.pools.hist_kv(shape, pids, device=dev)
        ctx.pool_register_blocks(R.RC_POOL_HIST_INT8, pids, [1] * len(pids), [int(protos.canon_pos[p]) for p in pids],
                                 hq, hs)
        pkv = rcgen.pools.prefix_kv(shape, wl.prefix_len, device=dev)
        ctx.pool_register_blocks(R.RC_POOL_PREFIX_BF16, [1], [wl.prefix_len], [0], pkv)
    lays = [ctx.decompose_prompt(sys_tok, r.hist_protos, r.hist_tokens, r.cand_items,
                                 [cat.tokens[int(i)] for i in r.cand_items], r.tail_tokens) for r in reqs]
    seqs = ctx.assemble(lays, prefix_id=1, gather_from=C)
    n_cand = sum(len(l["cand_idtok"]) for l in lays)
    out = ctx.selective_prefill(seqs, R_BP, R_BP, check_layer=C, hidden=True, n_cand=n_cand,
                                **(dict(gkw, sel_trace=True) if gkw else {}))
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}
    res["kv_last"] = {r: tuple(t.cpu().numpy().view(np.uint16) for t in ctx.read_kv(seqs[r], shape.n_layers - 1, n))
                      for r in check_reqs}
    cand_off = np.concatenate([[0], np.cumsum([len(l["cand_idtok"]) for l in lays])])
    ctx.release(seqs)
    # run-to-run determinism: the same batch assembled and prefilled again, in the default mode and
    # twice with every residual sum order-fixed (deterministic=1)
    for key, det in (() if gkw else (("rerun", False), ("det1", True), ("det2", True))):
        seqs = ctx.assemble(lays, prefix_id=1, gather_from=C)
        out2 = ctx.selective_prefill(seqs, R_BP, R_BP, check_layer=C, hidden=True, n_cand=n_cand, deterministic=det)
        torch.cuda.synchronize()
        res[key] = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out2.items()}
        ctx.release(seqs)
    ctx.close()
    Wh = {"embed": W["embed"].cpu(), "norm": W["norm"].cpu(), "lm_head": W["lm_head"].cpu(),
          "layers": [{k: v.cpu() for k, v in lw.items()} for lw in W["layers"]]}
    hist = {p: (hq[j].cpu().numpy(), hs[j].cpu().numpy(), int(protos.canon_pos[p])) for j, p in enumerate(pids)}
    ctxd = dict(wl=wl, shape=shape, W=Wh, cat=cat, sys=sys_tok, reqs=reqs, items=items, hist=hist,
                pkv=pkv.cpu(), cand_off=cand_off, item_kv=item_kv)
    del W
    torch.cuda.empty_cache()
    return res, ctxd


@pytest.fixture(scope="module")
def run():
    # the bench's default configuration: pools materialised by the model (bench.py --pools materialized)
    return _setup(rcgen.CFG3, rcgen.CFG3.batch, CHECK_REQS, materialize=True)


def _oracle(d, r, sel):
    wl, shape = d["wl"], d["shape"]
    req = d["reqs"][r]
    lay = layout_from_request(req, d["cat"], d["sys"])
    ids = [int(i) for i in req.cand_items]
    if d.get("item_kv") is not None:   # materialised pools: the registered bytes
        item_d = {it: (d["item_kv"][it], wl.prefix_len) for it in ids}
    else:
        ikv = rcgen.pools.item_kv(shape, wl.item_len, ids, device=torch.device("cuda", 0)).cpu()
        item_d = {it: (ikv[j], wl.prefix_len) for j, it in enumerate(ids)}
    K, V, dfn = assemble(shape, lay, item_d, d["hist"], d["pkv"], gather_from=C)
    forced = selective_prefill(OracleModel(shape, d["W"]), lay, K, V, R_BP, R_BP, check_layer=C, forced_sel=sel)
    # own selection from the 2-layer truncation (Sel is decided at the check layer c = 1)
    sub = dataclasses.replace(shape, n_layers=C + 1)
    Ws = dict(d["W"], layers=d["W"]["layers"][:C + 1])
    own = selective_prefill(OracleModel(sub, Ws), lay, K[:C + 1], V[:C + 1], R_BP, R_BP, check_layer=C)
    return lay, K, dfn, forced, own


@pytest.mark.parametrize("r", CHECK_REQS)
def test_cfg3_batch32_request_matches_oracle(run, r):
    res, d = run
    L = d["shape"].n_layers
    off = res["sel_off"]
    sel = res["sel_pos"][off[r]:off[r + 1]]
    assert len(sel) == len(set(sel.tolist())) and list(sel) == sorted(sel)
    lay, K_asm, dfn, forced, own = _oracle(d, r, sel)
    assert len(own["sel"]) == len(sel)  # same budgets (R5)
    jac = len(set(own["sel"].tolist()) & set(sel.tolist())) / len(set(own["sel"].tolist()) | set(sel.tolist()))
    Kg = bf16_to_f32(res["kv_last"][r][0])[sel].astype(np.float64)
    Vg = bf16_to_f32(res["kv_last"][r][1])[sel].astype(np.float64)
    err = {"request": r, "jaccard": jac, "logits": rel_l2(res["logits"][r], forced["logits"]),
           "hidden": rel_l2(res["hidden"][off[r]:off[r + 1]], forced["x_sel"]),
           "K_last": rel_l2(Kg, forced["K"][L - 1][sel]), "V_last": rel_l2(Vg, forced["V"][L - 1][sel])}
    print("fullsize parity", json.dumps(err))
    _LOGITS[r] = (res["logits"][r], forced["logits"])
    assert jac >= 0.95, err
    assert err["hidden"] < TOL and err["K_last"] < TOL and err["V_last"] < TOL, err
    # DESIGN.md R-TOL: per request the last-token logits sit at the bf16 floor of this 32-layer model
    # (0.90-1.02% measured; tests/test_gpu_accuracy_probe.py: torch bf16 with an fp32 residual 0.94%,
    # stock bf16 1.9%); the 1e-2 bound is asserted over the checked set (test below)
    assert err["logits"] < LOGITS_TOL_PER_REQUEST, err
    s = set(sel.tolist())
    keep = np.array([p for p in range(lay.n) if p not in s and dfn[L - 1, p]])
    assert len(keep) > 0 and np.array_equal(res["kv_last"][r][0][keep], K_asm[L - 1][keep])
    cs = res["cand_scores"][d["cand_off"][r]:d["cand_off"][r + 1]]
    ref = forced["cand_scores"]
    assert np.array_equal(cs, res["logits"][r][lay.cand_idtok])       # the readout itself is exact
    # each candidate score is a logit: within 5x the per-element RMS that rel-L2 <= 1e-2 allows
    assert np.max(np.abs(cs - ref)) <= 5 * TOL * np.sqrt(np.mean(forced["logits"] ** 2))
    print("fullsize ranking: resolvable top-10 positions checked",
          assert_top10_ranking(cs, ref, rms_err(res["logits"][r], forced["logits"])))


def test_cfg3_batch32_rerun_is_deterministic(run):
    """The same batch again (re-assembled). Default mode: the layers < c, which decide Sel, sum their
    partial tiles in K order, so the selection is identical; the later layers' split tiles meet in
    arrival order, so logits may differ in the last bits (bounded here far below the parity tolerance).
    deterministic=1: two runs are bitwise identical, and equal the default run's selection."""
    res, _ = run
    rr, d1, d2 = res["rerun"], res["det1"], res["det2"]
    assert np.array_equal(rr["sel_pos"], res["sel_pos"])
    assert np.array_equal(d1["sel_pos"], res["sel_pos"]) and np.array_equal(d2["sel_pos"], res["sel_pos"])
    drift = rel_l2(rr["logits"], res["logits"])
    same = {k: bool(np.array_equal(d1[k], d2[k])) for k in ("logits", "hidden", "cand_scores")}
    print("rerun: default-mode logits rel-L2 drift", drift, "deterministic bitwise", json.dumps(same))
    # default mode: last-bit differences of the split residual sums, amplified through 31 bf16 layers
    # (measured 2.5e-3 rel-L2 at cfg3 batch 32): bounded at half the parity tolerance
    assert drift < 5e-3
    assert all(same.values()), same
    assert rel_l2(d1["logits"], res["logits"]) < 5e-3


def test_cfg3_batch32_logits_over_checked_set():
    """rel-L2 <= 1e-2 of the last-token logits stacked over the checked requests (R-TOL)."""
    if len(_LOGITS) != len(CHECK_REQS):
        pytest.skip("per-request checks did not all run")
    got = np.concatenate([_LOGITS[r][0] for r in CHECK_REQS])
    ref = np.concatenate([_LOGITS[r][1] for r in CHECK_REQS])
    assert rel_l2(got, ref) < TOL


def test_cfg5_qwen2_8k_batch4_request_matches_oracle():
    """Config 5 shape at full size: Qwen2-7B (28 layers, GQA 7, QKV bias), 8192-token prompts -- the
    R6 key packing limit (positions up to 8191) -- in a batch of 4; the last request is checked end
    to end against the oracle (same bounds as cfg3)."""
    wl = rcgen.CFG5
    res, d = _setup(wl, 4, (3,))
    r = 3
    L = d["shape"].n_layers
    off = res["sel_off"]
    sel = res["sel_pos"][off[r]:off[r + 1]]
    assert sel[-1] == wl.n - 1 == 8191 and list(sel) == sorted(set(sel.tolist()))
    lay, K_asm, dfn, forced, own = _oracle(d, r, sel)
    jac = len(set(own["sel"].tolist()) & set(sel.tolist())) / len(set(own["sel"].tolist()) | set(sel.tolist()))
    Kg = bf16_to_f32(res["kv_last"][r][0])[sel].astype(np.float64)
    err = {"jaccard": jac, "logits": rel_l2(res["logits"][r], forced["logits"]),
           "hidden": rel_l2(res["hidden"][off[r]:off[r + 1]], forced["x_sel"]),
           "K_last": rel_l2(Kg, forced["K"][L - 1][sel])}
    print("fullsize cfg5 parity", json.dumps(err))
    assert jac >= 0.95, err
    assert err["hidden"] < TOL and err["K_last"] < TOL and err["logits"] < LOGITS_TOL_PER_REQUEST, err


@pytest.mark.parametrize("wl", [rcgen.CFG3, rcgen.CFG2], ids=["cfg3", "cfg2"])
def test_batch1_request_matches_oracle(wl):
    """BASELINE configs[1] (cfg2: 2560-token prompts) and configs[2] (cfg3: 4096) at batch 1, the TTFT
    launch configuration (single-tile attention over 160 CTAs at cfg3, 395-625 Sel rows on the
    small-M GEMM schedules, U = 2353-3889 rows in layer 0): request 0 end to end against the oracle,
    same bounds as at batch 32."""
    res, d = _setup(wl, 1, (0,))
    r = 0
    L = d["shape"].n_layers
    off = res["sel_off"]
    sel = res["sel_pos"][off[r]:off[r + 1]]
    lay, K_asm, dfn, forced, own = _oracle(d, r, sel)
    jac = len(set(own["sel"].tolist()) & set(sel.tolist())) / len(set(own["sel"].tolist()) | set(sel.tolist()))
    Kg = bf16_to_f32(res["kv_last"][r][0])[sel].astype(np.float64)
    err = {"jaccard": jac, "logits": rel_l2(res["logits"][r], forced["logits"]),
           "hidden": rel_l2(res["hidden"][off[r]:off[r + 1]], forced["x_sel"]),
           "K_last": rel_l2(Kg, forced["K"][L - 1][sel])}
    print(f"fullsize {wl.name} batch-1 parity", json.dumps(err))
    assert jac >= 0.95, err
    assert err["hidden"] < TOL and err["K_last"] < TOL and err["logits"] < LOGITS_TOL_PER_REQUEST, err


def test_cfg3_batch1_materialized_pools_matches_oracle():
    """BASELINE configs[2] prompt at batch 1 on pools the model materialised itself (R16/R17; item and
    prefix KV from full prefills, prototypes int8 at their canonical positions): the deviation scores
    now measure real context drift. Same bounds as on the seeded pools; the Jaccard is reported."""
    res, d = _setup(rcgen.CFG3, 1, (0,), materialize=True)
    r = 0
    off = res["sel_off"]
    sel = res["sel_pos"][off[r]:off[r + 1]]
    lay, K_asm, dfn, forced, own = _oracle(d, r, sel)
    jac = len(set(own["sel"].tolist()) & set(sel.tolist())) / len(set(own["sel"].tolist()) | set(sel.tolist()))
    Kg = bf16_to_f32(res["kv_last"][r][0])[sel].astype(np.float64)
    err = {"jaccard": jac, "logits": rel_l2(res["logits"][r], forced["logits"]),
           "hidden": rel_l2(res["hidden"][off[r]:off[r + 1]], forced["x_sel"]),
           "K_last": rel_l2(Kg, forced["K"][d["shape"].n_layers - 1][sel])}
    print("fullsize cfg3 batch-1 materialised-pool parity", json.dumps(err))
    assert jac >= 0.95, err
    assert err["hidden"] < TOL and err["K_last"] < TOL and err["logits"] < LOGITS_TOL_PER_REQUEST, err


def test_cfg3_batch1_gradual_filtering_matches_oracle():
    """Gradual filtering (R-GF) in the launch configuration `bench.py --batch 1 --gradual 2 --r-start
    3000` times: Sel at 30 % of each class at the check layer, 22.5 % at layer 2, 15 % from layer 3 on,
    on model-materialised pools. The oracle runs along the GPU's own trajectory (sel_trace): every step
    is nested with the step budgets, each step's members are the oracle's top-k of its own layer-l
    divergence among the previous step (Jaccard >= 0.95: bf16 noise may flip near ties), step 0 matches
    the oracle's one-shot choice at 30 %, and logits, x_L[Sel] and the last layer's K/V at Sel stay
    within the north-star bounds."""
    from oracle.select import select_sel, gradual_ratio_bp
    g, r0 = 2, 3000
    gkw = dict(gradual=g, r_start_rev_bp=r0, r_start_item_bp=r0)
    res, d = _setup(rcgen.CFG3, 1, (0,), materialize=True, gkw=gkw)
    L = d["shape"].n_layers
    off, trace = res["trace_off"], res["sel_trace"]
    steps = [trace[off[i]:off[i + 1]] for i in range(g + 1)]
    sel = res["sel_pos"]
    assert np.array_equal(steps[-1], sel)
    req = d["reqs"][0]
    lay = layout_from_request(req, d["cat"], d["sys"])
    ids = [int(i) for i in req.cand_items]
    item_d = {it: (d["item_kv"][it], d["wl"].prefix_len) for it in ids}
    K, V, _ = assemble(d["shape"], lay, item_d, d["hist"], d["pkv"], gather_from=C)
    forced = selective_prefill(OracleModel(d["shape"], d["W"]), lay, K, V, R_BP, R_BP, check_layer=C,
                               forced_steps=steps, **gkw)
    sub = dataclasses.replace(d["shape"], n_layers=C + 1)
    own0 = selective_prefill(OracleModel(sub, dict(d["W"], layers=d["W"]["layers"][:C + 1])), lay, K[:C + 1],
                             V[:C + 1], r0, r0, check_layer=C)["sel"]

    def jac(a, b):
        a, b = set(int(x) for x in a), set(int(x) for x in b)
        return len(a & b) / len(a | b)
    err = {"jaccard_step0": jac(steps[0], own0), "sizes": [len(x) for x in steps]}
    for i in range(1, g + 1):
        assert set(steps[i].tolist()) <= set(steps[i - 1].tolist())
        r_i = gradual_ratio_bp(r0, R_BP, i, g)
        ref = select_sel(lay.cls, forced["D_steps"][i], r_i, r_i, 0, among=steps[i - 1])
        assert len(ref) == len(steps[i])
        err[f"jaccard_step{i}"] = jac(steps[i], ref)
    Kg = bf16_to_f32(res["kv_last"][0][0])[sel].astype(np.float64)
    err.update(logits=rel_l2(res["logits"][0], forced["logits"]), hidden=rel_l2(res["hidden"], forced["x_sel"]),
               K_last=rel_l2(Kg, forced["K"][L - 1][sel]))
    print("fullsize cfg3 batch-1 gradual parity", json.dumps(err))
    assert all(err[f"jaccard_step{i}"] >= 0.95 for i in range(g + 1)), err
    assert err["hidden"] < TOL and err["K_last"] < TOL and err["logits"] < LOGITS_TOL_PER_REQUEST, err
