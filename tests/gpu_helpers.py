"""GPU-side test setup: the same generator outputs the oracle consumes, registered in librc."""
import numpy as np
import torch

import rcgen
from paper_2605_07443_b200.api import RcContext
from paper_2605_07443_b200 import _lib as R

PREFIX_ID = 1


def weights_to(W, device="cuda"):
    return {"embed": W["embed"].to(device), "norm": W["norm"].to(device), "lm_head": W["lm_head"].to(device),
            "layers": [{k: v.to(device).contiguous() for k, v in lw.items()} for lw in W["layers"]]}


def make_ctx(case, pools, n_req_tokens, arena_rows=None, remote_rows=0, Wd=None, extra_item_rows=0, items=None):
    wl, shape = case["wl"], case["shape"]
    Wd = Wd if Wd is not None else weights_to(case["W"])
    n_items = len(pools["item_ids"])
    ctx = RcContext(shape, Wd, item_rows=n_items * wl.item_len + remote_rows + extra_item_rows,
                    hist_rows=max(len(pools["proto_ids"]), 1), prefix_rows=max(wl.prefix_len, 1),
                    arena_rows=arena_rows or n_req_tokens, max_seq_len=max(wl.n, 256),
                    max_batch_tokens=n_req_tokens, remote_rows=remote_rows)
    register_pools(ctx, case, pools, items=items)
    return ctx, Wd


def register_pools(ctx, case, pools, items=None):
    wl, shape = case["wl"], case["shape"]
    L, Hk, dh = shape.n_layers, shape.n_kv_heads, shape.head_dim
    ids = pools["item_ids"] if items is None else items
    sel = [pools["item_ids"].index(i) for i in ids]
    if len(ids):
        kv = pools["item_kv"][sel].reshape(len(ids) * wl.item_len, L, 2, Hk, dh).contiguous().cuda()
        ctx.pool_register_blocks(R.RC_POOL_ITEM_BF16, ids, [wl.item_len] * len(ids), [wl.prefix_len] * len(ids), kv)
    pids = pools["proto_ids"]
    if len(pids):
        q = pools["hist_q"].contiguous().cuda()
        s = pools["hist_s"].contiguous().cuda()
        ctx.pool_register_blocks(R.RC_POOL_HIST_INT8, pids, [1] * len(pids),
                                 [int(case["protos"].canon_pos[p]) for p in pids], q, s)
    if wl.prefix_len:
        ctx.pool_register_blocks(R.RC_POOL_PREFIX_BF16, [PREFIX_ID], [wl.prefix_len], [0],
                                 pools["prefix"].contiguous().cuda())
    torch.cuda.synchronize()


def gpu_layouts(ctx, case, reqs=None):
    cat, sys_tok = case["cat"], case["sys"]
    reqs = reqs if reqs is not None else case["reqs"]
    return [ctx.decompose_prompt(sys_tok, r.hist_protos, r.hist_tokens, r.cand_items,
                                 [cat.tokens[int(i)] for i in r.cand_items], r.tail_tokens) for r in reqs]


def bits(t):
    return t.cpu().numpy().view(np.uint16)


def make_ctx_materialized(case, n_req_tokens, Wd=None, remote_rows=0):
    """Context whose pools are materialised by librc's dense path (SURVEY R16/R17, §8(d) "Pool
    contents"): prefix = full prefill of the system prompt, items = [system prompt; item] at P..,
    prototypes = their token at the canonical position of a review-corpus sequence, int8 (R15).
    Returns (ctx, pools) with pools in the oracle_pools format holding the registered bytes."""
    from paper_2605_07443_b200 import materialize as MZ
    wl, shape = case["wl"], case["shape"]
    Wd = Wd if Wd is not None else weights_to(case["W"])
    reqs = case["reqs"]
    items = sorted({int(i) for r in reqs for i in r.cand_items})
    protos = sorted({int(p) for r in reqs for p in r.hist_protos})
    corpus, seq_of, off_of = rcgen.proto_corpus(wl, case["protos"], protos)
    arena = max(n_req_tokens, 4 * (wl.prefix_len + max(corpus.shape[1], wl.item_len)))
    ctx = RcContext(shape, Wd, item_rows=len(items) * wl.item_len + remote_rows, hist_rows=max(len(protos), 1),
                    prefix_rows=max(wl.prefix_len, 1), arena_rows=arena, max_seq_len=max(wl.n, 256),
                    max_batch_tokens=arena, remote_rows=remote_rows)
    sys_tok = case["sys"]
    pkv = MZ.register_prefix(ctx, sys_tok, PREFIX_ID)
    kept = MZ.register_items(ctx, sys_tok, PREFIX_ID, items, [case["cat"].tokens[i] for i in items], keep=True)
    canon = [int(case["protos"].canon_pos[p]) for p in protos]
    q, s = MZ.register_protos(ctx, sys_tok, PREFIX_ID, protos, canon, corpus, seq_of, off_of)
    torch.cuda.synchronize()
    ikv = torch.stack([kept[i] for i in items]).cpu()
    hq, hs = q.cpu(), s.cpu()
    pools = dict(items={it: (ikv[j], wl.prefix_len) for j, it in enumerate(items)},
                 hist={pi: (hq[j].numpy(), hs[j].numpy(), canon[j]) for j, pi in enumerate(protos)},
                 prefix=pkv.cpu(), item_ids=items, proto_ids=protos, item_kv=ikv, hist_q=hq, hist_s=hs,
                 corpus=(corpus, seq_of, off_of))
    return ctx, pools, Wd
