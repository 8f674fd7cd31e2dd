"""Multi-GPU orchestration around librc: Alg. 1 placement and Eq. 2 routing
through the C-ABI (rc_place_items / rc_route, native C++), the item directory exchanged with
torch.distributed, and fetch planning for items resident on a peer (pulled over NVLink by
rc_fetch_remote). Host logic only; marshalling around librc.
"""
import ctypes as C

import numpy as np

from . import _lib as R
from ._lib import check, lib, np_ptr


def _csr(lists):
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in lists])
    flat = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int32) for x in lists]) if len(lists)
                                else np.zeros(0, np.int32), np.int32)
    return off, flat


def place_items(item_tokens, hist_requests, k, hot_bp=10, balance_eps=0.05, passes=10):
    """Alg. 1 -> (part [n_items] in -1..k-1 (-1 = replicated hot item), edge cut, heat)."""
    tok = np.ascontiguousarray(item_tokens, np.int32)
    off, flat = _csr(hist_requests)
    part = np.zeros(len(tok), np.int32)
    heat = np.zeros(len(tok), np.int64)
    cut = C.c_int64()
    check(lib().rc_place_items(len(tok), np_ptr(tok, C.c_int32), len(hist_requests), np_ptr(off, C.c_int64),
                               np_ptr(flat, C.c_int32), k, hot_bp, balance_eps, passes, np_ptr(part, C.c_int32),
                               C.byref(cut), np_ptr(heat, C.c_int64)))
    return part, int(cut.value), heat


def resident_matrix(part, k, heat=None, item_tokens=None, capacity_tokens=None):
    """C(p) per instance: its shard plus the replicated hot items. With a capacity (tokens per
    GPU), hot replicas first, then the shard's items by heat."""
    n = len(part)
    res = np.zeros((k, n), np.uint8)
    for p in range(k):
        mine = np.nonzero((part == p) | (part == -1))[0]
        if capacity_tokens is not None:
            pri = sorted(mine.tolist(), key=lambda i: (part[i] != -1, -(heat[i] if heat is not None else 0), i))
            used, keep = 0, []
            for i in pri:
                if used + item_tokens[i] > capacity_tokens:
                    continue
                used += item_tokens[i]
                keep.append(i)
            mine = np.array(keep, np.int64)
        res[p, mine] = 1
    return res


def route(requests, req_tokens, resident, alpha=0.7, beta=0.3, backlog=None):
    """Eq. 2 routing of requests (lists of candidate item ids) in arrival order."""
    k, n_items = resident.shape
    off, flat = _csr(requests)
    tok = np.ascontiguousarray(req_tokens, np.int64)
    bl = np.ascontiguousarray(backlog if backlog is not None else np.zeros(k), np.int64).copy()
    out = np.zeros(len(requests), np.int32)
    res = np.ascontiguousarray(resident, np.uint8)
    check(lib().rc_route(len(requests), np_ptr(off, C.c_int64), np_ptr(flat, C.c_int32), np_ptr(tok, C.c_int64), k,
                         n_items, np_ptr(res, C.c_uint8), alpha, beta, np_ptr(bl, C.c_int64), np_ptr(out, C.c_int32)))
    return out, bl


def exchange_directory(local_items, local_rows, rank, all_gather_object):
    """Global item -> (owner rank, pool row) directory; every rank contributes its resident items
    (hot replicas included: the first owner by rank order is used)."""
    mine = {int(i): int(r) for i, r in zip(local_items, local_rows)}
    gathered = all_gather_object({"rank": rank, "items": mine})  # callable: obj -> list over ranks
    directory = {}
    for g in sorted(gathered, key=lambda x: x["rank"]):
        for it, row in g["items"].items():
            directory.setdefault(it, (g["rank"], row))
    return directory


def share_directory(ctx, rank, all_gather_object):
    """Publish this rank's pool directory (rc_pool_list) and load every other rank's into the
    library (rc_peer_directory), so rc_fetch_remote resolves rows from (item id, owner) alone.
    Returns the global item -> (owner rank, pool row) map (first owner by rank order)."""
    ids, rows, nt, cp = ctx.pool_list()
    gathered = all_gather_object({"rank": rank, "ids": ids, "rows": rows, "nt": nt, "cp": cp})
    for g in gathered:
        if g["rank"] != rank:
            ctx.peer_directory(g["rank"], g["ids"], g["rows"], g["nt"], g["cp"])
    return exchange_directory(ids, rows, rank, lambda _: [{"rank": g["rank"], "items": dict(
        zip(g["ids"].tolist(), g["rows"].tolist()))} for g in gathered])


def plan_fetch(batch_candidates, resident_local, directory, rank):
    """Items of the batch not resident on this rank -> list of (item, owner, row). Raises if an
    item has no owner (it would become FORCED under RC_MISS_RECOMPUTE instead)."""
    need = sorted({int(i) for cands in batch_candidates for i in cands if not resident_local[int(i)]})
    plan = []
    for it in need:
        if it not in directory:
            continue
        owner, row = directory[it]
        if owner == rank:
            continue
        plan.append((it, owner, row))
    return plan


def hit_accounting(requests, routes, resident, item_bytes):
    """Per-request candidate classes under a placement: local (resident on the
    routed GPU), peer (resident on another GPU: one NVLink pull), miss (resident nowhere: recomputed
    as FORCED, or pulled from the host tier). Returns rates over all candidates, the fetch bytes per
    request and the resident fraction of the catalog."""
    k, n_items = resident.shape
    anywhere = resident.any(axis=0)
    loc = peer = miss = tot = 0
    for items, g in zip(requests, routes):
        items = np.asarray(items, np.int64)
        l = resident[g][items].astype(bool)
        a = anywhere[items]
        loc += int(l.sum())
        peer += int((a & ~l).sum())
        miss += int((~a).sum())
        tot += len(items)
    per = [int((np.asarray(routes) == p).sum()) for p in range(k)]
    return {"local_hit": loc / tot, "peer_hit": peer / tot, "miss": miss / tot,
            "resident_frac": float(anywhere.mean()), "resident_per_gpu": [int(x) for x in resident.sum(axis=1)],
            "fetch_mb_per_request": peer / len(requests) * item_bytes / 2 ** 20,
            "routed": per, "route_imbalance": max(per) / max(1.0, np.mean(per))}
