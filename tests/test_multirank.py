"""World-size-2 gloo run of the §8(e) host orchestration (placement, routing, directory
exchange, fetch planning) exactly as bench.py --gpus N composes it (not gpu)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import rcgen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_07443_b200 import cluster
    wl = rcgen.CFG2
    cat, protos = rcgen.gen_catalog(wl), rcgen.gen_protos(wl)
    hist = [r.cand_items.tolist() for r in rcgen.gen_requests(wl, cat, protos, 300, start=5_000_000)]
    part, cut, heat = cluster.place_items(np.full(wl.n_items, wl.item_len), hist, world, hot_bp=10)
    res = cluster.resident_matrix(part, world)
    reqs = rcgen.gen_requests(wl, cat, protos, 40)
    cands = [r.cand_items.tolist() for r in reqs]
    routes, backlog = cluster.route(cands, [wl.n] * len(cands), res)
    local = np.nonzero(res[rank])[0]
    rows = local * wl.item_len                       # this rank's pool rows (contiguous registration)

    def ago(obj):
        lst = [None] * world
        dist.all_gather_object(lst, obj)
        return lst
    directory = cluster.exchange_directory(local, rows, rank, ago)
    mine = [cands[i] for i in range(len(cands)) if routes[i] == rank]
    plan = cluster.plan_fetch(mine, res[rank], directory, rank)
    everything = ago({"part": part.tolist(), "routes": routes.tolist(), "plan": plan, "n_mine": len(mine),
                      "hit": float(np.mean([res[rank][c].mean() for c in mine])) if mine else 1.0})
    if rank == 0:
        out_q.put({"all": everything, "cut": cut, "res": res.tolist(), "n_items": wl.n_items, "dir_size": len(directory)})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_orchestration():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a, b = out["all"]
    assert a["part"] == b["part"] and a["routes"] == b["routes"]        # deterministic on every rank
    assert a["n_mine"] + b["n_mine"] == 40 and a["n_mine"] > 0 and b["n_mine"] > 0
    res = np.array(out["res"])
    assert out["dir_size"] == out["n_items"]                            # every item has an owner
    for r, info in enumerate((a, b)):
        for item, owner, row in info["plan"]:
            assert owner != r and res[owner][item] == 1 and not res[r][item]
            assert row == item * 64                                         # the owner's published pool row
    assert a["hit"] > 0.5 and b["hit"] > 0.5                            # affinity routing keeps most items local
