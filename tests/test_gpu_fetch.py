"""The NVLink exchange step of §8(e) on one GPU: two processes, each with its own librc context,
share item blocks through CUDA IPC exactly as the N > 1 bench does (rc_pool_export ->
rc_peer_attach -> rc_pool_list / rc_peer_directory -> rc_fetch_remote). The owner (rank 0) holds
every candidate item; the fetcher (rank 1) holds none, pulls them into a small LRU remote region --
small enough that later requests evict earlier blocks -- and the stitched KV of every request must
equal O-ASM bit for bit. Also the C-ABI's input validation of
the ADVICE round-1 findings (canonical-position range, last position recomputed)."""
import os
import socket

import numpy as np
import pytest
import torch

import rcgen

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2605_07443_b200 import cluster, _lib as R
    from paper_2605_07443_b200.api import RcContext
    from tests.helpers import make_case, oracle_pools, layouts
    from tests import gpu_helpers as G
    from oracle.assemble import assemble

    def ago(obj):
        lst = [None] * 2
        dist.all_gather_object(lst, obj)
        return lst

    wl = rcgen.MINI_L
    case = make_case(wl, n_req=4)
    pools = oracle_pools(case)
    shape = case["shape"]
    Wd = G.weights_to(case["W"])
    items = pools["item_ids"]
    per_req = [sorted({int(i) for i in r.cand_items}) for r in case["reqs"]]
    region = max(len(p) for p in per_req) * wl.item_len + wl.item_len  # one request's items + one spare block
    if rank == 0:
        ctx = RcContext(shape, Wd, item_rows=len(items) * wl.item_len, hist_rows=len(pools["proto_ids"]),
                        prefix_rows=wl.prefix_len, arena_rows=wl.n, max_seq_len=max(wl.n, 256), max_batch_tokens=wl.n)
        G.register_pools(ctx, case, pools)
    else:
        ctx = RcContext(shape, Wd, item_rows=region, remote_rows=region, hist_rows=len(pools["proto_ids"]),
                        prefix_rows=wl.prefix_len, arena_rows=wl.n, max_seq_len=max(wl.n, 256), max_batch_tokens=wl.n)
        G.register_pools(ctx, case, pools, items=[])
    handle, rows = ctx.pool_export()
    peers = [x for x in ago((rank, 0, handle, rows)) if x[0] != rank]
    ctx.peer_attach([p[0] for p in peers], [p[1] for p in peers], [p[2] for p in peers], [p[3] for p in peers])
    directory = cluster.share_directory(ctx, rank, ago)
    result = {}
    if rank == 1:
        assert set(directory) == set(items) and all(o == 0 for o, _ in directory.values())
        bad = []
        try:  # an id missing from the owner's directory: NOTFOUND, no partial effect
            ctx.fetch_remote([items[0], 10 ** 9], [0, 0])
        except R.RcError as e:
            bad.append(e.code)
        assert bad == [R.RC_E_NOTFOUND] and not ctx.pool_contains(R.RC_POOL_ITEM_BF16, [items[0]]).any()
        stream = torch.cuda.current_stream()
        checked, evicted = 0, 0
        prev = set()
        for r, lay in enumerate(layouts(case)):
            need = per_req[r]
            resident_before = ctx.pool_contains(R.RC_POOL_ITEM_BF16, need)
            ctx.fetch_remote(need + need[:3], [0] * (len(need) + 3), stream=stream)  # repeated ids are skipped
            assert ctx.pool_contains(R.RC_POOL_ITEM_BF16, need).all()
            gone = sorted(prev - set(need))
            if gone:   # blocks of the previous request that the LRU recycled for this one
                evicted += int((~ctx.pool_contains(R.RC_POOL_ITEM_BF16, gone)).sum())
            prev = set(need)
            gl = G.gpu_layouts(ctx, case, [case["reqs"][r]])
            seqs = ctx.assemble(gl, prefix_id=G.PREFIX_ID, gather_from=1, stream=stream)
            torch.cuda.synchronize()
            K, V, dfn = assemble(shape, lay, pools["items"], pools["hist"], pools["prefix"], 1)
            for l in range(1, shape.n_layers):
                k, v = ctx.read_kv(seqs[0], l, lay.n)
                m = dfn[l]
                assert np.array_equal(G.bits(k)[m], K[l][m]) and np.array_equal(G.bits(v)[m], V[l][m]), (r, l)
                checked += int(m.sum())
            ctx.release(seqs)
            assert resident_before.sum() <= len(need)
        result = {"checked": checked, "evicted": evicted}
    dist.barrier()   # the owner keeps its pool mapped until the fetcher is done
    ctx.close()
    if rank == 1:
        import json
        with open(out_path, "w") as f:
            json.dump(result, f)
    dist.destroy_process_group()


def test_fetch_remote_two_processes_bitexact(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07443_b200.build import build
    build()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    out = str(tmp_path / "fetch.json")
    procs = [ctx.Process(target=_worker, args=(r, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    import json
    res = json.load(open(out))
    assert res["checked"] > 0
    assert res["evicted"] > 0      # the LRU region really recycled blocks between requests


def _small_ctx():
    from tests.helpers import make_case, oracle_pools
    from tests import gpu_helpers as G
    wl = rcgen.MINI_L
    case = make_case(wl)
    pools = oracle_pools(case)
    ctx, _ = G.make_ctx(case, pools, wl.n, extra_item_rows=wl.item_len)
    return wl, case, pools, ctx


def test_register_rejects_canonical_positions_outside_the_prompt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07443_b200 import _lib as R
    wl, case, pools, ctx = _small_ctx()
    s = case["shape"]
    kv = torch.zeros((wl.item_len, s.n_layers, 2, s.n_kv_heads, s.head_dim), dtype=torch.bfloat16, device="cuda")
    max_seq = max(wl.n, 256)
    for canon in (-1, max_seq - wl.item_len + 1):
        with pytest.raises(R.RcError) as e:
            ctx.pool_register_blocks(R.RC_POOL_ITEM_BF16, [777777], [wl.item_len], [canon], kv)
        assert e.value.code == R.RC_E_INVALID
    ctx.pool_register_blocks(R.RC_POOL_ITEM_BF16, [777777], [wl.item_len], [max_seq - wl.item_len], kv)  # in range
    ctx.close()


def test_last_position_must_be_recomputed():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07443_b200 import _lib as R
    from tests import gpu_helpers as G
    wl, case, pools, ctx = _small_ctx()
    r = case["reqs"][0]
    # no instruction tail: the prompt ends inside the last item
    lay = ctx.decompose_prompt(case["sys"], r.hist_protos, r.hist_tokens, r.cand_items,
                               [case["cat"].tokens[int(i)] for i in r.cand_items], [])
    seqs = ctx.assemble([lay], prefix_id=G.PREFIX_ID, gather_from=1)
    with pytest.raises(R.RcError) as e:
        ctx.selective_prefill(seqs, 1500, 1500, check_layer=1, n_cand=len(lay["cand_idtok"]))
    assert e.value.code == R.RC_E_INVALID
    out = ctx.selective_prefill(seqs, 1500, 1500, check_layer=1, window=4, n_cand=len(lay["cand_idtok"]))
    torch.cuda.synchronize()
    n = len(lay["tokens"])
    assert int(out["sel_pos"][-1]) == n - 1          # a window makes the last position recomputed
    ctx.release(seqs)
    ctx.close()
