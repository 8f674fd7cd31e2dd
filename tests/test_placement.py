"""§8(e) host logic: Alg. 1 placement and Eq. 2 routing (native, through the C-ABI) against
the oracle and the SPEC worked examples (not gpu)."""
import itertools

import numpy as np
import pytest

from oracle import placement as O


def _cl():
    from tests.test_abi import _lib
    _lib()
    from paper_2605_07443_b200 import cluster
    return cluster


def test_two_disjoint_cliques_cut_zero(golden):
    g = golden("partition_spec155.json")
    cl = _cl()
    n = 2 * g["clique_size"]
    hist = [list(range(0, 10))] * 3 + [list(range(10, 20))] * 3
    part, cut, _ = cl.place_items(np.full(n, 8), hist, g["k"], hot_bp=0)
    assert cut == g["expected_cut"]
    assert len(set(part[:10])) == 1 and len(set(part[10:])) == 1 and part[0] != part[10]


def test_hot_replication_matches_oracle_and_coverage():
    cl = _cl()
    rng = np.random.default_rng(0)
    n_items, k = 3000, 4
    pop = 1.0 / np.arange(1, n_items + 1) ** 1.2
    hist = [rng.choice(n_items, size=20, replace=False, p=pop / pop.sum()).tolist() for _ in range(800)]
    tok = rng.integers(16, 128, n_items)
    part, cut, heat = cl.place_items(tok, hist, k, hot_bp=10)
    h = O.compute_heat(hist, n_items)
    assert np.array_equal(heat, h)
    hot, cold = O.split_hot_cold(h, 10)
    assert set(np.nonzero(part == -1)[0].tolist()) == hot and len(hot) == 3        # ceil(0.1% * 3000)
    assert set(np.unique(part[cold]).tolist()) <= set(range(k))                      # every cold item in one shard
    loads = [int(tok[part == p].sum()) for p in range(k)]
    assert max(loads) <= 1.05 * int(tok[cold].sum()) / k + 1                       # balance
    edges = O.cooccurrence(hist, cold)
    assert O.edge_cut({i: int(part[i]) for i in cold}, edges) == cut
    # cut no worse than the best of 100 seeded random balanced partitions
    best_rand = min(O.edge_cut({i: int(p) for i, p in zip(cold, np.random.default_rng(s).permutation(
        np.arange(len(cold)) % k))}, edges) for s in range(100))
    assert cut <= best_rand
    again, cut2, _ = cl.place_items(tok, hist, k, hot_bp=10)
    assert np.array_equal(part, again) and cut2 == cut                               # deterministic


@pytest.mark.parametrize("seed", range(6))
def test_planted_partition_reaches_bruteforce_optimum(seed):
    cl = _cl()
    rng = np.random.default_rng(seed)
    k, per = 2, 5
    n = k * per
    groups = [list(range(g * per, (g + 1) * per)) for g in range(k)]
    hist = []
    for _ in range(40):
        g = groups[rng.integers(k)]
        hist.append(rng.choice(g, size=3, replace=False).tolist())
    for _ in range(3):   # weak cross edges
        hist.append([int(rng.integers(0, per)), int(rng.integers(per, n))])
    tok = np.full(n, 10)
    part, cut, _ = cl.place_items(tok, hist, k, hot_bp=0, balance_eps=0.2)
    edges = O.cooccurrence(hist, range(n))
    _, opt = O.brute_force_partition(list(range(n)), {i: 10 for i in range(n)}, edges, k, 0.2)
    assert cut == opt


def test_k1_and_edgeless():
    cl = _cl()
    part, cut, _ = cl.place_items(np.full(50, 4), [[1, 2, 3]], 1, hot_bp=0)
    assert cut == 0 and set(part.tolist()) == {0}
    part, cut, _ = cl.place_items(np.arange(1, 41), [], 4, hot_bp=0, balance_eps=0.1)
    loads = [int(np.arange(1, 41)[part == p].sum()) for p in range(4)]
    assert cut == 0 and max(loads) <= 1.1 * 820 / 4


def test_route_matches_oracle_bitexact(golden):
    cl = _cl()
    g = golden("affinity_spec341.json")
    assert O.affinity(g["hit"], g["load"], g["alpha"], g["beta"]) == g["expected"]
    e = g["estimate_hit"]
    assert O.estimate_hit([0, 1, 2, 3], {0, 1, 2}) == e["expected"]
    rng = np.random.default_rng(2)
    n_items, k = 400, 8
    resident = (rng.random((k, n_items)) < 0.3).astype(np.uint8)
    reqs = [rng.choice(n_items, size=int(rng.integers(1, 30)), replace=False).tolist() for _ in range(500)]
    tok = rng.integers(500, 5000, len(reqs))
    for alpha, beta in ((0.7, 0.3), (1.0, 0.0), (0.0, 1.0), (0.5, 0.5)):
        got, bl = cl.route(reqs, tok, resident, alpha, beta)
        ref, bref = O.route(reqs, tok, [set(np.nonzero(resident[p])[0].tolist()) for p in range(k)], alpha, beta)
        assert got.tolist() == ref and bl.tolist() == bref
    # scale invariance of the argmax
    a, _ = cl.route(reqs, tok, resident, 0.7, 0.3)
    b, _ = cl.route(reqs, tok, resident, 1.4, 0.6)
    assert np.array_equal(a, b)


def test_route_spec_examples():
    cl = _cl()
    k, n_items = 8, 10
    resident = np.zeros((k, n_items), np.uint8)
    resident[7, :4] = 1
    out, _ = cl.route([[0, 1, 2, 3]], [100], resident, 0.5, 0.5)
    assert out.tolist() == [7]                              # items only on node 7, idle cluster
    resident[:, :] = 1
    out, bl = cl.route([[0]] * 6, [1] * 6, resident[:3], 0.0, 1.0)
    assert out.tolist() == [0, 1, 2, 0, 1, 2]               # LoadOnly on an equal cluster = round robin
    r_hit, _ = cl.route([[0, 1], [5]], [1, 1], resident[:3], 1.0, 0.0)
    assert r_hit.tolist() == [0, 0]                         # ties -> smallest node id


def test_resident_capacity_hot_first():
    cl = _cl()
    part = np.array([-1, 0, 0, 1, 1, 0])
    heat = np.array([9, 5, 1, 3, 2, 4])
    tok = np.array([10, 10, 10, 10, 10, 10])
    res = cl.resident_matrix(part, 2, heat, tok, capacity_tokens=30)
    assert res[0].tolist() == [1, 1, 0, 0, 0, 1] and res[1].tolist() == [1, 0, 0, 1, 1, 0]


def test_percentile_and_capacity_goldens(golden):
    g = golden("percentile_spec511.json")
    v = list(range(1, 101))
    assert [O.percentile_nearest_rank(v, q) for q in (50, 90, 99)] == [g["p50"], g["p90"], g["p99"]]
    c = golden("capacity_spec173.json")
    assert c["items"] * c["tokens_per_item"] * c["bytes_per_token"] / 1e9 == c["expected_gb"]


def test_config4_logical_scale_accounting_invariants():
    """SURVEY §8(e) / R27 accounting (profiles/config4_scale.py) on a reduced catalog: capacity-bounded
    resident sets (hot replicas first), Eq. 2 routing, local / peer / miss rates. The classes partition
    the candidates, no GPU holds more than its capacity, the hot replicas are resident everywhere, the
    resident fraction grows with k, and a catalog that fits entirely leaves no misses."""
    from paper_2605_07443_b200 import cluster
    from rcgen.catalog_scale import gen_catalog_struct, gen_candidate_lists
    cs = gen_catalog_struct(20_000, 200)
    hist = gen_candidate_lists(cs, 1500, 50, start=5_000_000)
    reqs = gen_candidate_lists(cs, 400, 50)
    tok = np.full(cs.n_items, 64, np.int32)
    prev = 0.0
    for k in (1, 2, 4):
        part, cut, heat = cluster.place_items(tok, [h.tolist() for h in hist], k, hot_bp=10)
        res = cluster.resident_matrix(part, k, heat, tok, capacity_tokens=3000 * 64)
        routes, _ = cluster.route([r.tolist() for r in reqs], [4096] * len(reqs), res)
        acc = cluster.hit_accounting(reqs, routes, res, 8 << 20)
        assert abs(acc["local_hit"] + acc["peer_hit"] + acc["miss"] - 1.0) < 1e-12
        assert max(acc["resident_per_gpu"]) <= 3000
        hot = np.nonzero(part == -1)[0]
        assert len(hot) == 20 and res[:, hot].all()             # top 0.1 % replicated on every GPU
        assert acc["resident_frac"] >= prev
        prev = acc["resident_frac"]
        if k == 1:
            assert acc["peer_hit"] == 0.0                         # no peer with one GPU
    # everything fits: no misses, and every candidate is local or one NVLink pull away
    part, cut, heat = cluster.place_items(tok, [h.tolist() for h in hist], 2, hot_bp=10)
    res = cluster.resident_matrix(part, 2, heat, tok)
    routes, _ = cluster.route([r.tolist() for r in reqs], [4096] * len(reqs), res)
    acc = cluster.hit_accounting(reqs, routes, res, 8 << 20)
    assert acc["miss"] == 0.0 and acc["resident_frac"] == 1.0
