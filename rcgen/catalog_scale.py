"""Seeded catalog structure and candidate lists at config-4 scale (SURVEY.md §8(d) "Items", §8(e)):
1M logical items in 10,000 latent clusters of 100 items, Zipf(1.2) popularity (
SPEC.md:60), co-selection within a request's cluster with probability 0.9.

Data arrangement only (no arithmetic of the method): no token ids are drawn -- placement (Alg. 1),
routing (Eq. 2) and hit accounting need only which items a request names. Samplers use cumulative
distributions (searchsorted), so a million-item catalog draws in seconds.
"""
from dataclasses import dataclass

import numpy as np


@dataclass
class CatalogStruct:
    n_items: int
    cluster: np.ndarray       # int32 [n_items]
    popularity: np.ndarray    # float64 [n_items], sums to 1
    members: list             # per cluster: item ids (int64 array)
    member_cdf: list          # per cluster: cdf of its members' popularity
    cluster_cdf: np.ndarray   # cdf of cluster popularity
    global_cdf: np.ndarray    # cdf of item popularity


def gen_catalog_struct(n_items: int, n_clusters: int, seed: int = 1, zipf_s: float = 1.2) -> CatalogStruct:
    rng = np.random.Generator(np.random.PCG64(seed))
    size = n_items // n_clusters
    cluster = (rng.permutation(n_items) // size).astype(np.int32)
    cluster = np.minimum(cluster, n_clusters - 1)
    rank = rng.permutation(n_items)
    pop = 1.0 / np.power(rank + 1.0, zipf_s)
    pop /= pop.sum()
    order = np.argsort(cluster, kind="stable")
    bounds = np.searchsorted(cluster[order], np.arange(n_clusters + 1))
    members, mcdf = [], []
    for c in range(n_clusters):
        ids = order[bounds[c]:bounds[c + 1]].astype(np.int64)
        members.append(ids)
        w = np.cumsum(pop[ids])
        mcdf.append(w / w[-1])
    cl_pop = np.bincount(cluster, weights=pop, minlength=n_clusters)
    ccdf = np.cumsum(cl_pop)
    gcdf = np.cumsum(pop)
    return CatalogStruct(n_items, cluster, pop, members, mcdf, ccdf / ccdf[-1], gcdf / gcdf[-1])


def gen_candidate_lists(cs: CatalogStruct, n_req: int, n_cand: int, start: int = 0, co: float = 0.9):
    """Per request (seed 1000 + i): a cluster by cluster popularity; Binomial(n_cand, co) candidates
    from that cluster, popularity-weighted without replacement (Gumbel top-k, equivalent to
    successive weighted draws), the rest from the whole catalog by popularity (rejecting repeats);
    the list randomly permuted. Returns a list of int64 arrays."""
    out = []
    for i in range(start, start + n_req):
        rng = np.random.Generator(np.random.PCG64(1000 + i))
        c = min(int(np.searchsorted(cs.cluster_cdf, rng.random(), side="right")), len(cs.members) - 1)
        ids = cs.members[c]
        n_c = min(int(rng.binomial(n_cand, co)), len(ids))
        keys = np.log(cs.popularity[ids]) + rng.gumbel(size=len(ids))
        chosen = ids[np.argsort(-keys, kind="stable")[:n_c]].tolist()
        taken = set(chosen)
        while len(chosen) < n_cand:
            it = min(int(np.searchsorted(cs.global_cdf, rng.random(), side="right")), cs.n_items - 1)
            if it not in taken:
                taken.add(it)
                chosen.append(it)
        out.append(np.array(chosen, np.int64)[rng.permutation(n_cand)])
    return out
