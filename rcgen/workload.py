"""Seeded synthetic recommendation workload (SURVEY.md §8(d) "Synthetic inputs").

Holds none of the method's arithmetic: it draws token ids, catalog structure, prototype
assignments and request contents. Seeds: catalog 1, prototypes 2,
system prompt 3, request i -> 1000 + i.

Recipe:
  * catalog: n_items items of item_len tokens; token 0 is a unique ID token
    (ids occupy the top n_items vocabulary entries), the rest uniform over the other
    ids. Popularity Zipf(s=1.2) over a random rank permutation (PAPER.md:469,
    SPEC.md:60); each item belongs to one of n_clusters latent clusters.
  * prototypes: n_protos position-aware prototypes. Prototype pi has
    a token and a log2 bucket b = pi mod NB of the history offset; its
    canonical position is P + an offset drawn uniformly inside that bucket.
  * history position t draws a prototype of bucket floor(log2(t+1)) by Zipf(1.1) rank;
    the token is the prototype's token with probability 0.93, else uniform
    (>93% of history tokens have a near-identical prototype).
  * candidates: n_cand items without replacement, each from the request's cluster with
    probability 0.9 else by global popularity, then randomly permuted
    (PAPER.md:59).
  * instruction tail: tail_len uniform tokens (FORCED).
"""
from dataclasses import dataclass
import math

import numpy as np

from .shapes import Workload


@dataclass
class Catalog:
    n_items: int
    item_len: int
    tokens: np.ndarray        # int32 [n_items][item_len]
    cluster: np.ndarray       # int32 [n_items]
    popularity: np.ndarray    # float64 [n_items], sums to 1
    id_base: int

    def idtok(self, item: int) -> int:
        return int(self.tokens[item, 0])


@dataclass
class Protos:
    n: int
    token: np.ndarray         # int32 [n]
    bucket: np.ndarray        # int32 [n]
    canon_pos: np.ndarray     # int32 [n]  absolute canonical position
    n_buckets: int


@dataclass
class Request:
    rid: int
    prefix_len: int
    hist_protos: np.ndarray   # int64 [hist_len]
    hist_tokens: np.ndarray   # int32 [hist_len]
    cand_items: np.ndarray    # int64 [n_cand], slot order
    tail_tokens: np.ndarray   # int32 [tail_len]


def _free_vocab(wl: Workload) -> int:
    return wl.shape.vocab - wl.n_items


def gen_catalog(wl: Workload, seed: int = 1) -> Catalog:
    rng = np.random.Generator(np.random.PCG64(seed))
    V, n = wl.shape.vocab, wl.n_items
    assert V > n, "vocabulary must hold one unique ID token per item"
    id_base = V - n
    toks = rng.integers(0, id_base, size=(n, wl.item_len), dtype=np.int64).astype(np.int32)
    toks[:, 0] = id_base + np.arange(n, dtype=np.int32)
    cluster = rng.integers(0, wl.n_clusters, size=n).astype(np.int32)
    rank = rng.permutation(n)
    pop = 1.0 / np.power(rank + 1.0, 1.2)
    pop /= pop.sum()
    return Catalog(n, wl.item_len, toks, cluster, pop, id_base)


def n_log_buckets(hist_len: int) -> int:
    return max(1, int(math.floor(math.log2(max(hist_len, 1)))) + 1)


def gen_protos(wl: Workload, seed: int = 2) -> Protos:
    rng = np.random.Generator(np.random.PCG64(seed))
    nb = n_log_buckets(wl.hist_len)
    pi = np.arange(wl.n_protos)
    bucket = (pi % nb).astype(np.int32)
    lo = (1 << bucket) - 1
    hi = np.minimum((1 << (bucket + 1)) - 1, wl.hist_len)
    off = lo + np.floor(rng.random(wl.n_protos) * np.maximum(hi - lo, 1)).astype(np.int64)
    token = rng.integers(0, _free_vocab(wl), size=wl.n_protos).astype(np.int32)
    return Protos(wl.n_protos, token, bucket, (wl.prefix_len + off).astype(np.int32), nb)


def gen_system_prompt(wl: Workload, seed: int = 3) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, _free_vocab(wl), size=wl.prefix_len).astype(np.int32)


_ZIPF_CDF = {}


def _zipf_pick(rng, m: int, s: float) -> int:
    """Same draw as rng.choice(m, p=zipf weights): one uniform, searched in the cdf."""
    cdf = _ZIPF_CDF.get((m, s))
    if cdf is None:
        w = 1.0 / np.power(np.arange(1, m + 1, dtype=np.float64), s)
        cdf = np.cumsum(w / w.sum())
        cdf /= cdf[-1]
        _ZIPF_CDF[(m, s)] = cdf
    return int(cdf.searchsorted(rng.random(), side="right"))


def gen_request(wl: Workload, cat: Catalog, protos: Protos, i: int) -> Request:
    rng = np.random.Generator(np.random.PCG64(1000 + i))
    V_free = _free_vocab(wl)
    # history
    hp = np.empty(wl.hist_len, dtype=np.int64)
    ht = np.empty(wl.hist_len, dtype=np.int32)
    nb = protos.n_buckets
    for t in range(wl.hist_len):
        b = int(math.floor(math.log2(t + 1)))
        b = min(b, nb - 1)
        members = np.arange(b, protos.n, nb)
        pi = int(members[_zipf_pick(rng, len(members), 1.1)]) if len(members) else t % protos.n
        hp[t] = pi
        ht[t] = protos.token[pi] if rng.random() < 0.93 else rng.integers(0, V_free)
    # candidates
    cl_pop = np.bincount(cat.cluster, weights=cat.popularity, minlength=wl.n_clusters)
    c = int(rng.choice(wl.n_clusters, p=cl_pop / cl_pop.sum()))
    chosen = []
    taken = np.zeros(cat.n_items, dtype=bool)
    in_c = cat.cluster == c
    for _ in range(wl.n_cand):
        use_c = rng.random() < 0.9 and np.any(in_c & ~taken)
        mask = (in_c if use_c else np.ones(cat.n_items, dtype=bool)) & ~taken
        p = np.where(mask, cat.popularity, 0.0)
        it = int(rng.choice(cat.n_items, p=p / p.sum()))
        taken[it] = True
        chosen.append(it)
    cand = np.array(chosen, dtype=np.int64)[rng.permutation(wl.n_cand)]
    tail = rng.integers(0, V_free, size=wl.tail_len).astype(np.int32)
    return Request(i, wl.prefix_len, hp, ht, cand, tail)


def gen_requests(wl: Workload, cat: Catalog, protos: Protos, n: int, start: int = 0):
    return [gen_request(wl, cat, protos, start + i) for i in range(n)]


def proto_corpus(wl: Workload, protos: Protos, proto_ids, seed: int = 4):
    """Synthetic review-corpus sequences that host the prototypes (a prototype is its
    medoid token at its canonical position in a synthetic review context). Data arrangement only:
    prototype pi is placed at history offset canon_pos[pi] - P of corpus sequence j, where j counts
    the earlier listed prototypes with the same offset; every other slot holds a seeded uniform
    token. Returns (tokens int32 [S][H], seq int32 [len(proto_ids)], offset int32 [len(proto_ids)]),
    H = 1 + the largest offset, S = the largest multiplicity of an offset."""
    ids = np.asarray(proto_ids, dtype=np.int64)
    off = (protos.canon_pos[ids] - wl.prefix_len).astype(np.int64)
    H = int(off.max()) + 1 if len(ids) else 1
    seq = np.zeros(len(ids), dtype=np.int32)
    used = {}
    for k, o in enumerate(off.tolist()):
        seq[k] = used.get(o, 0)
        used[o] = seq[k] + 1
    S = max(used.values()) if used else 1
    rng = np.random.Generator(np.random.PCG64(seed))
    toks = rng.integers(0, _free_vocab(wl), size=(S, H)).astype(np.int32)
    toks[seq, off] = protos.token[ids]
    return toks, seq, off.astype(np.int32)


def gen_mixed_requests(mix, cat: Catalog, protos: Protos, n: int, start: int = 0):
    """A mixed-length batch: n requests whose length classes follow the mix
    fractions (largest remainder, classes interleaved in a seeded order); request i is generated by its
    class's workload with seed 1000 + start + i over one shared catalog and prototype library.
    Returns (workload per request, requests)."""
    counts = [int(f * n) for _, f in mix]
    rem = sorted(range(len(mix)), key=lambda j: -(mix[j][1] * n - counts[j]))
    for j in rem[:n - sum(counts)]:
        counts[j] += 1
    cls = np.concatenate([np.full(c, j) for j, c in enumerate(counts)])
    cls = cls[np.random.Generator(np.random.PCG64(5)).permutation(n)]
    wls = [mix[int(j)][0] for j in cls]
    return wls, [gen_request(w, cat, protos, start + i) for i, w in enumerate(wls)]
