"""Alg. 1 placement pieces and the Eq. 2 router, plain and slow (test infrastructure only).

Alg. 1 ("Similarity-aware item placement algorithm with global replicas"):
  Phase 1  h_i = number of historical occurrences of item i
  Phase 2  the top 0.1% items by h (ties -> smaller id) are replicated on every
           instance (replica heat h_i / k)
  Phase 3  the remaining (cold) items are graph nodes
  Phase 4  edge (u, v) weight = number of historical requests in which u and v co-occur
           ("relevance derived from co-occurrence in historical requests")
  Phase 5  k-way partition minimising the edge cut with balanced memory (token weight)
The oracle gives the exact optimum only by brute force on tiny graphs (the product uses a
multilevel heuristic, as the paper uses METIS); placement results are compared on what is
unique (hot set, coverage, balance, cut of separable graphs) and validity.

Eq. 2: Affinity(R, p) = alpha * Hit(R, p) + beta * (1 - Load(p)),
Hit = |I(R) n C(p)| / |I(R)|, Load = backlog tokens / max(1, max backlog),
route = argmax, ties -> smallest p; the chosen node's backlog grows by the
request's tokens (arrival order).
"""
import itertools
import math

import numpy as np


def compute_heat(hist_requests, n_items):
    h = np.zeros(n_items, dtype=np.int64)
    for items in hist_requests:
        for i in items:
            h[int(i)] += 1
    return h


def split_hot_cold(h, hot_bp):
    """hot = ceil(hot_bp/10000 * |I|) items by heat desc, ties -> smaller id."""
    n = len(h)
    k = (int(hot_bp) * n + 9999) // 10000
    order = sorted(range(n), key=lambda i: (-int(h[i]), i))
    hot = set(order[:k])
    return hot, [i for i in range(n) if i not in hot]


def cooccurrence(hist_requests, cold):
    cold = set(cold)
    w = {}
    for items in hist_requests:
        s = sorted({int(i) for i in items if int(i) in cold})
        for a, b in itertools.combinations(s, 2):
            w[(a, b)] = w.get((a, b), 0) + 1
    return w


def edge_cut(part, edges):
    return sum(wt for (a, b), wt in edges.items() if part[a] != part[b])


def brute_force_partition(nodes, weights, edges, k, eps):
    """Exact min-cut k-way assignment of `nodes` with every part's weight <= (1+eps)*total/k."""
    total = sum(weights[v] for v in nodes)
    cap = (1 + eps) * total / k
    best, best_cut = None, math.inf
    for assign in itertools.product(range(k), repeat=len(nodes)):
        if assign[0] != 0:
            continue  # symmetry
        load = [0.0] * k
        for v, p in zip(nodes, assign):
            load[p] += weights[v]
        if max(load) > cap + 1e-9:
            continue
        part = dict(zip(nodes, assign))
        cut = edge_cut(part, edges)
        if cut < best_cut:
            best, best_cut = part, cut
    return best, best_cut


def estimate_hit(items, cached):
    return sum(1 for i in items if int(i) in cached) / len(items)


def affinity(hit, load, alpha, beta):
    return alpha * hit + beta * (1.0 - load)


def route(requests, req_tokens, cached_sets, alpha, beta, backlog=None):
    """requests: list of item lists; cached_sets: list (per instance) of sets C(p)."""
    k = len(cached_sets)
    backlog = list(backlog) if backlog is not None else [0] * k
    out = []
    for items, tok in zip(requests, req_tokens):
        mx = max(max(backlog), 1)
        scores = [affinity(estimate_hit(items, cached_sets[p]), backlog[p] / mx, alpha, beta) for p in range(k)]
        best = max(range(k), key=lambda p: (scores[p], -p))
        out.append(best)
        backlog[best] += int(tok)
    return out, backlog


def percentile_nearest_rank(values, q):
    """Nearest-rank percentile: the ceil(q/100 * n)-th smallest value."""
    v = sorted(values)
    r = max(1, math.ceil(q / 100.0 * len(v)))
    return v[r - 1]
