"""SURVEY §8(d) config 4 / §8(e) at its logical scale, on the host (no GPU needed): 1M items x 64
tokens in 10,000 clusters of 100 (Zipf 1.2 popularity, co-selection 0.9), Alg. 1 placement
(rc_place_items) from a 50K-request historical trace, capacity-bounded HBM item
pools per GPU (hot replicas first, then the shard by heat; reading R27), Eq. 2 routing (PAPER.md:539,
rc_route) of 10K requests, and the resulting local / peer / miss rates at k = 1, 2, 4, 8 GPUs.

  python profiles/config4_scale.py [--items N] [--hist H] [--reqs R] > profiles/r02_config4_scale.txt
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_07443_b200 import cluster  # noqa: E402
from rcgen.catalog_scale import gen_catalog_struct, gen_candidate_lists  # noqa: E402
import rcgen  # noqa: E402

# HBM budget per B200 for the item pool at the Llama-3-8B shape (DESIGN.md §5 layout at cfg3 batch 32):
# 180 GB - weights 16.1 GB - packed q|k|v and gate|up 9.4 GB - history pool 6.6 GB - stitched arena
# 17.2 GB - workspace 11 GB - headroom 2 GB = 117.7 GB; one 64-token item = 64 x 131,072 B = 8 MiB
ITEM_BYTES = 64 * rcgen.LLAMA3_8B.kv_bytes_per_token_bf16
BUDGET = 180e9 - 16.1e9 - 9.4e9 - 6.6e9 - 17.2e9 - 11e9 - 2e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=1_000_000)
    ap.add_argument("--clusters", type=int, default=0)
    ap.add_argument("--hist", type=int, default=50_000)
    ap.add_argument("--reqs", type=int, default=10_000)
    ap.add_argument("--cand", type=int, default=50)
    ap.add_argument("--capacity", type=int, default=0, help="items per GPU (default: HBM budget / 8 MiB)")
    a = ap.parse_args()
    n_cl = a.clusters or a.items // 100
    cap = a.capacity or int(BUDGET // ITEM_BYTES)
    t0 = time.time()
    cs = gen_catalog_struct(a.items, n_cl)
    hist = gen_candidate_lists(cs, a.hist, a.cand, start=5_000_000)
    reqs = gen_candidate_lists(cs, a.reqs, a.cand, start=0)
    print(f"# config 4 at logical scale: {a.items} items x 64 tokens ({a.items * ITEM_BYTES / 1e12:.2f} TB bf16 KV), "
          f"{n_cl} clusters, trace {a.hist} requests, {a.reqs} routed requests x {a.cand} candidates; "
          f"HBM item capacity {cap} items/GPU ({cap * ITEM_BYTES / 1e9:.1f} GB); generated in {time.time() - t0:.1f} s")
    tok = np.full(a.items, 64, np.int32)
    rows = []
    for k in (1, 2, 4, 8):
        t = time.time()
        part, cut, heat = cluster.place_items(tok, [h.tolist() for h in hist], k, hot_bp=10)
        t_place = time.time() - t
        res = cluster.resident_matrix(part, k, heat, tok, capacity_tokens=cap * 64)
        routes, backlog = cluster.route([r.tolist() for r in reqs], [4096] * len(reqs), res)
        acc = cluster.hit_accounting(reqs, routes, res, ITEM_BYTES)
        row = {"k": k, "placement_s": round(t_place, 1), "edge_cut": cut, "hot_replicated": int((part == -1).sum()),
               **{key: (round(v, 4) if isinstance(v, float) else v) for key, v in acc.items()}}
        rows.append(row)
        print(json.dumps(row))
    print()
    print(f"{'k':>2} {'resident':>9} {'local':>7} {'peer':>7} {'miss':>7} {'fetch MB/req':>13} {'imbalance':>9}")
    for r in rows:
        print(f"{r['k']:>2} {r['resident_frac']:9.4f} {r['local_hit']:7.3f} {r['peer_hit']:7.3f} {r['miss']:7.3f} "
              f"{r['fetch_mb_per_request']:13.1f} {r['route_imbalance']:9.3f}")


if __name__ == "__main__":
    main()
