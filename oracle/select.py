"""Eq. 3 importance score and heavy-hitter selection (test infrastructure only).

Eq. 3:
    S_i = (1 - lambda) ||A_i||_1 + lambda * sum_{M in {K,V}} ||M_i^new - M_i^cached||_1
Heavy hitters: the top tokens by S, plus the local sliding window; the
rest keep their cached state. Readings:
  R5  per-class budget k = ceil(r * count), r in basis points (r_rev for history tokens,
      r_item for item tokens)
  R6  order: larger score first, equal score -> lower position
  R7  window = the last w positions of the prompt; they are recomputed (added to Sel) and
      removed from the classes before the budgets are taken (reading D3)
  FORCED tokens (instruction tail, misses) are always in Sel.
"""
import numpy as np

from .layout import PREFIX, FORCED, HIST, ITEM, budget


def importance_scores(A, K_new, K_cached, V_new, V_cached, lam):
    """Eq. 3 in fp64 with plain L1 norms. A: [n]; the four matrices: [n][m]."""
    A = np.asarray(A, dtype=np.float64)
    mats = [np.asarray(M, dtype=np.float64) for M in (K_new, K_cached, V_new, V_cached)]
    n = A.shape[0]
    if any(M.ndim != 2 or M.shape[0] != n for M in mats) or mats[0].shape != mats[1].shape \
            or mats[2].shape != mats[3].shape:
        raise ValueError("DimensionMismatch")
    div = np.abs(mats[0] - mats[1]).sum(axis=1) + np.abs(mats[2] - mats[3]).sum(axis=1)
    return (1.0 - lam) * A + lam * div


MASS_FRAC_BITS = 24  # fixed point of the attention mass (NEXT-1 reading R2-FX)


def attention_mass_fixed(q, qpos, K, n_heads, n_kv_heads, head_dim):
    """||A_p||_1 of Eq. 3 as the column mass of the check-layer softmax (reading R2):
    A[p] = sum over heads h and queries q with pos_q >= p of P[h, q, p], P the causal softmax of
    q_h . K_{g(h)} / sqrt(d_h) over all keys at positions <= pos_q, g(h) = floor(h / (H / H_kv)).
    Fixed point (reading R2-FX): every term enters as floor(P * 2^24), summed exactly as integers.
    q: [T][H][dh] fp64 (fresh queries at layer c), qpos: [T], K: [n][Hk][dh] fp64 keys by position.
    Returns uint64 [n]."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    qpos = np.asarray(qpos, dtype=np.int64)
    n = K.shape[0]
    G = n_heads // n_kv_heads
    scale = 1.0 / np.sqrt(head_dim)
    kpos = np.arange(n)
    A = np.zeros(n, dtype=np.uint64)
    for t0 in range(0, len(qpos), 512):
        t1 = min(len(qpos), t0 + 512)
        mask = kpos[None, :] > qpos[t0:t1, None]
        for h in range(n_heads):
            sc = (q[t0:t1, h] @ K[:, h // G].T) * scale
            sc = np.where(mask, -np.inf, sc)
            sc = sc - sc.max(axis=1, keepdims=True)
            p = np.exp(sc)
            p /= p.sum(axis=1, keepdims=True)
            A += np.floor(p * float(1 << MASS_FRAC_BITS)).astype(np.uint64).sum(axis=0)
    return A


def combine_fixed(A_fx, D_fx, lam):
    """Eq. 3 on the fixed-point terms: S = rint((1 - lam) * A + lam * D) in IEEE fp64, round half to
    even (reading R2-FX: A and D both carry 24 fraction bits, so S does too). lam is the fp32
    parameter of the boundary (rc_prefill_params.lambda) widened to fp64. uint64 [n]."""
    A = np.asarray(A_fx, dtype=np.uint64).astype(np.float64)
    D = np.asarray(D_fx, dtype=np.uint64).astype(np.float64)
    lam = float(np.float32(lam))
    return np.rint((1.0 - lam) * A + lam * D).astype(np.uint64)


def topk_order(scores, idx):
    """Indices `idx` sorted by (score desc, index asc) -- the R6 order."""
    return sorted((int(i) for i in idx), key=lambda i: (-scores[i], i))


def select_heavy_hitters(scores, r_bp, window, n):
    """SPEC.md:423-431 semantics over one class: top ceil(r n) by score (ties -> lower index),
    unioned with the trailing `window` indices."""
    k = budget(r_bp, n)
    top = topk_order(list(scores), range(n))[:k]
    win = range(max(0, n - window), n)
    return sorted(set(top) | set(win))


def select_sel(cls, D, r_rev_bp, r_item_bp, window=0, among=None):
    """Sel for one request: FORCED u window u topk(HIST) u topk(ITEM), sorted by position.
    D: per-position integer deviation (only HIST/ITEM entries are read).
    among (gradual filtering, reading R-GF): the previous step's Sel; the top-k of a class is taken
    over its positions in `among` only, with the budget still ceil(r * |class|) over the whole class."""
    n = len(cls)
    win = set(range(max(0, n - window), n)) if window > 0 else set()
    win = {p for p in win if cls[p] != PREFIX}
    sel = {p for p in range(n) if cls[p] == FORCED} | win
    D = [int(d) for d in D]
    pool = None if among is None else {int(p) for p in among}
    for c, r_bp in ((HIST, r_rev_bp), (ITEM, r_item_bp)):
        members = [p for p in range(n) if cls[p] == c and p not in win]
        k = budget(r_bp, len(members))
        cand = members if pool is None else [p for p in members if p in pool]
        assert k <= len(cand), "a gradual step cannot grow a class"
        sel |= set(topk_order(D, cand)[:k])
    return np.array(sorted(sel), dtype=np.int32)


def gradual_ratio_bp(r_start_bp, r_bp, i, g):
    """Reading R-GF: the ratio of gradual step i in [0, g], linear from r_start (check layer c) to r
    (layer c + g), truncated: r_start - floor((r_start - r) * i / g)."""
    if g == 0:
        return int(r_bp)
    return int(r_start_bp) - (int(r_start_bp) - int(r_bp)) * int(i) // int(g)


def sel_count(cls, r_rev_bp, r_item_bp, window=0):
    """|Sel| is fixed by the layout (no data dependence): used to size outputs."""
    n = len(cls)
    win = {p for p in range(max(0, n - window), n) if cls[p] != PREFIX} if window > 0 else set()
    forced = sum(1 for p in range(n) if cls[p] == FORCED and p not in win)
    nh = sum(1 for p in range(n) if cls[p] == HIST and p not in win)
    ni = sum(1 for p in range(n) if cls[p] == ITEM and p not in win)
    return forced + len(win) + budget(r_rev_bp, nh) + budget(r_item_bp, ni)
