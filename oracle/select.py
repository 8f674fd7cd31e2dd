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


def select_sel(cls, D, r_rev_bp, r_item_bp, window=0):
    """Sel for one request: FORCED u window u topk(HIST) u topk(ITEM), sorted by position.
    D: per-position integer deviation (only HIST/ITEM entries are read)."""
    n = len(cls)
    win = set(range(max(0, n - window), n)) if window > 0 else set()
    win = {p for p in win if cls[p] != PREFIX}
    sel = {p for p in range(n) if cls[p] == FORCED} | win
    D = [int(d) for d in D]
    for c, r_bp in ((HIST, r_rev_bp), (ITEM, r_item_bp)):
        members = [p for p in range(n) if cls[p] == c and p not in win]
        k = budget(r_bp, len(members))
        sel |= set(topk_order(D, members)[:k])
    return np.array(sorted(sel), dtype=np.int32)


def sel_count(cls, r_rev_bp, r_item_bp, window=0):
    """|Sel| is fixed by the layout (no data dependence): used to size outputs."""
    n = len(cls)
    win = {p for p in range(max(0, n - window), n) if cls[p] != PREFIX} if window > 0 else set()
    forced = sum(1 for p in range(n) if cls[p] == FORCED and p not in win)
    nh = sum(1 for p in range(n) if cls[p] == HIST and p not in win)
    ni = sum(1 for p in range(n) if cls[p] == ITEM and p not in win)
    return forced + len(win) + budget(r_rev_bp, nh) + budget(r_item_bp, ni)
