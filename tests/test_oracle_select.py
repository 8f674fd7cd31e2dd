"""Pins of oracle/layout.py and oracle/select.py (not gpu)."""
import itertools

import numpy as np
import pytest

from oracle.layout import decompose_prompt, budget, PREFIX, FORCED, HIST, ITEM
from oracle.select import importance_scores, select_heavy_hitters, select_sel, sel_count, topk_order


def test_layout_worked_example(golden):
    g = golden("layout_spec68.json")
    lay = decompose_prompt(np.zeros(g["instruction"], int), np.arange(g["history"][0]),
                           np.ones(g["history"][0], int), [7], [np.arange(g["items"][0]) + 3],
                           np.zeros(g["tail"], int))
    assert lay.seg_start[:3] == g["segment_offsets"] and lay.n == g["total"]
    assert (lay.cls[:207] == PREFIX).all() and (lay.cls[207:257] == HIST).all() and (lay.cls[257:] == ITEM).all()
    assert list(lay.src_off[257:260]) == [0, 1, 2] and lay.cand_idtok[0] == 3


def test_layout_conservation():
    rng = np.random.default_rng(0)
    for _ in range(20):
        P, H, T = rng.integers(0, 50, 3)
        lens = rng.integers(1, 30, rng.integers(0, 6))
        lay = decompose_prompt(np.zeros(P, int), np.arange(H), np.zeros(H, int), list(range(len(lens))),
                               [np.arange(k) for k in lens], np.zeros(T, int))
        assert lay.n == P + H + sum(lens) + T
        assert np.bincount(lay.cls, minlength=4).tolist() == [P, T, H, sum(lens)]


def test_budget_examples(golden):
    g = golden("budget_spec413.json")
    assert budget(g["r_bp"], g["cached_items"] * g["item_len"]) == g["expected_heavy_hitters"]
    assert budget(1500, 1280) == 192          # integer basis points, not 0.15f
    assert budget(10000, 77) == 77 and budget(0, 77) == 0 and budget(1, 1) == 1


def test_select_heavy_hitters_spec(golden):
    for c in golden("topk_spec431.json")["cases"]:
        assert select_heavy_hitters(c["scores"], c["r_bp"], c["window"], len(c["scores"])) == c["expected"]


def test_topk_is_unique_dominating_subset_bruteforce():
    # brute force over all k-subsets: exactly one subset has every member ahead (score desc,
    # position asc) of every non-member; it is the oracle's top-k
    rng = np.random.default_rng(1)
    for _ in range(30):
        n = 9
        sc = rng.integers(0, 4, n).tolist()
        for k in range(n + 1):
            top = set(topk_order(sc, range(n))[:k])
            ok = []
            for sub in itertools.combinations(range(n), k):
                s = set(sub)
                if all((sc[a] > sc[b]) or (sc[a] == sc[b] and a < b) for a in s for b in range(n) if b not in s):
                    ok.append(s)
            assert ok == [top]


def test_select_sel_classes_nesting_and_bounds():
    rng = np.random.default_rng(2)
    cls = np.array([PREFIX] * 5 + [HIST] * 40 + [ITEM] * 60 + [FORCED] * 6, np.uint8)
    D = rng.integers(0, 1000, len(cls))
    prev = set()
    for r in (0, 500, 1500, 3000, 10000):
        sel = select_sel(cls, D, r, r)
        assert len(sel) == sel_count(cls, r, r) == 6 + budget(r, 40) + budget(r, 60)
        assert list(sel) == sorted(sel) and set(range(105, 111)) <= set(sel)
        assert not any(cls[p] == PREFIX for p in sel)
        assert prev <= set(sel)                        # nested in r
        prev = set(sel)
    assert set(select_sel(cls, D, 10000, 10000)) == set(range(5, 111))   # r = 1 -> all of U
    assert set(select_sel(cls, D, 0, 0)) == set(range(105, 111))         # r = 0 -> FORCED only
    # per-class ordering: the chosen history tokens carry the largest D of their class
    sel = set(select_sel(cls, D, 2000, 0))
    hs = [p for p in range(5, 45) if p in sel]
    assert min(D[hs]) >= max(D[[p for p in range(5, 45) if p not in sel]])
    # window: trailing positions become recomputed, outside the budgets
    selw = select_sel(cls, D, 0, 0, window=10)
    assert set(selw) == set(range(101, 111)) and sel_count(cls, 0, 0, 10) == 10


def test_importance_scores_reductions_and_brute_force():
    rng = np.random.default_rng(3)
    n, m = 64, 32
    A = rng.random(n)
    Kn, Kc, Vn, Vc = (rng.standard_normal((n, m)) for _ in range(4))
    assert np.array_equal(importance_scores(A, Kn, Kc, Vn, Vc, 0.0), A)          # lambda = 0
    assert np.all(importance_scores(A, Kn, Kn, Vn, Vn, 1.0) == 0)               # vanishing divergence
    S = importance_scores(A, Kn, Kc, Vn, Vc, 0.5)
    for i in range(n):
        t = 0.5 * A[i]
        for j in range(m):
            t += 0.5 * (abs(Kn[i, j] - Kc[i, j]) + abs(Vn[i, j] - Vc[i, j]))
        assert abs(S[i] - t) < 1e-12
    with pytest.raises(ValueError):
        importance_scores(A[:-1], Kn, Kc, Vn, Vc, 0.5)


# ----------------------------------------------------------------------------- NEXT-1: attention mass
from oracle.select import attention_mass_fixed, combine_fixed, MASS_FRAC_BITS  # noqa: E402

ONE = 1 << MASS_FRAC_BITS


def _mass_case(seed, n=40, P=8, H=4, Hk=2, dh=16):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n - P, H, dh)) * 2.0
    K = rng.standard_normal((n, Hk, dh))
    return q, np.arange(P, n), K


def test_attention_mass_rows_sum_to_one():
    """Every softmax row sums to 1 over its keys: sum_p A[p] = H |U| 2^24 minus the floor losses."""
    q, qpos, K = _mass_case(1)
    H = q.shape[1]
    A = attention_mass_fixed(q, qpos, K, H, K.shape[1], q.shape[2])
    total = int(A.sum())
    terms = H * int(sum(p + 1 for p in qpos))
    assert H * len(qpos) * ONE - terms <= total <= H * len(qpos) * ONE
    assert A[qpos[-1] + 1:].sum() == 0 if qpos[-1] + 1 < len(A) else True


def test_attention_mass_uniform_closed_form():
    """q = 0: every visible key gets 1/(pos_q + 1), so A[p] = H * sum_{pos_q >= p} floor(2^24 / (pos_q + 1))."""
    _, qpos, K = _mass_case(2)
    H = 4
    q = np.zeros((len(qpos), H, K.shape[2]))
    A = attention_mass_fixed(q, qpos, K, H, K.shape[1], K.shape[2])
    ref = [H * sum(ONE // (int(t) + 1) for t in qpos if t >= p) for p in range(K.shape[0])]
    assert [int(a) for a in A] == ref


def test_attention_mass_gqa_grouping():
    """Heads h use kv head floor(h / G): zero keys in kv head 1 make heads 2, 3 uniform, heads 0, 1 equal
    the single-kv-head computation on kv head 0 (a wrong h -> kv map fails this)."""
    q, qpos, K = _mass_case(3)
    K[:, 1] = 0.0
    A = attention_mass_fixed(q, qpos, K, 4, 2, K.shape[2])
    A01 = attention_mass_fixed(q[:, :2], qpos, K[:, :1], 2, 1, K.shape[2])
    unif = np.array([2 * sum(ONE // (int(t) + 1) for t in qpos if t >= p) for p in range(K.shape[0])], np.uint64)
    assert np.array_equal(A, A01 + unif)


def test_attention_mass_brute_force_tiny():
    """Independent scalar evaluation with math.exp / math.fsum on a 7-token instance."""
    import math
    rng = np.random.default_rng(4)
    n, P, H, Hk, dh = 7, 2, 2, 1, 4
    q = rng.standard_normal((n - P, H, dh))
    K = rng.standard_normal((n, Hk, dh))
    qpos = list(range(P, n))
    ref = [0] * n
    for h in range(H):
        for i, t in enumerate(qpos):
            sc = [math.fsum(q[i, h, d] * K[p, 0, d] for d in range(dh)) / math.sqrt(dh) for p in range(t + 1)]
            mx = max(sc)
            e = [math.exp(x - mx) for x in sc]
            z = math.fsum(e)
            for p in range(t + 1):
                ref[p] += math.floor(e[p] / z * ONE)
    A = attention_mass_fixed(q, qpos, K, H, Hk, dh)
    assert [int(a) for a in A] == ref


def test_combine_fixed_reductions_and_rounding():
    A = np.array([3, 1, 0, 7, 2 ** 40], np.uint64)
    D = np.array([4, 4, 9, 7, 2 ** 50], np.uint64)
    assert np.array_equal(combine_fixed(A, D, 1.0), D)
    assert np.array_equal(combine_fixed(A, D, 0.0), A)
    # 3.5 -> 4, 2.5 -> 2 (half to even), 4.5 -> 4, 7 -> 7
    assert combine_fixed(A, D, 0.5)[:4].tolist() == [4, 2, 4, 7]
    assert int(combine_fixed(A, D, 0.5)[4]) == (2 ** 40 + 2 ** 50) // 2


def test_top10_ranking_helper():
    from tests.helpers import assert_top10_ranking
    ref = np.array([5.0, 4.0, 3.9999, 1.0, 0.5, 9.0, 2.0, 2.5, 3.0, 0.1, 0.2, 7.0])
    assert assert_top10_ranking(ref + 1e-6, ref, 1e-3) >= 8     # all resolvable gaps agree
    near = ref.copy(); near[1], near[2] = ref[2], ref[1]       # swap inside a near-tie: allowed
    assert_top10_ranking(near, ref, 1e-3)
    bad = ref.copy(); bad[5], bad[11] = ref[11], ref[5]        # a candidate far off its logit error: caught
    with pytest.raises(AssertionError):
        assert_top10_ranking(bad, ref, 1e-3)
