"""Pins of oracle/semlib.py (NEXT-3 LSH prototype matching; not gpu)."""
import math

import numpy as np

from oracle.semlib import (D, T, B, Library, bucket, dot_rows, embed, lexical, signatures, splitmix64,
                           splitmix64_np)

SEED = 11


def _H(seed=5):
    return np.random.default_rng(seed).standard_normal((T * B, D)).astype(np.float32)


def test_splitmix_vectorised_equals_scalar_reference_values():
    # splitmix64 reference outputs for seed 0, 1, 2 (the published generator's first values)
    assert splitmix64(0) == 0xE220A8397B1DCDAF
    xs = np.array([0, 1, 12345, 2 ** 63 + 7], dtype=np.uint64)
    assert [int(v) for v in splitmix64_np(xs)] == [splitmix64(int(x)) for x in xs]


def test_embedding_unit_norm_and_bucket_identity():
    for tok, off in [(3, 0), (3, 1), (99, 5), (7, 600)]:
        v = embed(tok, off, 10, SEED).astype(np.float64)
        assert abs(np.linalg.norm(v) - 1.0) < 1e-6
    assert bucket(3, 10) == bucket(5, 10) == 2 and bucket(6, 10) == 2 and bucket(7, 10) == 3
    assert np.array_equal(embed(42, 3, 10, SEED), embed(42, 5, 10, SEED))  # same log bucket
    a, b = embed(42, 3, 10, SEED), embed(42, 40, 10, SEED)
    assert float(np.dot(a.astype(np.float64), b)) < 1.0 - 1e-3
    assert set(np.unique(lexical(5, SEED))) <= {-1.0, 1.0}


def test_tree_dot_within_fp32_error_bound_of_exact():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((500, D)).astype(np.float32)
    b = rng.standard_normal((500, D)).astype(np.float32)
    exact = (a.astype(np.float64) * b.astype(np.float64)).sum(axis=1)
    bound = 7 * 2.0 ** -24 * (np.abs(a.astype(np.float64) * b)).sum(axis=1) * 2  # 6 rounding levels
    assert np.all(np.abs(dot_rows(a, b).astype(np.float64) - exact) <= bound)
    assert dot_rows(a, b).dtype == np.float32


def test_signature_of_negated_vector_is_complement():
    H = _H()
    rng = np.random.default_rng(1)
    v = rng.standard_normal((50, D)).astype(np.float32)
    s, sn = signatures(v, H), signatures(-v, H)
    assert np.array_equal(sn, (~s) & np.uint32(0xFFFF))


def test_match_self_and_exact_nn_among_candidates():
    rng = np.random.default_rng(2)
    toks = rng.integers(0, 5000, 300)
    offs = rng.integers(0, 640, 300)
    lib = Library(toks, offs, 10, _H(), SEED)
    for i in range(0, 300, 7):  # a prototype's own (token, offset): its embedding, cosine ~1, smallest equal id
        pid, cos = lib.match(int(toks[i]), int(offs[i]))
        assert np.array_equal(lib.C[pid], lib.C[i]) and pid <= i and abs(cos - 1.0) < 1e-6
    hits = 0
    for q in range(60):  # the exact NN wins whenever it is among the LSH candidates
        if q % 2 == 0:   # a prototype's token at another offset of its bucket: same embedding
            i = int(rng.integers(0, 300))
            b = bucket(int(offs[i]), 10)
            tok, off = int(toks[i]), int(rng.integers(2 ** b - 1, min(2 ** (b + 1) - 1, 640)))
            assert bucket(off, 10) == b
        else:            # an unrelated (token, offset)
            tok, off = int(rng.integers(0, 5000)), int(rng.integers(0, 640))
        v = embed(tok, off, 10, SEED)
        exact = dot_rows(np.broadcast_to(v, lib.C.shape), lib.C)
        nn = int(np.argmax(exact))
        sig = signatures(v, lib.H)
        cand = {p for t in range(T) for p in lib.maps[t].get(int(sig[t]), [])}
        pid, cos = lib.match(tok, off)
        if nn in cand:
            hits += 1
            assert pid == nn and cos == exact[nn]
        elif not cand:  # fallback: the best of the query's bucket (or of all prototypes)
            same = np.nonzero(lib.bucket == bucket(off, 10))[0]
            pool = same if len(same) else np.arange(len(lib.C))
            assert pid == int(pool[np.argmax(exact[pool])])
    assert hits >= 30   # every same-embedding query hashes into its prototype's buckets


def test_positional_code_values():
    from oracle.semlib import positional
    p = positional(3)
    assert p.dtype == np.float32 and p[0] == np.float32(math.sin(3.0)) and p[1] == np.float32(math.cos(3.0))
    assert p[2] == np.float32(math.sin(3 * 10000.0 ** (-1 / 8)))
