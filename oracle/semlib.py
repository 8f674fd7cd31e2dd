"""NEXT-3: online LSH matching of history tokens to semantic prototypes
(test infrastructure only).

PAPER.md:549: review tokens "are mapped to the nearest pre-computed semantic prototype using
LSH-based matching"; prototypes are position-aware token embeddings clustered
by LSH. SPEC.md:237-263 fixes the operations this follows:
  embed_token(t, p)  = normalize(lexical(t) (+) positional(bucket(p)))
  match_token(t, p)  = probe every LSH table, union the candidates, return the max-cosine
                       prototype, ties -> smaller id; no candidate -> best prototype of the same
                       position bucket by linear scan
Readings (DESIGN.md R-LSH), chosen so that every integer decision (a signature bit, an argmax)
is taken in fp32 with one fixed operation order on both sides:
  * D = 64 = 48 lexical + 16 positional dims; T = 8 tables x B = 16 bits (SPEC LshConfig defaults).
  * lexical_j(t) = +1 if bit 63 of splitmix64(seed * 2^32 XOR (64 t + j)) is 0 else -1 (a seeded
    feature hash).
  * bucket(p) = min(floor(log2(p + 1)), n_buckets - 1), p = offset inside the review history
    (the log buckets of the generator); positional = [sin(b w_k), cos(b w_k)]_{k<8},
    w_k = 10000^(-k/8), evaluated in fp64 by the C library and rounded once to fp32.
  * dot(a, b) over 64 fp32 values: s_l = (a_l b_l) + (a_{l+32} b_{l+32}) for l < 32, then
    s_l <- s_l + s_{l XOR o} for o = 16, 8, 4, 2, 1; every product and sum rounded to fp32 (no FMA).
  * normalize: v / sqrt(dot(v, v)), fp32 correctly rounded sqrt and division.
  * signature_t(v) = sum_b [dot(h_{t,b}, v) > 0] 2^b; hyperplanes h are inputs (seeded Gaussians).
  * a prototype's centroid = embed(token(pi), offset(pi)) (its medoid token at its canonical
    position); the fallback scans the prototypes of the query's bucket, and all
    prototypes if that bucket has none.
"""
import math

import numpy as np

D, D_LEX, D_POS, T, B = 64, 48, 16, 8, 16
MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64_np(x):
    """splitmix64 on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        z = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def lexical(token: int, seed: int) -> np.ndarray:
    base = np.uint64(((seed & 0xFFFFFFFF) << 32) & MASK64)
    x = base ^ (np.uint64(64) * np.uint64(int(token)) + np.arange(D_LEX, dtype=np.uint64))
    return np.where((splitmix64_np(x) >> np.uint64(63)) == 0, 1.0, -1.0).astype(np.float32)


def bucket(offset: int, n_buckets: int) -> int:
    return min(int(math.floor(math.log2(int(offset) + 1))), n_buckets - 1)


def positional(b: int) -> np.ndarray:
    out = []
    for k in range(D_POS // 2):
        w = 10000.0 ** (-k / (D_POS // 2))
        out += [math.sin(b * w), math.cos(b * w)]
    return np.array(out, dtype=np.float32)


def dot_rows(a, b):
    """The fixed fp32 reduction order of R-LSH, row-wise over [..., 64] float32 arrays."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    s = (a[..., :32] * b[..., :32]) + (a[..., 32:] * b[..., 32:])
    idx = np.arange(32)
    for o in (16, 8, 4, 2, 1):
        s = s + s[..., idx ^ o]
    return s[..., 0]


def embed(token: int, offset: int, n_buckets: int, seed: int) -> np.ndarray:
    v = np.concatenate([lexical(token, seed), positional(bucket(offset, n_buckets))])
    n = np.sqrt(dot_rows(v, v))
    return (v / n).astype(np.float32)


def signatures(v, H):
    """[.., T] uint32 signatures of unit vectors v [.., 64] under hyperplanes H [T*B][64]."""
    v = np.asarray(v, dtype=np.float32)
    bits = np.stack([dot_rows(v, H[i]) > 0 for i in range(T * B)], axis=-1).astype(np.uint32)
    bits = bits.reshape(*bits.shape[:-1], T, B)
    return (bits << np.arange(B, dtype=np.uint32)).sum(axis=-1).astype(np.uint32)


class Library:
    """Prototype centroids, their buckets and the T bucket maps signature -> prototype ids."""

    def __init__(self, proto_token, proto_offset, n_buckets, H, seed):
        self.n_buckets = n_buckets
        self.seed = seed
        self.H = np.asarray(H, dtype=np.float32)
        self.C = np.stack([embed(t, o, n_buckets, seed) for t, o in zip(proto_token, proto_offset)])
        self.bucket = np.array([bucket(o, n_buckets) for o in proto_offset], dtype=np.int32)
        self.sig = signatures(self.C, self.H)  # [n][T]
        self.maps = []
        for t in range(T):
            m = {}
            for pid, s in enumerate(self.sig[:, t]):
                m.setdefault(int(s), []).append(pid)
            self.maps.append(m)

    def match(self, token: int, offset: int):
        """(prototype id, cosine) of SPEC match_token under R-LSH."""
        v = embed(token, offset, self.n_buckets, self.seed)
        sig = signatures(v, self.H)
        cand = sorted({pid for t in range(T) for pid in self.maps[t].get(int(sig[t]), [])})
        if not cand:
            b = bucket(offset, self.n_buckets)
            cand = [int(p) for p in np.nonzero(self.bucket == b)[0]] or list(range(len(self.C)))
        cos = dot_rows(np.broadcast_to(v, (len(cand), D)), self.C[cand])
        best = int(np.argmax(cos))  # first maximum = smallest id (cand ascending)
        return cand[best], float(cos[best])
