"""O-FULL: textbook Llama / Qwen2 decoder prefill in fp64 (test infrastructure only).

Follows Eq. 1, softmax(Q K^T / sqrt(d_k)) V, inside the standard decoder
block of the served models (SURVEY.md §8(c) O-FULL):
    x0 = E[t]
    a = RMSNorm(x) * g1,  RMSNorm(x) = x / sqrt(mean(x^2) + eps)
    q, k, v = a Wq (+bq), a Wk (+bk), a Wv (+bv); RoPE at the token position on q and k
    o_h = softmax(q_h K_{g(h)}[0..p]^T / sqrt(d_h)) V_{g(h)}[0..p],  g(h) = floor(h / (H/H_kv))
    x += o Wo;  m = RMSNorm(x) * g2;  x += (silu(m Wg) * (m Wu)) Wd
    logits = RMSNorm(x_L[n-1]) * g_f  W_lm
Weights are the bf16 generator tensors widened exactly to fp64. RoPE uses the fp32 tables
of numerics.RopeTable, widened.
"""
import numpy as np

from .numerics import RopeTable, rope_rotate_f64


def _np64(t):
    return t.detach().to("cpu").float().numpy().astype(np.float64)


class OracleModel:
    def __init__(self, shape, weights):
        self.s = shape
        self.w = weights
        self.rope_table = RopeTable(shape.rope_theta, shape.head_dim)
        self._cache_l, self._cache = None, {}
        self._glob = {}

    def g(self, name):
        if name not in self._glob:
            self._glob[name] = _np64(self.w[name])
        return self._glob[name]

    def lw(self, l, name):
        if self._cache_l != l:
            self._cache_l, self._cache = l, {}
        if name not in self._cache:
            self._cache[name] = _np64(self.w["layers"][l][name])
        return self._cache[name]

    # --- block pieces -------------------------------------------------------------------
    def rmsnorm(self, x, gain):
        return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + self.s.rms_eps) * gain

    def rope(self, x, pos):
        c, s = self.rope_table.get(pos)
        return rope_rotate_f64(x, c[:, None, :], s[:, None, :])

    def qkv(self, l, x, pos):
        """q [T,H,dh], k [T,Hk,dh] (both RoPE'd at pos), v [T,Hk,dh]."""
        s = self.s
        a = self.rmsnorm(x, self.lw(l, "ln1"))
        q = a @ self.lw(l, "wq").T
        k = a @ self.lw(l, "wk").T
        v = a @ self.lw(l, "wv").T
        if s.qkv_bias:
            q = q + self.lw(l, "bq")
            k = k + self.lw(l, "bk")
            v = v + self.lw(l, "bv")
        T = x.shape[0]
        q = q.reshape(T, s.n_heads, s.head_dim)
        k = k.reshape(T, s.n_kv_heads, s.head_dim)
        v = v.reshape(T, s.n_kv_heads, s.head_dim)
        return self.rope(q, pos), self.rope(k, pos), v

    def attend(self, q, qpos, K, V):
        """Causal by true position: query at p attends keys at positions 0..p.
        K, V: [n_ctx, Hk, dh] indexed by position."""
        s = self.s
        G = s.group
        T = q.shape[0]
        o = np.empty((T, s.n_heads, s.head_dim))
        kpos = np.arange(K.shape[0])
        scale = 1.0 / np.sqrt(s.head_dim)
        for t0 in range(0, T, 1024):
            t1 = min(T, t0 + 1024)
            mask = kpos[None, :] > np.asarray(qpos[t0:t1])[:, None]
            for h in range(s.n_heads):
                kv = h // G
                sc = (q[t0:t1, h] @ K[:, kv].T) * scale
                sc = np.where(mask, -np.inf, sc)
                sc = sc - sc.max(axis=1, keepdims=True)
                p = np.exp(sc)
                p /= p.sum(axis=1, keepdims=True)
                o[t0:t1, h] = p @ V[:, kv]
        return o

    def post(self, l, x, o):
        s = self.s
        x = x + o.reshape(x.shape[0], s.q_dim) @ self.lw(l, "wo").T
        m = self.rmsnorm(x, self.lw(l, "ln2"))
        gt = m @ self.lw(l, "wg").T
        up = m @ self.lw(l, "wu").T
        return x + ((gt / (1.0 + np.exp(-gt))) * up) @ self.lw(l, "wd").T

    def embed(self, tokens):
        return self.g("embed")[np.asarray(tokens, dtype=np.int64)].copy()

    def logits(self, x_last):
        a = self.rmsnorm(x_last, self.g("norm"))
        return a @ self.g("lm_head").T


def forward(m: OracleModel, tokens, start_pos=0, past_K=None, past_V=None):
    """Prefill `tokens` at positions start_pos.. over an optional past KV cache
    (lists per layer of [start_pos, Hk, dh]). Returns dict(logits_last, logits_all, K, V, x)."""
    s = m.s
    T = len(tokens)
    pos = np.arange(start_pos, start_pos + T)
    x = m.embed(tokens)
    Ks, Vs = [], []
    for l in range(s.n_layers):
        q, k, v = m.qkv(l, x, pos)
        if past_K is not None:
            K = np.concatenate([past_K[l], k], axis=0)
            V = np.concatenate([past_V[l], v], axis=0)
        else:
            K, V = k, v
        Ks.append(K)
        Vs.append(V)
        o = m.attend(q, pos, K, V)
        x = m.post(l, x, o)
    return {"logits_last": m.logits(x[-1]), "K": Ks, "V": Vs, "x": x,
            "logits_fn": lambda: m.logits(x)}


def full_prefill(m: OracleModel, tokens):
    """O-FULL of the whole prompt from position 0."""
    return forward(m, tokens, 0)
