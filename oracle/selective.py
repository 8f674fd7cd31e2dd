"""O-SEL: selective recomputation over the stitched KV, one request (test infrastructure only).

Follows PAPER.md:557-566 step by step (SURVEY.md §8(c) O-SEL), with U the non-PREFIX
positions and c the check layer (reading R1):
  1. O-ASM (assemble.py) gives the stitched cache KV_st (bf16 values).
  2. Layers l < c: the full layer for every p in U over prefix + U, causal ("full attention
     computation in the first decoder layer"); KV_st[l][U] := fresh.
  3. Check layer c: K_new, V_new for U (RoPE at p); for HIST/ITEM tokens the Eq. 3 divergence
     in the R4 fixed point, on K_new/V_new rounded to the bf16 value they would be stored as vs
     the stitched bf16 value. lambda = 1 (R3) scores by D alone; lambda < 1 (NEXT-1) adds the
     attention-mass term: the fresh queries of U attend, causally, over the fresh keys (prefix
     cache + K_new of U) -- "full attention computation in the first decoder layer"
      -- and S = (1 - lambda) A + lambda D (Eq. 3) in the R2-FX fixed point.
  4. Sel = FORCED u window u topk per class (select.select_sel; R5-R7), or a forced Sel.
  5. Layers c..L-1 on Sel only: q, k, v at the true positions, KV_st[l][Sel] := (k, v),
     non-selected tokens keep their stitched state (R9), attention of every selected query
     over all stitched keys at positions <= its own (R11), O-proj, residual, MLP.
  6. Logits of the last position (always FORCED: the instruction tail), candidate scores =
     logits[ID token of the candidate], ranked by score desc, ties -> lower slot (R19).

Gradual filtering (NEXT-1 variant, reading R-GF; the CacheBlend scheme PAPER.md:557 cites for
"token importance persists across layers"): with gradual = g > 0, step 4 takes Sel_0 at the
ratios r_start, and each layer l = c + i (i = 1..g) runs q, k, v for every row of Sel_{i-1},
scores the HIST/ITEM rows of Sel_{i-1} by the Eq. 3 divergence (R4 fixed point) of that layer's
fresh K/V against the stitched K/V still in KV_st[l], writes the fresh K/V of all of Sel_{i-1}
into KV_st[l], keeps Sel_i = FORCED u window u per-class top-k_i among Sel_{i-1} (R5-R7, the
budget k_i = ceil(r_i * |class|) at r_i = select.gradual_ratio_bp), and runs the attention,
O-proj and MLP of layer l for the rows of Sel_i only. Layers > c + g run on Sel_g.
"""
import numpy as np

from .layout import PREFIX, HIST, ITEM
from .numerics import bf16_to_f32, round_bf16, deviation_fixed
from .select import select_sel, attention_mass_fixed, combine_fixed, gradual_ratio_bp


def selective_prefill(m, layout, K_bits, V_bits, r_rev_bp, r_item_bp, check_layer=1,
                      window=0, forced_sel=None, keep_kv=True, exact_kv=False, lam=1.0,
                      gradual=0, r_start_rev_bp=None, r_start_item_bp=None, forced_steps=None):
    """K_bits, V_bits: stitched cache per layer [n][Hk][dh] as bf16 bit patterns (O-ASM), or
    fp64 values when exact_kv (lossless test mode of the exact-cache invariant).
    gradual, r_start_*: gradual filtering (R-GF); forced_steps: Sel_0..Sel_g given (test mode)."""
    s = m.s
    n, L, c = layout.n, s.n_layers, check_layer
    cls = layout.cls
    U = np.array([p for p in range(n) if cls[p] != PREFIX], dtype=np.int64)
    assert len(U) == 0 or U[0] == n - len(U), "PREFIX must be the leading positions"
    if exact_kv:
        K = [np.array(K_bits[l], dtype=np.float64) for l in range(L)]
        V = [np.array(V_bits[l], dtype=np.float64) for l in range(L)]
    else:
        K = [bf16_to_f32(K_bits[l]).astype(np.float64) for l in range(L)]
        V = [bf16_to_f32(V_bits[l]).astype(np.float64) for l in range(L)]

    x = m.embed(layout.tokens[U])
    for l in range(c):
        q, k, v = m.qkv(l, x, U)
        K[l][U], V[l][U] = k, v
        o = m.attend(q, U, K[l], V[l])
        x = m.post(l, x, o)

    # check layer c: deviation of the fresh K/V from the stitched cache
    q_new, k_new, v_new = m.qkv(c, x, U)
    D = np.zeros(n, dtype=np.uint64)
    reuse = np.array([cls[p] in (HIST, ITEM) for p in U])
    if reuse.any():
        ur = U[reuse]
        kb = round_bf16(k_new[reuse]).reshape(len(ur), -1)
        vb = round_bf16(v_new[reuse]).reshape(len(ur), -1)
        D[ur] = deviation_fixed(kb, round_bf16(K[c][ur]).reshape(len(ur), -1)) + \
            deviation_fixed(vb, round_bf16(V[c][ur]).reshape(len(ur), -1))
    A = None
    S = D
    if lam < 1.0:  # NEXT-1: attention mass of the fresh layer-c softmax (prefix keys are exact)
        K_fresh = K[c].copy()
        K_fresh[U] = k_new
        A = attention_mass_fixed(q_new, U, K_fresh, s.n_heads, s.n_kv_heads, s.head_dim)
        S = np.zeros(n, dtype=np.uint64)
        ru = U[reuse] if len(U) else U
        S[ru] = combine_fixed(A[ru], D[ru], lam)
    g = int(gradual)
    if g:
        assert 0 < g and c + g <= L - 1, "gradual steps must end inside the model"
        r0h = r_rev_bp if r_start_rev_bp is None else r_start_rev_bp
        r0i = r_item_bp if r_start_item_bp is None else r_start_item_bp
        assert r_rev_bp <= r0h <= 10000 and r_item_bp <= r0i <= 10000
    else:
        r0h, r0i = r_rev_bp, r_item_bp

    def ratios(i):
        return gradual_ratio_bp(r0h, r_rev_bp, i, g), gradual_ratio_bp(r0i, r_item_bp, i, g)

    if forced_steps is not None:
        sel = np.array(sorted(int(p) for p in forced_steps[0]), dtype=np.int32)
    elif forced_sel is None:
        sel = select_sel(cls, S, *ratios(0), window)
    else:
        sel = np.array(sorted(int(p) for p in forced_sel), dtype=np.int32)
    steps, D_steps = [sel], [D]
    row_of = {int(p): i for i, p in enumerate(U)}
    xs = x[[row_of[int(p)] for p in sel]]
    sp = sel.astype(np.int64)
    for l in range(c, L):
        q, k, v = m.qkv(l, xs, sp)
        i = l - c
        if 1 <= i <= g:   # gradual step i: score Sel_{i-1} against the stitched K/V of this layer
            Dl = np.zeros(n, dtype=np.uint64)
            ru = np.array([cls[p] in (HIST, ITEM) and not (window > 0 and p >= n - window) for p in sp])
            if ru.any():
                pr = sp[ru]
                Dl[pr] = deviation_fixed(round_bf16(k[ru]).reshape(len(pr), -1),
                                         round_bf16(K[l][pr]).reshape(len(pr), -1)) + \
                    deviation_fixed(round_bf16(v[ru]).reshape(len(pr), -1),
                                    round_bf16(V[l][pr]).reshape(len(pr), -1))
            K[l][sp], V[l][sp] = k, v
            if forced_steps is not None:
                nxt = np.array(sorted(int(p) for p in forced_steps[i]), dtype=np.int32)
                assert set(nxt.tolist()) <= set(sp.tolist()), "forced step must be a subset"
            else:
                nxt = select_sel(cls, Dl, *ratios(i), window, among=sp)
            keep = np.isin(sp, nxt)
            q, xs, sp = q[keep], xs[keep], sp[keep]
            steps.append(nxt)
            D_steps.append(Dl)
        else:
            K[l][sp], V[l][sp] = k, v
        o = m.attend(q, sp, K[l], V[l])
        xs = m.post(l, xs, o)
    sel = sp.astype(np.int32)
    assert sp[-1] == n - 1, "the last position must be selected (FORCED tail)"
    logits = m.logits(xs[-1])
    cand = logits[layout.cand_idtok.astype(np.int64)]
    rank = sorted(range(len(cand)), key=lambda i: (-cand[i], i))
    out = {"logits": logits, "cand_scores": cand, "rank": np.array(rank), "sel": sel,
           "D": D, "A": A, "S": S, "x_sel": xs, "sel_steps": steps, "D_steps": D_steps}
    if keep_kv:
        out["K"], out["V"] = K, V
    return out
