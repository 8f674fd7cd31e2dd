"""O-ASM: KV block retrieval + alignment (test infrastructure only).

PAPER.md:548-551 (retrieval: history tokens from the prototype library, item tokens by item
ID) and PAPER.md:566 ((i) Assembly, (ii) Alignment: "Reused blocks undergo positional
adjustment (e.g., RoPE rotation) to align with the current request's indices").
SURVEY.md §8(c) O-ASM table, per layer l and position p:
  PREFIX             K, V = prefix-cache KV (exact copy)
  HIST  proto pi     K = bf16(rot(p - o_pi, deq(Kq))),       V = bf16(deq(Vq))
  ITEM  item i, off j K = bf16(rot(p - (s_i + j), K_item)),  V = V_item (copy)
  FORCED             undefined until recomputed
deq / rot / bf16 are the exact fp32 sequences of numerics (R13, R15). Pools store K
post-RoPE at canonical positions (R14), so alignment is a rotation by the offset Delta.
Layers below `gather_from` hold only the prefix (they are recomputed for all of U).
"""
import numpy as np

from .layout import PREFIX, FORCED, HIST, ITEM
from .numerics import RopeTable, rope_rotate_f32, bf16_bits, bf16_to_f32, dequant_int8


def _bits(t):
    """torch bf16 tensor or uint16 array -> uint16 numpy."""
    if hasattr(t, "view") and hasattr(t, "dtype") and "bfloat16" in str(t.dtype):
        import torch
        return t.detach().to("cpu").view(torch.int16).numpy().view(np.uint16)
    return np.asarray(t, dtype=np.uint16)


def assemble(shape, layout, items, hist, prefix, gather_from=0, rope=None):
    """items: {item_id: (kv [len][L][2][Hk][dh] bf16, canon_start)};
    hist: {proto: (q int8 [L][2][Hk][dh], scale f32 [L][2][Hk], canon_pos)};
    prefix: kv [P][L][2][Hk][dh] bf16.
    Returns (K bits uint16 [L][n][Hk][dh], V bits, defined bool [L][n])."""
    L, Hk, dh = shape.n_layers, shape.n_kv_heads, shape.head_dim
    n = layout.n
    rope = rope or RopeTable(shape.rope_theta, dh)
    K = np.zeros((L, n, Hk, dh), np.uint16)
    V = np.zeros((L, n, Hk, dh), np.uint16)
    defined = np.zeros((L, n), bool)
    pre = _bits(prefix) if prefix is not None else None
    item_bits = {}
    lay = slice(gather_from, L)
    for p in range(n):
        c = int(layout.cls[p])
        if c == PREFIX:
            K[:, p] = pre[p, :, 0]
            V[:, p] = pre[p, :, 1]
            defined[:, p] = True
        elif c == HIST:
            q, sc, o = hist[int(layout.src_id[p])]
            q = np.asarray(q)[lay]
            sc = np.asarray(sc, dtype=np.float32)[lay]
            kd = dequant_int8(q[:, 0], sc[:, 0])          # [L', Hk, dh] fp32
            vd = dequant_int8(q[:, 1], sc[:, 1])
            cs, sn = rope.get([p - int(o)])
            K[lay, p] = bf16_bits(rope_rotate_f32(kd, cs[0], sn[0]))
            V[lay, p] = bf16_bits(vd)
            defined[lay, p] = True
        elif c == ITEM:
            it = int(layout.src_id[p])
            if it not in item_bits:
                item_bits[it] = (_bits(items[it][0]), int(items[it][1]))
            kv, s0 = item_bits[it]
            j = int(layout.src_off[p])
            kf = bf16_to_f32(kv[j, lay, 0])
            cs, sn = rope.get([p - (s0 + j)])
            K[lay, p] = bf16_bits(rope_rotate_f32(kf, cs[0], sn[0]))
            V[lay, p] = kv[j, lay, 1]
            defined[lay, p] = True
        elif c == FORCED:
            pass
        else:
            raise ValueError(f"bad token class {c} at {p}")
    return K, V, defined
