"""Offline pool materialisation through librc's own dense path (SURVEY.md §8(d) "Pool contents",
readings R16/R17; PAPER.md:384 "canonical representative token", :458 "precomputes their KV blocks
offline").

  prefix      full prefill of the system prompt (every position recomputed) -> bf16 KV rows 0..P-1
  items (R16) full prefill of [system prompt; item tokens] at positions 0..P+len-1 over the exact
              prefix cache; the item rows' K (post-RoPE at P+j, R14) and V, bf16 -> canonical start P
  prototypes  (R17) full prefill of [system prompt; review-corpus sequence] (rcgen.proto_corpus puts
              each prototype's token at its canonical position); the prototype's row, quantised to
              int8 with fp32 scales by rc_seq_export_kv (R15)

Every step is a librc call (rc_assemble + rc_selective_prefill at r = 100%, then rc_seq_export_kv):
this module only builds layouts and chunks the work. The returned tensors are in the registration
layout of rc_pool_register_blocks ([n_tok][L][2][H_kv][d_h]).
"""
import numpy as np
import torch

from . import _lib as R

FORCED, PREFIX = 1, 0


def _layout(tokens, n_prefix):
    n = len(tokens)
    cls = np.full(n, FORCED, np.uint8)
    cls[:n_prefix] = PREFIX
    return dict(tokens=np.ascontiguousarray(tokens, np.int32), cls=cls, src_id=np.full(n, -1, np.int64),
                src_off=np.zeros(n, np.int32), cand_idtok=np.zeros(0, np.int32))


def _prefill(ctx, layouts, prefix_id, stream):
    seqs = ctx.assemble(layouts, prefix_id=prefix_id, gather_from=0, stream=stream)
    ctx.selective_prefill(seqs, 10000, 10000, check_layer=0, logits=False, cand_scores=False, sel_pos=False,
                          stream=stream)
    return seqs


def _chunk(ctx, n_seq_tokens, n_u_tokens):
    """Requests per call: the stitched arena and the batch-token workspace bound a chunk."""
    return max(1, min(ctx.arena_rows // n_seq_tokens, ctx.max_batch_tokens // max(n_u_tokens, 1), 256))


def prefix_kv(ctx, sys_tokens, stream=None):
    """bf16 [P][L][2][Hk][dh]: the exact prefix cache (R8)."""
    seqs = _prefill(ctx, [_layout(sys_tokens, 0)], 0, stream)
    kv = ctx.export_kv(seqs[0], 0, len(sys_tokens), stream=stream)
    ctx.release(seqs)
    return kv


def register_prefix(ctx, sys_tokens, prefix_id=1, stream=None):
    kv = prefix_kv(ctx, sys_tokens, stream)
    ctx.pool_register_blocks(R.RC_POOL_PREFIX_BF16, [prefix_id], [len(sys_tokens)], [0], kv, stream=stream)
    return kv


def item_kv_chunks(ctx, sys_tokens, prefix_id, item_ids, item_tokens, stream=None):
    """Yields (ids, bf16 [n][len][L][2][Hk][dh]) chunk by chunk (R16: canonical start P)."""
    P = len(sys_tokens)
    ln = len(item_tokens[0])
    k = _chunk(ctx, P + ln, ln)
    for i0 in range(0, len(item_ids), k):
        ids = list(item_ids[i0:i0 + k])
        lays = [_layout(np.concatenate([sys_tokens, item_tokens[j]]), P) for j in range(i0, i0 + len(ids))]
        seqs = _prefill(ctx, lays, prefix_id, stream)
        kv = torch.stack([ctx.export_kv(s, P, ln, stream=stream) for s in seqs])
        ctx.release(seqs)
        yield ids, kv


def register_items(ctx, sys_tokens, prefix_id, item_ids, item_tokens, kind=R.RC_POOL_ITEM_BF16, stream=None,
                   keep=False):
    """Materialise and register item blocks; returns {id: bf16 kv [len][L][2][Hk][dh]} if keep."""
    kept = {}
    P = len(sys_tokens)
    for ids, kv in item_kv_chunks(ctx, sys_tokens, prefix_id, item_ids, item_tokens, stream):
        ln = kv.shape[1]
        ctx.pool_register_blocks(kind, ids, [ln] * len(ids), [P] * len(ids),
                                 kv.reshape(len(ids) * ln, *kv.shape[2:]).contiguous(), stream=stream)
        if keep:
            kept.update({int(i): kv[j] for j, i in enumerate(ids)})
    return kept


def proto_kv(ctx, sys_tokens, prefix_id, corpus, seq_of, off_of, stream=None):
    """int8 [n][L][2][Hk][dh] + fp32 scales [n][L][2][Hk] for prototypes sitting at (seq_of, off_of)
    of the corpus sequences (R15 quantisation of the token's K/V at its canonical position)."""
    P = len(sys_tokens)
    S, H = corpus.shape
    k = _chunk(ctx, P + H, H)
    seq_of = np.asarray(seq_of, np.int64)
    off_of = np.asarray(off_of, np.int64)
    L, Hk, dh = ctx.shape.n_layers, ctx.shape.n_kv_heads, ctx.shape.head_dim
    dev = torch.device("cuda", ctx.device)
    q = torch.empty((len(seq_of), L, 2, Hk, dh), dtype=torch.int8, device=dev)
    sc = torch.empty((len(seq_of), L, 2, Hk), dtype=torch.float32, device=dev)
    for s0 in range(0, S, k):
        lays = [_layout(np.concatenate([sys_tokens, corpus[j]]), P) for j in range(s0, min(S, s0 + k))]
        seqs = _prefill(ctx, lays, prefix_id, stream)
        for j, sq in enumerate(seqs):
            mine = np.nonzero(seq_of == s0 + j)[0]
            if len(mine) == 0:
                continue
            qj, sj = ctx.export_kv(sq, P, H, int8=True, stream=stream)
            idx = torch.as_tensor(mine, device=dev)
            oi = torch.as_tensor(off_of[mine], device=dev)
            q[idx] = qj[oi]
            sc[idx] = sj[oi]
        ctx.release(seqs)
    return q, sc


def register_protos(ctx, sys_tokens, prefix_id, proto_ids, canon_pos, corpus, seq_of, off_of, stream=None):
    q, sc = proto_kv(ctx, sys_tokens, prefix_id, corpus, seq_of, off_of, stream)
    ctx.pool_register_blocks(R.RC_POOL_HIST_INT8, list(proto_ids), [1] * len(proto_ids),
                             [int(c) for c in canon_pos], q, sc, stream=stream)
    return q, sc
