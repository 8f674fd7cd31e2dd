"""Prompt decomposition and budgets (test infrastructure only).

decompose_prompt follows PAPER.md:548-551 (§III-C-2 a): the prompt is the fixed system
prompt (an exact, shared prefix), then the history (review) tokens, then one block
per candidate item in request order, then the instance-specific instruction tail, which is
always recomputed (FORCED). SPEC.md:62-70 gives the segment order and the worked example
(207 + 50 + 87 -> offsets 0, 207, 257, total 344).

Token classes (include/rc.h): PREFIX=0, FORCED=1, HIST=2, ITEM=3.
"""
from dataclasses import dataclass
import numpy as np

PREFIX, FORCED, HIST, ITEM = 0, 1, 2, 3


@dataclass
class Layout:
    tokens: np.ndarray     # int32 [n]
    cls: np.ndarray        # uint8 [n]
    src_id: np.ndarray     # int64 [n]: prototype id (HIST), item id (ITEM), -1 otherwise
    src_off: np.ndarray    # int32 [n]: offset inside the item block (ITEM), else 0
    seg_start: list        # segment start positions: prefix, history, item_1..item_k, tail
    cand_idtok: np.ndarray  # int32 [n_cand]: first (ID) token of every candidate, slot order

    @property
    def n(self) -> int:
        return int(self.tokens.shape[0])


def decompose_prompt(sys_tokens, hist_protos, hist_tokens, cand_items, cand_tokens, tail_tokens) -> Layout:
    """cand_tokens: list of int arrays, one per candidate (its catalog token ids)."""
    toks, cls, sid, soff, seg = [], [], [], [], []
    pos = 0
    seg.append(pos)
    for t in sys_tokens:
        toks.append(int(t)); cls.append(PREFIX); sid.append(-1); soff.append(0)
    pos += len(sys_tokens)
    seg.append(pos)
    for pi, t in zip(hist_protos, hist_tokens):
        toks.append(int(t)); cls.append(HIST); sid.append(int(pi)); soff.append(0)
    pos += len(hist_tokens)
    idtok = []
    for it, ct in zip(cand_items, cand_tokens):
        seg.append(pos)
        for j, t in enumerate(ct):
            toks.append(int(t)); cls.append(ITEM); sid.append(int(it)); soff.append(j)
        idtok.append(int(ct[0]))
        pos += len(ct)
    seg.append(pos)
    for t in tail_tokens:
        toks.append(int(t)); cls.append(FORCED); sid.append(-1); soff.append(0)
    return Layout(np.array(toks, np.int32), np.array(cls, np.uint8), np.array(sid, np.int64),
                  np.array(soff, np.int32), seg, np.array(idtok, np.int32))


def layout_from_request(req, catalog, sys_tokens) -> Layout:
    return decompose_prompt(sys_tokens, req.hist_protos, req.hist_tokens, req.cand_items,
                            [catalog.tokens[int(i)] for i in req.cand_items], req.tail_tokens)


def classify_tokens(layout: Layout, resident_items=None) -> Layout:
    """Item tokens of non-resident items become FORCED (PAPER.md:551 'cache misses are
    computed on-the-fly')."""
    if resident_items is None:
        return layout
    cls = layout.cls.copy()
    for p in range(layout.n):
        if cls[p] == ITEM and int(layout.src_id[p]) not in resident_items:
            cls[p] = FORCED
    return Layout(layout.tokens, cls, layout.src_id, layout.src_off, layout.seg_start, layout.cand_idtok)


def budget(r_bp: int, count: int) -> int:
    """k = ceil(r * count) with r in basis points."""
    return (int(r_bp) * int(count) + 9999) // 10000
