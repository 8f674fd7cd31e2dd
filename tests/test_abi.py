"""The C-ABI library loads and exports every symbol include/rc.h declares; host-only entry
points agree with the oracle (not gpu: no compute calls need a device)."""
import os
import re

import numpy as np
import pytest

import rcgen
from oracle.layout import decompose_prompt, layout_from_request

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2605_07443_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2605_07443_b200.build import build
        build()
    return _lib


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "rc.h")).read()
    return sorted(set(re.findall(r"^\s*(?:rc_status|void|const char\*|int32_t|int64_t)\s+(rc_\w+)\(", txt, re.M)))


def test_exports_match_header():
    L = _lib()
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(L.EXPORTED) == syms
    assert lib.rc_abi_version() == 1


def test_decompose_prompt_worked_example(golden):
    _lib()
    from paper_2605_07443_b200.api import RcContext
    g = golden("layout_spec68.json")
    out = RcContext.decompose_prompt(np.zeros(g["instruction"]), np.arange(50), np.ones(50), [7],
                                     [np.arange(87) + 3], np.zeros(0))
    assert list(out["seg_start"][:3]) == g["segment_offsets"] and len(out["tokens"]) == g["total"]


@pytest.mark.parametrize("wl", [rcgen.CFG1, rcgen.CFG1_Q7, rcgen.CFG2])
def test_decompose_matches_oracle(wl):
    _lib()
    from paper_2605_07443_b200.api import RcContext
    cat, protos, sys_tok = rcgen.gen_catalog(wl), rcgen.gen_protos(wl), rcgen.gen_system_prompt(wl)
    for r in rcgen.gen_requests(wl, cat, protos, 3):
        ref = layout_from_request(r, cat, sys_tok)
        out = RcContext.decompose_prompt(sys_tok, r.hist_protos, r.hist_tokens, r.cand_items,
                                         [cat.tokens[int(i)] for i in r.cand_items], r.tail_tokens)
        assert np.array_equal(out["tokens"], ref.tokens) and np.array_equal(out["cls"], ref.cls)
        assert np.array_equal(out["src_id"][ref.cls >= 2], ref.src_id[ref.cls >= 2])
        assert np.array_equal(out["src_off"], ref.src_off)
        assert list(out["seg_start"]) == ref.seg_start and np.array_equal(out["cand_idtok"], ref.cand_idtok)


def test_error_paths_without_device():
    L = _lib()
    import ctypes as C
    lib = L.lib()
    # invalid prompt: negative lengths -> RC_E_INVALID, message set
    pr = L.Prompt()
    pr.prefix_len = -1
    n = C.c_int32()
    assert lib.rc_decompose_prompt(C.byref(pr), 0, C.byref(n), None, None, None, None, None) == L.RC_E_INVALID
    assert b"negative" in lib.rc_last_error()
    # null context arguments fail cleanly
    assert lib.rc_create(None, None, None, 0, None) == L.RC_E_INVALID
    assert lib.rc_sel_count(None, 0, None, None, None) == L.RC_E_INVALID
