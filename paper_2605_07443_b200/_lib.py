"""ctypes binding of librc (include/rc.h). Argument marshalling only: every step of the hot
path runs in librc's CUDA kernels. Fails loudly when the library is missing -- there is no
CPU or eager fallback.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librc.so")

RC_OK, RC_E_INVALID, RC_E_NOMEM, RC_E_CAPACITY, RC_E_NOTFOUND, RC_E_EXISTS, RC_E_CUDA, RC_E_PEER, RC_E_UNSUPPORTED = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
RC_POOL_ITEM_BF16, RC_POOL_HIST_INT8, RC_POOL_PREFIX_BF16, RC_POOL_ITEM_HOST_BF16 = 0, 1, 2, 3
RC_TOK_PREFIX, RC_TOK_FORCED, RC_TOK_HIST, RC_TOK_ITEM = 0, 1, 2, 3
RC_MISS_ERROR, RC_MISS_RECOMPUTE = 0, 1

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
U64P = C.POINTER(C.c_uint64)
U8P = C.POINTER(C.c_uint8)


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32), ("rope_theta", C.c_double),
                ("rms_eps", C.c_float), ("qkv_bias", C.c_int32)]


class Weights(C.Structure):
    _fields_ = [("embed", P), ("final_norm", P), ("lm_head", P)] + \
        [(n, PP) for n in ("ln1", "wq", "wk", "wv", "bq", "bk", "bv", "wo", "ln2", "wg", "wu", "wd")]


class PoolDesc(C.Structure):
    _fields_ = [("item_rows", C.c_int64), ("remote_rows", C.c_int64), ("hist_rows", C.c_int64),
                ("prefix_rows", C.c_int64), ("arena_rows", C.c_int64), ("max_seq_len", C.c_int32),
                ("max_batch_tokens", C.c_int32), ("host_item_rows", C.c_int64)]


class Request(C.Structure):
    _fields_ = [("n", C.c_int32), ("token_ids", I32P), ("cls", U8P), ("src_id", I64P), ("src_off", I32P),
                ("prefix_id", C.c_uint64), ("n_cand", C.c_int32), ("cand_idtok", I32P), ("hist_proto_dev", C.c_void_p)]


class Prompt(C.Structure):
    _fields_ = [("prefix_len", C.c_int32), ("prefix_tokens", I32P), ("n_hist", C.c_int32), ("hist_proto", I64P),
                ("hist_tokens", I32P), ("n_cand", C.c_int32), ("cand_item", I64P), ("cand_len", I32P),
                ("cand_tokens", I32P), ("n_tail", C.c_int32), ("tail_tokens", I32P)]


RC_ATTN_AUTO, RC_ATTN_SINGLE, RC_ATTN_PAIRED, RC_ATTN_SPLIT2, RC_ATTN_ADAPTIVE, RC_ATTN_CHUNKED = 0, 1, 2, 3, 4, 5


class PrefillParams(C.Structure):
    _fields_ = [("r_rev_bp", C.c_int32), ("r_item_bp", C.c_int32), ("lambda_", C.c_float),
                ("check_layer", C.c_int32), ("window", C.c_int32), ("forced_sel", I32P), ("forced_sel_off", I32P),
                ("attn_kernel", C.c_int32), ("score_out", C.c_void_p), ("deterministic", C.c_int32),
                ("gradual_layers", C.c_int32), ("r_start_rev_bp", C.c_int32), ("r_start_item_bp", C.c_int32),
                ("sel_trace", C.c_void_p)]


_LIB = None


class RcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"librc error {code}: {msg}")
        self.code = code


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"librc.so not built at {LIB_PATH}; run python -m paper_2605_07443_b200.build "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        sig = {
            "rc_create": (C.c_int32, [C.POINTER(ModelDesc), C.POINTER(Weights), C.POINTER(PoolDesc), C.c_int32, C.POINTER(P)]),
            "rc_destroy": (None, [P]),
            "rc_last_error": (C.c_char_p, []),
            "rc_abi_version": (C.c_int32, []),
            "rc_decompose_prompt": (C.c_int32, [C.POINTER(Prompt), C.c_int32, I32P, I32P, U8P, I64P, I32P, I32P]),
            "rc_pool_register_blocks": (C.c_int32, [P, C.c_int32, C.c_int32, U64P, I32P, I32P, P, P, P]),
            "rc_pool_contains": (C.c_int32, [P, C.c_int32, C.c_int32, U64P, U8P]),
            "rc_pool_locate": (C.c_int32, [P, C.c_int32, U64P, I64P]),
            "rc_assemble": (C.c_int32, [P, C.c_int32, C.POINTER(Request), C.c_int32, C.c_int32, U64P, U64P, I32P, P]),
            "rc_sel_count": (C.c_int32, [P, C.c_int32, U64P, C.POINTER(PrefillParams), I32P]),
            "rc_selective_prefill": (C.c_int32, [P, C.c_int32, U64P, C.POINTER(PrefillParams), P, P, P, P, P]),
            "rc_release": (None, [P, C.c_int32, U64P]),
            "rc_pool_export": (C.c_int32, [P, P, I64P]),
            "rc_peer_attach": (C.c_int32, [P, C.c_int32, I32P, I32P, PP, I64P]),
            "rc_fetch_remote": (C.c_int32, [P, C.c_int32, U64P, I32P, P]),
            "rc_pool_list": (C.c_int32, [P, C.c_int32, U64P, I64P, I32P, I32P, I32P]),
            "rc_peer_directory": (C.c_int32, [P, C.c_int32, C.c_int32, U64P, I64P, I32P, I32P]),
            "rc_fetch_host": (C.c_int32, [P, C.c_int32, U64P, P]),
            "rc_semlib_build": (C.c_int32, [P, C.c_int32, I32P, I32P, C.c_int32, C.POINTER(C.c_float), C.c_uint64]),
            "rc_semlib_match": (C.c_int32, [P, C.c_int32, P, P, P, P, P]),
            "rc_seq_read_kv": (C.c_int32, [P, C.c_uint64, C.c_int32, P, P, P]),
            "rc_seq_export_kv": (C.c_int32, [P, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, P, P, P]),
            "rc_diag_deviation_select": (C.c_int32, [C.c_int32, C.c_int32, P, P, P, P, U8P, C.c_int32, C.c_int32,
                                                     C.c_int32, C.c_int32, P, P, I32P, P]),
            "rc_diag_gemm": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, P, P, P, C.c_int32, P]),
            "rc_diag_gemm_add": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, P, P, P, C.c_int32, P]),
            "rc_launch_count": (C.c_int64, [P]),
            "rc_device_error_count": (C.c_int64, [P]),
            "rc_place_items": (C.c_int32, [C.c_int32, I32P, C.c_int32, I64P, I32P, C.c_int32, C.c_int32, C.c_double,
                                           C.c_int32, I32P, I64P, I64P]),
            "rc_route": (C.c_int32, [C.c_int32, I64P, I32P, I64P, C.c_int32, C.c_int32, U8P, C.c_double, C.c_double,
                                     I64P, I32P]),
            "rc_profile_begin": (C.c_int32, [P]),
            "rc_profile_end": (C.c_int32, [P, C.c_int32, C.POINTER(C.c_double), I64P, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def check(code):
    if code != RC_OK:
        raise RcError(code, lib().rc_last_error().decode())
    return code


def np_ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


EXPORTED = ["rc_create", "rc_destroy", "rc_last_error", "rc_abi_version", "rc_decompose_prompt",
            "rc_pool_register_blocks", "rc_pool_contains", "rc_pool_locate", "rc_assemble", "rc_sel_count",
            "rc_selective_prefill", "rc_release", "rc_pool_export", "rc_peer_attach", "rc_fetch_remote",
            "rc_seq_read_kv", "rc_diag_deviation_select", "rc_diag_gemm", "rc_launch_count", "rc_profile_begin",
            "rc_profile_end", "rc_place_items", "rc_route", "rc_fetch_host", "rc_semlib_build", "rc_semlib_match",
            "rc_pool_list", "rc_peer_directory", "rc_seq_export_kv", "rc_diag_gemm_add",
            "rc_device_error_count"]
KINDS = ["gemm", "attention", "gather", "select", "small", "lm_head", "fetch"]
