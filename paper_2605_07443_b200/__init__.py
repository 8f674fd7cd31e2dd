"""B200-native RcLLM selective-attention prefill (arxiv 2605.07443).

The hot path lives in librc.so (csrc/, C-ABI in include/rc.h); `api` is the thin ctypes face.
"""
from ._lib import LIB_PATH, lib, RcError  # noqa: F401
from . import _lib as abi  # noqa: F401


def __getattr__(name):
    if name in ("RcContext", "diag_gemm", "diag_deviation_select"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
