"""ctypes loader for libroundpipe_b200.so (the product C-ABI, include/rp/*.h).

The library is built in-tree by ``make`` (``__graft_entry__.build()``); there
is no Python or PyTorch fallback for anything it exports — a missing library
is an ImportError at first use.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# RP_LIB: an alternative build of the same library (same-box A/B measurements)
LIB_PATH = os.environ.get("RP_LIB") or os.path.join(_HERE, "libroundpipe_b200.so")
_lock = threading.Lock()
_lib: C.CDLL | None = None


class NativeError(RuntimeError):
    """A non-zero status from the C-ABI (code follows include/rp/cabi.h)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[rp status {code}] {msg}")
        self.code = code


class InputError(NativeError, ValueError):
    pass


class InfeasibleError(NativeError):
    pass


class ProtocolViolation(NativeError):
    pass


class CapExceededError(NativeError):
    pass


class CudaError(NativeError):
    pass


_ERRORS = {2: InputError, 3: InfeasibleError, 4: ProtocolViolation,
           5: CapExceededError, 6: CudaError}


def load(path: str = LIB_PATH) -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None or path != LIB_PATH:
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} not built; run `make` (or __graft_entry__.build())")
            lib = C.CDLL(path)
            if path != LIB_PATH:
                return lib
            _lib = lib
        return _lib


def check(lib: C.CDLL, prefix: str, code: int) -> int:
    if code != 0:
        msg = getattr(lib, prefix + "last_error")
        msg.restype = C.c_char_p
        text = (msg() or b"").decode(errors="replace")
        raise _ERRORS.get(code, NativeError)(code, text)
    return code
