"""ctypes loader for libactnn.so (the C ABI declared in include/actnn.h).

Argument marshalling only.  The library is built in-tree by
``paper_2104_14129_b200/csrc/Makefile`` (``__graft_entry__.build()``); if it
is missing this module raises -- there is no fallback implementation.
"""
from __future__ import annotations

import ctypes
import os
import re
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libactnn.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "actnn.h")

_lib = None
_lock = threading.Lock()

P = ctypes.c_void_p
I32, I64, U32, U64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
SIZE = ctypes.c_size_t

# name -> (restype, argtypes), mirroring include/actnn.h
SIGNATURES = {
    "actnn_last_error": (ctypes.c_char_p, []),
    "actnn_abi_version": (ctypes.c_int, []),
    "actnn_workspace_bytes": (SIZE, [ctypes.c_int, I64, I64, I32]),
    "actnn_packed_bytes": (I64, [I64, I64, I32, P]),
    "actnn_group_stats": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, P, P, P, SIZE, P]),
    "actnn_allocate_bits": (ctypes.c_int, [P, P, I64, I64, U32, I64, I32, P, P, P, SIZE, P]),
    "actnn_uniform_bits": (ctypes.c_int, [I64, I64, I32, I32, P, P, P]),
    "actnn_quantize": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, P, U64, I64, P, P, P,
                                      P, P, P]),
    "actnn_dequantize": (ctypes.c_int, [P, P, P, P, P, I64, I64, I32, P, ctypes.c_int, P]),
    "actnn_quantize_bf16meta": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, P, U64, I64,
                                               P, P, P, P, P]),
    "actnn_dequantize_bf16meta": (ctypes.c_int, [P, P, P, P, I64, I64, I32, P, ctypes.c_int,
                                                 P]),
    "actnn_relu_pack": (ctypes.c_int, [P, ctypes.c_int, I64, P, P, P]),
    "actnn_relu_backward": (ctypes.c_int, [P, P, ctypes.c_int, I64, P, P]),
    "actnn_maxpool2d_forward": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I64] + [I32] * 8
                                + [P, P, P]),
    "actnn_maxpool2d_backward": (ctypes.c_int, [P, P, ctypes.c_int, I64, I64, I64] + [I32] * 8
                                 + [P, P]),
    "actnn_grad_sqnorm": (ctypes.c_int, [P, ctypes.c_int, I64, I64, I32, P, P, SIZE, P]),
    "actnn_gradmag_ema": (ctypes.c_int, [P, I64, ctypes.c_double, P, P]),
    "actnn_gradmag_gather": (ctypes.c_int, [P, I64, P, I64, P, P]),
    "actnn_gradmag_scatter": (ctypes.c_int, [P, I64, P, P, I64, P]),
    "actnn_allocate_layers_ws_bytes": (SIZE, [I64, I64, U32]),
    "actnn_allocate_layers": (ctypes.c_int, [P, P, P, P, I64, I64, I64, U32, P, P, P, SIZE, P]),
}


class ActnnError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"actnn status {status}: {message}")
        self.status = status


def header_symbols():
    """Function names declared in include/actnn.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(actnn_[a-z0-9_]+)\s*\(", txt)))


def load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ActnnError(-4, f"{LIB_PATH} is missing: build it with "
                                 "`python -c 'import __graft_entry__ as g; g.build()'` "
                                 "(no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int):
    if status != 0:
        msg = load().actnn_last_error()
        raise ActnnError(status, msg.decode() if msg else "")
