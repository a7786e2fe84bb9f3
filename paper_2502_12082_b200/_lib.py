"""ctypes loader for libentmax_attn.so (the C ABI declared in include/entmax_attn.h and
include/entmax_rowwise.h).

The library is built in-tree (``make`` at the repo root, or ``__graft_entry__.build()``).
If it is missing or fails to load, every entry point raises: there is no fallback path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ENTMAX_ATTN_LIB: diagnostics only (e.g. the -DENTMAX_TRACE build under tests/probe)
LIB_PATH = os.environ.get("ENTMAX_ATTN_LIB", os.path.join(_HERE, "libentmax_attn.so"))

ENTMAX_OK, ENTMAX_ERR_INVALID_ARG, ENTMAX_ERR_UNSUPPORTED, ENTMAX_ERR_WORKSPACE, ENTMAX_ERR_CUDA = range(5)
ENTMAX_BF16, ENTMAX_FP32 = 0, 1


class EntmaxAttnError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


class Shape(ctypes.Structure):
    """entmax_shape_t"""
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("N", ctypes.c_int32), ("d", ctypes.c_int32),
                ("sb", ctypes.c_int64), ("sh", ctypes.c_int64), ("sn", ctypes.c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `make` (or __graft_entry__.build()); "
                          "this package has no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, f32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_float
    pshape = ctypes.POINTER(Shape)
    L.entmax_attn_status_string.restype = ctypes.c_char_p
    L.entmax_attn_status_string.argtypes = [i32]
    L.entmax_attn_last_error.restype = ctypes.c_char_p
    L.entmax_attn_last_error.argtypes = []
    L.entmax_attn_block_size.restype = ctypes.c_int
    L.entmax_attn_block_size.argtypes = [ctypes.c_int32, ctypes.c_int, ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_int32)]
    for fn in (L.entmax_attn_fwd_workspace_bytes, L.entmax_attn_bwd_workspace_bytes):
        fn.restype = sz
        fn.argtypes = [pshape, i32, i32]
    L.entmax_attn_fwd.restype = i32
    L.entmax_attn_fwd.argtypes = [vp, vp, vp, pshape, i32, f32, i32, i32, f32,
                                  vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.entmax_attn_bwd.restype = i32
    L.entmax_attn_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, pshape, i32, f32, i32, f32,
                                  vp, vp, vp, vp, sz, vp]
    L.entmax_attn_profile_enable.restype = None
    L.entmax_attn_profile_enable.argtypes = [i32]
    L.entmax_attn_profile_reset.restype = None
    L.entmax_attn_profile_reset.argtypes = []
    L.entmax_attn_profile_collect.restype = i32
    L.entmax_attn_profile_collect.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_int32),
                                              ctypes.POINTER(ctypes.c_double), i32]
    L.entmax_attn_impl_for.restype = i32
    L.entmax_attn_impl_for.argtypes = [pshape, i32]
    i64 = ctypes.c_int64
    L.entmax_attn_pack_mask.restype = i32
    L.entmax_attn_pack_mask.argtypes = [vp, i64, ctypes.c_int32, vp, vp]
    L.entmax_rowwise_fwd.restype = i32          # include/entmax_rowwise.h
    L.entmax_rowwise_fwd.argtypes = [vp, i64, ctypes.c_int32, i64, i32, f32, i32, i32, vp, vp, vp]
    L.entmax_rowwise_bwd.restype = i32
    L.entmax_rowwise_bwd.argtypes = [vp, vp, i64, ctypes.c_int32, i64, i32, f32, vp, vp]
    _lib = L
    return L


def check(status: int, where: str):
    if status != ENTMAX_OK:
        L = lib()
        detail = L.entmax_attn_last_error().decode() or L.entmax_attn_status_string(status).decode()
        raise EntmaxAttnError(status, where, detail)
