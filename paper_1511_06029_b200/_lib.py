"""ctypes declarations for include/qtt.h (argument marshalling only).

Loads the in-tree ``libqtt_b200.so``; there is no fallback -- if the library
is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqtt_b200.so")
# A/B experiments may point at another in-tree build of the same library
LIB_PATH = os.environ.get("QTT_LIB_PATH", LIB_PATH)

QTT_SUCCESS = 0
QTT_ERROR_INVALID_VALUE = 1
QTT_ERROR_NOT_SUPPORTED = 2
QTT_ERROR_OUT_OF_MEMORY = 3
QTT_ERROR_CUDA = 4

# every symbol include/qtt.h declares
SYMBOLS = (
    "qtt_status_string", "qtt_create", "qtt_create_ex", "qtt_plan_stages", "qtt_plan_stages_split", "qtt_apply", "qtt_workspace_size", "qtt_apply_ws",
    "qtt_apply_host", "qtt_get_info", "qtt_get_stage", "qtt_get_stage_split", "qtt_get_apply_plan", "qtt_set_fused", "qtt_set_stage_timing",
    "qtt_stage_times", "qtt_destroy", "qtt_morton_pack", "qtt_morton_unpack", "qtt_apply_grid",
    "qtt_product_create", "qtt_product_workspace_size", "qtt_product_apply", "qtt_product_apply_ws",
    "qtt_product_destroy", "qtt_compressed_matvec", "qtt_compressed_matvec_cores",
    "qtt_create_shard", "qtt_shard_apply", "qtt_shard_apply_ws", "qtt_shard_projection",
    "qtt_stage_super_core", "qtt_shard_set_peers", "qtt_shard_apply_fused", "qtt_shard_reduce",
    "qtt_ipc_alloc", "qtt_ipc_free", "qtt_ipc_get_handle", "qtt_ipc_open", "qtt_ipc_close",
)

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1511_06029_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    h = C.c_void_p
    st = C.c_int
    i64 = C.c_int64
    dp = C.c_void_p
    lib.qtt_status_string.restype = C.c_char_p
    lib.qtt_status_string.argtypes = [st]
    lib.qtt_create.restype = st
    lib.qtt_create.argtypes = [C.POINTER(h), C.c_int, C.POINTER(i64), C.POINTER(C.c_void_p)]
    lib.qtt_create_ex.restype = st
    lib.qtt_create_ex.argtypes = [C.POINTER(h), C.c_int, C.POINTER(i64), C.POINTER(C.c_void_p), C.c_int]
    ip = C.POINTER(C.c_int)
    lib.qtt_plan_stages.restype = st
    lib.qtt_plan_stages.argtypes = [C.c_int, C.POINTER(i64), C.c_size_t, C.c_int, ip, ip, ip, ip]
    lib.qtt_plan_stages_split.restype = st
    lib.qtt_plan_stages_split.argtypes = [C.c_int, C.POINTER(i64), C.c_size_t, C.c_int, ip, ip, ip, ip, ip]
    lib.qtt_apply.restype = st
    lib.qtt_apply.argtypes = [h, dp, dp, i64, C.c_void_p]
    lib.qtt_workspace_size.restype = st
    lib.qtt_workspace_size.argtypes = [h, i64, C.POINTER(C.c_size_t)]
    lib.qtt_apply_ws.restype = st
    lib.qtt_apply_ws.argtypes = [h, dp, dp, i64, dp, C.c_size_t, C.c_void_p]
    lib.qtt_apply_host.restype = st
    lib.qtt_apply_host.argtypes = [h, dp, dp, i64, C.c_void_p]
    lib.qtt_get_info.restype = st
    lib.qtt_get_info.argtypes = [h, C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(i64),
                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.qtt_get_stage.restype = st
    lib.qtt_get_stage.argtypes = [h, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.qtt_get_stage_split.restype = st
    lib.qtt_get_stage_split.argtypes = [h, C.c_int, C.c_int64, C.POINTER(C.c_int)]
    lib.qtt_set_fused.restype = st
    lib.qtt_set_fused.argtypes = [h, C.c_int]
    lib.qtt_get_apply_plan.restype = st
    lib.qtt_get_apply_plan.argtypes = [h, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                       C.c_void_p]
    lib.qtt_set_stage_timing.restype = st
    lib.qtt_set_stage_timing.argtypes = [h, C.c_int]
    lib.qtt_stage_times.restype = st
    lib.qtt_stage_times.argtypes = [h, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int)]
    for name in ("qtt_morton_pack", "qtt_morton_unpack"):
        fn = getattr(lib, name)
        fn.restype = st
        fn.argtypes = [dp, dp, C.c_int, C.c_int, i64, C.c_void_p]
    lib.qtt_apply_grid.restype = st
    lib.qtt_apply_grid.argtypes = [h, dp, dp, C.c_int, i64, C.c_void_p]
    lib.qtt_product_create.restype = st
    lib.qtt_product_create.argtypes = [C.POINTER(h), C.c_int, C.POINTER(h)]
    lib.qtt_product_workspace_size.restype = st
    lib.qtt_product_workspace_size.argtypes = [h, i64, C.POINTER(C.c_size_t)]
    lib.qtt_product_apply.restype = st
    lib.qtt_product_apply.argtypes = [h, dp, dp, i64, C.c_void_p]
    lib.qtt_product_apply_ws.restype = st
    lib.qtt_product_apply_ws.argtypes = [h, dp, dp, i64, dp, C.c_size_t, C.c_void_p]
    lib.qtt_product_destroy.restype = st
    lib.qtt_product_destroy.argtypes = [h]
    lib.qtt_compressed_matvec.restype = st
    lib.qtt_compressed_matvec.argtypes = [h, C.POINTER(i64), C.POINTER(C.c_void_p), dp, C.POINTER(i64), C.c_void_p]
    lib.qtt_compressed_matvec_cores.restype = st
    lib.qtt_compressed_matvec_cores.argtypes = [h, C.POINTER(i64), C.POINTER(C.c_void_p), dp, C.c_size_t,
                                                C.POINTER(i64), C.c_void_p]
    lib.qtt_create_shard.restype = st
    lib.qtt_create_shard.argtypes = [C.POINTER(h), C.c_int, C.POINTER(i64), C.POINTER(C.c_void_p), C.c_int, C.c_int]
    lib.qtt_shard_apply.restype = st
    lib.qtt_shard_apply.argtypes = [h, dp, dp, i64, C.c_void_p]
    lib.qtt_shard_apply_ws.restype = st
    lib.qtt_shard_apply_ws.argtypes = [h, dp, dp, i64, dp, C.c_size_t, C.c_void_p]
    lib.qtt_shard_projection.restype = st
    lib.qtt_shard_projection.argtypes = [C.c_int, C.POINTER(i64), C.POINTER(C.c_void_p), C.c_int, C.c_int, dp]
    lib.qtt_stage_super_core.restype = st
    lib.qtt_stage_super_core.argtypes = [C.c_int, C.POINTER(i64), C.POINTER(C.c_void_p), C.c_int, C.c_int, dp]
    lib.qtt_shard_set_peers.restype = st
    lib.qtt_shard_set_peers.argtypes = [h, C.POINTER(C.c_void_p), C.c_int]
    lib.qtt_shard_apply_fused.restype = st
    lib.qtt_shard_apply_fused.argtypes = [h, dp, i64, C.c_void_p]
    lib.qtt_shard_reduce.restype = st
    lib.qtt_shard_reduce.argtypes = [dp, dp, C.c_int, i64, C.c_void_p]
    vpp = C.POINTER(C.c_void_p)
    lib.qtt_ipc_alloc.restype = st
    lib.qtt_ipc_alloc.argtypes = [C.c_size_t, vpp]
    lib.qtt_ipc_free.restype = st
    lib.qtt_ipc_free.argtypes = [dp]
    lib.qtt_ipc_get_handle.restype = st
    lib.qtt_ipc_get_handle.argtypes = [dp, dp]
    lib.qtt_ipc_open.restype = st
    lib.qtt_ipc_open.argtypes = [dp, vpp]
    lib.qtt_ipc_close.restype = st
    lib.qtt_ipc_close.argtypes = [dp]
    lib.qtt_destroy.restype = st
    lib.qtt_destroy.argtypes = [h]
    _lib = lib
    return lib


class QttError(RuntimeError):
    def __init__(self, fn, code):
        self.code = code
        name = load().qtt_status_string(code).decode()
        super().__init__(f"{fn} failed: {name} ({code})")


def check(fn, code):
    if code != QTT_SUCCESS:
        raise QttError(fn, code)
