"""ctypes binding of the C ABI in include/ss_b200.h (libss_b200.so, built in-tree).

This is the only way the package reaches the GPU. There is no CPU fallback: if the shared
library is missing, importing the executor raises immediately (build with
``python __graft_entry__.py`` or ``make -C paper_2507_03220_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SS_B200_LIB: load a differently built copy of the library (kernel-variant experiments)
LIB_PATH = os.environ.get("SS_B200_LIB") or os.path.join(_HERE, "libss_b200.so")

SS_OK = 0
SS_E_ARG = -1
SS_E_CUDA = -2
SS_E_NOLAYER = -3
SS_E_NOMEM = -4
SS_E_UNSUPPORTED = -5
SS_E_PROTOCOL = -6

SS_SEG_OK = 0
SS_SEG_BAD_WIDTH = 1
SS_SEG_BAD_PTR = 2
SS_SEG_NO_ADAPTER = 3
SS_SEG_UNSUPPORTED = 5

SS_GRADF_ACCUMULATE = 1 << 0
SS_GRADF_X_BF16 = 1 << 1
SS_GRADF_DY_BF16 = 1 << 2
SS_GRADF_BASE_BF16 = 1 << 3

SS_MEM_DEVICE = 1 << 0
SS_DT_BF16 = 1 << 1

SS_ADAPTER_LORA = 1
SS_ADAPTER_IA3 = 2

SS_SEGF_SRC_BF16 = 1 << 0
SS_SEGF_DST_BF16 = 1 << 1
SS_SEGF_BASE_BF16 = 1 << 2
SS_SEGF_ADAPTER = 1 << 3
SS_SEGF_PINNED = 1 << 4
SS_SEGF_CLASS_DECODE = 1 << 5
SS_SEGF_CLASS_PREFILL = 1 << 6

# Every symbol include/ss_b200.h declares (checked by tests/test_lib_abi.py).
EXPORTED = (
    "ss_ctx_create", "ss_ctx_destroy", "ss_last_error", "ss_version", "ss_load_layer",
    "ss_unload_layer", "ss_set_adapter", "ss_clear_adapter", "ss_clear_client",
    "ss_compute_batch", "ss_memory_stats", "ss_kernel_launches", "ss_set_option",
    "ss_profile", "ss_profile_read", "ss_adapter_grads", "ss_plan_create", "ss_plan_launch",
    "ss_plan_destroy", "ss_compute_batch_host", "ss_serve_frames", "ss_ctx_epoch",
    "ss_ipc_last_error", "ss_ipc_export", "ss_ipc_alloc", "ss_ipc_free", "ss_ipc_open",
    "ss_ipc_close", "ss_ipc_event_create", "ss_ipc_event_open", "ss_ipc_event_record",
    "ss_ipc_event_wait", "ss_ipc_event_sync", "ss_ipc_event_destroy",
    "ss_layer_dims", "ss_ctx_device", "ss_sched_create", "ss_sched_destroy", "ss_sched_set_policy",
    "ss_sched_register", "ss_sched_deregister", "ss_sched_submit", "ss_sched_wait",
    "ss_sched_request", "ss_sched_next_done", "ss_sched_log", "ss_sched_queued",
    "ss_sched_last_error",
)

SS_SCHED_NOLOCKSTEP = 0
SS_SCHED_LOCKSTEP = 1
SS_SCHED_OPPORTUNISTIC = 2
SS_REQ_BAD_PASS = 16
SS_REQ_BAD_ID = 17
SS_REQ_NO_LAYER = 18
SS_REQ_FAILED = 19

SS_KERNEL_GATHER = 0
SS_KERNEL_SHRINK = 1
SS_KERNEL_GEMM = 2
SS_KERNEL_GRAD = 3


class SsSeg(ctypes.Structure):
    _fields_ = [
        ("client_id", ctypes.c_uint32),
        ("rows", ctypes.c_uint32),
        ("width", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("src", ctypes.c_void_p),
        ("src_ld", ctypes.c_int64),
        ("dst", ctypes.c_void_p),
        ("dst_ld", ctypes.c_int64),
        ("dst_base", ctypes.c_void_p),
        ("base_ld", ctypes.c_int64),
    ]


class SsGradSeg(ctypes.Structure):
    _fields_ = [
        ("client_id", ctypes.c_uint32),
        ("rows", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("x", ctypes.c_void_p),
        ("x_ld", ctypes.c_int64),
        ("dy", ctypes.c_void_p),
        ("dy_ld", ctypes.c_int64),
        ("y_base", ctypes.c_void_p),
        ("base_ld", ctypes.c_int64),
        ("grad_a", ctypes.c_void_p),
        ("grad_b", ctypes.c_void_p),
        ("grad_l", ctypes.c_void_p),
    ]


class SsRequest(ctypes.Structure):
    _fields_ = [
        ("client_id", ctypes.c_uint32),
        ("pass_kind", ctypes.c_uint32),
        ("block", ctypes.c_int32),
        ("role", ctypes.c_int32),
        ("request_id", ctypes.c_uint64),
        ("seg", SsSeg),
        ("ready", ctypes.c_void_p),
    ]


class SsSchedPolicy(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("wait_per_token", ctypes.c_double),
        ("wait_cap", ctypes.c_double),
        ("max_batch_tokens", ctypes.c_int64),
    ]


class SsSchedRec(ctypes.Structure):
    _fields_ = [
        ("dispatch", ctypes.c_uint64),
        ("block", ctypes.c_int32),
        ("role", ctypes.c_int32),
        ("pass_kind", ctypes.c_int32),
        ("rows", ctypes.c_int32),
        ("wait_s", ctypes.c_double),
    ]


class SsIpcMem(ctypes.Structure):
    """ss_ipc_mem: an exported device buffer (CUDA IPC handle + offset in its allocation)."""
    _fields_ = [
        ("handle", ctypes.c_uint8 * 64),
        ("offset", ctypes.c_uint64),
        ("bytes", ctypes.c_uint64),
        ("device", ctypes.c_int32),
        ("reserved", ctypes.c_uint32),
    ]


class SsIpcEvt(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_uint8 * 64)]


class LibraryMissing(RuntimeError):
    """libss_b200.so is not built; the executor has no other compute path."""


class SsError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"ss_b200 error {code}: {message}")
        self.code = code


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: the CUDA extension is not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32
        sig = {
            "ss_ctx_create": (i32, [i32, i32, i32, ctypes.POINTER(vp)]),
            "ss_ctx_destroy": (i32, [vp]),
            "ss_last_error": (ctypes.c_char_p, [vp]),
            "ss_version": (ctypes.c_char_p, []),
            "ss_load_layer": (i32, [vp, i32, i32, i32, i32, vp, i64, vp, u32]),
            "ss_unload_layer": (i32, [vp, i32, i32]),
            "ss_set_adapter": (i32, [vp, u32, i32, i32, u32, i32, ctypes.c_float, vp, vp, vp, u32]),
            "ss_clear_adapter": (i32, [vp, u32, i32, i32]),
            "ss_clear_client": (i32, [vp, u32]),
            "ss_compute_batch": (i32, [vp, i32, i32, i32, i32, ctypes.POINTER(SsSeg), vp,
                                       ctypes.POINTER(ctypes.c_int32)]),
            "ss_adapter_grads": (i32, [vp, i32, i32, i32, ctypes.POINTER(SsGradSeg), vp,
                                       ctypes.POINTER(ctypes.c_int32)]),
            "ss_compute_batch_host": (i32, [vp, i32, i32, i32, i32, ctypes.POINTER(SsSeg), vp,
                                            ctypes.POINTER(ctypes.c_int32)]),
            "ss_serve_frames": (i32, [vp, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), vp,
                                      ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), vp]),
            "ss_plan_create": (i32, [vp, i32, i32, i32, i32, ctypes.POINTER(SsSeg),
                                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(vp)]),
            "ss_plan_launch": (i32, [vp, vp]),
            "ss_plan_destroy": (i32, [vp]),
            "ss_memory_stats": (i32, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                      ctypes.POINTER(i64)]),
            "ss_kernel_launches": (i64, [vp]),
            "ss_ctx_epoch": (ctypes.c_uint64, [vp]),
            "ss_set_option": (i32, [vp, ctypes.c_char_p, i64]),
            "ss_profile": (i32, [vp, i32]),
            "ss_profile_read": (i32, [vp, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64),
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
            "ss_layer_dims": (i32, [vp, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
            "ss_ctx_device": (i32, [vp]),
            "ss_sched_create": (i32, [vp, ctypes.POINTER(SsSchedPolicy), vp, ctypes.POINTER(vp)]),
            "ss_sched_destroy": (i32, [vp, i32]),
            "ss_sched_set_policy": (i32, [vp, ctypes.POINTER(SsSchedPolicy)]),
            "ss_sched_register": (i32, [vp, u32, i32]),
            "ss_sched_deregister": (i32, [vp, u32]),
            "ss_sched_submit": (i32, [vp, ctypes.POINTER(SsRequest), i32, ctypes.POINTER(ctypes.c_uint64)]),
            "ss_sched_wait": (i32, [vp, ctypes.c_uint64, vp, i64, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(i64)]),
            "ss_sched_request": (i32, [vp, ctypes.POINTER(SsRequest), vp, i64, ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(i64)]),
            "ss_sched_next_done": (i32, [vp, vp, i64, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(i64)]),
            "ss_sched_log": (i32, [vp, ctypes.POINTER(SsSchedRec), i32, ctypes.POINTER(i32)]),
            "ss_sched_queued": (i64, [vp]),
            "ss_sched_last_error": (ctypes.c_char_p, [vp]),
            "ss_ipc_last_error": (ctypes.c_char_p, []),
            "ss_ipc_export": (i32, [vp, ctypes.c_uint64, ctypes.POINTER(SsIpcMem)]),
            "ss_ipc_alloc": (i32, [i32, ctypes.c_uint64, ctypes.POINTER(vp), ctypes.POINTER(SsIpcMem)]),
            "ss_ipc_free": (i32, [vp]),
            "ss_ipc_open": (i32, [i32, ctypes.POINTER(SsIpcMem), ctypes.POINTER(vp)]),
            "ss_ipc_close": (i32, [vp]),
            "ss_ipc_event_create": (i32, [i32, ctypes.POINTER(vp), ctypes.POINTER(SsIpcEvt)]),
            "ss_ipc_event_open": (i32, [i32, ctypes.POINTER(SsIpcEvt), ctypes.POINTER(vp)]),
            "ss_ipc_event_record": (i32, [vp, vp]),
            "ss_ipc_event_wait": (i32, [vp, vp]),
            "ss_ipc_event_sync": (i32, [vp]),
            "ss_ipc_event_destroy": (i32, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check_ipc(rc: int) -> None:
    if rc != SS_OK:
        msg = load().ss_ipc_last_error() or b""
        raise SsError(rc, msg.decode("utf-8", "replace"))


def check(ctx, rc: int) -> None:
    if rc != SS_OK:
        lib = load()
        msg = lib.ss_last_error(ctx) if ctx else b"(no context)"
        raise SsError(rc, (msg or b"").decode("utf-8", "replace"))
