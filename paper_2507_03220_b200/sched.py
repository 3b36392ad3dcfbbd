"""NativeScheduler — the executor's batch formation on a C++ thread (ss_sched_*, csrc/ss_sched.cu).

The reference's executor forms batches in a Python scheduler thread (executor.py:162-178
``submit``, 235-283 ``_loop`` / ``_pick_ready``, 285-300 ``_dispatch``); ``GpuBaseExecutor``
keeps that loop (scheduler="python"). With scheduler="native" the same policies run in the
library: a request is one ctypes call that blocks without the GIL until its batch is launched,
so tens of client threads no longer serialise on the interpreter. Request statuses map back to
the reference's error messages here (``status_message``).
"""

from __future__ import annotations

import ctypes
import struct

import torch

from . import _lib
from ._lib import SsRequest, SsSchedPolicy, SsSchedRec

_MODES = {"nolockstep": _lib.SS_SCHED_NOLOCKSTEP, "lockstep": _lib.SS_SCHED_LOCKSTEP,
          "opportunistic": _lib.SS_SCHED_OPPORTUNISTIC}
_REQ_FMT = struct.Struct("<IIiiQ4IQqQqQqQ")     # ss_request (include/ss_b200.h)
assert _REQ_FMT.size == ctypes.sizeof(SsRequest)


def policy_struct(policy) -> SsSchedPolicy:
    """Any BatchPolicy-like object (ours or the reference's, executor.py:32-56)."""
    return SsSchedPolicy(_MODES[policy.mode], 0, float(policy.wait_per_token), float(policy.wait_cap),
                         int(policy.max_batch_tokens))


def raw_event(ev) -> int:
    """cudaEvent_t of a torch.cuda.Event or an ipc.IpcEvent (0: none)."""
    if ev is None:
        return 0
    if hasattr(ev, "cuda_event"):
        return int(ev.cuda_event)
    ptr = getattr(ev, "_ptr", None)
    return int(ptr.value or 0) if ptr is not None else 0


def pack_request(buf, client_id, pass_kind, block, role, request_id, seg_fields, ready) -> None:
    """Fill an SsRequest in place; ``seg_fields`` = device.seg_fields(...) (client_id first)."""
    _REQ_FMT.pack_into(buf, 0, client_id, pass_kind, block, role, request_id, *seg_fields, ready)


def status_message(status: int, aux: int, env_like, expected: int | None, scheduler=None) -> str:
    """The reference's message for a rejected request (executor.py:162-178, 196-213)."""
    if status == _lib.SS_REQ_BAD_PASS:
        return f"unknown pass {env_like.pass_kind}"
    if status == _lib.SS_REQ_BAD_ID:
        return f"request_id {env_like.request_id} not increasing (last {aux})"
    if status == _lib.SS_REQ_NO_LAYER:
        return f"unknown layer {env_like.layer}"
    if status == _lib.SS_SEG_BAD_WIDTH:
        return f"row width {env_like.width} does not match layer {env_like.layer} expected {expected}"
    if status == _lib.SS_REQ_FAILED:
        why = scheduler.last_error() if scheduler is not None else ""
        return f"executor failure: {why}"
    return f"executor rejected segment (status {status}) for layer {env_like.layer}"


CUDA_STREAM_LEGACY = 0x1   # cudaStreamLegacy: the legacy default stream as an explicit handle


def stream_handle(cuda_stream):
    """The handle to give the scheduler's ``wait_stream`` for a torch ``Stream.cuda_stream``.

    The C ABI reads NULL as "no stream to order" (ss_b200.h, ss_sched_wait), while torch reports
    its default stream -- the legacy default stream -- as 0: passed through, a client on the
    default stream would read its reply before the batch's kernels finished. None stays "no
    wait"; 0 becomes cudaStreamLegacy."""
    if cuda_stream is None:
        return None
    return int(cuda_stream) or CUDA_STREAM_LEGACY


class NativeScheduler:
    def __init__(self, ctx, policy, stream: torch.cuda.Stream | None = None):
        self.lib = ctx.lib
        self.ctx = ctx
        pol = policy_struct(policy)
        h = ctypes.c_void_p()
        raw = stream.cuda_stream if stream is not None else None
        _lib.check(ctx.h, self.lib.ss_sched_create(ctx.h, ctypes.byref(pol), raw, ctypes.byref(h)))
        self.h = h
        self._status = ctypes.c_int32()
        self._aux = ctypes.c_int64()

    def set_policy(self, policy) -> None:
        pol = policy_struct(policy)
        self.lib.ss_sched_set_policy(self.h, ctypes.byref(pol))

    def register(self, client_id: int, sends_backward: bool) -> None:
        self.lib.ss_sched_register(self.h, int(client_id), 1 if sends_backward else 0)

    def deregister(self, client_id: int) -> None:
        self.lib.ss_sched_deregister(self.h, int(client_id))

    def submit(self, req: SsRequest, notify: bool = True) -> int:
        t = ctypes.c_uint64()
        rc = self.lib.ss_sched_submit(self.h, ctypes.byref(req), 1 if notify else 0, ctypes.byref(t))
        if rc != _lib.SS_OK:
            raise _lib.SsError(rc, "ss_sched_submit")
        return t.value

    def request(self, req: SsRequest, wait_stream: int, timeout_s: float) -> tuple[int, int]:
        """Queue + block until launched (GIL released); ``wait_stream`` then waits for the batch."""
        st, aux = ctypes.c_int32(), ctypes.c_int64()
        rc = self.lib.ss_sched_request(self.h, ctypes.byref(req), stream_handle(wait_stream), int(timeout_s * 1e6),
                                       ctypes.byref(st), ctypes.byref(aux))
        if rc == 1:
            raise TimeoutError("timed out waiting for executor reply")
        if rc != _lib.SS_OK:
            raise _lib.SsError(rc, "ss_sched_request")
        return st.value, aux.value

    def next_done(self, wait_stream: int, timeout_s: float):
        """(ticket, status, aux) of the next completed notify-request, or None on timeout."""
        t, st, aux = ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_int64()
        rc = self.lib.ss_sched_next_done(self.h, stream_handle(wait_stream), int(timeout_s * 1e6), ctypes.byref(t),
                                         ctypes.byref(st), ctypes.byref(aux))
        if rc == 1:
            return None
        if rc != _lib.SS_OK:
            raise _lib.SsError(rc, "ss_sched_next_done")
        return t.value, st.value, aux.value

    def drain_log(self) -> list:
        """[(dispatch, block, role, pass, rows, wait_s)] since the last call."""
        out = []
        cap = 4096
        arr = (SsSchedRec * cap)()
        n = ctypes.c_int32()
        while True:
            self.lib.ss_sched_log(self.h, arr, cap, ctypes.byref(n))
            out.extend((r.dispatch, r.block, r.role, r.pass_kind, r.rows, r.wait_s) for r in arr[: n.value])
            if n.value < cap:
                return out

    def queued(self) -> int:
        return int(self.lib.ss_sched_queued(self.h))

    def last_error(self) -> str:
        return (self.lib.ss_sched_last_error(self.h) or b"").decode("utf-8", "replace")

    def close(self, drain: bool = True) -> None:
        if self.h:
            self.lib.ss_sched_destroy(self.h, 1 if drain else 0)
            self.h = None
