"""DeviceChannel — the co-located client <-> executor hand-off, device-resident.

Implements the reference channel duck type (transport.py:52-101: ``request(block, role,
pass_kind, payload) -> array``, ``register(sends_backward)``, ``deregister()``, ``close()``,
``reply_is_view``, ``extra_payload_copies``) over a per-client DEVICE exchange buffer that
follows SharedBuffer's rule (transport.py:28-49): capacity batch*seq*max_width elements,
grows to exactly the requested size and never shrinks. The request is written into the
request buffer, the executor reads it in place and writes the reply into a reply buffer of
the same size and rule, and the client receives a view of it — no host round trip. (The
reference reuses ONE buffer for both; the executor supports that too — aliased sources are
gathered before the GEMM writes — but two buffers let it read the request rows in place.)
When the client sits on another GPU the buffers live on the client's GPU and the executor reads/writes it over NVLink peer access
(the C ABI takes plain device pointers; enable peer access with ``enable_peer_access``).

Ordering (payload visible before the control message): the request carries a
CUDA event recorded after the payload write; the reply carries the executor's completion
event, and the client's stream waits on it before the view is read.
"""

from __future__ import annotations

import itertools
import queue

import numpy as np
import torch

from . import _lib
from .errors import ProtocolError, TransportError
from .protocol import PASS_BACKWARD, PASS_ERROR, Envelope, error_message

REQUEST_TIMEOUT_S = 60.0


class DeviceBuffer:
    """Grow-only device exchange tensor (SharedBuffer on the GPU)."""

    def __init__(self, capacity: int, dtype=torch.bfloat16, device="cuda"):
        self.dtype = dtype
        self.device = torch.device(device)
        self.buf = torch.empty(max(1, int(capacity)), dtype=dtype, device=self.device)
        self.resizes = 0

    @property
    def capacity(self) -> int:
        return self.buf.numel()

    def ensure(self, n: int) -> None:
        if n > self.capacity:
            self.buf = torch.empty(int(n), dtype=self.dtype, device=self.device)
            self.resizes += 1

    def view(self, rows: int, cols: int) -> torch.Tensor:
        return self.buf[: rows * cols].view(rows, cols)


def enable_peer_access(dev_a: int, dev_b: int) -> bool:
    """Let kernels on dev_a dereference dev_b's memory (NVLink peer path)."""
    if dev_a == dev_b:
        return True
    if not torch.cuda.can_device_access_peer(dev_a, dev_b):
        return False
    # torch enables peer access lazily for copies; touching a cross-device copy does it
    with torch.cuda.device(dev_a):
        a = torch.empty(1, device=f"cuda:{dev_b}")
        a.to(f"cuda:{dev_a}")
    return True


class DeviceChannel:
    reply_is_view = True

    def __init__(self, executor, client_id: int, batch_size: int, seq_len: int, max_width: int,
                 dtype=torch.bfloat16, device=None):
        self.executor = executor
        self.client_id = client_id
        self.max_width = max_width
        dev = device if device is not None else executor.device
        self.buffer = DeviceBuffer(batch_size * seq_len * max_width, dtype, dev)
        self.reply_buffer = DeviceBuffer(batch_size * seq_len * max_width, dtype, dev)
        self.base_buffer: DeviceBuffer | None = None
        self.extra_payload_copies = 0
        self.last_base: torch.Tensor | None = None
        self._replies: queue.Queue = queue.Queue()
        self._ids = itertools.count(1)
        self._ready_ev: torch.cuda.Event | None = None
        self._native_cache: dict = {}

    def register(self, sends_backward: bool = False) -> None:
        self.executor.register(self.client_id, sends_backward)

    def deregister(self) -> None:
        self.executor.deregister(self.client_id)

    def register_adapter(self, adapter, addresses=None) -> set:
        """Fuse this client's adapter into the executor; returns the fused addresses."""
        self.executor.register_adapter(self.client_id, adapter, addresses)
        return self.executor.fused_addresses(self.client_id)

    def request(self, block: int, role: int, pass_kind: int, payload, want_base: bool = False):
        if getattr(self.executor, "_native", None) is not None and isinstance(payload, torch.Tensor):
            return self._native_request(block, role, pass_kind, payload, want_base)
        rows, cols = int(payload.shape[0]), int(payload.shape[1])
        d_in, d_out = self.executor.layer_dims(block, role)
        out_cols = d_in if pass_kind == PASS_BACKWARD else d_out
        self.buffer.ensure(rows * self.max_width)
        self.reply_buffer.ensure(rows * self.max_width)
        sent = self.buffer.view(rows, cols)
        if isinstance(payload, torch.Tensor):
            if payload.data_ptr() != sent.data_ptr():
                sent.copy_(payload, non_blocking=True)
        else:
            sent.copy_(torch.from_numpy(np.ascontiguousarray(payload, dtype=np.float32)))
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.buffer.device))
        reply_to = self.reply_buffer.view(rows, out_cols)
        base_to = None
        if want_base and pass_kind != PASS_BACKWARD:
            if self.base_buffer is None:
                self.base_buffer = DeviceBuffer(self.buffer.capacity, self.buffer.dtype, self.buffer.device)
            self.base_buffer.ensure(rows * self.max_width)
            base_to = self.base_buffer.view(rows, out_cols)
        env = Envelope(self.client_id, next(self._ids), block, role, pass_kind, sent,
                       reply_to=reply_to, base_to=base_to, ready=ready)
        self.executor.submit(env, self._deliver)
        try:
            kind, value = self._replies.get(timeout=REQUEST_TIMEOUT_S)
        except queue.Empty:
            raise TransportError("timed out waiting for executor reply") from None
        if kind == "error":
            raise ProtocolError(value)
        if value is not None:
            torch.cuda.current_stream(self.buffer.device).wait_event(value)
        self.last_base = base_to
        return reply_to

    def _native_request(self, block, role, pass_kind, payload, want_base):
        """The native scheduler's path (GpuBaseExecutor(scheduler="native")): one library call
        queues the request and returns once its batch is launched, the GIL released meanwhile;
        the request struct of a recurring (layer, pass, shape) is built once."""
        from .device import Seg, seg_fields
        from .sched import pack_request, status_message
        ex = self.executor
        rows, cols = int(payload.shape[0]), int(payload.shape[1])
        dims = ex._dims.get((int(block), int(role)))
        expected, out_cols = (None, cols) if dims is None else \
            ((dims[1], dims[0]) if pass_kind == PASS_BACKWARD else (dims[0], dims[1]))
        self.buffer.ensure(rows * self.max_width)
        self.reply_buffer.ensure(rows * self.max_width)
        want_base = bool(want_base) and pass_kind != PASS_BACKWARD
        if want_base:
            if self.base_buffer is None:
                self.base_buffer = DeviceBuffer(self.buffer.capacity, self.buffer.dtype, self.buffer.device)
            self.base_buffer.ensure(rows * self.max_width)
        key = (block, role, pass_kind, rows, cols, want_base, payload.dtype, self.buffer.resizes,
               self.reply_buffer.resizes, self.base_buffer.resizes if want_base else -1, ex._fused_ver)
        hit = self._native_cache.get(key)
        if hit is None:
            if len(self._native_cache) > 1024:
                self._native_cache.clear()
            sent = self.buffer.view(rows, cols)
            reply_to = self.reply_buffer.view(rows, out_cols)
            base_to = self.base_buffer.view(rows, out_cols) if want_base else None
            req = _lib.SsRequest()
            if self._ready_ev is None:
                self._ready_ev = torch.cuda.Event()
                self._ready_ev.record(torch.cuda.current_stream(self.buffer.device))
            fields = seg_fields(Seg(self.client_id, sent, reply_to, base_to,
                                    adapter=(int(block), int(role)) in ex._fused.get(self.client_id, ())))
            pack_request(memoryview(req).cast("B"), self.client_id, pass_kind, block, role, 0, fields,
                         int(self._ready_ev.cuda_event))
            hit = self._native_cache[key] = (sent, reply_to, base_to, req)
        sent, reply_to, base_to, req = hit
        stream = torch.cuda.current_stream(self.buffer.device)
        if payload.data_ptr() != sent.data_ptr():
            sent.copy_(payload, non_blocking=True)
        self._ready_ev.record(stream)
        req.request_id = next(self._ids)
        try:
            status, aux = ex._native.request(req, stream.cuda_stream, REQUEST_TIMEOUT_S)
        except TimeoutError:
            raise TransportError("timed out waiting for executor reply") from None
        if status != _lib.SS_SEG_OK:
            env = Envelope(self.client_id, req.request_id, block, role, pass_kind, sent)
            raise ProtocolError(status_message(status, aux, env, expected, ex._native))
        self.last_base = base_to
        return reply_to

    def _deliver(self, reply: Envelope) -> None:
        if reply.pass_kind == PASS_ERROR:
            self._replies.put(("error", error_message(reply)))
        else:
            self._replies.put(("ok", reply.done))

    def close(self) -> None:
        pass
