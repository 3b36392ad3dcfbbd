"""Cross-process device hand-off: client processes share their exchange buffers with the
executor process through CUDA IPC instead of serialising payloads through host memory.

The paper's co-located mode shares one pre-allocated CUDA tensor between a client process and
the executor process (``share_memory_()`` / ``rebuild_cuda_tensor()``). The
reference package's process mode (harness.py:243-260 ``_process_worker``, :367-394
``_run_processes``) instead connects each client process with ``RemoteChannel`` to an
``ExecutorServer`` (transport.py:104-275), which frames every payload (LSV1) through host memory
and a socket. This module keeps that process topology and those two duck types:

* ``IpcChannel(host, port, client_id, ...)`` — the ``RemoteChannel`` surface (``register``,
  ``deregister``, ``request``, ``close``, ``reply_is_view``, ``extra_payload_copies``). Its
  request / reply / y_base buffers are device buffers owned by the client process, grow-only
  like ``SharedBuffer`` (transport.py:28-49), exported once per grow (``ss_ipc_alloc``);
* ``IpcExecutorServer(executor, host, port)`` — the ``ExecutorServer`` surface (``start``,
  ``stop``, ``host``, ``port``, context manager). It maps each client's buffers once
  (``ss_ipc_open``) and submits envelopes whose payload / reply / y_base are views into the
  client's memory, so the executor's kernels read the request rows and write the reply rows
  in place: no host staging, no frames. A client on another GPU is mapped as peer memory and
  served over NVLink (the executor's peer-GPU routing, channel.py).

Only small control messages (envelope header fields, buffer / event handles, acks) cross the
socket (``multiprocessing.connection`` with an HMAC handshake: a mapped buffer is device memory
of the client, so only holders of the server's ``authkey`` may connect). Ordering (SPEC.md:465,
payload visible before the control message): the client records an interprocess event after
writing the request and the executor's stream waits on it; the executor records its own
interprocess event after the reply and the client's stream waits on that before the view is
read. A request is synchronous per client (as in the reference), so both buffers are free
again when the next request is sent.
"""

from __future__ import annotations

import ctypes
import itertools
import os
import threading
from multiprocessing.connection import Client, Listener

import numpy as np
import torch

from . import _lib
from .errors import ProtocolError, TransportError
from .protocol import PASS_BACKWARD, PASS_ERROR, Envelope, error_message

REQUEST_TIMEOUT_S = 60.0
_DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}
_TAGS = {v: k for k, v in _DTYPES.items()}


# ---------------------------------------------------------------------------- raw memory
class _Cai:
    """__cuda_array_interface__ over a raw device pointer (torch.as_tensor keeps it alive)."""

    def __init__(self, ptr: int, nbytes: int, owner=None):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 2}
        self.owner = owner


def _tensor_at(ptr: int, nbytes: int, dtype: torch.dtype, owner=None) -> torch.Tensor:
    return torch.as_tensor(_Cai(ptr, nbytes, owner)).view(dtype)


def _mem_bytes(m: _lib.SsIpcMem) -> bytes:
    return bytes(ctypes.string_at(ctypes.addressof(m), ctypes.sizeof(m)))


def _mem_from(b: bytes) -> _lib.SsIpcMem:
    m = _lib.SsIpcMem()
    ctypes.memmove(ctypes.addressof(m), b, ctypes.sizeof(m))
    return m


class IpcEvent:
    """Interprocess CUDA event. ``wait(stream)`` makes it usable as ``Envelope.ready`` and with
    ``torch.cuda.Stream.wait_event`` (duck typed)."""

    def __init__(self, device: int, handle: bytes | None = None):
        lib = _lib.load()
        self.device = device
        self._ptr = ctypes.c_void_p()
        if handle is None:
            h = _lib.SsIpcEvt()
            _lib.check_ipc(lib.ss_ipc_event_create(device, ctypes.byref(self._ptr), ctypes.byref(h)))
            self.handle = bytes(h.handle)
        else:
            h = _lib.SsIpcEvt()
            ctypes.memmove(h.handle, handle, 64)
            _lib.check_ipc(lib.ss_ipc_event_open(device, ctypes.byref(h), ctypes.byref(self._ptr)))
            self.handle = bytes(handle)

    @staticmethod
    def _raw(stream) -> int:
        if stream is None:
            return 0
        return int(stream.cuda_stream)

    def record(self, stream=None) -> None:
        _lib.check_ipc(_lib.load().ss_ipc_event_record(self._ptr, self._raw(stream)))

    def wait(self, stream=None) -> None:
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        _lib.check_ipc(_lib.load().ss_ipc_event_wait(self._raw(stream), self._ptr))

    def synchronize(self) -> None:
        _lib.check_ipc(_lib.load().ss_ipc_event_sync(self._ptr))

    def close(self) -> None:
        if self._ptr.value:
            _lib.load().ss_ipc_event_destroy(self._ptr)
            self._ptr = ctypes.c_void_p()


class IpcBuffer:
    """Client side: a grow-only device exchange buffer (SharedBuffer, transport.py:28-49) in its
    own allocation, exportable to another process."""

    def __init__(self, capacity: int, dtype=torch.bfloat16, device: int = 0):
        self.dtype = dtype
        self.device = int(device)
        self.resizes = 0
        self._ptr = ctypes.c_void_p()
        self.buf: torch.Tensor | None = None
        self.mem: bytes = b""
        self._alloc(max(1, int(capacity)))

    def _alloc(self, n: int) -> None:
        esz = torch.empty((), dtype=self.dtype).element_size()
        ptr, m = ctypes.c_void_p(), _lib.SsIpcMem()
        _lib.check_ipc(_lib.load().ss_ipc_alloc(self.device, n * esz, ctypes.byref(ptr), ctypes.byref(m)))
        self._ptr = ptr
        self.buf = _tensor_at(ptr.value, n * esz, self.dtype)
        self.mem = _mem_bytes(m)

    @property
    def capacity(self) -> int:
        return self.buf.numel()

    def ensure(self, n: int):
        """Grow to exactly ``n`` elements if needed; returns the old allocation (free it with
        ``release`` once the executor has unmapped it) or None."""
        if n <= self.capacity:
            return None
        old = (self._ptr, self.buf)
        self._alloc(int(n))
        self.resizes += 1
        return old

    @staticmethod
    def release(old) -> None:
        if old is not None and old[0].value:
            torch.cuda.synchronize()
            _lib.load().ss_ipc_free(old[0])

    def view(self, rows: int, cols: int) -> torch.Tensor:
        return self.buf[: rows * cols].view(rows, cols)

    def close(self) -> None:
        self.release((self._ptr, self.buf))
        self._ptr, self.buf = ctypes.c_void_p(), None


class _Mapped:
    """Executor side: one client buffer mapped into this process."""

    def __init__(self, device: int, mem: bytes, dtype: torch.dtype):
        m = _mem_from(mem)
        self._ptr = ctypes.c_void_p()
        _lib.check_ipc(_lib.load().ss_ipc_open(device, ctypes.byref(m), ctypes.byref(self._ptr)))
        self.nbytes = int(m.bytes)
        self.dtype = dtype
        self.tensor = _tensor_at(self._ptr.value, self.nbytes, dtype)

    def view(self, rows: int, cols: int) -> torch.Tensor:
        if rows * cols > self.tensor.numel():
            raise ProtocolError(f"request of {rows}x{cols} exceeds the exported buffer "
                                f"({self.tensor.numel()} elements)")
        return self.tensor[: rows * cols].view(rows, cols)

    def close(self) -> None:
        if self._ptr.value:
            self.tensor = None
            _lib.load().ss_ipc_close(self._ptr)
            self._ptr = ctypes.c_void_p()


# ---------------------------------------------------------------------------- client side
class _ExecutorProxy:
    """What ``fusion.fuse_client_model`` / ``VirtLayer`` need of ``channel.executor``:
    adapter (re-)registration and layer dims, carried over the control connection."""

    def __init__(self, channel: "IpcChannel"):
        self._ch = channel
        self.device = channel.device

    def layer_dims(self, block: int, role: int) -> tuple[int, int]:
        return self._ch._dims[(int(block), int(role))]

    def register_adapter(self, client_id: int, adapter, addresses=None) -> None:
        from .config import addr_key
        lora = {addr_key(a): (np.asarray(v[0], np.float32), np.asarray(v[1], np.float32))
                for a, v in (getattr(adapter, "lora", {}) or {}).items()}
        ia3 = {addr_key(a): np.asarray(v, np.float32) for a, v in (getattr(adapter, "ia3", {}) or {}).items()}
        keys = None if addresses is None else sorted(addr_key(a) for a in addresses)
        reply = self._ch._call(("adapter", lora, ia3, float(adapter.alpha), int(adapter.rank), keys))
        self._ch._fused = set(reply[1])

    refresh_adapter = register_adapter

    def deregister_adapter(self, client_id: int) -> None:
        self._ch._call(("adapter_clear",))
        self._ch._fused = set()

    def fused_addresses(self, client_id: int) -> set:
        return set(self._ch._fused)


class IpcChannel:
    """RemoteChannel's surface (transport.py:104-161) over CUDA-IPC-shared device buffers.

    ``request`` accepts a numpy payload (the reference ClientModel's f32 activations: copied
    into the device request buffer, the reply read back to numpy) or a CUDA tensor (a GPU
    client: device-to-device write, the reply returned as a view of the reply buffer, valid
    until the next request — ``reply_is_view``)."""

    reply_is_view = True

    def __init__(self, host: str, port: int, client_id: int, timeout: float = REQUEST_TIMEOUT_S,
                 *, authkey: bytes | None = None, batch_size: int = 1, seq_len: int = 1,
                 dtype=torch.bfloat16, device: int | None = None):
        self.client_id = int(client_id)
        self.timeout = timeout
        self.extra_payload_copies = 0
        self._ids = itertools.count(1)
        self._fused: set = set()
        if authkey is None:
            authkey = os.environ.get("SS_IPC_AUTHKEY", "").encode() or None
        try:
            self._conn = Client((host, int(port)), authkey=authkey)
        except OSError as exc:
            raise TransportError(f"connect to {host}:{port} failed: {exc}") from exc
        self.device = int(device if device is not None else torch.cuda.current_device())
        self._ready = IpcEvent(self.device)
        try:
            hello = self._call(("hello", self.client_id, self._ready.handle, os.getpid()))
        except ProtocolError:
            self._ready.close()
            self._conn.close()
            raise
        _, self.max_width, self.executor_device, done_handle, dims = hello
        self._dims = {tuple(k): tuple(v) for k, v in dims}
        self._done = IpcEvent(self.device, done_handle)
        cap = batch_size * seq_len * self.max_width
        self.dtype = dtype
        self.buffer = IpcBuffer(cap, dtype, self.device)
        self.reply_buffer = IpcBuffer(cap, dtype, self.device)
        self.base_buffer: IpcBuffer | None = None
        self.last_base: torch.Tensor | None = None
        for slot, b in (("req", self.buffer), ("rep", self.reply_buffer)):
            self._call(("map", slot, b.mem, _TAGS[dtype]))
        self.executor = _ExecutorProxy(self)

    # -- control ----------------------------------------------------------------------
    def _call(self, msg):
        try:
            self._conn.send(msg)
            if not self._conn.poll(self.timeout):
                raise TransportError("timed out waiting for executor reply")
            reply = self._conn.recv()
        except (OSError, EOFError) as exc:
            raise TransportError(f"transport failure: {exc}") from exc
        if reply[0] == "err":
            raise ProtocolError(reply[-1])
        return reply

    def register(self, sends_backward: bool = False) -> None:
        self._call(("register", bool(sends_backward)))

    def deregister(self) -> None:
        self._call(("deregister",))

    def register_adapter(self, adapter, addresses=None) -> set:
        self.executor.register_adapter(self.client_id, adapter, addresses)
        return set(self._fused)

    def _grow(self, slot: str, buf: IpcBuffer, n: int) -> None:
        old = buf.ensure(n)
        if old is not None:
            self._call(("map", slot, buf.mem, _TAGS[buf.dtype]))   # the executor unmapped the old one
            IpcBuffer.release(old)

    # -- data -------------------------------------------------------------------------
    def request(self, block: int, role: int, pass_kind: int, payload, want_base: bool = False):
        rows, cols = int(payload.shape[0]), int(payload.shape[1])
        dims = self._dims.get((int(block), int(role)))
        out_cols = (dims[0] if pass_kind == PASS_BACKWARD else dims[1]) if dims else cols
        self._grow("req", self.buffer, rows * self.max_width)
        self._grow("rep", self.reply_buffer, rows * self.max_width)
        want_base = bool(want_base) and pass_kind != PASS_BACKWARD
        if want_base:
            if self.base_buffer is None:
                self.base_buffer = IpcBuffer(self.buffer.capacity, self.dtype, self.device)
                self._call(("map", "base", self.base_buffer.mem, _TAGS[self.dtype]))
            self._grow("base", self.base_buffer, rows * self.max_width)
        stream = torch.cuda.current_stream(self.device)
        sent = self.buffer.view(rows, cols)
        is_torch = isinstance(payload, torch.Tensor)
        if is_torch:
            if payload.data_ptr() != sent.data_ptr():
                sent.copy_(payload, non_blocking=True)
        else:
            sent.copy_(torch.from_numpy(np.ascontiguousarray(payload, dtype=np.float32)))
        self._ready.record(stream)
        request_id = next(self._ids)
        reply = self._call(("req", request_id, int(block), int(role), int(pass_kind), rows, cols, want_base))
        if reply[0] == "fail":
            raise ProtocolError(reply[2])
        if reply[1] != request_id:
            raise ProtocolError(f"reply id {reply[1]} does not match request {request_id}")
        self._done.wait(stream)
        out = self.reply_buffer.view(rows, out_cols)
        self.last_base = self.base_buffer.view(rows, out_cols) if want_base else None
        if is_torch:
            return out
        if want_base:
            self.last_base = self.last_base.float().cpu().numpy()
        return out.float().cpu().numpy()

    def close(self) -> None:
        conn = getattr(self, "_conn", None)
        if conn is None:
            return
        try:
            self._call(("close",))
        except (TransportError, ProtocolError):
            pass
        try:
            conn.close()
        except OSError:
            pass
        self._conn = None
        for b in (self.buffer, self.reply_buffer, self.base_buffer):
            if b is not None:
                b.close()
        self._ready.close()
        self._done.close()


# ---------------------------------------------------------------------------- executor side
class _Adapter:
    def __init__(self, lora, ia3, alpha, rank):
        self.lora, self.ia3, self.alpha, self.rank = lora, ia3, alpha, rank


class IpcExecutorServer:
    """ExecutorServer's surface (transport.py:164-275) for IpcChannel clients: accepts many
    connections and multiplexes them onto one executor. A client disconnect fails only that
    client (its registration is dropped, its mappings closed once the executor is done with
    them); the executor and the other connections are unaffected."""

    def __init__(self, executor, host: str = "127.0.0.1", port: int = 0, authkey: bytes | None = None):
        self.executor = executor
        self.authkey = authkey if authkey is not None else os.urandom(16)
        self._listener = Listener((host, port), authkey=self.authkey)
        self.host, self.port = self._listener.address
        dev = executor.device
        self.device = dev if isinstance(dev, int) else (torch.device(dev).index or 0)
        self._threads: list[threading.Thread] = []
        self._conns: list = []
        self._lock = threading.Lock()
        self._running = False
        self.requests_served = 0

    def start(self) -> "IpcExecutorServer":
        self._running = True
        t = threading.Thread(target=self._accept_loop, daemon=True, name="ipc-server-accept")
        t.start()
        self._threads.append(t)
        return self

    def _accept_loop(self) -> None:
        while self._running:
            try:
                conn = self._listener.accept()
            except Exception:   # noqa: BLE001 — AuthenticationError (wrong key), EOF, closed listener
                if not self._running:
                    return
                continue   # a failed handshake refuses that connection only
            with self._lock:
                self._conns.append(conn)
            t = threading.Thread(target=self._serve_conn, args=(conn,), daemon=True, name="ipc-server-conn")
            t.start()
            self._threads.append(t)

    def _serve_conn(self, conn) -> None:
        ex = self.executor
        send_lock = threading.Lock()
        mapped: dict[str, _Mapped] = {}
        client_id = None
        registered = False
        ready = None
        done = IpcEvent(self.device)
        side = torch.cuda.Stream(self.device)     # records `done` behind the dispatch's completion

        def send(msg) -> None:
            with send_lock:
                try:
                    conn.send(msg)
                except OSError:
                    pass

        def quiesce() -> None:
            done.synchronize()
            side.synchronize()

        try:
            while True:
                try:
                    msg = conn.recv()
                except (EOFError, OSError):
                    break
                op = msg[0]
                if op == "hello":
                    if msg[3] == os.getpid():
                        # CUDA IPC handles cannot be opened by the process that exported them
                        send(("err", "IpcChannel needs a client in another process "
                                     "(in-process clients use DeviceChannel)"))
                        break
                    client_id = int(msg[1])
                    ready = IpcEvent(self.device, msg[2])
                    dims = [(k, v) for k, v in ex._dims.items()]
                    width = max(max(v) for v in ex._dims.values())
                    send(("hello", width, self.device, done.handle, dims))
                elif op == "register":
                    ex.register(client_id, sends_backward=bool(msg[1]))
                    registered = True
                    send(("ack",))
                elif op == "deregister":
                    ex.deregister(client_id)
                    registered = False
                    send(("ack",))
                elif op == "map":
                    _, slot, mem, tag = msg
                    quiesce()
                    old = mapped.pop(slot, None)
                    if old is not None:
                        old.close()
                    try:
                        mapped[slot] = _Mapped(self.device, mem, _DTYPES[tag])
                    except Exception as exc:   # noqa: BLE001 — reported to this client only
                        send(("err", f"cannot map {slot} buffer: {exc}"))
                        continue
                    send(("ack",))
                elif op == "adapter":
                    _, lora, ia3, alpha, rank, keys = msg
                    try:
                        ex.register_adapter(client_id, _Adapter(lora, ia3, alpha, rank), keys)
                    except Exception as exc:   # noqa: BLE001
                        send(("err", str(exc)))
                        continue
                    send(("ack", sorted(ex.fused_addresses(client_id))))
                elif op == "adapter_clear":
                    ex.deregister_adapter(client_id)
                    send(("ack",))
                elif op == "req":
                    self._request(msg, client_id, mapped, ready, done, side, send)
                elif op == "close":
                    send(("ack",))
                    break
                else:
                    send(("err", f"unknown control message {op!r}"))
        finally:
            if client_id is not None and registered:
                ex.deregister(client_id)
            try:
                quiesce()
            except Exception:   # noqa: BLE001
                pass
            for m in mapped.values():
                m.close()
            done.close()
            if ready is not None:
                ready.close()
            try:
                conn.close()
            except OSError:
                pass

    def _request(self, msg, client_id, mapped, ready, done, side, send) -> None:
        _, request_id, block, role, pass_kind, rows, cols, want_base = msg
        ex = self.executor
        try:
            src = mapped["req"].view(rows, cols)
            dims = ex._dims.get((block, role))
            reply_to = base_to = None
            if dims is not None:
                out_cols = dims[0] if pass_kind == PASS_BACKWARD else dims[1]
                reply_to = mapped["rep"].view(rows, out_cols)
                if want_base:
                    base_to = mapped["base"].view(rows, out_cols)
        except (ProtocolError, KeyError) as exc:
            send(("fail", request_id, str(exc)))
            return
        env = Envelope(client_id, request_id, block, role, pass_kind, src,
                       reply_to=reply_to, base_to=base_to, ready=ready)

        def reply_fn(reply: Envelope) -> None:
            if reply.pass_kind == PASS_ERROR:
                send(("fail", reply.request_id, error_message(reply)))
                return
            if reply.done is not None:
                side.wait_event(reply.done)
            else:
                side.wait_stream(torch.cuda.current_stream(self.device))
            done.record(side)
            self.requests_served += 1
            send(("ok", reply.request_id))

        ex.submit(env, reply_fn)

    def stop(self) -> None:
        self._running = False
        try:
            self._listener.close()
        except OSError:
            pass
        with self._lock:
            for conn in self._conns:
                try:
                    conn.close()
                except OSError:
                    pass
        for t in self._threads:
            t.join(timeout=2.0)

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.stop()
