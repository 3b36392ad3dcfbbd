"""GpuBaseExecutor — drop-in for splitserve.executor.BaseExecutor on one B200.

Same surface as the reference (pkg/src/splitserve/executor.py:95-300): constructor
``(layers, policy=None, save_activations=False)``, ``start/stop`` / context manager,
``register/deregister``, ``submit(env, reply_fn)``, ``serve_forward / serve_backward /
serve_noise_effect``, attributes ``layers, policy, metrics, ledger``. Validation messages,
batch formation (FIFO segment order, pass-keyed queues, the three policies) and the
error-isolation rule ("a malformed envelope fails alone") are the reference's.

What changes is ``_compute_batch``: instead of concat -> einsum -> split on the host it
builds one segment table and makes ONE C-ABI call (ss_compute_batch), which gathers the
segments on the device, runs the tcgen05 GEMM with each client's LoRA / IA3 delta fused in
the epilogue, and scatters every segment straight into its destination. Adapters move
executor-side through a new control call, ``register_adapter`` (SURVEY §7 "adapter
registration needs a new control message").

Payloads may be host arrays (numpy / CPU tensors: staged through pinned memory, results
returned as numpy f32 like the reference) or device tensors (zero-copy; results are device
tensors, written into ``env.reply_to`` when the client supplies its exchange buffer).
"""

from __future__ import annotations

import csv
import os
import threading
import time
import weakref
from collections import defaultdict, deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ledger as ledger_mod
from .config import Role, addr_key
from .device import Seg, SegmentTable, SsContext
from .errors import ConfigError, ProtocolError
from .protocol import (COMPUTE_PASSES, PASS_BACKWARD, PASS_FORWARD, PASS_NOISE_EFFECT,
                       Envelope, error_envelope)
from . import _lib

POLICY_MODES = ("nolockstep", "lockstep", "opportunistic")


@dataclass
class BatchPolicy:
    """Dispatch policy (executor.py:32-56): a queue ripens for
    min(wait_cap, wait_per_token * smallest member's tokens) or until max_batch_tokens."""

    mode: str = "opportunistic"
    wait_per_token: float = 0.0001
    wait_cap: float = 0.050
    max_batch_tokens: int = 8192
    dispatch_cost: float = 0.0

    def __post_init__(self):
        if self.mode not in POLICY_MODES:
            raise ConfigError(f"unknown policy mode {self.mode!r}")
        if self.wait_per_token < 0 or self.wait_cap < 0:
            raise ConfigError("wait durations must be non-negative")

    def wait_budget(self, token_counts) -> float:
        return min(self.wait_cap, self.wait_per_token * min(token_counts))


@dataclass
class ExecutorMetrics:
    """Per-(block, role, pass) dispatch records (executor.py:59-92)."""

    batch_sizes: dict = field(default_factory=lambda: defaultdict(list))
    batch_tokens: dict = field(default_factory=lambda: defaultdict(list))
    wait_times: dict = field(default_factory=lambda: defaultdict(list))
    dispatches: int = 0

    def record(self, key, size: int, tokens: int, waits) -> None:
        self.batch_sizes[key].append(size)
        self.batch_tokens[key].append(tokens)
        self.wait_times[key].extend(waits)
        self.dispatches += 1

    def mean_batch_size(self) -> float:
        sizes = [s for v in self.batch_sizes.values() for s in v]
        return float(np.mean(sizes)) if sizes else 0.0

    def max_wait(self) -> float:
        return max((w for v in self.wait_times.values() for w in v), default=0.0)

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            out = csv.writer(fh)
            out.writerow(["block", "role", "pass", "batch_size", "tokens", "mean_wait_s"])
            for key in sorted(self.batch_sizes):
                block, role, pass_kind = key
                waits = self.wait_times[key]
                mean_wait = float(np.mean(waits)) if waits else 0.0
                for size, tokens in zip(self.batch_sizes[key], self.batch_tokens[key]):
                    out.writerow([block, Role(role).name, pass_kind, size, tokens, mean_wait])


@dataclass
class _LayerShape:
    d_in: int
    d_out: int

    @property
    def nbytes(self) -> int:
        return 2 * self.d_in * self.d_out + 4 * self.d_out


class Dispatch:
    """A prebuilt dispatch over fixed device buffers: one ss_plan (routing tables built once,
    resident on the device), so each ``run`` is a kernel launch sequence with no table work.

    For device-resident clients whose exchange buffers do not move (DeviceChannel after its
    first grow). ``run`` is capturable in a CUDA graph (``GpuBaseExecutor.capture``)."""

    def __init__(self, ctx: SsContext, pass_kind: int, key, segs, segments=None, lock=None):
        self.ctx, self.pass_kind, self.key = ctx, pass_kind, key
        self._lock = lock if lock is not None else threading.RLock()
        self.segments = segments          # the (client, src, dst, base) tuples it was built from
        self.plan = ctx.plan(pass_kind, key[0], key[1], segs)
        self.rows = sum(int(s.src.shape[0]) for s in segs)
        bad = [s for s in self.plan.status if s != _lib.SS_SEG_OK]
        if bad:
            raise ProtocolError(f"dispatch {self.key} pass {self.pass_kind}: segment status {bad}")

    def run(self, stream: torch.cuda.Stream | None = None) -> None:
        with self._lock:
            self.plan.launch(stream)


class CapturedStep:
    """A sequence of prebuilt dispatches captured as one CUDA graph (``GpuBaseExecutor.capture``).

    Captured kernels bake the context's workspace / LoRA-pack / IA3 addresses. Any later call
    that frees or moves one of them (a larger eager dispatch growing the workspace, an adapter
    rank / kind / scale change, ...) moves ``ss_ctx_epoch``; ``replay`` then re-captures
    (eagerly running the dispatches once, which rebuilds their plans) instead of replaying
    freed memory. Adapter VALUE refreshes at the same rank write the packs in place and need
    no re-capture."""

    def __init__(self, executor: "GpuBaseExecutor", dispatches, stream: torch.cuda.Stream | None = None):
        self.executor = executor
        self.dispatches = list(dispatches)
        self.stream = stream if stream is not None else torch.cuda.Stream(executor.device)
        self.graph: torch.cuda.CUDAGraph | None = None
        self.epoch = -1
        self.recaptures = -1
        self._capture()

    def _capture(self) -> None:
        ex, s = self.executor, self.stream
        with ex._lock, torch.cuda.device(ex.device):
            self.graph = None          # (the old graph's memory may be what just moved)
            for d in self.dispatches:
                d.run(s)
            torch.cuda.synchronize(ex.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for d in self.dispatches:
                    d.run(s)
            self.graph = g
            self.epoch = ex.ctx.epoch()
            self.recaptures += 1

    @property
    def stale(self) -> bool:
        return self.executor.ctx.epoch() != self.epoch

    def replay(self) -> None:
        with self.executor._lock:
            if self.stale:
                self._capture()
            self.graph.replay()


def _is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def _out_dtype(payload) -> torch.dtype:
    if isinstance(payload, torch.Tensor) and payload.dtype == torch.bfloat16:
        return torch.bfloat16
    return torch.float32


def _host_tensor_info(t: torch.Tensor):
    """(dtype, shape) of a contiguous pinned-host bf16/f32 tensor, else None. Cached per tensor
    object by the executor (a tensor's placement, dtype and shape do not change)."""
    if t.is_cuda or t.dtype not in (torch.bfloat16, torch.float32) or not t.is_contiguous() or not t.is_pinned():
        return None
    return (t.dtype, tuple(t.shape))


def _host_tensor(a: np.ndarray) -> torch.Tensor:
    """Zero-copy CPU tensor over a numpy array (read-only arrays too: the library only reads
    request rows)."""
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)   # non-writable arrays (frozen payloads)
        return torch.from_numpy(a)


def _cached_info(cache: dict, t: torch.Tensor):
    hit = cache.get(id(t))
    ptr = t.data_ptr()
    if hit is not None and hit[0]() is t and hit[2] == ptr:    # same object, same storage
        return hit[1]
    if len(cache) > 4096:
        cache.clear()
    v = _host_tensor_info(t)
    cache[id(t)] = (weakref.ref(t), v, ptr)
    return v


class GpuBaseExecutor:
    """Stateless layer server: one scheduler thread, compute on the B200 via libss_b200."""

    def __init__(self, layers, policy: BatchPolicy | None = None, save_activations: bool = False,
                 *, device: int = 0, stream: torch.cuda.Stream | None = None,
                 context: SsContext | None = None, retain_layers: bool = True,
                 scheduler: str | None = None):
        """``layers``: mapping (or iterable of pairs) LayerAddress -> AffineParams. Weights are
        copied to the device as bf16 (bias f32). With ``retain_layers=False`` the host-side
        parameters are dropped after upload (``layers`` then holds shape-only records), so a
        generator of pairs streams a large model through without a second copy.

        ``scheduler``: "python" (the reference's scheduler loop in a Python thread) or "native"
        (batch formation and dispatch on a library thread, ss_sched_*: same policies, same
        messages; client threads block without the GIL). Default: $SS_SCHEDULER or "native"."""
        self.policy = policy or BatchPolicy()
        scheduler = scheduler or os.environ.get("SS_SCHEDULER", "native")
        if scheduler not in ("python", "native"):
            raise ConfigError(f"unknown scheduler {scheduler!r}")
        self.scheduler = scheduler
        self._native = None                 # NativeScheduler while started (scheduler="native")
        self._native_pending: dict = {}     # ticket -> (env, reply_fn, dst, host_reply, expected)
        self._native_thread: threading.Thread | None = None
        self.save_activations = save_activations
        # Serialises every call into the library context: the scheduler thread's dispatches,
        # adapter (re-)registration from client threads, plans, graphs, gradient jobs. The
        # library itself is single-threaded per context (pack growth frees what a concurrent
        # table build would read).
        self._lock = threading.RLock()
        self._saved_debug: list = []
        self.ctx = context if context is not None else SsContext(device)
        self.device = self.ctx.device
        self.stream = stream
        self._dims: dict[tuple[int, int], tuple[int, int]] = {}
        self.layers = {}
        for addr, params in (layers.items() if hasattr(layers, "items") else layers):
            key = addr_key(addr)
            self.ctx.load_layer(key[0], key[1], params.weight, getattr(params, "bias", None))
            self._dims[key] = (int(params.weight.shape[0]), int(params.weight.shape[1]))
            self.layers[addr] = params if retain_layers else _LayerShape(*self._dims[key])
        self._fused: dict[int, set] = defaultdict(set)   # client -> {(block, role)} fused
        self._queues: dict[tuple, deque] = defaultdict(deque)
        self._cond = threading.Condition()
        self._clients: dict[int, bool] = {}
        self._last_request_id: dict[int, int] = {}
        self._running = False
        self._thread: threading.Thread | None = None
        self._metrics = ExecutorMetrics()
        self.ledger = ledger_mod.MemoryLedger("executor")
        self._pinned: dict[str, torch.Tensor] = {}
        self._np_pool: list = []         # (pinned tensor, its numpy base) reply arrays (_numpy_out)
        # pinned-host checks of client payload / reply tensors, per live tensor object:
        # id -> (weakref, info) (tensors compare elementwise, so they cannot be dict keys)
        self._host_info: dict[int, tuple] = {}
        # recurring host dispatches (decode: the same client buffers every step) -> their packed
        # segment table; see _host_memo_get
        self._host_memo: dict[tuple, tuple] = {}
        self._fused_ver = 0
        self._dev_staging: dict = {}
        self._host_replies: list = []
        self.last_event: torch.cuda.Event | None = None
        self._sync_ledger()

    # -- lifecycle ------------------------------------------------------------------------
    def start(self) -> "GpuBaseExecutor":
        with self._cond:
            if self._running:
                return self
            self._running = True
        if self.scheduler == "native":
            from .sched import NativeScheduler
            # a torch stream object, so staged request tensors can be tied to it (record_stream)
            self._native_stream = self.stream if self.stream is not None else torch.cuda.Stream(self.device)
            self._native = NativeScheduler(self.ctx, self.policy, self._native_stream)
            for cid, bwd in self._clients.items():
                self._native.register(cid, bwd)
            self._reply_stream = torch.cuda.Stream(self.device)
            self._native_thread = threading.Thread(target=self._native_completions, daemon=True,
                                                   name="gpu-base-executor-replies")
            self._native_thread.start()
            return self
        self._thread = threading.Thread(target=self._loop, daemon=True, name="gpu-base-executor")
        self._thread.start()
        return self

    def stop(self, drain: bool = True) -> None:
        if self._native is not None:
            if drain:
                while self._native.queued() or self._native_pending:
                    time.sleep(0.005)
            with self._cond:
                self._running = False
            self._native_thread.join()
            self._native_thread = None
            self._pull_native_log()
            self._native.close(drain=False)
            self._native = None
            return
        if drain:
            with self._cond:
                while self._running and any(self._queues.values()):
                    self._cond.wait(0.01)
        with self._cond:
            self._running = False
            self._cond.notify_all()
        if self._thread is not None:
            self._thread.join()
            self._thread = None

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.stop()

    def close(self) -> None:
        self.stop(drain=False)
        self.ctx.close()

    # -- registry -------------------------------------------------------------------------
    def register(self, client_id: int, sends_backward: bool = False) -> None:
        with self._cond:
            self._clients[client_id] = sends_backward
            if self._native is not None:
                self._native.register(client_id, sends_backward)
            self._cond.notify_all()

    def deregister(self, client_id: int) -> None:
        with self._cond:
            self._clients.pop(client_id, None)
            if self._native is not None:
                self._native.deregister(client_id)
            self._cond.notify_all()
        self._host_memo.clear()   # (drops the memo's references to the client's buffers)

    def layer_dims(self, block: int, role: int) -> tuple[int, int]:
        return self._dims[(int(block), int(role))]

    # -- adapters (new control surface) ---------------------------------------------------
    def register_adapter(self, client_id: int, adapter, addresses=None) -> None:
        """Move a client's adapter executor-side. ``adapter`` is AdapterState-like
        (adapters.py:44-60: ``lora {addr: (A, B)}``, ``ia3 {addr: l}``, ``alpha``, ``rank``).
        Call again after every optimizer step to refresh the device copy. From then on the
        client must NOT apply the adapter itself on these addresses (client.py:206-209)."""
        with self._lock:
            self._register_adapter(client_id, adapter, addresses)

    def _register_adapter(self, client_id: int, adapter, addresses) -> None:
        lora = getattr(adapter, "lora", {}) or {}
        ia3 = getattr(adapter, "ia3", {}) or {}
        keys = {addr_key(a) for a in list(lora) + list(ia3)}
        if addresses is not None:
            keys &= {addr_key(a) for a in addresses}
        by_key_lora = {addr_key(a): v for a, v in lora.items()}
        by_key_ia3 = {addr_key(a): v for a, v in ia3.items()}
        for key in sorted(keys):
            if key not in self._dims:
                raise ConfigError(f"adapter targets unknown layer {key}")
            lo = None
            if key in by_key_lora:
                a, b = by_key_lora[key]
                lo = (a, b, float(adapter.alpha) / float(adapter.rank))
            self.ctx.set_adapter(client_id, key[0], key[1], lora=lo, ia3=by_key_ia3.get(key))
            if key not in self._fused[client_id]:
                self._fused[client_id].add(key)
                self._fused_ver += 1
        self._sync_ledger()

    refresh_adapter = register_adapter

    def deregister_adapter(self, client_id: int) -> None:
        with self._lock:
            self.ctx.clear_adapter(client_id)
            self._fused.pop(client_id, None)
            self._fused_ver += 1
            self._host_memo.clear()
            self._sync_ledger()

    def fused_addresses(self, client_id: int) -> set:
        return set(self._fused.get(client_id, ()))

    def compile_dispatch(self, pass_kind: int, block: int, role: int, segments) -> Dispatch:
        """Prebuild a dispatch: ``segments`` = [(client_id, src, dst, base_or_None)] over
        device tensors, in batch order. Adapters registered for (client, layer) are fused."""
        key = (int(block), int(role))
        if key not in self._dims:
            raise ProtocolError(f"unknown layer {key}")
        segs = [Seg(client_id=c, src=src, dst=dst,
                    base=base if pass_kind != PASS_BACKWARD else None,
                    adapter=key in self._fused.get(c, ()))
                for c, src, dst, base in segments]
        with self._lock:
            return Dispatch(self.ctx, pass_kind, key, segs, list(segments), self._lock)

    def capture(self, dispatches, stream: torch.cuda.Stream | None = None) -> CapturedStep:
        """Capture a sequence of prebuilt dispatches into one CUDA graph (replay = one launch
        for the whole sequence). Runs them once eagerly first so every plan's workspace is at
        its high-water mark. The returned ``CapturedStep.replay()`` re-captures by itself when
        the context freed or moved anything the graph references since (ss_ctx_epoch)."""
        return CapturedStep(self, dispatches, stream)

    def adapter_grads(self, block: int, role: int, jobs, stream: torch.cuda.Stream | None = None) -> list:
        """LoRA / IA3 weight gradients of one layer on the GPU (ss_adapter_grads) for the
        client-side half of ``_layer_backward`` (client.py:286-305): ``jobs`` is a list of
        ``device.GradSeg``. Returns one status per job (0 = computed)."""
        key = (int(block), int(role))
        if key not in self._dims:
            raise ProtocolError(f"unknown layer {key}")
        with self._lock:
            return self.ctx.adapter_grads(key[0], key[1], jobs, stream)

    def _sync_ledger(self) -> None:
        w, a, _ = self.ctx.memory_stats()
        self.ledger.set(ledger_mod.WEIGHTS, w)
        self.ledger.set(ledger_mod.ADAPTER, a)

    # -- intake ---------------------------------------------------------------------------
    def submit(self, env, reply_fn) -> None:
        if self._native is not None:
            self._native_submit(env, reply_fn)
            return
        if env.pass_kind not in COMPUTE_PASSES:
            reply_fn(error_envelope(env, f"unknown pass {env.pass_kind}"))
            return
        with self._cond:
            last = self._last_request_id.get(env.client_id)
            if last is not None and env.request_id <= last:
                bad = f"request_id {env.request_id} not increasing (last {last})"
            else:
                bad = None
                self._last_request_id[env.client_id] = env.request_id
        if bad is not None:
            reply_fn(error_envelope(env, bad))
            return
        if (int(env.block), int(env.role)) not in self._dims:
            reply_fn(error_envelope(env, f"unknown layer {env.layer}"))
            return
        with self._cond:
            self._queues[(env.block, env.role, env.pass_kind)].append((env, reply_fn, time.monotonic()))
            self._cond.notify_all()

    # -- native scheduler (scheduler="native") ---------------------------------------------
    @property
    def metrics(self) -> ExecutorMetrics:
        self._pull_native_log()
        return self._metrics

    def _pull_native_log(self) -> None:
        nat = self._native
        if nat is None:
            return
        recs = nat.drain_log()
        i = 0
        while i < len(recs):           # requests of one dispatch are contiguous in the log
            j = i
            while j < len(recs) and recs[j][0] == recs[i][0]:
                j += 1
            _, block, role, pass_kind, _, _ = recs[i]
            self._metrics.record((block, role, pass_kind), j - i, sum(r[4] for r in recs[i:j]),
                                 [r[5] for r in recs[i:j]])
            i = j

    def _native_request_fields(self, env, out_w):
        """(segment fields, dst tensor, host reply target or None) of a native request. Device
        payloads are served in place; host payloads are staged to the device here (the library
        scheduler only sees device pointers) and their reply read back by the reply thread."""
        p = env.payload
        host_reply = None
        if _is_device(p):
            src = p if p.dtype in (torch.float32, torch.bfloat16) else p.float()
            if src.dim() != 2 or src.stride(-1) != 1:
                src = src.contiguous()
        else:
            a = p if isinstance(p, torch.Tensor) else _host_tensor(np.ascontiguousarray(p, dtype=np.float32))
            if a.dtype not in (torch.float32, torch.bfloat16):
                a = a.float()
            if a.dim() != 2:
                a = a.reshape(a.shape[0] if a.dim() else 0, -1)
            src = a.to(self.device, non_blocking=False)
        reply = getattr(env, "reply_to", None)
        if _is_device(reply):
            dst = reply
        else:
            dst = torch.empty((src.shape[0], out_w), dtype=_out_dtype(p), device=self.device)
            host_reply = reply if reply is not None else True
        base = getattr(env, "base_to", None) if env.pass_kind != PASS_BACKWARD else None
        if base is not None and not _is_device(base):
            base = None
        key = (int(env.block), int(env.role))
        seg = Seg(client_id=env.client_id, src=src, dst=dst, base=base,
                  adapter=key in self._fused.get(env.client_id, ()), width=env.width)
        from .device import seg_fields
        return seg_fields(seg), src, dst, host_reply

    def _native_submit(self, env, reply_fn) -> None:
        from .sched import pack_request, raw_event
        key = (int(env.block), int(env.role))
        dims = self._dims.get(key)
        expected = out_w = None
        if dims is not None:
            expected = dims[1] if env.pass_kind == PASS_BACKWARD else dims[0]
            out_w = dims[0] if env.pass_kind == PASS_BACKWARD else dims[1]
        else:
            out_w = env.width
        with torch.cuda.device(self.device):
            fields, src, dst, host_reply = self._native_request_fields(env, max(out_w, 1))
            ready = raw_event(getattr(env, "ready", None))
            keep = None
            if not ready:
                # the payload write (or the staging copy above) is ordered on this thread's
                # stream: the scheduler's stream waits for this point
                keep = torch.cuda.Event()
                keep.record()
                ready = raw_event(keep)
            if src is not env.payload:
                src.record_stream(self._native_stream)   # staged copy: freed only after the batch
        req = _lib.SsRequest()
        pack_request(memoryview(req).cast("B"), env.client_id, env.pass_kind, env.block, env.role,
                     env.request_id, fields, ready)
        with self._cond:   # the reply thread looks the ticket up under the same lock
            ticket = self._native.submit(req, notify=True)
            self._native_pending[ticket] = (env, reply_fn, src, dst, host_reply, expected, keep)
            self._cond.notify_all()

    def _native_completions(self) -> None:
        from .sched import status_message
        torch.cuda.set_device(self.device)
        nat, rs = self._native, self._reply_stream
        while True:
            got = nat.next_done(rs.cuda_stream, 0.02)
            if got is None:
                with self._cond:
                    if not self._running:
                        return
                continue
            ticket, status, aux = got
            with self._cond:
                while ticket not in self._native_pending:   # submit() is between its two steps
                    self._cond.wait(0.01)
                env, reply_fn, src, dst, host_reply, expected, _ = self._native_pending.pop(ticket)
            if status != _lib.SS_SEG_OK:
                reply_fn(error_envelope(env, status_message(status, aux, env, expected, nat)))
                continue
            with torch.cuda.stream(rs):
                done = torch.cuda.Event()
                if host_reply is None:
                    res = dst
                else:
                    h = dst.cpu()          # rs waits for the batch (next_done), then D2H
                    if isinstance(host_reply, torch.Tensor):
                        host_reply.copy_(h)
                        res = host_reply
                    else:
                        res = h.float().numpy() if h.dtype == torch.float32 else h
                done.record(rs)
            reply_fn(Envelope(env.client_id, env.request_id, env.block, env.role, env.pass_kind, res,
                              done=done))

    # -- batch surface --------------------------------------------------------------------
    def serve_forward(self, envelopes) -> list:
        return self._compute_batch(PASS_FORWARD, envelopes)

    def serve_backward(self, envelopes) -> list:
        return self._compute_batch(PASS_BACKWARD, envelopes)

    def serve_noise_effect(self, envelope):
        return self._compute_batch(PASS_NOISE_EFFECT, [envelope])[0]

    def _pinned_buf(self, name: str, nbytes: int) -> torch.Tensor:
        buf = self._pinned.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
            self._pinned[name] = buf
        return buf

    def _compute_batch(self, pass_kind: int, envelopes) -> list:
        """One dispatch; per-envelope result is an array/tensor or a ProtocolError.

        Validation and its messages follow executor.py:196-213; the compute is one
        ss_compute_batch call (gather + GEMM + fused adapter + scatter)."""
        if not envelopes:
            return []
        with self._lock:
            return self._compute_batch_locked(pass_kind, envelopes)

    def _compute_batch_locked(self, pass_kind: int, envelopes) -> list:
        addr = envelopes[0].layer
        key = addr_key(addr)
        d_in, d_out = self._dims[key]
        expected = d_out if pass_kind == PASS_BACKWARD else d_in
        out_w = d_in if pass_kind == PASS_BACKWARD else d_out
        results: list = [None] * len(envelopes)
        good: list[int] = []
        for i, env in enumerate(envelopes):
            if (int(env.block), int(env.role)) != key:      # == addr_key(env.layer), no enum
                results[i] = ProtocolError(f"layer mismatch in batch: {env.layer} != {addr}")
            elif env.pass_kind != pass_kind:
                results[i] = ProtocolError(f"pass mismatch in batch: {env.pass_kind}")
            elif env.width != expected:
                results[i] = ProtocolError(
                    f"row width {env.width} does not match layer {addr} expected {expected}")
            else:
                good.append(i)
        if not good:
            return results
        stream = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        memo = self._host_memo_get(pass_kind, key, envelopes, good)
        if (memo is not None and memo[2] is not None) or self._all_pinned_host(envelopes, good, out_w):
            with torch.cuda.device(self.device):
                status = self._pipelined_host(pass_kind, key, envelopes, good, out_w, stream, memo)
            for j, i in enumerate(good):
                results[i] = (ProtocolError(f"executor rejected segment (status {status[j]}) for layer {addr}")
                              if status[j] != _lib.SS_SEG_OK else envelopes[i].reply_to)
            rows = sum(envelopes[i].token_count for i in good)
            self.ledger.set(ledger_mod.TRANSIENT_BUFFER, rows * (expected + out_w) * 2)
            self.ledger.set(ledger_mod.TRANSIENT_BUFFER, 0)
            return results
        if self.numpy_native and self._all_numpy(envelopes, good):
            with torch.cuda.device(self.device):
                return self._numpy_host(pass_kind, key, envelopes, good, out_w, stream, results, addr,
                                        expected)
        with torch.cuda.device(self.device), torch.cuda.stream(stream):
            for i in good:
                ev = getattr(envelopes[i], "ready", None)
                if ev is not None:
                    stream.wait_event(ev)
            srcs, host_idx = self._stage_inputs(envelopes, good, stream)
            dsts, host_out = self._stage_outputs(envelopes, good, out_w, stream)
            fused = self._fused
            segs = []
            for j, i in enumerate(good):
                env = envelopes[i]
                base = getattr(env, "base_to", None) if pass_kind != PASS_BACKWARD else None
                segs.append(Seg(client_id=env.client_id, src=srcs[j], dst=dsts[j], base=base,
                                adapter=key in fused.get(env.client_id, ())))
            status = self.ctx.compute(pass_kind, key[0], key[1], segs, stream)
            rows = sum(envelopes[i].token_count for i in good)
            esz = 2 if all(s.src.dtype == torch.bfloat16 for s in segs) else 4
            self.ledger.set(ledger_mod.TRANSIENT_BUFFER, rows * (expected + out_w) * esz)
            self.ledger.set(ledger_mod.TRANSIENT_BUFFER, 0)
            if self.save_activations and pass_kind == PASS_FORWARD:
                saved = [(s.src.clone(), s.dst.clone()) for s in segs]
                self._saved_debug.append(saved)
                self.ledger.add(ledger_mod.SAVED_ACTIVATIONS, rows * (expected + out_w) * esz)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.last_event = ev
            host_results = self._finish_outputs(host_out, ev)
        for j, i in enumerate(good):
            st = status[j]
            if st != _lib.SS_SEG_OK:
                results[i] = ProtocolError(f"executor rejected segment (status {st}) for layer {addr}")
            elif j in host_results:
                results[i] = host_results[j]
            else:
                results[i] = dsts[j]
        return results

    # -- pipelined host path ----------------------------------------------------------------
    pipeline_rows = 4096          # max rows per sub-batch of a host-payload dispatch
    pipeline_bytes = 24 << 20     # target bytes of the wider side per sub-batch

    def _all_pinned_host(self, envelopes, good, out_w) -> bool:
        if self.save_activations:
            return False
        info = self._host_info
        dtype = None
        for i in good:
            e = envelopes[i]
            p, r = e.payload, getattr(e, "reply_to", None)
            if not isinstance(p, torch.Tensor) or not isinstance(r, torch.Tensor) or \
                    getattr(e, "base_to", None) is not None:
                return False
            ip, ir = _cached_info(info, p), _cached_info(info, r)
            if not ip or not ir or ip[0] != ir[0] or ir[1] != (e.token_count, out_w):
                return False
            # the native host pipeline needs one payload / reply dtype per dispatch; a mixed
            # batch takes the staged path (every valid envelope still computes)
            if dtype is None:
                dtype = ip[0]
            elif ip[0] != dtype:
                return False
        return True

    def _host_memo_get(self, pass_kind, key, envelopes, good):
        """(signature, fingerprint, table) of a host dispatch identical to an earlier one — the
        same payload / reply tensor objects (held by the memo, so their ids stay theirs), the
        same clients, storage and shapes, and no adapter-set change since — else (signature,
        fingerprint, None). Decode clients send from the same buffers every step, and the
        per-envelope checks and segment packing cost more than the dispatch's kernels."""
        if self.save_activations:
            return None
        sig = [pass_kind, key, self._fused_ver]
        fp = []
        for i in good:
            e = envelopes[i]
            p, r = e.payload, getattr(e, "reply_to", None)
            if not isinstance(p, torch.Tensor) or not isinstance(r, torch.Tensor) or \
                    getattr(e, "base_to", None) is not None:
                return None
            sig += (id(p), id(r), e.client_id)
            fp += (p.data_ptr(), r.data_ptr(), p.shape, r.shape)
        sig, fp = tuple(sig), tuple(fp)
        hit = self._host_memo.get(sig)
        if hit is not None and hit[1] == fp:
            return sig, fp, hit[2]
        return sig, fp, None

    def _pipelined_host(self, pass_kind, key, envelopes, good, out_w, stream, memo=None) -> list[int]:
        """Host clients (pinned payload + pinned reply buffer): one ss_compute_batch_host call.
        The library splits the dispatch into row sub-batches so the H2D copy of sub-batch j+1
        and the D2H copy of j-1 overlap the kernels of j (its own copy streams and device
        staging ring). Rows are independent and the kernels never mix rows (tensor_ops.py:1-8),
        so results are bitwise those of one device-resident batch."""
        knobs = (int(self.pipeline_rows), int(self.pipeline_bytes))
        if knobs != getattr(self, "_pipeline_knobs", None):
            self.ctx.set_option("pipeline_rows", knobs[0])
            self.ctx.set_option("pipeline_bytes", knobs[1])
            self._pipeline_knobs = knobs
        self.last_event = None
        if memo is not None and memo[2] is not None:
            return self.ctx.compute_host_table(pass_kind, key[0], key[1], memo[2], stream)
        fused = self._fused
        in_w = envelopes[good[0]].width
        # _all_pinned_host verified every payload / reply is page-locked: tell the library
        segs = [Seg(client_id=envelopes[i].client_id, src=envelopes[i].payload, dst=envelopes[i].reply_to,
                    width=in_w, adapter=key in fused.get(envelopes[i].client_id, ()), pinned=True)
                for i in good]
        table = SegmentTable(segs, self.ctx._seg_cache)
        status = self.ctx.compute_host_table(pass_kind, key[0], key[1], table, stream)
        if memo is not None:
            if len(self._host_memo) > 2048:
                self._host_memo.clear()
            self._host_memo[memo[0]] = (table._keep, memo[1], table)   # (table holds the tensors)
        return status

    # -- numpy clients (the reference's LocalChannel / RemoteChannel payloads) ----------------
    numpy_native = True   # False: the staged path below (one H2D / D2H per dispatch, synchronous)

    def _all_numpy(self, envelopes, good) -> bool:
        if self.save_activations:
            return False
        for i in good:
            e = envelopes[i]
            if not isinstance(e.payload, np.ndarray) or getattr(e, "reply_to", None) is not None or \
                    getattr(e, "base_to", None) is not None or getattr(e, "ready", None) is not None:
                return False
        return True

    def _numpy_host(self, pass_kind, key, envelopes, good, out_w, stream, results, addr, expected) -> list:
        """f32 numpy payloads (what the reference's channels carry, transport.py:36, 78) through
        the native host pipeline (ss_compute_batch_host): the H2D of row sub-batch j+1, the
        kernels of j and the D2H of j-1 overlap, straight from / into the client arrays (no
        executor-side host copy). The replies are row views of ONE fresh f32 array per dispatch,
        like split_rows' views of the reference's ``out`` (tensor_ops.py:149-156)."""
        rows = sum(envelopes[i].token_count for i in good)
        out = self._numpy_out(rows, out_w)
        fused = self._fused
        segs, views, seg_of, pos = [], [], [], 0
        for i in good:
            e = envelopes[i]
            t = e.token_count
            view = out[pos:pos + t]
            views.append(view)
            pos += t
            if t == 0:                 # (empty arrays have zero strides; nothing to compute)
                seg_of.append(-1)
                continue
            p = e.payload
            if p.dtype != np.float32 or not p.flags.c_contiguous:
                p = np.ascontiguousarray(p, dtype=np.float32)
            seg_of.append(len(segs))
            segs.append(Seg(client_id=e.client_id, src=_host_tensor(p), dst=torch.from_numpy(view),
                            width=e.width, adapter=key in fused.get(e.client_id, ())))
        status = self.ctx.compute_host(pass_kind, key[0], key[1], segs, stream) if segs else []
        self.last_event = None
        for j, i in enumerate(good):
            st = status[seg_of[j]] if seg_of[j] >= 0 else _lib.SS_SEG_OK
            results[i] = (ProtocolError(f"executor rejected segment (status {st}) for layer {addr}")
                          if st != _lib.SS_SEG_OK else views[j])
        self.ledger.set(ledger_mod.TRANSIENT_BUFFER, rows * (expected + out_w) * 4)
        self.ledger.set(ledger_mod.TRANSIENT_BUFFER, 0)
        return results

    numpy_out_pool = 8    # page-locked reply arrays kept for reuse (0: fresh pageable arrays)

    def _numpy_out(self, rows: int, width: int) -> np.ndarray:
        """A [rows, width] f32 reply array in PAGE-LOCKED memory, recycled: an entry is reused
        only when no view of it is alive any more (numpy views keep their base array referenced,
        so the base's reference count says whether a caller still holds a reply). The reference
        LocalChannel copies each reply into its shared buffer at once (transport.py:91-98), so
        its replies free their entry immediately; D2H copies into page-locked memory run at
        copy-engine speed instead of through the driver's pageable staging + page faults."""
        import sys
        need = rows * width
        pool = self._np_pool
        for entry in pool:
            base = entry[1]
            if base.size >= need and sys.getrefcount(base) <= 3:   # pool list + local + getrefcount arg
                return base[:need].reshape(rows, width)
        if len(pool) >= self.numpy_out_pool or need == 0:
            return np.empty((rows, width), dtype=np.float32)
        cap = 1 << max(20, (need - 1).bit_length())
        t = torch.empty(cap, dtype=torch.float32, pin_memory=True)
        base = t.numpy()
        pool.append((t, base))
        return base[:need].reshape(rows, width)

    # -- staging helpers --------------------------------------------------------------------
    def _stage_inputs(self, envelopes, good, stream):
        """Device views of every good payload; host payloads go through one pinned buffer and
        one H2D copy (the only host->device crossing of a dispatch). Payloads that already sit
        in pinned host memory are copied straight from there."""
        srcs: list = [None] * len(good)
        host = []
        pinned = []
        for j, i in enumerate(good):
            p = envelopes[i].payload
            if _is_device(p):
                if p.dtype not in (torch.float32, torch.bfloat16):
                    p = p.float()
                if p.stride(-1) != 1:
                    p = p.contiguous()
                srcs[j] = p
            elif (isinstance(p, torch.Tensor) and p.is_pinned() and p.is_contiguous()
                  and p.dtype in (torch.float32, torch.bfloat16)):
                pinned.append(j)
            else:
                host.append(j)
        if pinned:
            sizes = [envelopes[good[j]].payload.numel() for j in pinned]
            dts = {envelopes[good[j]].payload.dtype for j in pinned}
            dt = dts.pop() if len(dts) == 1 else torch.float32
            dev = self._dev_buf("in", sum(sizes), dt)
            pos = 0
            for j, n in zip(pinned, sizes):
                p = envelopes[good[j]].payload
                view = dev[pos:pos + n].view(p.shape)
                view.copy_(p, non_blocking=True)
                srcs[j] = view
                pos += n
        if host:
            arrays = []
            for j in host:
                p = envelopes[good[j]].payload
                if isinstance(p, torch.Tensor):
                    a = p if p.dtype in (torch.float32, torch.bfloat16) else p.float()
                else:
                    a = torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32))
                arrays.append(a.contiguous())
            sizes = [a.numel() * a.element_size() for a in arrays]
            offs = np.cumsum([0] + [(s + 255) // 256 * 256 for s in sizes])
            total = int(offs[-1])
            pin = self._pinned_buf("in", total)
            stream.synchronize()  # the pinned staging buffer may still feed an earlier copy
            for a, o, s in zip(arrays, offs, sizes):
                pin[o:o + s].copy_(a.view(-1).view(torch.uint8))
            dev = torch.empty(total, dtype=torch.uint8, device=self.device)
            dev.copy_(pin[:total], non_blocking=True)
            for j, a, o, s in zip(host, arrays, offs, sizes):
                srcs[j] = dev[o:o + s].view(a.dtype).view(a.shape)
        return srcs, host

    def _dev_buf(self, name: str, numel: int, dtype) -> torch.Tensor:
        """Grow-only device staging (reported through the ledger's transient category)."""
        key = (name, dtype)
        buf = self._dev_staging.get(key)
        if buf is None or buf.numel() < numel:
            if buf is not None:
                # the old buffer may still feed copies / kernels on other streams
                torch.cuda.synchronize(self.device)
            buf = torch.empty(max(numel, 1 << 20), dtype=dtype, device=self.device)
            self._dev_staging[key] = buf
        return buf[:numel]

    def _stage_outputs(self, envelopes, good, out_w, stream):
        dsts: list = [None] * len(good)
        host_out = {}
        need = []
        self._host_replies = []
        for j, i in enumerate(good):
            env = envelopes[i]
            r = getattr(env, "reply_to", None)
            if r is not None:
                if tuple(r.shape) != (env.token_count, out_w) or not isinstance(r, torch.Tensor):
                    raise ProtocolError(f"reply_to must be a tensor of shape {(env.token_count, out_w)}")
                if r.is_cuda:
                    dsts[j] = r
                else:
                    # host reply buffer: compute into device staging, then one D2H into it
                    n = r.numel()
                    dev = self._dev_buf(f"out{j}", n, r.dtype if r.dtype == torch.bfloat16 else torch.float32)
                    dsts[j] = dev.view(r.shape)
                    self._host_replies.append((r, dsts[j]))
            else:
                need.append(j)
        if need:
            dts = {_out_dtype(envelopes[good[j]].payload) for j in need}
            dt = torch.float32 if torch.float32 in dts else torch.bfloat16
            rows = sum(envelopes[good[j]].token_count for j in need)
            out = torch.empty((rows, out_w), dtype=dt, device=self.device)
            pos = 0
            for j in need:
                t = envelopes[good[j]].token_count
                dsts[j] = out[pos:pos + t]
                if not _is_device(envelopes[good[j]].payload):
                    host_out[j] = (pos, t)
                pos += t
            if host_out:
                host_out["__out__"] = out
        return dsts, host_out

    def _finish_outputs(self, host_out, ev):
        if self._host_replies:
            for host, dev in self._host_replies:
                host.copy_(dev, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            self._host_replies = []
        if not host_out:
            return {}
        out = host_out.pop("__out__")
        pin = self._pinned_buf("out", out.numel() * 4)
        hv = pin[:out.numel() * 4].view(torch.float32).view(out.shape)
        hv.copy_(out.float(), non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        full = hv.numpy().copy()   # one array; slots are views of it, like split_rows
        return {j: full[pos:pos + t] for j, (pos, t) in host_out.items()}

    # -- scheduler (executor.py:235-300 semantics) ------------------------------------------
    def _loop(self) -> None:
        torch.cuda.set_device(self.device)
        while True:
            with self._cond:
                while True:
                    if not self._running:
                        return
                    picked, timeout = self._pick_ready(time.monotonic())
                    if picked is not None:
                        break
                    self._cond.wait(timeout)
            self._dispatch(*picked)

    def _pick_ready(self, now: float):
        """((key, entries), None) when some queue should dispatch now, else
        (None, seconds until the earliest opportunistic deadline or None)."""
        soonest = None
        for key, q in self._queues.items():
            if not q:
                continue
            pass_kind = key[2]
            if pass_kind == PASS_NOISE_EFFECT or self.policy.mode == "nolockstep":
                return (key, [q.popleft()]), None
            if self.policy.mode == "lockstep":
                need = {c for c, bwd in self._clients.items() if pass_kind == PASS_FORWARD or bwd}
                have = {e.client_id for e, _, _ in q}
                if need <= have:
                    return (key, self._drain(q)), None
                continue
            tokens = [e.token_count for e, _, _ in q]
            if sum(tokens) >= self.policy.max_batch_tokens:
                return (key, self._drain(q)), None
            deadline = min(t for _, _, t in q) + self.policy.wait_budget(tokens)
            if now >= deadline:
                return (key, self._drain(q)), None
            left = deadline - now
            soonest = left if soonest is None else min(soonest, left)
        return None, soonest

    @staticmethod
    def _drain(q: deque) -> list:
        entries = list(q)
        q.clear()
        return entries

    def _dispatch(self, key, entries) -> None:
        now = time.monotonic()
        if self.policy.dispatch_cost > 0:
            time.sleep(self.policy.dispatch_cost)
        envs = [e for e, _, _ in entries]
        try:
            results = self._compute_batch(key[2], envs)
        except Exception as exc:  # a CUDA failure fails the batch, not the scheduler
            results = [ProtocolError(f"executor failure: {exc}")] * len(envs)
        self._metrics.record(key, len(entries), sum(e.token_count for e in envs),
                            [now - t for _, _, t in entries])
        done = self.last_event
        for (env, reply_fn, _), res in zip(entries, results):
            if isinstance(res, ProtocolError):
                reply_fn(error_envelope(env, str(res)))
            else:
                reply_fn(Envelope(env.client_id, env.request_id, env.block, env.role,
                                  env.pass_kind, res, done=done))
        with self._cond:
            self._cond.notify_all()
