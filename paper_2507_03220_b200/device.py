"""SsContext — owner of one libss_b200 context (one CUDA device, one TP rank).

Thin, allocation-free translation from torch/numpy objects to the C ABI of
include/ss_b200.h. The executor (executor.py) drives it; benchmarks may drive it directly
with prebuilt segment tables (``SegmentTable``) to keep host overhead per dispatch at one
ctypes call.
"""

from __future__ import annotations

import ctypes
import struct
import weakref
from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import SsSeg, check


def _host_or_device(arr) -> tuple[Any, int, int, Any]:
    """Returns (pointer, flags, row_stride_elems, keepalive) for an upload source."""
    if isinstance(arr, torch.Tensor):
        t = arr
        if t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
        if t.dim() == 2 and t.stride(1) != 1:
            t = t.contiguous()
        if t.dim() == 1:
            t = t.contiguous()
        flags = _lib.SS_DT_BF16 if t.dtype == torch.bfloat16 else 0
        if t.is_cuda:
            flags |= _lib.SS_MEM_DEVICE
        ld = t.stride(0) if t.dim() == 2 else t.numel()
        return t.data_ptr(), flags, ld, t
    a = np.ascontiguousarray(arr, dtype=np.float32)
    ld = a.shape[1] if a.ndim == 2 else a.size
    return a.ctypes.data, 0, ld, a


def tensor_flags(t: torch.Tensor) -> int:
    dt = t.dtype
    if dt is _BF16:
        return 1
    if dt is _F32:
        return 0
    raise TypeError(f"activations must be float32 or bfloat16, got {t.dtype}")


@dataclass
class Seg:
    """One envelope's slice of a dispatch (device tensors, caller-owned)."""

    client_id: int
    src: torch.Tensor          # [rows, width] (row stride may exceed width)
    dst: torch.Tensor          # [rows, out_width]
    base: torch.Tensor | None = None
    adapter: bool = False
    width: int | None = None   # declared width (defaults to src.shape[1])
    pinned: bool = False       # host tensors verified page-locked by the caller (SS_SEGF_PINNED)


_SEG_FMT = struct.Struct("<4I QqQqQq")          # ss_seg layout (include/ss_b200.h)
assert _SEG_FMT.size == ctypes.sizeof(SsSeg)
_BF16, _F32 = torch.bfloat16, torch.float32


class SegmentTable:
    """A ctypes ss_seg array for one dispatch (prebuilt tables reuse it every step). Packed
    with one struct.pack_into per segment into the array's buffer: a decode dispatch has tens
    of segments and the per-field ctypes setters cost more than the dispatch's GPU work."""

    def __init__(self, segs: Sequence[Seg], cache: dict | None = None):
        self.n = len(segs)
        self.arr = (SsSeg * max(1, self.n))()
        self.status = (ctypes.c_int32 * max(1, self.n))()
        self._keep = list(segs)
        buf = memoryview(self.arr).cast("B")
        for i, s in enumerate(segs):
            _SEG_FMT.pack_into(buf, i * _SEG_FMT.size, *(seg_fields(s) if cache is None else _cached_fields(cache, s)))

    def statuses(self) -> list[int]:
        return list(self.status)[: self.n]


def _cached_fields(cache: dict, s: Seg) -> tuple:
    """seg_fields of a segment whose tensors recur across dispatches (clients reuse their
    buffers): keyed by the tensor objects' ids, validated through weak references."""
    key = (id(s.src), id(s.dst), id(s.base), s.client_id, s.adapter, s.width, s.pinned)
    hit = cache.get(key)
    # same live objects AND same storage (in-place set_ / resize_ could move a tensor)
    if (hit is not None and hit[0]() is s.src and hit[1]() is s.dst and (s.base is None or hit[2]() is s.base)
            and hit[3][4] == s.src.data_ptr() and hit[3][6] == s.dst.data_ptr()):
        return hit[3]
    if len(cache) > 4096:
        cache.clear()
    f = seg_fields(s)
    cache[key] = (weakref.ref(s.src), weakref.ref(s.dst), weakref.ref(s.base) if s.base is not None else None, f)
    return f


def _row_ld(stride: tuple, shape) -> int:
    return stride[0] if shape[0] > 1 else max(stride[0], shape[1])


def seg_fields(s: Seg) -> tuple:
    """The ss_seg field values of one segment (client_id, rows, width, flags, src, src_ld, dst,
    dst_ld, dst_base, base_ld)."""
    src, dst, base = s.src, s.dst, s.base
    ss, sd = src.stride(), dst.stride()
    if len(ss) != 2 or len(sd) != 2 or ss[1] != 1 or sd[1] != 1:
        raise ValueError("segment tensors must be 2-d with unit column stride")
    shs, shd = src.shape, dst.shape
    flags = ((_lib.SS_SEGF_SRC_BF16 if tensor_flags(src) else 0) |
             (_lib.SS_SEGF_DST_BF16 if tensor_flags(dst) else 0))
    if s.adapter:
        flags |= _lib.SS_SEGF_ADAPTER
    if s.pinned:
        flags |= _lib.SS_SEGF_PINNED
    if base is not None:
        if tensor_flags(base):
            flags |= _lib.SS_SEGF_BASE_BF16
        bptr, bld = base.data_ptr(), _row_ld(base.stride(), base.shape)
    else:
        bptr, bld = 0, 0
    return (int(s.client_id), shs[0], int(s.width if s.width is not None else shs[1]), flags,
            src.data_ptr(), _row_ld(ss, shs), dst.data_ptr(), _row_ld(sd, shd), bptr, bld)


class Plan:
    """A prebuilt dispatch (ss_plan_*): routing tables live on the device; ``launch`` only
    launches kernels (CUDA-graph capturable). Keeps its segment tensors alive."""

    def __init__(self, ctx: "SsContext", pass_kind: int, block: int, role: int, segs: Sequence[Seg]):
        self.ctx, self.pass_kind, self.key = ctx, int(pass_kind), (int(block), int(role))
        table = SegmentTable(segs)
        self._table = table
        h = ctypes.c_void_p()
        check(ctx.h, ctx.lib.ss_plan_create(ctx.h, self.pass_kind, self.key[0], self.key[1], table.n,
                                            table.arr, table.status, ctypes.byref(h)))
        self.h = h
        self.status = table.statuses()
        ctx._plans.add(self)

    def launch(self, stream: torch.cuda.Stream | None = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.ctx.device)
        check(self.ctx.h, self.ctx.lib.ss_plan_launch(self.h, ctypes.c_void_p(s.cuda_stream)))

    def destroy(self) -> None:
        if getattr(self, "h", None):
            self.ctx.lib.ss_plan_destroy(self.h)
            self.h = None
            self.ctx._plans.discard(self)

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


@dataclass
class GradSeg:
    """One client's adapter-gradient job for one layer (ss_adapter_grads): device tensors.

    LoRA: ``x`` (the layer's forward input, bf16) and ``dy`` (bf16) -> ``grad_a`` [d_in, r],
    ``grad_b`` [r, d_out] (f32). IA3: ``dy`` and ``y_base`` -> ``grad_l`` [d_out] (f32).
    ``accumulate`` adds into the gradient tensors like the reference's ``_accumulate``."""

    client_id: int
    dy: torch.Tensor
    x: torch.Tensor | None = None
    y_base: torch.Tensor | None = None
    grad_a: torch.Tensor | None = None
    grad_b: torch.Tensor | None = None
    grad_l: torch.Tensor | None = None
    accumulate: bool = False


def _ld(t: torch.Tensor) -> int:
    return t.stride(0) if t.shape[0] > 1 else max(t.stride(0), t.shape[1])


def _f32_out(t: torch.Tensor | None, name: str):
    if t is None:
        return None
    if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return t.data_ptr()


def fill_grad_seg(c, g: GradSeg) -> None:
    for t in (g.dy, g.x, g.y_base):
        if t is not None and (t.dim() != 2 or t.stride(1) != 1 or not t.is_cuda):
            raise ValueError("gradient-job activations must be 2-d CUDA tensors with unit column stride")
    c.client_id = int(g.client_id)
    c.rows = int(g.dy.shape[0])
    flags = _lib.SS_GRADF_ACCUMULATE if g.accumulate else 0
    if tensor_flags(g.dy):
        flags |= _lib.SS_GRADF_DY_BF16
    c.dy, c.dy_ld = g.dy.data_ptr(), _ld(g.dy)
    if g.x is not None:
        if tensor_flags(g.x):
            flags |= _lib.SS_GRADF_X_BF16
        c.x, c.x_ld = g.x.data_ptr(), _ld(g.x)
    else:
        c.x, c.x_ld = None, 0
    if g.y_base is not None:
        if tensor_flags(g.y_base):
            flags |= _lib.SS_GRADF_BASE_BF16
        c.y_base, c.base_ld = g.y_base.data_ptr(), _ld(g.y_base)
    else:
        c.y_base, c.base_ld = None, 0
    c.grad_a = _f32_out(g.grad_a, "grad_a")
    c.grad_b = _f32_out(g.grad_b, "grad_b")
    c.grad_l = _f32_out(g.grad_l, "grad_l")
    c.flags = flags


class SsContext:
    def __init__(self, device: int | torch.device = 0, tp_rank: int = 0, tp_size: int = 1):
        self.lib = _lib.load()
        self.device = torch.device("cuda", device if isinstance(device, int) else device.index or 0)
        if not torch.cuda.is_available():
            raise RuntimeError("GpuBaseExecutor needs a CUDA device (no CPU fallback by design)")
        torch.cuda.set_device(self.device)
        torch.cuda.init()
        h = ctypes.c_void_p()
        rc = self.lib.ss_ctx_create(self.device.index, tp_rank, tp_size, ctypes.byref(h))
        if rc != _lib.SS_OK:
            raise _lib.SsError(rc, f"ss_ctx_create(device={self.device.index}) failed "
                                   "(needs an sm_100 GPU)")
        self.h = h
        self.dims: dict[tuple[int, int], tuple[int, int]] = {}
        import weakref
        self._plans = weakref.WeakSet()
        self._seg_cache: dict = {}      # ss_seg fields of recurring host segments (compute_host)

    # -- weights --------------------------------------------------------------------------
    def load_layer(self, block: int, role: int, weight, bias=None) -> None:
        wp, wf, wld, wk = _host_or_device(weight)
        bp, bk = None, None
        if bias is not None:
            # one flag set covers both uploads: bring the bias to the weight's dtype / memory
            if isinstance(weight, torch.Tensor):
                b = torch.as_tensor(bias).to(device=weight.device, dtype=wk.dtype).contiguous()
            else:
                b = np.ascontiguousarray(bias.detach().cpu().float().numpy()
                                         if isinstance(bias, torch.Tensor) else bias, dtype=np.float32)
            bp, _, _, bk = _host_or_device(b)
        d_in, d_out = int(weight.shape[0]), int(weight.shape[1])
        check(self.h, self.lib.ss_load_layer(self.h, int(block), int(role), d_in, d_out, wp, wld, bp, wf))
        del wk, bk
        self.dims[(int(block), int(role))] = (d_in, d_out)

    # -- adapters -------------------------------------------------------------------------
    def set_adapter(self, client_id: int, block: int, role: int, lora=None, ia3=None) -> None:
        """lora = (A [d_in, r], B [r, d_out], scale) ; ia3 = l [d_out]."""
        parts = [p for p in ((lora[0], lora[1]) if lora is not None else ()) + ((ia3,) if ia3 is not None else ())]
        on_dev = any(isinstance(p, torch.Tensor) and p.is_cuda for p in parts)

        def norm(p):  # one dtype / memory kind for every pointer of this call
            if on_dev:
                return torch.as_tensor(p, device=self.device).float().contiguous()
            if isinstance(p, torch.Tensor):
                p = p.float().numpy()
            return np.ascontiguousarray(p, dtype=np.float32)

        kind, rank, scale = 0, 0, 0.0
        ap = bp = lp = None
        keep = []
        if lora is not None:
            a, b = norm(lora[0]), norm(lora[1])
            scale = float(lora[2])
            ap, flags, _, _ = _host_or_device(a)
            bp, _, _, _ = _host_or_device(b)
            keep += [a, b]
            kind |= _lib.SS_ADAPTER_LORA
            rank = int(a.shape[1])
        if ia3 is not None:
            lv = norm(ia3)
            lp, flags, _, _ = _host_or_device(lv)
            keep.append(lv)
            kind |= _lib.SS_ADAPTER_IA3
        if kind:
            self._set(client_id, block, role, kind, rank, scale, ap, bp, lp, flags)
        del keep

    def _set(self, client_id, block, role, kind, rank, scale, ap, bp, lp, flags):
        check(self.h, self.lib.ss_set_adapter(self.h, int(client_id), int(block), int(role), kind,
                                              rank, ctypes.c_float(scale), ap, bp, lp, flags or 0))

    def clear_adapter(self, client_id: int, block: int | None = None, role: int | None = None) -> None:
        if block is None:
            check(self.h, self.lib.ss_clear_client(self.h, int(client_id)))
        else:
            rc = self.lib.ss_clear_adapter(self.h, int(client_id), int(block), int(role))
            if rc not in (_lib.SS_OK, _lib.SS_E_NOLAYER):
                check(self.h, rc)

    # -- compute --------------------------------------------------------------------------
    def compute(self, pass_kind: int, block: int, role: int, segs: Sequence[Seg],
                stream: torch.cuda.Stream | None = None) -> list[int]:
        table = SegmentTable(segs)
        self.compute_table(pass_kind, block, role, table, stream)
        return table.statuses()

    def compute_table(self, pass_kind: int, block: int, role: int, table: SegmentTable,
                      stream: torch.cuda.Stream | None = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.ss_compute_batch(self.h, int(pass_kind), int(block), int(role), table.n,
                                       table.arr, ctypes.c_void_p(s.cuda_stream), table.status)
        check(self.h, rc)

    def compute_host(self, pass_kind: int, block: int, role: int, segs: Sequence[Seg],
                     stream: torch.cuda.Stream | None = None) -> list[int]:
        """One dispatch over HOST (pinned) tensors: ss_compute_batch_host pipelines the H2D
        copies, kernels and D2H copies natively and returns when the replies are in place."""
        return self.compute_host_table(pass_kind, block, role, SegmentTable(segs, self._seg_cache), stream)

    def compute_host_table(self, pass_kind: int, block: int, role: int, table: SegmentTable,
                           stream: torch.cuda.Stream | None = None) -> list[int]:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(self.h, self.lib.ss_compute_batch_host(self.h, int(pass_kind), int(block), int(role), table.n,
                                                     table.arr, ctypes.c_void_p(s.cuda_stream), table.status))
        return table.statuses()

    def plan(self, pass_kind: int, block: int, role: int, segs: Sequence[Seg]) -> "Plan":
        """Prebuild a dispatch over fixed device buffers (ss_plan_create)."""
        return Plan(self, pass_kind, block, role, segs)

    def adapter_grads(self, block: int, role: int, jobs: Sequence[GradSeg],
                      stream: torch.cuda.Stream | None = None) -> list[int]:
        """LoRA / IA3 weight gradients of one layer for every job (ss_adapter_grads)."""
        n = len(jobs)
        arr = (_lib.SsGradSeg * max(1, n))()
        status = (ctypes.c_int32 * max(1, n))()
        for i, g in enumerate(jobs):
            fill_grad_seg(arr[i], g)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(self.h, self.lib.ss_adapter_grads(self.h, int(block), int(role), n, arr,
                                                ctypes.c_void_p(s.cuda_stream), status))
        return [int(status[i]) for i in range(n)]

    # -- introspection --------------------------------------------------------------------
    def memory_stats(self) -> tuple[int, int, int]:
        w, a, ws = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self.h, self.lib.ss_memory_stats(self.h, ctypes.byref(w), ctypes.byref(a), ctypes.byref(ws)))
        return w.value, a.value, ws.value

    def kernel_launches(self) -> int:
        return int(self.lib.ss_kernel_launches(self.h))

    def epoch(self) -> int:
        """ss_ctx_epoch: moves whenever a buffer captured kernels may reference was freed."""
        return int(self.lib.ss_ctx_epoch(self.h))

    def profile(self, enable: bool) -> None:
        """Start (and reset) / stop in-stream CUDA-event timing of every kernel launch."""
        check(self.h, self.lib.ss_profile(self.h, 1 if enable else 0))

    def profile_read(self, kernel: int) -> dict:
        ms, n = ctypes.c_double(), ctypes.c_int64()
        fl, by = ctypes.c_double(), ctypes.c_double()
        check(self.h, self.lib.ss_profile_read(self.h, int(kernel), ctypes.byref(ms), ctypes.byref(n),
                                               ctypes.byref(fl), ctypes.byref(by)))
        return {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}

    def set_option(self, key: str, value: int) -> None:
        check(self.h, self.lib.ss_set_option(self.h, key.encode(), int(value)))

    def close(self) -> None:
        if getattr(self, "h", None):
            torch.cuda.synchronize(self.device)
            for p in list(self._plans):
                p.destroy()
            self.lib.ss_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
