"""LSV1 frames served on the GPU without a host-side decode.

The reference's byte-stream path (protocol.py:96-153 encode / try_decode, ExecutorServer
transport.py:168-275) decodes every request frame into a numpy array, batches, and re-encodes
each reply — ~1 GB/s of host codec work per direction. ``FrameServer.serve`` hands a run of
received bytes to ``ss_serve_frames``: the library parses the headers in place, applies the
executor's intake checks (same messages), copies each f32 payload to the GPU straight out of
the receive buffer, runs one fused dispatch per (layer, pass) group, and writes complete reply
frames (header + f32 payload straight from the GPU) into a pinned send buffer, in request order.
Sockets stay the caller's business (out of scope here); this is the codec + compute boundary an
``ExecutorServer._serve_conn`` loop would call instead of ``try_decode`` / ``submit`` / ``encode``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check


class FrameServer:
    def __init__(self, executor, in_capacity: int = 1 << 20, out_capacity: int = 1 << 20):
        self.ctx = executor.ctx
        self._in = torch.empty(max(1, in_capacity), dtype=torch.uint8, pin_memory=True)
        self._out = torch.empty(max(1, out_capacity), dtype=torch.uint8, pin_memory=True)

    def _grow(self, name: str, n: int) -> torch.Tensor:
        buf = getattr(self, name)
        if buf.numel() < n:
            buf = torch.empty(max(n, 2 * buf.numel()), dtype=torch.uint8, pin_memory=True)
            setattr(self, name, buf)
        return buf

    def serve(self, data) -> tuple[bytes, int]:
        """Serve every whole request frame at the head of ``data`` (bytes-like). Returns the
        concatenated reply frames and the number of input bytes consumed (a trailing partial
        frame is left for the next call). Raises SsError(SS_E_PROTOCOL) on a corrupt stream."""
        mv = memoryview(data).cast("B")
        n = mv.nbytes
        buf = self._grow("_in", n)
        if n:
            buf[:n].numpy()[:] = np.frombuffer(mv, dtype=np.uint8)
        out, used = self.serve_pinned(buf, n)
        return bytes(out.numpy()), used

    def serve_pinned(self, buf: torch.Tensor, n: int) -> tuple[torch.Tensor, int]:
        """Same, reading the frames from a caller-owned pinned uint8 tensor and returning the reply
        stream as a view of the server's pinned send buffer (valid until the next call, like the
        reference LocalChannel's reply view) — no host-side copy of either stream."""
        lib = self.ctx.lib
        consumed, out_len = ctypes.c_size_t(), ctypes.c_size_t()
        stream = torch.cuda.current_stream(self.ctx.device)
        for _ in range(2):
            out = self._out
            rc = lib.ss_serve_frames(self.ctx.h, buf.data_ptr(), n, ctypes.byref(consumed), out.data_ptr(),
                                     out.numel(), ctypes.byref(out_len), ctypes.c_void_p(stream.cuda_stream))
            if rc == _lib.SS_E_NOMEM and out_len.value > out.numel():
                self._grow("_out", out_len.value)
                continue
            check(self.ctx.h, rc)
            return self._out[: out_len.value], consumed.value
        check(self.ctx.h, rc)
        return self._out[:0], 0
