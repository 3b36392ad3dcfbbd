"""Layer-interception surface, kept intact (reference client.py:48-98, 206-209, 286-305).

``VirtLayer`` is the reference's stand-in for one frozen layer: same constructor, same
shape checks and error messages, same copy-out of a view reply. It works over any channel
(the reference LocalChannel/RemoteChannel duck type or ``DeviceChannel``) with numpy or
torch activations.

The only client-side change fused adapters require is in ``_apply`` / ``_layer_backward``:
for addresses the executor fuses, the client must not apply the adapter again, and an IA3
fine-tune client takes y_base from the executor's second output. ``client_forward`` and
``client_backward_input`` below are those two call sites restated against the fused
executor (the LoRA/IA3 *weight* gradients stay client-side, adapters.py:36-39).
"""

from __future__ import annotations

import numpy as np
import torch

from .config import addr_key
from .errors import ProtocolError
from .protocol import PASS_BACKWARD, PASS_FORWARD


class VirtLayer:
    def __init__(self, addr, d_in: int, d_out: int, channel, noise=None):
        if noise is not None:
            raise NotImplementedError(
                "activation blinding is incompatible with executor-fused adapters; privacy "
                "clients use the reference's unfused path (SURVEY §7)")
        self.addr = addr
        self.d_in = d_in
        self.d_out = d_out
        self.channel = channel

    def forward(self, x, iteration: int = 0, want_base: bool = False):
        if x.shape[1] != self.d_in:
            raise ProtocolError(f"{self.addr}: input width {x.shape[1]} != d_in {self.d_in}")
        kw = {"want_base": True} if want_base else {}
        y = self.channel.request(self.addr.block, int(self.addr.role), PASS_FORWARD, x, **kw)
        y = self._checked(y, x.shape[0], self.d_out)
        base = getattr(self.channel, "last_base", None) if want_base else None
        if self.channel.reply_is_view:
            y = _detach(y)
            base = None if base is None else _detach(base)
        return (y, base) if want_base else y

    def backward(self, grad_y):
        if grad_y.shape[1] != self.d_out:
            raise ProtocolError(f"{self.addr}: grad width {grad_y.shape[1]} != d_out {self.d_out}")
        gx = self.channel.request(self.addr.block, int(self.addr.role), PASS_BACKWARD, grad_y)
        gx = self._checked(gx, grad_y.shape[0], self.d_in)
        return _detach(gx) if self.channel.reply_is_view else gx

    def _checked(self, y, rows: int, cols: int):
        if tuple(y.shape) != (rows, cols):
            raise ProtocolError(f"{self.addr}: executor returned shape {tuple(y.shape)}, "
                                f"expected {(rows, cols)}")
        return y


def _detach(y):
    return y.clone() if isinstance(y, torch.Tensor) else np.array(y, copy=True)


def client_forward(layer: VirtLayer, fused: set, adapter, x, iteration: int = 0):
    """``ClientModel._apply`` (client.py:206-209) for a fused executor: returns (y, y_base).

    Fused address: the executor already produced (y_base + lora) * l, and y_base for IA3.
    Unfused address: identical to the reference (apply_adapter client-side)."""
    key = addr_key(layer.addr)
    if key in fused:
        needs_base = adapter is not None and any(addr_key(a) == key for a in getattr(adapter, "ia3", {}))
        if needs_base:
            return layer.forward(x, iteration, want_base=True)
        y = layer.forward(x, iteration)
        return y, y
    y = layer.forward(x, iteration)
    if adapter is None:
        return y, y
    from .adapters_host import apply_adapter_host
    return apply_adapter_host(adapter, layer.addr, x, y), y


def client_backward_input(layer: VirtLayer, fused: set, grad_y):
    """The grad_x part of ``_layer_backward`` (client.py:286-305) for a fused address: the
    executor applies g = dy * l, dx = g W^T and the LoRA grad_x term in one dispatch."""
    if addr_key(layer.addr) not in fused:
        raise ValueError("client_backward_input is for executor-fused addresses")
    return layer.backward(grad_y)
