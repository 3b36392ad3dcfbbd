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
    """Client-side stand-in for one frozen layer (client.py:48-98). With ``noise`` (a
    ``privacy.DeviceNoiseSet``, or the reference's NoiseSet for numpy clients) forward payloads
    are blinded and replies de-noised (privacy.py:1-12); for executor-fused adapters the
    effect includes the adapter (privacy.py here), so blinding and fusion compose."""

    def __init__(self, addr, d_in: int, d_out: int, channel, noise=None):
        self.addr = addr
        self.d_in = d_in
        self.d_out = d_out
        self.channel = channel
        self.noise = noise

    def forward(self, x, iteration: int = 0, want_base: bool = False):
        if x.shape[1] != self.d_in:
            raise ProtocolError(f"{self.addr}: input width {x.shape[1]} != d_in {self.d_in}")
        if self.noise is not None:
            payload, index = self.noise.blind(self.addr, x, iteration)
        else:
            payload, index = x, None
        kw = {"want_base": True} if want_base else {}
        y = self.channel.request(self.addr.block, int(self.addr.role), PASS_FORWARD, payload, **kw)
        y = self._checked(y, x.shape[0], self.d_out)
        base = getattr(self.channel, "last_base", None) if want_base else None
        if index is not None:
            # unblind() returns a fresh array: nothing aliases the channel's shared buffer
            y = self.noise.unblind(self.addr, y, index)
            if base is not None:
                base = self.noise.unblind_base(self.addr, base, index)
        elif self.channel.reply_is_view:
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


def client_layer_backward(layer: VirtLayer, fused: set, executor, client_id: int, adapter,
                          x_saved, grad_y, grads: dict, y_base=None):
    """``ClientModel._layer_backward`` (client.py:286-305) for an executor-fused address, with
    the adapter weight gradients on the GPU as well.

    grad_x = one fused backward dispatch (g = dy * l, g W^T, + the LoRA grad_x term); then
    ss_adapter_grads adds grad_l = sum_rows(dy * y_base) (IA3) or grad_a / grad_b
    (lora_backward, adapters.py:26-41) into ``grads`` under the reference's keys
    ``(addr, "l" | "a" | "b")``, accumulating like the reference's ``_accumulate``.
    Activations are device tensors (bf16 for LoRA's x and dy)."""
    from .device import GradSeg

    grad_x = client_backward_input(layer, fused, grad_y)
    if adapter is None:
        return grad_x
    addr = layer.addr
    key = addr_key(addr)
    dev = grad_y.device
    job = GradSeg(client_id=client_id, dy=grad_y)
    lora = {addr_key(a): v for a, v in (getattr(adapter, "lora", {}) or {}).items()}
    ia3 = {addr_key(a): v for a, v in (getattr(adapter, "ia3", {}) or {}).items()}

    def slot(part, shape):
        g = grads.get((addr, part))
        if g is None:
            g = torch.zeros(shape, dtype=torch.float32, device=dev)
            grads[(addr, part)] = g
        return g

    if key in ia3:
        if y_base is None:
            raise ValueError(f"{addr}: IA3 backward needs the forward's y_base")
        job.y_base = y_base
        job.grad_l = slot("l", (layer.d_out,))
    elif key in lora:
        a, _ = lora[key]
        job.x = x_saved
        job.grad_a = slot("a", (layer.d_in, int(a.shape[1])))
        job.grad_b = slot("b", (int(a.shape[1]), layer.d_out))
    else:
        return grad_x
    job.accumulate = True
    status = executor.adapter_grads(addr.block, int(addr.role), [job])
    if status[0] != 0:
        raise ProtocolError(f"{addr}: adapter gradient job rejected (status {status[0]})")
    return grad_x
