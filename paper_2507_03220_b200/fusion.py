"""Executor-side adapters for an existing client model (reference client.py:147-351).

``fuse_client_model`` takes a client model built the reference's way
(``ClientModel.virtualize(model, base_layer_set, channel)``, client.py:159-178) and moves its
LoRA adapter into the base executor's GEMM epilogue, touching only the two call sites that
decide where the adapter is applied:

* ``_apply`` (client.py:206-209): for a fused address the executor's reply already is
  ``y_base + (alpha/r)·(x·A)·B``, so the client returns it instead of calling apply_adapter;
* ``_layer_backward`` (client.py:286-305): the executor's backward reply already is
  ``g·Wᵀ + (alpha/r)·(g·Bᵀ)·Aᵀ``; the client keeps only the LoRA *weight* gradients
  (adapters.py:36-39, they need the client-saved x), computed by the client module's own
  ``lora_backward`` exactly as the reference does.

The adapter is (re-)registered before every forward, so optimizer steps between iterations
(ClientJob.train_step, client.py:491-508) reach the executor. Works with any channel whose
``executor`` attribute is a ``GpuBaseExecutor`` (the reference LocalChannel with numpy
payloads, or ``DeviceChannel``) — duck typed, no import of the client's package.

IA3 is fused only through ``DeviceChannel`` (the client needs the pre-IA3 ``y_base`` for
``grad_l``, client.py:291-294, which the executor writes as a second output); with other
channels IA3 addresses stay client-side, unchanged from the reference.
"""

from __future__ import annotations

import inspect
import sys
import types

import numpy as np

from .config import addr_key


def _lora_backward_numpy(x, grad_y, a, b, alpha, rank):
    """adapters.py:26-41, used only when the client module does not expose lora_backward."""
    s = np.float32(alpha / rank)
    xa = x @ a
    gyb = grad_y @ b.T
    return s * (x.T @ gyb), s * (xa.T @ grad_y), s * (gyb @ a.T)


def fuse_client_model(cm, client_id: int, adapter, executor=None, ia3: bool | None = None) -> set:
    """Fuse ``adapter`` (AdapterState-like: ``lora``, ``ia3``, ``alpha``, ``rank``) of the
    client ``client_id`` into the executor behind ``cm``'s virtual layers. Returns the set of
    fused addresses (keys ``(block, role)``). Idempotent per client model."""
    virt = {addr: layer for addr, layer in cm.layers.items() if hasattr(layer, "channel")}
    if not virt:
        return set()
    channel = next(iter(virt.values())).channel
    ex = executor if executor is not None else getattr(channel, "executor", None)
    if ex is None or not hasattr(ex, "register_adapter"):
        raise TypeError("fuse_client_model needs a GpuBaseExecutor behind the client's channel")
    if ia3 is None:                                  # DeviceChannel + VirtLayer return y_base
        layer = next(iter(virt.values()))
        ia3 = hasattr(channel, "base_buffer") and \
            "want_base" in inspect.signature(layer.forward).parameters
    lora = getattr(adapter, "lora", {}) or {}
    ia3_map = (getattr(adapter, "ia3", {}) or {}) if ia3 else {}
    targets = [a for a in list(lora) + list(ia3_map) if a in virt]
    if not targets:
        return set()
    fused = {addr_key(a) for a in targets}
    ex.register_adapter(client_id, adapter, targets)
    client_mod = sys.modules.get(type(cm).__module__)
    lora_backward = getattr(client_mod, "lora_backward", None) or _lora_backward_numpy
    orig_apply, orig_backward, orig_forward = cm._apply, cm._layer_backward, cm.forward

    def _apply(self, adapter_, addr, x, iteration):
        if adapter_ is adapter and addr_key(addr) in fused:
            layer = self.layers[addr]
            if addr in ia3_map:
                return layer.forward(x, iteration, want_base=True)
            y = layer.forward(x, iteration)
            return y, y
        return orig_apply(adapter_, addr, x, iteration)

    def _layer_backward(self, adapter_, addr, x_saved, grad_y, grads, y_base=None):
        if adapter_ is not adapter or addr_key(addr) not in fused:
            return orig_backward(adapter_, addr, x_saved, grad_y, grads, y_base)
        if addr in ia3_map:                              # client.py:291-294, g*l is executor-side
            _acc(grads, (addr, "l"), _sum_rows(grad_y, y_base))
            return self.layers[addr].backward(grad_y)
        grad_x = self.layers[addr].backward(grad_y)      # g·Wᵀ + s·(g·Bᵀ)·Aᵀ, one dispatch
        a, b = lora[addr]
        ga, gb, _ = lora_backward(x_saved, grad_y, a, b, adapter.alpha, adapter.rank)
        _acc(grads, (addr, "a"), ga)
        _acc(grads, (addr, "b"), gb)
        return grad_x

    def forward(self, adapter_, *args, **kw):
        if adapter_ is adapter:                          # values move after each optimizer step
            ex.refresh_adapter(client_id, adapter, targets)
        return orig_forward(adapter_, *args, **kw)

    cm._apply = types.MethodType(_apply, cm)
    cm._layer_backward = types.MethodType(_layer_backward, cm)
    cm.forward = types.MethodType(forward, cm)
    return fused


def _sum_rows(g, y_base):
    if hasattr(g, "is_cuda"):
        return (g.float() * y_base.float()).sum(0)
    return np.sum(g * y_base, axis=0)


def _acc(grads: dict, key, value) -> None:
    prev = grads.get(key)
    grads[key] = value if prev is None else prev + value
