"""Client-side adapter step for UNFUSED addresses (reference adapters.py:127-145).

Used only when a client keeps an adapter client-side (e.g. a blinded/privacy client);
fused addresses never reach this. Works on numpy or torch tensors.
"""

from __future__ import annotations

import numpy as np
import torch

from .config import addr_key


def apply_adapter_host(adapter, addr, x, y_base):
    key = addr_key(addr)
    lora = {addr_key(a): v for a, v in (getattr(adapter, "lora", {}) or {}).items()}
    ia3 = {addr_key(a): v for a, v in (getattr(adapter, "ia3", {}) or {}).items()}
    y = y_base
    if key in lora:
        a, b = lora[key]
        scale = adapter.alpha / adapter.rank
        if isinstance(x, torch.Tensor):
            a_t = torch.as_tensor(a, device=x.device, dtype=torch.float32)
            b_t = torch.as_tensor(b, device=x.device, dtype=torch.float32)
            y = (y.float() + ((x.float() @ a_t) @ b_t) * scale).to(y.dtype)
        else:
            y = y + (np.asarray(x) @ a @ b) * np.float32(scale)
    if key in ia3:
        l = ia3[key]
        if isinstance(y, torch.Tensor):
            y = (y.float() * torch.as_tensor(l, device=y.device, dtype=torch.float32)).to(y.dtype)
        else:
            y = y * l
    return y
