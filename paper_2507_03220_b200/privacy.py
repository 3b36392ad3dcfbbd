"""Activation blinding with executor-fused adapters.

The reference's scheme (privacy.py:1-12): the client adds a precomputed noise matrix n to its
forward activations and removes the noise's effect from the reply, y = (W(x+n) + b) - Wn; the
effect Wn comes from the bias-nullified NOISE pass (executor.py:221-222), precomputed once per
layer and fetched twice to check it is reproducible (privacy.py:79-106).

With the adapter applied executor-side the reply is ((x+n)W + b + s(x+n)AB) * l, so the effect
to subtract is (nW + s nAB) * l. The C ABI computes exactly that when a NOISE segment carries
the adapter flag (include/ss_b200.h SS_SEGF_ADAPTER), and the executor sets it for every client
whose adapter is fused on the layer — so ``precompute_noise`` through a fused client's channel
returns the right effect with no client-side math, and the IA3 pre-scale output y_base (which
an IA3 fine-tune client needs for grad_l) is unblinded with the pre-IA3 part of the same effect
(the NOISE pass's dst_base output). Effects depend on the adapter: after an optimizer step
refreshes a fused adapter, its effects must be recomputed (``refresh``).

Semantics follow the reference: ``rotate`` picks the noise index per (layer, iteration) from
``default_rng([seed, block, role, iteration])`` (privacy.py:33-44); ``draw_noise`` draws
uniform[-scale, scale] from ``default_rng([seed, block, role, index, 7])`` (privacy.py:72-76);
``precompute_noise`` needs k >= 2 and rejects an irreproducible effect (privacy.py:79-106).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .config import addr_key
from .errors import ConfigError, ProtocolError
from .protocol import PASS_NOISE_EFFECT


def rotate(seed: int, addr, iteration: int, k: int) -> int:
    if k < 1:
        raise ConfigError(f"noise set size must be >= 1, got {k}")
    rng = np.random.default_rng([seed, addr.block, int(addr.role), iteration])
    return int(rng.integers(k))


def draw_noise(seed: int, addr, index: int, t_max: int, d_in: int, scale: float) -> np.ndarray:
    rng = np.random.default_rng([seed, addr.block, int(addr.role), index, 7])
    return rng.uniform(-scale, scale, size=(t_max, d_in)).astype(np.float32)


@dataclass
class DeviceNoiseSet:
    """Per-layer noise matrices and their (adapter-aware) effects, resident on the device."""

    seed: int
    k: int
    t_max: int
    noises: dict = field(default_factory=dict)        # addr -> [tensor [t_max, d_in]]
    effects: dict = field(default_factory=dict)       # addr -> [tensor [t_max, d_out]]
    base_effects: dict = field(default_factory=dict)  # addr -> [pre-IA3 effect] (IA3 clients)

    def pick(self, addr, iteration: int) -> int:
        return rotate(self.seed, addr, iteration, self.k)

    def blind(self, addr, x, iteration: int):
        t = int(x.shape[0])
        if t > self.t_max:
            raise ConfigError(f"token count {t} exceeds noise row budget t_max={self.t_max}")
        i = self.pick(addr, iteration)
        n = self.noises[addr][i][:t]
        return (x.to(n.dtype) + n if isinstance(x, torch.Tensor)
                else torch.as_tensor(np.asarray(x, np.float32), device=n.device) + n), i

    def unblind(self, addr, y_noisy, index: int):
        t = int(y_noisy.shape[0])
        return y_noisy.to(torch.float32) - self.effects[addr][index][:t]

    def unblind_base(self, addr, base_noisy, index: int):
        t = int(base_noisy.shape[0])
        return base_noisy.to(torch.float32) - self.base_effects[addr][index][:t]


def precompute_noise(channel, dims: dict, k: int, scale: float, seed: int, t_max: int,
                     layers=None, want_base: bool = False, device=None) -> DeviceNoiseSet:
    """``privacy.precompute_noise`` (privacy.py:79-106) over a device channel. ``dims`` maps
    each layer address to (d_in, d_out). Noise is uploaded as f32 (the executor rounds its
    GEMM operands to bf16; effects come back in the channel's dtype and are kept as f32)."""
    if k < 2:
        raise ConfigError(f"need at least 2 noise values per layer, got {k}")
    addrs = list(layers) if layers is not None else list(dims)
    ns = DeviceNoiseSet(seed=seed, k=k, t_max=t_max)
    for addr in addrs:
        d_in, _ = dims[addr]
        ns.noises[addr], ns.effects[addr], ns.base_effects[addr] = [], [], []
        for j in range(k):
            n = torch.as_tensor(draw_noise(seed, addr, j, t_max, d_in, scale), device=device)
            kw = {"want_base": True} if want_base else {}
            eff = channel.request(addr.block, int(addr.role), PASS_NOISE_EFFECT, n, **kw)
            eff = eff.to(torch.float32).clone()
            base = channel.last_base.to(torch.float32).clone() if want_base else None
            check = channel.request(addr.block, int(addr.role), PASS_NOISE_EFFECT, n)
            if not torch.allclose(eff, check.to(torch.float32), atol=1e-5):
                raise ProtocolError(f"noise effect for {addr} not reproducible across requests")
            ns.noises[addr].append(n.to(torch.float32))
            ns.effects[addr].append(eff)
            ns.base_effects[addr].append(base)
    return ns


def refresh(noise: DeviceNoiseSet, channel, dims: dict, layers=None, want_base: bool = False) -> None:
    """Recompute the effects of existing noises after the client's fused adapter changed (an
    optimizer step): the adapter is part of the effect, the noises stay the same."""
    for addr in (list(layers) if layers is not None else list(noise.noises)):
        for j, n in enumerate(noise.noises[addr]):
            kw = {"want_base": True} if want_base else {}
            eff = channel.request(addr.block, int(addr.role), PASS_NOISE_EFFECT, n, **kw)
            noise.effects[addr][j] = eff.to(torch.float32).clone()
            if want_base:
                noise.base_effects[addr][j] = channel.last_base.to(torch.float32).clone()


__all__ = ["DeviceNoiseSet", "draw_noise", "precompute_noise", "refresh", "rotate", "addr_key"]
