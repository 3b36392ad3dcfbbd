"""Byte ledger of the executor (reference: pkg/src/splitserve/ledger.py:18-53).

Same categories and semantics: WEIGHTS is set at load, SAVED_ACTIVATIONS must stay 0
(statelessness), TRANSIENT_BUFFER is set/cleared per batch with a high-water mark. Bytes
here are the device bytes actually held (bf16 weights, f32 bias, adapter packs, workspace).
"""

from __future__ import annotations

WEIGHTS = "weights"
ADAPTER = "adapter"
KV_CACHE = "kv_cache"
OPTIMIZER = "optimizer"
SAVED_ACTIVATIONS = "saved_activations"
TRANSIENT_BUFFER = "transient_buffer"
CATEGORIES = (WEIGHTS, ADAPTER, KV_CACHE, OPTIMIZER, SAVED_ACTIVATIONS, TRANSIENT_BUFFER)


class MemoryLedger:
    def __init__(self, owner: str):
        self.owner = owner
        self._bytes = dict.fromkeys(CATEGORIES, 0)
        self.transient_high_water = 0

    def set(self, category: str, nbytes: int) -> None:
        self._bytes[category] = int(nbytes)
        if category == TRANSIENT_BUFFER and nbytes > self.transient_high_water:
            self.transient_high_water = int(nbytes)

    def add(self, category: str, delta: int) -> None:
        self.set(category, self._bytes[category] + int(delta))

    def get(self, category: str) -> int:
        return self._bytes[category]

    def total(self, include_transient: bool = True) -> int:
        held = sum(v for c, v in self._bytes.items() if c != TRANSIENT_BUFFER)
        return held + (self.transient_high_water if include_transient else 0)

    def snapshot(self) -> dict:
        return dict(self._bytes)
