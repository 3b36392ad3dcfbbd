"""AffineParams — one frozen layer as handed to the executor (reference tensor_ops.py:39-68).

Only the parameter container lives here; the arithmetic runs in the CUDA library.
``weight`` is [d_in, d_out] (numpy f32/bf16-as-f32, or a torch tensor on the executor's
device), ``bias`` [d_out] or None.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any

from .errors import ShapeMismatchError


@dataclass
class AffineParams:
    weight: Any
    bias: Any = None

    def __post_init__(self):
        if len(self.weight.shape) != 2:
            raise ShapeMismatchError(f"weight must be 2-d, got shape {tuple(self.weight.shape)}")
        if self.bias is not None and tuple(self.bias.shape) != (self.weight.shape[1],):
            raise ShapeMismatchError(
                f"bias shape {tuple(self.bias.shape)} does not match d_out={self.weight.shape[1]}")

    @property
    def d_in(self) -> int:
        return int(self.weight.shape[0])

    @property
    def d_out(self) -> int:
        return int(self.weight.shape[1])

    @property
    def nbytes(self) -> int:
        def nb(a):
            if a is None:
                return 0
            return int(a.nbytes) if hasattr(a, "nbytes") else a.numel() * a.element_size()
        return nb(self.weight) + nb(self.bias)
