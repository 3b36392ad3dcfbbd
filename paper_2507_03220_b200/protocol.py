"""Envelope — the per-request routing record (reference: pkg/src/splitserve/protocol.py:37-89).

Pass values and the reply/error conventions are the reference's. Two optional device-side
extensions ride along for the fused executor and are ignored by the reference:

* ``reply_to``  – caller-owned device tensor [token_count, out_width] that receives the
  result (the client's exchange buffer); without it the executor allocates the output.
* ``base_to``   – caller-owned device tensor receiving the pre-IA3 output y_base, which an
  IA3 fine-tuning client needs for dl = sum(dy * y_base) (client.py:241-242, 291-294).
* ``ready``     – a torch.cuda.Event the executor's stream waits on before reading payload
  (the "payload visible before the control message" rule).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

import numpy as np

from .config import LayerAddress, Role

PASS_FORWARD = 0
PASS_BACKWARD = 1
PASS_NOISE_EFFECT = 2
PASS_REGISTER = 16
PASS_DEREGISTER = 17
PASS_ACK = 32
PASS_ERROR = 255

COMPUTE_PASSES = (PASS_FORWARD, PASS_BACKWARD, PASS_NOISE_EFFECT)


@dataclass
class Envelope:
    client_id: int
    request_id: int
    block: int
    role: int
    pass_kind: int
    payload: Any                      # [token_count, width]: numpy f32, or torch tensor
    reply_to: Any = field(default=None, repr=False)
    base_to: Any = field(default=None, repr=False)
    ready: Any = field(default=None, repr=False)
    done: Any = field(default=None, repr=False)   # set on replies: torch.cuda.Event

    @property
    def token_count(self) -> int:
        return int(self.payload.shape[0])

    @property
    def width(self) -> int:
        return int(self.payload.shape[1]) if len(self.payload.shape) == 2 else 0

    @property
    def layer(self) -> LayerAddress:
        return LayerAddress(int(self.block), Role(int(self.role)))


def error_envelope(like, message: str) -> Envelope:
    """PASS_ERROR reply carrying a UTF-8 message (protocol.py:86-89)."""
    data = np.frombuffer(message.encode("utf-8"), dtype=np.uint8)
    return Envelope(like.client_id, like.request_id, like.block, like.role, PASS_ERROR, data)


def error_message(env) -> str:
    return bytes(np.asarray(env.payload, dtype=np.uint8)).decode("utf-8", errors="replace")


def control_envelope(client_id: int, request_id: int, pass_kind: int, flag: int = 0) -> Envelope:
    return Envelope(client_id, request_id, 0, flag, pass_kind, np.empty((0, 0), dtype=np.float32))
