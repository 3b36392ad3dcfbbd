"""B200-native Symbiosis base executor (the splitserve hot path on sm_100a).

Public surface (drop-in for the reference's executor / channel / interception layer):

* ``GpuBaseExecutor``, ``BatchPolicy``, ``ExecutorMetrics``  — executor.py
* ``DeviceChannel``, ``DeviceBuffer``                          — channel.py
* ``IpcChannel``, ``IpcExecutorServer`` (client processes, CUDA IPC) — ipc.py
* ``VirtLayer``                                                — client.py
* ``Envelope`` / ``PASS_*``, ``LayerAddress`` / ``Role``, ``AffineParams``, ``MemoryLedger``
* ``SsContext`` — the raw C-ABI context (libss_b200.so, include/ss_b200.h)

Importing the package does not touch the GPU; creating an executor loads the CUDA library
and fails loudly if it is missing or no sm_100 device is present (there is no CPU path).
"""

from .config import (BLOCK_ROLES, IA3_ROLES, LayerAddress, ModelConfig, Role,  # noqa: F401
                     base_addresses, layer_dims, max_layer_width)
from .errors import (ConfigError, JobStateError, ProtocolError,  # noqa: F401
                     ShapeMismatchError, TransportError)
from .ledger import MemoryLedger  # noqa: F401
from .protocol import (COMPUTE_PASSES, PASS_BACKWARD, PASS_ERROR, PASS_FORWARD,  # noqa: F401
                       PASS_NOISE_EFFECT, Envelope, error_envelope, error_message)
from .tensor_ops import AffineParams  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):  # lazy: torch-heavy modules load on first use
    if name in ("GpuBaseExecutor", "BatchPolicy", "ExecutorMetrics"):
        from . import executor
        return getattr(executor, name)
    if name in ("DeviceChannel", "DeviceBuffer"):
        from . import channel
        return getattr(channel, name)
    if name in ("IpcChannel", "IpcExecutorServer", "IpcBuffer", "IpcEvent"):
        from . import ipc
        return getattr(ipc, name)
    if name == "VirtLayer":
        from .client import VirtLayer
        return VirtLayer
    if name in ("SsContext", "Seg", "SegmentTable"):
        from . import device
        return getattr(device, name)
    raise AttributeError(name)
