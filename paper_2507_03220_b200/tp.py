"""Tensor-parallel base executor: one rank of a TP group (north-star mode).

Each rank holds its column / row shard of every frozen layer (parallel_plan.plan_layer) in its
own libss_b200 context, computes its part of every dispatch through the same C-ABI call as the
single-GPU executor — column-sharded inputs and outputs are strided VIEWS of the full-width
client buffers (the ABI takes a row stride), so slicing costs nothing — and finishes the
dispatch with one collective over torch.distributed (NCCL over NVLink on a B200 box):
all-gather for column layers in forward / row layers in backward, all-reduce (sum) for row
layers in forward / column layers in backward. Adapters shard with their layer
(parallel_plan.shard_adapter).

Reduce-type partials are produced in fp32 by default (`reduce_dtype`), so the only bf16
rounding is the final one, as on one GPU.
"""

from __future__ import annotations

import torch

from . import parallel_plan as P
from .config import Role, addr_key
from .executor import GpuBaseExecutor
from .protocol import PASS_BACKWARD, Envelope
from .tensor_ops import AffineParams


class TensorParallelExecutor:
    def __init__(self, layers, rank: int, world: int, *, device: int = 0, group=None,
                 reduce_dtype=torch.float32):
        self.rank, self.world, self.group = rank, world, group
        self.reduce_dtype = reduce_dtype
        self.specs: dict[tuple[int, int], P.ShardSpec] = {}
        shards = []
        for addr, p in (layers.items() if hasattr(layers, "items") else layers):
            key = addr_key(addr)
            d_in, d_out = int(p.weight.shape[0]), int(p.weight.shape[1])
            spec = P.plan_layer(Role(key[1]), d_in, d_out, rank, world)
            self.specs[key] = spec
            w, b = P.shard_params(spec, p.weight, p.bias)
            shards.append((addr, AffineParams(_contig(w), None if b is None else _contig(b))))
        self.ex = GpuBaseExecutor(shards, device=device, retain_layers=False)
        self.device = self.ex.device
        self._rid = 0

    def register_adapter(self, client_id: int, adapter) -> None:
        class _Shard:
            pass
        sh = _Shard()
        sh.alpha, sh.rank = getattr(adapter, "alpha", 0.0), getattr(adapter, "rank", 1)
        sh.lora, sh.ia3 = {}, {}
        for addr, (a, b) in (getattr(adapter, "lora", {}) or {}).items():
            lo, _ = P.shard_adapter(self.specs[addr_key(addr)], (a, b), None)
            sh.lora[addr] = (_contig(lo[0]), _contig(lo[1]))
        for addr, l in (getattr(adapter, "ia3", {}) or {}).items():
            _, li = P.shard_adapter(self.specs[addr_key(addr)], None, l)
            sh.ia3[addr] = _contig(li)
        self.ex.register_adapter(client_id, sh)

    # ------------------------------------------------------------------------- dispatch
    def dispatch_local(self, pass_kind: int, block: int, role: int, payloads, client_ids):
        """This rank's share: returns (spec, local [M, w] tensor, row counts). Column-split
        inputs are strided views of the full payloads (no copy)."""
        key = (int(block), int(role))
        spec = self.specs[key]
        reduce = spec.collective(pass_kind) == "all_reduce"
        out_w = spec.shard_in if pass_kind == PASS_BACKWARD else spec.shard_out
        if reduce:
            out_w = spec.d_in if pass_kind == PASS_BACKWARD else spec.d_out
        counts = [int(x.shape[0]) for x in payloads]
        # a single rank has nothing to sum: its "partials" are the final bf16 rows
        dt = self.reduce_dtype if (reduce and self.world > 1) else payloads[0].dtype
        local = torch.empty((sum(counts), out_w), dtype=dt, device=self.device)
        envs, pos = [], 0
        for cid, x, t in zip(client_ids, payloads, counts):
            self._rid += 1
            envs.append(Envelope(cid, self._rid, block, role, pass_kind, P.shard_input(spec, pass_kind, x),
                                 reply_to=local[pos:pos + t]))
            pos += t
        res = self.ex._compute_batch(pass_kind, envs)
        for r in res:
            if not isinstance(r, torch.Tensor):
                raise r
        return spec, local, counts

    def dispatch(self, pass_kind: int, block: int, role: int, payloads, client_ids):
        """Full-width outputs for every segment on every rank (one collective)."""
        spec, local, counts = self.dispatch_local(pass_kind, block, role, payloads, client_ids)
        full = P.combine(spec, pass_kind, local, self.group) if self.world > 1 else local
        if full.dtype != payloads[0].dtype:
            full = full.to(payloads[0].dtype)
        out, pos = [], 0
        for t in counts:
            out.append(full[pos:pos + t])
            pos += t
        return out


def combine_local(spec_parts, pass_kind: int):
    """Collective of one dispatch emulated in-process: spec_parts = [(spec, local)] for every
    rank in rank order (used to test the sharded CUDA path on a single GPU)."""
    spec0 = spec_parts[0][0]
    if spec0.collective(pass_kind) == "all_reduce":
        out = spec_parts[0][1].clone()
        for _, loc in spec_parts[1:]:
            out += loc
        return out
    return torch.cat([loc for _, loc in spec_parts], dim=1)


def _contig(x):
    if isinstance(x, torch.Tensor):
        return x.contiguous()
    import numpy as np
    return np.ascontiguousarray(x)
