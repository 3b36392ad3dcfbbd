"""Multi-GPU planning for the base executor.

Two modes, both one process per GPU over ``torch.distributed``:

* **Segment-parallel replicas** (default; what ``bench.py --gpus N`` measures). The executor is
  stateless and rows are independent (tensor_ops.py:1-8), so every rank holds a full bf16 replica
  and serves a disjoint subset of clients. No collective on the data path. ``partition_clients``
  assigns clients to ranks (greedy on token load, deterministic).

* **Tensor parallel** (the north star's mode). Column split (shard d_out) for Q, K, V, FF_UP and
  LM_HEAD, row split (shard d_in) for O and FF_DOWN. Because the client does attention / SiLU
  between layers (client.py:240-269), activations cannot stay sharded between layers, so each
  dispatch ends in one collective:

  ============  ===============================  ===============================
  layer split   forward                          backward (input gradient)
  ============  ===============================  ===============================
  column (N)    each rank: y[:, n-slice] -> all-gather over N     partial dx -> all-reduce
  row (K)       each rank: partial y (bias on rank 0) -> all-reduce   dx[:, k-slice] -> all-gather
  ============  ===============================  ===============================

  Adapters shard with their layer: column layers keep A replicated and slice B[:, n] and l[n];
  row layers slice A[k, :] and keep B replicated (the LoRA delta is linear in the K-partials,
  so it rides the same all-reduce; IA3 only targets column-split roles K/V/FF_UP).

The per-rank compute is a plain executor dispatch over the shard (C ABI, device pointers); this
module only plans shapes and runs the collectives, so it is testable on CPU with gloo
(tests/test_parallel_plan.py) by passing a reference compute function.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import Role

COLUMN_ROLES = frozenset((Role.Q, Role.K, Role.V, Role.FF_UP, Role.LM_HEAD))
ROW_ROLES = frozenset((Role.O, Role.FF_DOWN))


def partition_clients(tokens: dict, world: int) -> dict[int, list]:
    """Greedy longest-processing-time assignment of clients (id -> token count) to ranks.
    Deterministic: ties broken by client id. Every client lands on exactly one rank."""
    load = [0] * world
    out: dict[int, list] = {r: [] for r in range(world)}
    for cid in sorted(tokens, key=lambda c: (-tokens[c], c)):
        r = min(range(world), key=lambda i: (load[i], i))
        out[r].append(cid)
        load[r] += tokens[cid]
    for r in out:
        out[r].sort()
    return out


def shard_bounds(n: int, rank: int, world: int, align: int = 64) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n for `rank`; slice sizes are multiples of `align` except
    the last (d_ff / 8 = 1728 for 13B is not a multiple of 128 — ragged tiles are handled by
    the kernel's TMA bounds)."""
    per = -(-n // world)
    per = -(-per // align) * align
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


@dataclass(frozen=True)
class ShardSpec:
    role: Role
    split: str          # "column" | "row"
    lo: int
    hi: int
    d_in: int
    d_out: int
    rank: int
    world: int

    @property
    def shard_in(self) -> int:
        return self.hi - self.lo if self.split == "row" else self.d_in

    @property
    def shard_out(self) -> int:
        return self.hi - self.lo if self.split == "column" else self.d_out

    def collective(self, pass_kind: int) -> str:
        """'all_gather' | 'all_reduce' for this layer and pass (table in the module doc)."""
        fwd = pass_kind != 1
        if self.split == "column":
            return "all_gather" if fwd else "all_reduce"
        return "all_reduce" if fwd else "all_gather"


def plan_layer(role, d_in: int, d_out: int, rank: int, world: int) -> ShardSpec:
    role = Role(role)
    if role in COLUMN_ROLES:
        lo, hi = shard_bounds(d_out, rank, world)
        return ShardSpec(role, "column", lo, hi, d_in, d_out, rank, world)
    lo, hi = shard_bounds(d_in, rank, world)
    return ShardSpec(role, "row", lo, hi, d_in, d_out, rank, world)


def shard_params(spec: ShardSpec, weight, bias):
    """This rank's (weight, bias) for the layer. Row split keeps the bias on rank 0 only, so
    the all-reduce adds it exactly once."""
    if spec.split == "column":
        w = weight[:, spec.lo:spec.hi]
        b = None if bias is None else bias[spec.lo:spec.hi]
    else:
        w = weight[spec.lo:spec.hi, :]
        b = bias if spec.rank == 0 else None
    return w, b


def shard_adapter(spec: ShardSpec, lora=None, ia3=None):
    """Shard one layer's adapter: lora = (A [d_in, r], B [r, d_out]), ia3 = l [d_out]."""
    out_lora, out_ia3 = None, None
    if lora is not None:
        a, b = lora
        out_lora = (a, b[:, spec.lo:spec.hi]) if spec.split == "column" else (a[spec.lo:spec.hi, :], b)
    if ia3 is not None:
        if spec.split != "column":
            raise ValueError("IA3 targets K/V/FF_UP, which are column-split")
        out_ia3 = ia3[spec.lo:spec.hi]
    return out_lora, out_ia3


def shard_input(spec: ShardSpec, pass_kind: int, x):
    """The slice of a full-width request payload this rank consumes."""
    if pass_kind == 1:      # backward: payload is dy [t, d_out]
        return x[:, spec.lo:spec.hi] if spec.split == "column" else x
    return x[:, spec.lo:spec.hi] if spec.split == "row" else x


def combine(spec: ShardSpec, pass_kind: int, local, group=None):
    """Run the layer's collective on this rank's output (torch tensor [t, *]) and return the
    full-width result on every rank."""
    import torch
    import torch.distributed as dist

    kind = spec.collective(pass_kind)
    if kind == "all_reduce":
        out = local.contiguous()
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
        return out
    sizes = [shard_bounds(spec.d_out if spec.split == "column" else spec.d_in, r, spec.world)
             for r in range(spec.world)]
    width = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((local.shape[0], width), dtype=local.dtype, device=local.device)
    pad[:, : local.shape[1]] = local
    parts = [torch.empty_like(pad) for _ in range(spec.world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:, : hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=1)


def tp_dispatch(spec: ShardSpec, pass_kind: int, payloads, compute, group=None):
    """One tensor-parallel dispatch: slice each segment's payload for this rank, run `compute`
    (rank-local batch over the shard: list of [t_i, shard_in] -> list of [t_i, shard_out]
    (fwd) / [t_i, d_in or slice] (bwd)), then the collective per segment batch.

    Segments are concatenated for the collective (one call per dispatch, in batch order) and
    split back with the reference's prefix offsets (split_rows, tensor_ops.py:149-156)."""
    import torch

    local_in = [shard_input(spec, pass_kind, p) for p in payloads]
    local_out = compute(local_in)
    counts = [int(p.shape[0]) for p in payloads]
    cat = torch.cat([torch.as_tensor(o) for o in local_out], dim=0) if local_out else None
    if cat is None:
        return []
    full = combine(spec, pass_kind, cat, group)
    out, pos = [], 0
    for c in counts:
        out.append(full[pos:pos + c])
        pos += c
    return out


def comm_bytes_per_token(d_in: int, d_out: int, role, pass_kind: int, world: int, esz: int = 2) -> float:
    """Ring-algorithm bytes each rank sends per token for one dispatch (SURVEY §8e budget)."""
    spec = plan_layer(role, d_in, d_out, 0, world)
    width = spec.d_out if pass_kind != 1 else spec.d_in
    f = (world - 1) / world
    if spec.collective(pass_kind) == "all_reduce":
        # reduce-scatter of fp32 partials + all-gather of the bf16 rows (dispatch_buffers)
        return f * width * (4 + esz)
    return f * width * esz


def ratio_check(a, b, rtol=1e-5, atol=1e-5) -> bool:
    return np.allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), rtol=rtol, atol=atol)


def dispatch_buffers(spec: ShardSpec, pass_kind: int, rows: int, world: int, rank: int, alloc, tag=""):
    """Buffers of one prebuilt tensor-parallel dispatch: returns (kind, local, gbuf, reply).

    `local` is what this rank's kernels write:
    * all-reduce layers: fp32 partials [rows, full] (rows of a buffer padded to a multiple of
      the world size). The collective is a REDUCE-SCATTER of the fp32 partials (each rank sums
      1/world of the rows exactly, in fp32), one bf16 rounding, then an ALL-GATHER of bf16 rows
      straight into the reply: (world-1)/world x (4 + 2) bytes per element instead of an fp32
      all-reduce's 2 x 4, and the same single rounding as on one GPU;
    * all-gather layers: a column view of a padded bf16 shard buffer;
    * world size 1: the reply itself.
    `alloc(tag, shape, dtype)` provides (possibly shared) tensors; `tag` separates the buffers of
    pipelined slabs of one dispatch."""
    import torch
    full = spec.d_in if pass_kind == 1 else spec.d_out
    kind = spec.collective(pass_kind) if world > 1 else "none"
    if kind == "all_reduce":
        rows_pad = -(-rows // world) * world
        part = alloc("partial" + tag, (rows_pad, full), torch.float32)
        rs = alloc("rs" + tag, (rows_pad // world, full), torch.float32)
        rs_bf = alloc("rs_bf16" + tag, (rows_pad // world, full), torch.bfloat16)
        gathered = alloc("gathered_rows" + tag, (rows_pad, full), torch.bfloat16)
        return kind, part[:rows], (part, rs, rs_bf, gathered), gathered[:rows]
    reply = alloc("reply" + tag, (rows, full), torch.bfloat16)
    if kind == "all_gather":
        sizes = [shard_bounds(spec.d_out if spec.split == "column" else spec.d_in, q, world) for q in range(world)]
        wmax = max(hi - lo for lo, hi in sizes)
        pad = alloc("shard" + tag, (rows, wmax), torch.bfloat16)
        local = pad[:, : sizes[rank][1] - sizes[rank][0]]
        return kind, local, (pad, alloc("gathered" + tag, (world * rows, wmax), torch.bfloat16), sizes), reply
    return kind, reply, None, reply


def finish_dispatch(kind: str, local, gbuf, reply, group=None) -> None:
    """The dispatch's collective, landing the full-width result in `reply` on every rank:
    reduce-scatter the fp32 partials, round once to bf16, all-gather the rows (all-reduce
    layers); or all-gather the padded column shards and reassemble them (all-gather layers).
    Runs on the caller's current CUDA stream (a comm stream when slabs are pipelined)."""
    import torch.distributed as dist
    if kind == "all_reduce":
        part, rs, rs_bf, gathered = gbuf
        dist.reduce_scatter_tensor(rs, part, op=dist.ReduceOp.SUM, group=group)
        rs_bf.copy_(rs)
        dist.all_gather_into_tensor(gathered, rs_bf, group=group)   # `reply` is a view of it
    elif kind == "all_gather":
        pad, out, sizes = gbuf
        dist.all_gather_into_tensor(out, pad, group=group)
        m = pad.shape[0]
        for q, (lo, hi) in enumerate(sizes):
            reply[:, lo:hi].copy_(out[q * m:(q + 1) * m, : hi - lo])
