"""Multi-GPU host logic on CPU: client partitioning (segment-parallel replicas) and the
tensor-parallel shard / collective plan, run as world-size-2 gloo process groups with the
oracle standing in for the per-rank device compute (test-only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import splitserve_oracle as O
from paper_2507_03220_b200 import parallel_plan as P
from paper_2507_03220_b200.config import Role


def test_partition_clients_balanced_and_complete():
    tokens = {c: t for c, t in enumerate([1024] * 16 + [2] * 16 + [512] * 3)}
    for world in (1, 2, 4, 8):
        parts = P.partition_clients(tokens, world)
        flat = sorted(c for cs in parts.values() for c in cs)
        assert flat == sorted(tokens)
        loads = [sum(tokens[c] for c in cs) for cs in parts.values()]
        assert max(loads) - min(loads) <= max(tokens.values())
        assert P.partition_clients(tokens, world) == parts  # deterministic


@pytest.mark.parametrize("n,world", [(5120, 2), (13824, 8), (32000, 4), (8, 2), (1728, 8)])
def test_shard_bounds_cover_exactly(n, world):
    spans = [P.shard_bounds(n, r, world) for r in range(world)]
    covered = np.zeros(n, int)
    for lo, hi in spans:
        covered[lo:hi] += 1
    assert (covered == 1).all()


def test_collective_table_matches_survey():
    # forward all-reduce only at row-parallel layers; backward mirrored
    assert P.plan_layer(Role.Q, 8, 8, 0, 2).collective(0) == "all_gather"
    assert P.plan_layer(Role.O, 8, 8, 0, 2).collective(0) == "all_reduce"
    assert P.plan_layer(Role.FF_UP, 8, 16, 0, 2).collective(1) == "all_reduce"
    assert P.plan_layer(Role.FF_DOWN, 16, 8, 0, 2).collective(1) == "all_gather"
    # 13B, TP=8: per-token bytes of O fwd: fp32 reduce-scatter + bf16 all-gather, 7/8 x 5120 x 6
    b = P.comm_bytes_per_token(5120, 5120, Role.O, 0, 8)
    assert b == 7 / 8 * 5120 * 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [(Role.Q, 48, 40), (Role.O, 40, 48), (Role.FF_UP, 48, 72), (Role.FF_DOWN, 72, 48),
         (Role.LM_HEAD, 48, 100), (Role.K, 40, 40)]


def _reference(role, d_in, d_out):
    w, b = O.layer_params(5, 0, int(role), d_in, d_out)
    ads = {0: O.lora_params(5, 0, 0, int(role), d_in, d_out, 4, 8.0)}
    if role in (Role.K, Role.FF_UP):
        ads[1] = O.ia3_params(5, 1, 0, int(role), d_out)
    rng = np.random.default_rng(int(role))
    rows = [3, 5, 2]
    xs = {0: [rng.standard_normal((t, d_in)).astype(np.float32) for t in rows],
          1: [rng.standard_normal((t, d_out)).astype(np.float32) for t in rows]}
    return w, b, ads, xs


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for role, d_in, d_out in CASES:
            w, b, ads, xs = _reference(role, d_in, d_out)
            spec = P.plan_layer(role, d_in, d_out, rank, world)
            ws, bs = P.shard_params(spec, w, b)
            sads = {}
            for c, ad in ads.items():
                lora = (ad.a, ad.b) if ad.a is not None else None
                sl, si = P.shard_adapter(spec, lora, ad.ia3)
                sads[c] = O.OracleAdapter(a=None if sl is None else np.ascontiguousarray(sl[0]),
                                          b=None if sl is None else np.ascontiguousarray(sl[1]),
                                          alpha=ad.alpha, rank=ad.rank,
                                          ia3=None if si is None else np.ascontiguousarray(si))
            for pass_kind in (0, 1):

                def compute(local_in):
                    envs = [O.OracleEnvelope(c, 1, 0, int(role), pass_kind,
                                             np.ascontiguousarray(x.numpy())) for c, x in enumerate(local_in)]
                    res = O.fused_compute_batch(pass_kind, envs, np.ascontiguousarray(ws),
                                                None if bs is None else np.ascontiguousarray(bs), sads)
                    return [torch.from_numpy(np.ascontiguousarray(r[0])) for r in res]

                got = P.tp_dispatch(spec, pass_kind, [torch.from_numpy(x) for x in xs[pass_kind]], compute)
                full = O.fused_compute_batch(pass_kind, [O.OracleEnvelope(c, 1, 0, int(role), pass_kind, x)
                                                         for c, x in enumerate(xs[pass_kind])], w, b, ads)
                for c, (g, f) in enumerate(zip(got, full)):
                    if not np.allclose(g.numpy(), f[0], rtol=1e-4, atol=1e-4):
                        q.put((rank, f"{role.name} pass {pass_kind} client {c}: max err "
                                     f"{np.abs(g.numpy() - f[0]).max():.3e}"))
                        return
        q.put((rank, "ok"))
    finally:
        dist.destroy_process_group()


def test_tensor_parallel_world2_matches_unsharded_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(60)
    assert all(msg == "ok" for _, msg in results), results


def _finish_worker(rank, world, port, q):
    """Each rank writes its share of a known full-width output into the buffers
    dispatch_buffers hands out (what its plan's kernels write), then finish_dispatch must
    leave the full result in `reply` on every rank: bitwise for the all-gather layers, the
    one bf16 rounding of the fp32 sum for the all-reduce layers."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pool = {}

        def alloc(tag, shape, dtype):
            key = (tag, shape, dtype)
            if key not in pool:
                pool[key] = torch.full(shape, float("nan"), dtype=dtype)
            return pool[key]

        rows = 7
        for role, d_in, d_out in CASES + [(Role.FF_UP, 48, 200)]:
            spec = P.plan_layer(role, d_in, d_out, rank, world)
            for pass_kind in (0, 1):
                full_w = d_in if pass_kind == 1 else d_out
                g = torch.Generator().manual_seed(int(role) * 10 + pass_kind)
                want = torch.randn(rows, full_w, generator=g).to(torch.bfloat16)
                kind, local, gbuf, reply = P.dispatch_buffers(spec, pass_kind, rows, world, rank, alloc)
                if kind == "all_reduce":
                    parts = [want.float() * 0.5 for _ in range(world)]     # exact halves
                    local.copy_(parts[rank])
                elif kind == "all_gather":
                    lo, hi = spec.lo, spec.hi
                    assert local.shape == (rows, hi - lo)
                    local.copy_(want[:, lo:hi])
                P.finish_dispatch(kind, local, gbuf, reply)
                if not torch.equal(reply, want):
                    q.put((rank, f"{role.name} pass {pass_kind} ({kind}) mismatch"))
                    return
        q.put((rank, "ok"))
    finally:
        dist.destroy_process_group()


def test_plan_collectives_world2_reassemble_full_rows():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_finish_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(60)
    assert all(msg == "ok" for _, msg in results), results
