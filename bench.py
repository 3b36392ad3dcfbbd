"""Aggregate adapter tokens/sec of the B200 base executor (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 13b|7b] [--impl ours|reference]

One STEP = one executor pass of the workload: a forward dispatch of every one of
the 6L+1 frozen layers over all clients' token segments (LoRA / IA3 deltas fused), then a
backward (input-gradient) dispatch of every layer in reverse over the fine-tuning clients'
segments. Every client token counts once; fine-tune tokens cost fwd + bwd.

Default workload (BASELINE configs[2], the metric's Llama2-13B shape, on one GPU): d 5120,
d_ff 13824, L 40, V 32000; 32 clients = 24 LoRA (ranks 8/16/32/64, alpha = 2r, Q/K/V/O) + 8
IA3 (K, V, FF_UP); 16 fine-tune + 16 inference clients, 2 x 512 tokens each -> 32 768 rows per
forward dispatch, 16 384 per backward dispatch. Multi-GPU: one process per GPU, each a full
replica serving its own 32 clients (segment-parallel, no collective on the data path):
weak scaling, value = all ranks' tokens / max-over-ranks time.

Legs reported on one JSON line (rank 0):
  value   device-resident exchange buffers, one prebuilt C-ABI dispatch per layer and pass;
  e2e     the reference-facing API (GpuBaseExecutor._compute_batch with pinned HOST payloads
          and host reply buffers): H2D + compute + D2H per dispatch, like host clients;
  roofline  fused GEMM kernel, CUDA events around every launch in the timed region;
  cpu_baseline  the reference algorithm (oracle port) on host cores, bounded sample.
``--impl reference`` times only the reference algorithm on the host (rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aggregate adapter tokens/sec (fwd+bwd), Llama2-13B shape, N clients, 1/2/4/8 B200"

WORKLOADS = {
    # BASELINE configs[2] on one GPU (the metric's model shape)
    "13b": dict(name="llama2-13b-shape, 32 mixed LoRA(r8-64)+IA3 clients, 16 FT + 16 inference, 2x512 tok",
                d=5120, d_ff=13824, L=40, V=32000, clients=32, tokens=1024, seq=512, batch=2),
    # BASELINE configs[1]
    "7b": dict(name="llama2-7b-shape, 8 LoRA r16 fine-tune clients, 2x512 tok",
               d=4096, d_ff=11008, L=32, V=32000, clients=8, tokens=1024, seq=512, batch=2),
    # BASELINE configs[2]'s inference clients in their decode phase: every client sends one
    # token per sequence (batch 2) per layer -> 64-row forward dispatches, weight-streaming bound
    "13b-decode": dict(name="llama2-13b-shape, 32 mixed LoRA(r8-64)+IA3 inference clients, decode (2 tok/client/step)",
                       d=5120, d_ff=13824, L=40, V=32000, clients=32, tokens=2, seq=1, batch=2),
    # BASELINE configs[4]: adapter-count sweep with --clients {8,16,32,64}
    "granite20b": dict(name="granite-20b-shape, N LoRA r8 fine-tune clients, 1x2048 tok",
                       d=6144, d_ff=24576, L=52, V=49152, clients=64, tokens=2048, seq=2048, batch=1),
}
Q, K, V, O, FF_UP, FF_DOWN, LM_HEAD = range(7)


def client_specs(wl_key: str, n: int):
    """[(kind, rank, finetune)] per client."""
    if wl_key == "7b":
        return [("lora", 16, True) for _ in range(n)]
    if wl_key == "granite20b":
        return [("lora", 8, True) for _ in range(n)]
    if wl_key == "13b-decode":
        return [(k, r, False) for k, r, _ in client_specs("13b", n)]
    specs = []
    for c in range(n):
        if c < 24:
            specs.append(("lora", (8, 16, 32, 64)[c % 4], c % 2 == 0))
        else:
            specs.append(("ia3", 0, c % 2 == 0))
    return specs


def layer_list(wl):
    d, f, L, Vv = wl["d"], wl["d_ff"], wl["L"], wl["V"]
    dims = {Q: (d, d), K: (d, d), V: (d, d), O: (d, d), FF_UP: (d, f), FF_DOWN: (f, d), LM_HEAD: (d, Vv)}
    out = [(b, r) for b in range(L) for r in (Q, K, V, O, FF_UP, FF_DOWN)] + [(L, LM_HEAD)]
    return out, dims


def flops_per_step(wl, specs):
    """Algorithmic FLOPs of one step: 2*d_in*d_out per token per layer (fwd), the same again
    for fine-tune tokens (bwd), plus each client's LoRA 2*r*(d_in+d_out) per targeted layer."""
    layers, dims = layer_list(wl)
    t = wl["tokens"]
    total = 0.0
    for (_, r) in layers:
        di, do = dims[r]
        for kind, rank, ft in specs:
            passes = 2 if ft else 1
            f = 2.0 * di * do
            if kind == "lora" and r in (Q, K, V, O):
                f += 2.0 * rank * (di + do)
            total += passes * t * f
    return total


# ============================================================================ GPU leg

def cublas_same_shapes(wl_key, specs, device, reps=2):
    """torch.matmul (cuBLAS) bf16 over the step's GEMM shapes — every layer forward at the
    dispatch's M, then backward (dy.W^T) at the fine-tune clients' M — without adapters,
    gather/scatter or epilogue, on the same box right after the timed region: the library
    baseline the fused kernel is compared against (box-to-box power-state variance cancels)."""
    import torch
    wl = WORKLOADS[wl_key]
    layers, dims = layer_list(wl)
    t = wl["tokens"]
    m_f = len(specs) * t
    m_b = sum(1 for _, _, ft in specs if ft) * t
    g = torch.Generator(device=device).manual_seed(7)
    W = {r: (torch.randn(di, do, generator=g, device=device) / math.sqrt(di)).to(torch.bfloat16)
         for r, (di, do) in dims.items()}
    wmax = max(max(di, do) for di, do in dims.values())
    X = torch.randn(m_f * wmax, generator=g, device=device).to(torch.bfloat16)
    Y = torch.empty(m_f * wmax, dtype=torch.bfloat16, device=device)

    def step():
        for (_, r) in layers:
            di, do = dims[r]
            torch.matmul(X[: m_f * di].view(m_f, di), W[r], out=Y[: m_f * do].view(m_f, do))
        if m_b:
            for (_, r) in reversed(layers):
                di, do = dims[r]
                torch.matmul(X[: m_b * do].view(m_b, do), W[r].t(), out=Y[: m_b * di].view(m_b, di))

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = sum(2.0 * m_f * dims[r][0] * dims[r][1] + 2.0 * m_b * dims[r][0] * dims[r][1] for (_, r) in layers)
    del X, Y, W
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "tflops": flops / (ms / 1e3) / 1e12, "gemms_per_step": len(layers) * (2 if m_b else 1),
            "what": "torch.matmul bf16 (cuBLAS), the step's GEMM shapes without adapters, same box, after the timed region"}


def nvsmi_sampler(stop: threading.Event, out: list, index: int):
    cmd = ["nvidia-smi", f"--id={index}",
           "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
           "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
           "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"]
    try:
        p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except OSError:
        return
    try:
        while not stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            out.append([x.strip() for x in line.split(",")])
    finally:
        p.kill()
        p.wait()


def summarize_clocks(samples):
    if not samples:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
    sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
    mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({n for s in samples for n, v in zip(names, s[3:7]) if v.strip().lower() == "active"})
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": reasons, "samples": len(samples)}


INPLACE = False   # --inplace: replies written over the request buffers (SharedBuffer style)


def build_gpu_workload(wl_key, device, rank):
    import torch
    from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role

    wl = WORKLOADS[wl_key]
    layers, dims = layer_list(wl)
    specs = client_specs(wl_key, wl["clients"])
    seed = 1234 + 7919 * rank

    def gen_layers():
        g = torch.Generator(device=device)
        for (b, r) in layers:
            di, do = dims[r]
            g.manual_seed(seed * 1000 + b * 8 + r)
            w = torch.randn(di, do, generator=g, device=device, dtype=torch.float32)
            w = (w * (1.0 / math.sqrt(di))).to(torch.bfloat16)
            bias = 0.05 * torch.randn(do, generator=g, device=device)
            yield LayerAddress(b, Role(r)), AffineParams(w, bias)
            del w, bias

    ex = GpuBaseExecutor(gen_layers(), device=device.index, retain_layers=False)

    class Ad:
        def __init__(self):
            self.lora, self.ia3, self.alpha, self.rank = {}, {}, 0.0, 1

    g = torch.Generator(device=device)
    for c, (kind, rank_, ft) in enumerate(specs):
        ad = Ad()
        g.manual_seed(seed + 17 * c + 5)
        if kind == "lora":
            ad.alpha, ad.rank = 2.0 * rank_, rank_
            for b in range(wl["L"]):
                for r in (Q, K, V, O):
                    di, do = dims[r]
                    a = torch.randn(di, rank_, generator=g, device=device) / math.sqrt(di)
                    bm = 0.05 * torch.randn(rank_, do, generator=g, device=device)
                    ad.lora[LayerAddress(b, Role(r))] = (a, bm)
        else:
            for b in range(wl["L"]):
                for r in (K, V, FF_UP):
                    ad.ia3[LayerAddress(b, Role(r))] = 1.0 + 0.1 * torch.randn(dims[r][1], generator=g, device=device)
        ex.register_adapter(c, ad)
        del ad

    # per-client device exchange buffers (DeviceChannel sizing: tokens x max layer width)
    t = wl["tokens"]
    maxw = max(wl["d"], wl["d_ff"], wl["V"])
    # request and reply buffers per client (DeviceChannel keeps them apart: a reply written over
    # its own request rows would force the gather path, SharedBuffer semantics)
    bufs = [torch.randn(t * maxw, generator=g, device=device).to(torch.bfloat16) for _ in specs]
    outs = ([torch.empty(t * maxw, dtype=torch.bfloat16, device=device) for _ in specs]
            if not INPLACE else bufs)
    base_bufs = {c: torch.empty(t * wl["d_ff"], dtype=torch.bfloat16, device=device)
                 for c, (k, _, ft) in enumerate(specs) if k == "ia3" and ft}
    fwd, bwd = [], []
    for (b, r) in layers:
        di, do = dims[r]
        segs = []
        for c, (kind, _, ft) in enumerate(specs):
            base = None
            if c in base_bufs and r in (K, V, FF_UP):
                base = base_bufs[c][: t * do].view(t, do)
            segs.append((c, bufs[c][: t * di].view(t, di), outs[c][: t * do].view(t, do), base))
        fwd.append(ex.compile_dispatch(0, b, r, segs))
        segs = [(c, bufs[c][: t * do].view(t, do), outs[c][: t * di].view(t, di), None)
                for c, (kind, _, ft) in enumerate(specs) if ft]
        if segs:
            bwd.append(ex.compile_dispatch(1, b, r, segs))
    bwd.reverse()
    # adapter weight gradients of the fine-tune clients (ss_adapter_grads), per layer in backward
    # order: LoRA grad_a / grad_b from the layer input x and dy, IA3 grad_l from dy and y_base
    from paper_2507_03220_b200.device import GradSeg
    grads = []
    for (b, r) in reversed(layers):
        di, do = dims[r]
        jobs = []
        for c, (kind, rank_, ft) in enumerate(specs):
            if not ft:
                continue
            if kind == "lora" and r in (Q, K, V, O):
                jobs.append(GradSeg(c, dy=bufs[c][: t * do].view(t, do), x=bufs[c][: t * di].view(t, di),
                                    grad_a=torch.zeros(di, rank_, device=device),
                                    grad_b=torch.zeros(rank_, do, device=device), accumulate=True))
            elif kind == "ia3" and r in (K, V, FF_UP):
                jobs.append(GradSeg(c, dy=bufs[c][: t * do].view(t, do), y_base=base_bufs[c][: t * do].view(t, do),
                                    grad_l=torch.zeros(do, device=device), accumulate=True))
        if jobs:
            grads.append((b, r, jobs))
    ex._bench_grads = grads
    return ex, fwd + bwd, specs, wl


def run_step(plan, stream):
    for d in plan:
        d.run(stream)


def build_tp_workload(wl_key, device, rank, world):
    """--parallel tp: every rank serves ALL clients with its column / row shard of every layer
    (paper_2507_03220_b200.tp); each dispatch ends in one NCCL all-gather or all-reduce.
    All ranks generate the same full layers (rank-independent seeds) and keep their shard."""
    import torch
    from paper_2507_03220_b200 import AffineParams, LayerAddress, Role
    from paper_2507_03220_b200.tp import TensorParallelExecutor

    wl = WORKLOADS[wl_key]
    layers, dims = layer_list(wl)
    specs = client_specs(wl_key, wl["clients"])
    seed = 1234

    def gen_layers():
        g = torch.Generator(device=device)
        for (b, r) in layers:
            di, do = dims[r]
            g.manual_seed(seed * 1000 + b * 8 + r)
            w = (torch.randn(di, do, generator=g, device=device) * (1.0 / math.sqrt(di))).to(torch.bfloat16)
            yield LayerAddress(b, Role(r)), AffineParams(w, 0.05 * torch.randn(do, generator=g, device=device))

    tp = TensorParallelExecutor(gen_layers(), rank, world, device=device.index)

    class Ad:
        def __init__(self):
            self.lora, self.ia3, self.alpha, self.rank = {}, {}, 0.0, 1

    g = torch.Generator(device=device)
    for c, (kind, rank_, ft) in enumerate(specs):
        ad = Ad()
        g.manual_seed(seed + 17 * c + 5)
        if kind == "lora":
            ad.alpha, ad.rank = 2.0 * rank_, rank_
            for b in range(wl["L"]):
                for r in (Q, K, V, O):
                    di, do = dims[r]
                    ad.lora[LayerAddress(b, Role(r))] = (torch.randn(di, rank_, generator=g, device=device) / math.sqrt(di),
                                                         0.05 * torch.randn(rank_, do, generator=g, device=device))
        else:
            for b in range(wl["L"]):
                for r in (K, V, FF_UP):
                    ad.ia3[LayerAddress(b, Role(r))] = 1.0 + 0.1 * torch.randn(dims[r][1], generator=g, device=device)
        tp.register_adapter(c, ad)
    t = wl["tokens"]
    maxw = max(wl["d"], wl["d_ff"], wl["V"])
    # request and reply buffers per client (DeviceChannel keeps them apart: a reply written over
    # its own request rows would force the gather path, SharedBuffer semantics)
    bufs = [torch.randn(t * maxw, generator=g, device=device).to(torch.bfloat16) for _ in specs]
    outs = ([torch.empty(t * maxw, dtype=torch.bfloat16, device=device) for _ in specs]
            if not INPLACE else bufs)
    # Prebuilt per-rank dispatches (ss_plan_*): each rank computes its shard of every dispatch
    # straight from the clients' full-width buffers (column slices are strided views) into a
    # dispatch-wide output; then ONE collective finishes the dispatch: all-reduce of fp32
    # partials (converted to bf16 into the reply rows) or all-gather of the column shards
    # (reassembled into the reply rows). World size 1: the shard IS the layer, no collective.
    from paper_2507_03220_b200 import parallel_plan as P
    ft = [c for c, s_ in enumerate(specs) if s_[2]]
    plan = []
    pool = {}   # dispatch-wide buffers, shared by every dispatch of the same shape (reused)

    def buf(tag, shape, dtype):
        key = (tag, shape, dtype)
        if key not in pool:
            pool[key] = torch.empty(shape, dtype=dtype, device=device)
        return pool[key]

    def add(pass_kind, b, r, cids):
        """One dispatch as `slabs` prebuilt sub-dispatches over consecutive client groups (rows
        are independent: bitwise the same rows as one dispatch), each with its own collective,
        so the collective of slab k runs on the comm stream under the GEMM of slab k+1."""
        di, do = dims[r]
        spec = tp.specs[(b, r)]
        w_in = do if pass_kind == 1 else di
        parts = []
        n = 1 if world == 1 else max(1, min(TP_SLABS, len(cids)))   # (nothing to overlap alone)
        groups = [cids[i * len(cids) // n:(i + 1) * len(cids) // n] for i in range(n)]
        for k, grp in enumerate(groups):
            kind, local, gbuf, reply = P.dispatch_buffers(spec, pass_kind, len(grp) * t, world, rank, buf, tag=f"/{k}")
            segs = [(c, P.shard_input(spec, pass_kind, bufs[c][: t * w_in].view(t, w_in)), local[j * t:(j + 1) * t], None)
                    for j, c in enumerate(grp)]
            parts.append((tp.ex.compile_dispatch(pass_kind, b, r, segs), kind, local, gbuf, reply))
        plan.append(parts)

    for (b, r) in layers:
        add(0, b, r, list(range(len(specs))))
    for (b, r) in reversed(layers):
        if ft:
            add(1, b, r, ft)
    tp.comm_stream = torch.cuda.Stream(device)
    return tp, plan, specs, wl


TP_SLABS = 4   # sub-dispatches per TP dispatch (collective of slab k overlaps the GEMM of slab k+1)


def run_step_tp(tp, plan):
    import torch
    from paper_2507_03220_b200.parallel_plan import finish_dispatch
    stream = torch.cuda.current_stream(tp.device)
    comm = tp.comm_stream
    for parts in plan:
        for disp, kind, local, gbuf, reply in parts:
            disp.run(stream)
            if kind == "none":
                continue
            comm.wait_stream(stream)           # this slab's partials / shards are written
            with torch.cuda.stream(comm):
                finish_dispatch(kind, local, gbuf, reply, tp.group)
        stream.wait_stream(comm)               # the dispatch's replies are complete


def tp_leg(wl_key, device, rank, world, steps, warmup):
    """Beside the replicas line at N > 1: the north star's tensor-parallel executor over the
    same N GPUs (strong scaling: the SAME 32 clients served by N column/row shards, one
    reduce-scatter+all-gather or all-gather per slab), timed like the main leg (barrier, CUDA
    events, max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2507_03220_b200 import parallel_plan as P
    tp, plan, specs, wl = build_tp_workload(wl_key, device, rank, world)
    stream = torch.cuda.current_stream(device)
    for _ in range(max(3, warmup)):
        run_step_tp(tp, plan)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        run_step_tp(tp, plan)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    layers, dims = layer_list(wl)
    tok = wl["tokens"]
    n_all, n_ft = len(specs), sum(1 for s_ in specs if s_[2])
    comm = sum(P.comm_bytes_per_token(dims[r][0], dims[r][1], r, 0, world) * n_all * tok +
               P.comm_bytes_per_token(dims[r][0], dims[r][1], r, 1, world) * n_ft * tok for (_, r) in layers)
    tp.ex.close()
    return {"value": n_all * tok / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms, "scaling": "strong",
            "n_gpus": world, "slabs_per_dispatch": TP_SLABS,
            "comm_bytes_per_rank_per_step": comm,
            "what": "tensor-parallel executor (column split Q/K/V/FF_UP/LM_HEAD, row split O/FF_DOWN), "
                    "same 32 clients on all ranks; fp32 reduce-scatter + bf16 all-gather / bf16 all-gather "
                    "per slab on a comm stream overlapping the next slab's GEMM"}


def e2e_leg(ex, wl_key, specs, steps, device):
    """Reference-facing path: numpy-like HOST clients. Each dispatch: pinned host payloads ->
    H2D -> fused compute -> D2H into pinned host reply buffers (in place, like LocalChannel's
    SharedBuffer), all inside the timed region."""
    import torch
    from paper_2507_03220_b200 import Envelope

    wl = WORKLOADS[wl_key]
    layers, dims = layer_list(wl)
    t = wl["tokens"]
    maxw = max(wl["d"], wl["d_ff"], wl["V"])
    host = [torch.empty(t * maxw, dtype=torch.bfloat16, pin_memory=True) for _ in specs]
    reply = [torch.empty(t * maxw, dtype=torch.bfloat16, pin_memory=True) for _ in specs]
    for h in host:
        h.normal_()
    rid = [0]
    h2d = d2h = 0
    views = {}

    def view(bufs, c, w):
        # clients reuse their exchange buffers (SharedBuffer style): one view per (client, width)
        key = (id(bufs), c, w)
        v = views.get(key)
        if v is None:
            v = views[key] = bufs[c][: t * w].view(t, w)
        return v

    def step():
        nonlocal h2d, d2h
        h2d = d2h = 0
        for (b, r) in layers:
            di, do = dims[r]
            envs = []
            for c in range(len(specs)):
                rid[0] += 1
                envs.append(Envelope(c, rid[0], b, r, 0, view(host, c, di), reply_to=view(reply, c, do)))
                h2d += t * di * 2
                d2h += t * do * 2
            ex.serve_forward(envs)
        for (b, r) in reversed(layers):
            di, do = dims[r]
            envs = []
            for c, (_, _, ft) in enumerate(specs):
                if not ft:
                    continue
                rid[0] += 1
                envs.append(Envelope(c, rid[0], b, r, 1, view(host, c, do), reply_to=view(reply, c, di)))
                h2d += t * do * 2
                d2h += t * di * 2
            ex.serve_backward(envs)

    step()  # warm-up (allocates the device staging)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return dt, h2d, d2h


def submit_leg(ex, wl_key, specs, steps, mode="lockstep", scheduler="python"):
    """The full client path: one thread per client, each driving its layer sequence through
    ``DeviceChannel.request`` -> ``GpuBaseExecutor.submit`` -> the scheduler thread's batch
    formation (``BatchPolicy`` ``mode``) -> one fused dispatch per layer -> reply + completion
    event (executor.py:162-178, 235-300 in the reference). Wall clock around ``steps`` steps of
    every client (after one warm-up step), synchronized: this is what the Python scheduler and
    per-request host work cost next to the graph-replayed ``value``."""
    import torch
    from paper_2507_03220_b200 import BatchPolicy, DeviceChannel

    wl = WORKLOADS[wl_key]
    layers, dims = layer_list(wl)
    t = wl["tokens"]
    maxw = max(wl["d"], wl["d_ff"], wl["V"])
    old_policy, old_sched = ex.policy, ex.scheduler
    ex.policy = BatchPolicy(mode=mode)
    ex.scheduler = scheduler
    ex._metrics = type(ex._metrics)()
    ex.start()
    chans = []
    for c, (kind, _, ft) in enumerate(specs):
        ch = DeviceChannel(ex, c, 1, t, maxw)
        ch.buffer.buf.normal_()
        ch.register(sends_backward=ft)
        chans.append(ch)
    n_req = [0]
    barrier = threading.Barrier(len(specs) + 1)
    errors = []

    def client(c):
        kind, _, ft = specs[c]
        ch = chans[c]
        try:
            for _ in range(steps + 1):
                barrier.wait()
                for (b, r) in layers:
                    di, do = dims[r]
                    want = kind == "ia3" and ft and r in (K, V, FF_UP)
                    # the payload is the channel's own request buffer: no client-side copy
                    ch.request(b, r, 0, ch.buffer.view(t, di), want_base=want)
                if ft:
                    for (b, r) in reversed(layers):
                        di, do = dims[r]
                        ch.request(b, r, 1, ch.buffer.view(t, do))
                barrier.wait()
        except Exception as exc:   # noqa: BLE001
            errors.append(repr(exc))
            barrier.abort()

    threads = [threading.Thread(target=client, args=(c,), daemon=True) for c in range(len(specs))]
    for th in threads:
        th.start()
    times = []
    try:
        for i in range(steps + 1):
            barrier.wait()
            t0 = time.perf_counter()
            barrier.wait()
            torch.cuda.synchronize()
            if i:
                times.append(time.perf_counter() - t0)
    except threading.BrokenBarrierError:
        pass
    for th in threads:
        th.join(timeout=60)
    for ch in chans:
        ch.deregister()
    ex.stop()
    ex.policy, ex.scheduler = old_policy, old_sched
    if errors:
        raise RuntimeError(errors[0])
    n_req = sum(len(layers) * (2 if ft else 1) for _, _, ft in specs)
    dispatches = len(ex.metrics.batch_sizes) and sum(len(v) for v in ex.metrics.batch_sizes.values())
    return float(np.mean(times)), n_req, dispatches


def e2e_numpy_leg(ex, wl_key, specs, steps):
    """The reference's own payload type: f32 NUMPY activations (transport.py:36, 78), sent
    through GpuBaseExecutor.serve_forward / serve_backward with no reply buffer (the executor
    returns f32 numpy row views, like split_rows). Each dispatch runs the native host pipeline
    (ss_compute_batch_host: H2D of sub-batch j+1 / kernels of j / D2H of j-1 overlapped, from
    the pageable client arrays into recycled page-locked reply arrays). A full step moves
    ~630 GB over PCIe at 13B, so this leg times a bounded sample — block 0 (6 layers) and
    LM_HEAD, forward for every client and backward for the fine-tune clients, `steps` times
    after one warm-up — and scales it like the CPU baseline: step = L x t_block + t_head
    (blocks are identical)."""
    from paper_2507_03220_b200 import Envelope

    wl = WORKLOADS[wl_key]
    layers, dims = layer_list(wl)
    t = wl["tokens"]
    maxw = max(wl["d"], wl["d_ff"], wl["V"])
    rng = np.random.default_rng(5)
    host = [rng.standard_normal(t * maxw, dtype=np.float32) for _ in specs]
    rid = [0]
    moved = [0, 0]

    def run(layer_set):
        for (b, r) in layer_set:
            di, do = dims[r]
            envs = []
            for c in range(len(specs)):
                rid[0] += 1
                envs.append(Envelope(c, rid[0], b, r, 0, host[c][: t * di].reshape(t, di)))
                moved[0] += t * di * 4
                moved[1] += t * do * 4
            ex.serve_forward(envs)
        for (b, r) in reversed(layer_set):
            di, do = dims[r]
            envs = []
            for c, (_, _, ft) in enumerate(specs):
                if ft:
                    rid[0] += 1
                    envs.append(Envelope(c, rid[0], b, r, 1, host[c][: t * do].reshape(t, do)))
                    moved[0] += t * do * 4
                    moved[1] += t * di * 4
            ex.serve_backward(envs)

    block = [l for l in layers if l[0] == 0]
    head = [l for l in layers if l[0] == wl["L"]]
    run(block + head)
    tb = th = 0.0
    for _ in range(steps):
        t0 = time.perf_counter()
        run(block)
        tb += time.perf_counter() - t0
        t0 = time.perf_counter()
        run(head)
        th += time.perf_counter() - t0
    tb, th = tb / steps, th / steps
    moved[0] = moved[1] = 0
    run([])
    # byte count of one full step (no compute). Request rows cross PCIe as bf16: the library
    # converts pageable f32 rows on host threads (`host_convert`), except backward IA3 rows (dy
    # is scaled by l in f32 on the device first: copied as f32); replies are f32.
    n_ft = sum(1 for s_ in specs if s_[2])
    n_ft_ia3 = sum(1 for s_ in specs if s_[2] and s_[0] == "ia3")
    for l in layers:
        di, do = dims[l[1]]
        f32_rows = n_ft_ia3 if l[1] in (K, V, FF_UP) else 0      # backward IA3 rows stay f32
        moved[0] += t * len(specs) * di * 2 + t * ((n_ft - f32_rows) * do * 2 + f32_rows * do * 4)
        moved[1] += t * (len(specs) * do + n_ft * di) * 4
    return wl["L"] * tb + th, moved[0], moved[1], (tb, th)


# ============================================================================ CPU leg (oracle)

_CPU = {}


def _cpu_task(args):
    """One (layer, pass, row-chunk) task of the reference algorithm: the batched base GEMM
    (executor.py:191-231 via the oracle's einsum) plus each client's own adapter step."""
    from oracle import splitserve_oracle as Or
    li, pass_kind, clients, rows = args
    w, bias, ads = _CPU["layers"][li]
    xs = [_CPU["x"][pass_kind][li][c][:rows] for c in clients]
    envs = [Or.OracleEnvelope(c, 1, 0, 0, pass_kind, x) for c, x in zip(clients, xs)]
    t0 = time.perf_counter()
    if pass_kind == 0:
        out = Or.compute_batch(0, envs, w, bias)
        for c, x, y in zip(clients, xs, out):
            Or.apply_adapter(ads.get(c), x, y)
    else:
        gs = [x * ads[c].ia3 if (c in ads and ads[c].ia3 is not None) else x for c, x in zip(clients, xs)]
        envs = [Or.OracleEnvelope(c, 1, 0, 0, 1, gx) for c, gx in zip(clients, gs)]
        out = Or.compute_batch(1, envs, w, bias)
        for c, gx, dx in zip(clients, gs, out):
            ad = ads.get(c)
            if ad is not None and ad.a is not None:
                dx + Or.lora_backward_dx(gx, ad.a, ad.b, ad.alpha, ad.rank)
    return time.perf_counter() - t0


class CpuReference:
    """Bounded sample of the same workload on host cores: block 0's six layers + LM_HEAD,
    `tokens_per_client` tokens for every client (fwd for all, bwd for fine-tune clients),
    through the reference algorithm (oracle port, np.einsum optimize=False). Tasks are
    (layer, pass, 4-client chunk) spread over a fork pool (rows are independent, so this is
    the same arithmetic). ``sample()`` returns tokens/s for the full 6L+1-layer workload."""

    def __init__(self, wl_key, tokens_per_client=1, procs=None):
        from oracle import splitserve_oracle as Or

        self.wl = wl = WORKLOADS[wl_key]
        layers, dims = layer_list(wl)
        self.specs = specs = client_specs(wl_key, wl["clients"])
        self.tpc = tokens_per_client
        sample = [(0, r) for r in (Q, K, V, O, FF_UP, FF_DOWN)] + [(wl["L"], LM_HEAD)]
        rng = np.random.default_rng(0)
        _CPU["layers"], _CPU["x"] = [], {0: [], 1: []}
        for (b, r) in sample:
            di, do = dims[r]
            w, bias = Or.layer_params(99, b, r, di, do)
            ads = {}
            for c, (kind, rank, ft) in enumerate(specs):
                if kind == "lora" and r in (Q, K, V, O):
                    ads[c] = Or.lora_params(99, c, b, r, di, do, rank, 2.0 * rank)
                elif kind == "ia3" and r in (K, V, FF_UP):
                    ads[c] = Or.ia3_params(99, c, b, r, do)
            _CPU["layers"].append((w, bias, ads))
            # 2x the sample's rows: the linearity check times the doubled token count too
            _CPU["x"][0].append({c: rng.standard_normal((2 * tokens_per_client, di)).astype(np.float32)
                                 for c in range(len(specs))})
            _CPU["x"][1].append({c: rng.standard_normal((2 * tokens_per_client, do)).astype(np.float32)
                                 for c in range(len(specs))})
        all_c = list(range(len(specs)))
        self.ft_c = ft_c = [c for c, s in enumerate(specs) if s[2]]
        chunk = lambda cs: [cs[i:i + 4] for i in range(0, len(cs), 4)]  # noqa: E731
        self.block_tasks = self._tasks(range(6), all_c, ft_c, chunk, tokens_per_client)
        self.head_tasks = self._tasks([6], all_c, ft_c, chunk, tokens_per_client)
        ncpu = procs or os.cpu_count() or 1
        self.n = max(1, min(ncpu, len(self.block_tasks)))
        for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"
        import multiprocessing as mp
        self.pool = mp.get_context("fork").Pool(self.n)
        self.pool.map(_cpu_task, self.head_tasks[:1])  # fork + import warm-up, untimed

    @staticmethod
    def _tasks(layer_idx, all_c, ft_c, chunk, rows):
        return [(li, 0, cs, rows) for li in layer_idx for cs in chunk(all_c)] + \
               [(li, 1, cs, rows) for li in layer_idx for cs in chunk(ft_c)]

    def linearity(self) -> dict:
        """time the sample (block 0 + LM_HEAD) at n and 2n tokens per client;
        the full-step model scales by tokens, so t(2n) / (2 t(n)) must be ~1 (reported)."""
        times = {}
        for rows in (self.tpc, 2 * self.tpc):
            tasks = [(li, p, cs, rows) for li, p, cs, _ in self.block_tasks + self.head_tasks]
            t0 = time.perf_counter()
            self.pool.map(_cpu_task, tasks, chunksize=1)
            times[rows] = time.perf_counter() - t0
        n = self.tpc
        return {"tokens_per_client": [n, 2 * n], "sample_s": [times[n], times[2 * n]],
                "ratio_t2n_over_2tn": times[2 * n] / (2 * times[n])}

    def sample(self):
        wl = self.wl
        t0 = time.perf_counter()
        self.pool.map(_cpu_task, self.block_tasks, chunksize=1)
        t_block = time.perf_counter() - t0
        t0 = time.perf_counter()
        self.pool.map(_cpu_task, self.head_tasks, chunksize=1)
        t_head = time.perf_counter() - t0
        step_s = wl["tokens"] / self.tpc * (wl["L"] * t_block + t_head)
        tok_s = len(self.specs) * wl["tokens"] / step_s
        info = (f"block 0 (6 layers) + LM_HEAD, {self.tpc} tok x {len(self.specs)} clients "
                f"(fwd all, bwd {len(self.ft_c)} FT), {len(self.block_tasks) + len(self.head_tasks)} "
                f"tasks on {self.n} procs: block {t_block:.2f}s head {t_head:.2f}s per sample, "
                f"scaled x{wl['L']} blocks x{wl['tokens']}/{self.tpc} tok")
        return tok_s, info

    def close(self):
        self.pool.close()
        self.pool.join()


def config_dict(wl, tokens_per_rank, world, tp_mode, step_flops, ms):
    """The workload description both arms print (the driver compares the two dicts)."""
    tokens = tokens_per_rank * (1 if tp_mode else world)
    return {"workload": wl["name"], "model": f"d{wl['d']}-ff{wl['d_ff']}-L{wl['L']}-V{wl['V']}",
            "clients": wl["clients"], "global_batch": tokens, "seq_len": wl["seq"],
            "batch_per_client": wl["batch"], "rows_per_fwd_dispatch": tokens_per_rank,
            "parallelism": (f"tensor-parallel x{world} (column/row shards, NCCL per dispatch)" if tp_mode
                            else f"segment-parallel replicas x{world}" if world > 1 else "single GPU"),
            "l2": "inputs larger than L2 (every step streams all 6L+1 weight matrices)",
            "step_tflop": step_flops / 1e12}


def self_launch(args) -> int | None:
    """`python bench.py --gpus N` without a launcher: re-exec under torch.distributed.run with
    N ranks (one per GPU) on 127.0.0.1, exactly as the driver launches N > 1; returns the
    launcher's exit code. None when already inside a launcher or N == 1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args) -> None:
    """--dry-run: the launcher / rendezvous / barrier / max-over-ranks / JSON contract of an
    N-rank run on the HOST (gloo), with a small numpy GEMM standing in for the step: what the
    CPU test suite can check without a GPU."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    a = np.random.default_rng(rank).standard_normal((256, 256)).astype(np.float32)
    for _ in range(args.warmup):
        a @ a
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a @ a
    dt = time.perf_counter() - t0
    if world > 1:
        import torch
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        dist.barrier()
    if rank == 0:
        toks = 256 * args.steps * world
        print(json.dumps({"metric": METRIC, "value": toks / dt, "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
                          "higher_is_better": True, "scaling": "weak", "dry_run": True}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ============================================================================ main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="13b", choices=sorted(WORKLOADS))
    ap.add_argument("--clients", type=int, default=0, help="override the workload's client count")
    ap.add_argument("--opt", action="append", default=[],
                    help="library tuning option key=value (ss_set_option), e.g. gemm_2cta=1, group_m=8")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="timed e2e steps (0: 1 for the prefill workloads, 10 for decode)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=8,
                    help="tokens per client in each CPU-reference sample (~5 s of host work at 8)")
    ap.add_argument("--graph", type=int, default=1,
                    help="1: replay the step's prebuilt dispatch plans as one CUDA graph (the kernel "
                         "roofline is still measured on an eager, event-bracketed pass)")
    ap.add_argument("--inplace", action="store_true",
                    help="device clients reuse one buffer for request and reply (SharedBuffer style; "
                         "aliased sources are gathered before the GEMM)")
    ap.add_argument("--dry-run", action="store_true",
                    help="host-only (gloo) run of the launcher / timing / JSON contract (CPU tests)")
    ap.add_argument("--no-tp-leg", action="store_true",
                    help="N > 1 replicas run: skip the tensor-parallel leg reported beside it")
    ap.add_argument("--e2e-numpy-steps", type=int, default=2,
                    help="timed samples of the f32-numpy e2e leg (0: skip)")
    ap.add_argument("--submit-steps", type=int, default=2,
                    help="timed steps of the client-thread submit() leg (0: skip)")
    ap.add_argument("--parallel", default="replicas", choices=("replicas", "tp"),
                    help="replicas: segment-parallel full replicas (weak scaling, no data-path "
                         "collective); tp: column/row-sharded layers + NCCL per dispatch (strong)")
    args = ap.parse_args()
    global INPLACE
    INPLACE = args.inplace
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.dry_run:
        dry_run(args)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.clients:
        WORKLOADS[args.workload] = dict(WORKLOADS[args.workload], clients=args.clients)
    wl = WORKLOADS[args.workload]
    specs = client_specs(args.workload, wl["clients"])
    tokens_per_rank = wl["clients"] * wl["tokens"]

    if args.impl == "reference":
        if rank != 0:
            return
        cpu_ref = CpuReference(args.workload, args.cpu_tokens)
        lin = cpu_ref.linearity()
        vals, walls = [], []
        for i in range(max(0, args.warmup) + args.steps):
            t0 = time.perf_counter()
            tok_s, info = cpu_ref.sample()
            if i >= args.warmup:
                vals.append(tok_s)
                walls.append(time.perf_counter() - t0)
        cpu_ref.close()
        cores = cpu_ref.n
        v = float(np.mean(vals))
        world = args.gpus
        # the reference arm serves the same workload: same config dict as our arm at this N
        cfg = config_dict(wl, tokens_per_rank, world, args.parallel == "tp", flops_per_step(wl, specs), 0)
        line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                # wall time of one bounded sample (a step of this arm); the full step it stands
                # for would take full_step_s_modelled
                "ms_per_step": 1e3 * float(np.mean(walls)), "higher_is_better": True,
                "scaling": "strong" if args.parallel == "tp" else "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded N(0,1) activations, reference-style random init)",
                "impl": "reference", "config": cfg,
                "reference_execution": f"reference algorithm (oracle port, np.einsum optimize=False) on a "
                                       f"{cores}-process host pool, rank 0 only",
                "full_step_s_modelled": tokens_per_rank * (1 if args.parallel == "tp" else world) / v,
                "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                                 "sample": info, "cpu": cpu_model(), "linearity": lin},
                "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    tp_mode = args.parallel == "tp"
    if world > 1 or tp_mode:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                rank=rank, world_size=world)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    from paper_2507_03220_b200 import _lib

    if tp_mode:
        tp, tp_plan, specs, wl = build_tp_workload(args.workload, device, rank, world)
        ex, plan = tp.ex, None
        step_fn = lambda: run_step_tp(tp, tp_plan)  # noqa: E731
    else:
        ex, plan, specs, wl = build_gpu_workload(args.workload, device, rank)
        step_fn = lambda: run_step(plan, stream)  # noqa: E731
    ctx = ex.ctx
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    if args.opt and not tp_mode:   # options change kernel / tile choice: rebuild the plans
        ex, plan, specs, wl = ex, [ex.compile_dispatch(d.pass_kind, d.key[0], d.key[1], d.segments) for d in plan], specs, wl
        step_fn = lambda: run_step(plan, stream)  # noqa: E731
    stream = torch.cuda.current_stream(device)
    for _ in range(max(3, args.warmup)):
        step_fn()
    torch.cuda.synchronize()
    eager_step_fn = step_fn
    graph = None
    if args.graph and not tp_mode:
        graph = ex.capture(plan, stream=torch.cuda.Stream(device))
        step_fn = lambda: graph.replay()  # noqa: E731  (replays on torch's current stream)
        for _ in range(max(3, args.warmup)):
            step_fn()
        torch.cuda.synchronize()

    samples, stop = [], threading.Event()
    sampler = threading.Thread(target=nvsmi_sampler, args=(stop, samples, local), daemon=True)
    sampler.start()
    time.sleep(0.5)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches()
    if graph is None:
        ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step_fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stop.set()
    launches = ctx.kernel_launches() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    prof_steps = args.steps
    if graph is not None:
        # graph replays launch no host-side kernels: count the captured launches per step, and
        # take the per-kernel roofline from an eager pass of the same plans, event-bracketed
        ctx.profile(True)
        l0 = ctx.kernel_launches()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        eager_step_fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = (ctx.kernel_launches() - l0) * args.steps
        eager_ms = ev0.elapsed_time(ev1)
        prof_steps = 1
    gemm = ctx.profile_read(_lib.SS_KERNEL_GEMM)
    shrink = ctx.profile_read(_lib.SS_KERNEL_SHRINK)
    gather = ctx.profile_read(_lib.SS_KERNEL_GATHER)
    ctx.profile(False)

    # adapter weight-gradient leg (fine-tune clients' grad_a / grad_b / grad_l, every layer)
    grads_leg = None
    if not tp_mode and getattr(ex, "_bench_grads", None):
        def grads_pass():
            for b, r, jobs in ex._bench_grads:
                ex.adapter_grads(b, r, jobs, stream)
        for _ in range(2):
            grads_pass()
        torch.cuda.synchronize()
        # wall time of the passes without per-launch profiling events, then one profiled pass
        # per step for the kernel-only time and bytes
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            grads_pass()
        g1.record(stream)
        torch.cuda.synchronize()
        g_ms = g0.elapsed_time(g1) / args.steps
        ctx.profile(True)
        for _ in range(args.steps):
            grads_pass()
        torch.cuda.synchronize()
        gk = ctx.profile_read(_lib.SS_KERNEL_GRAD)
        ctx.profile(False)
        grads_leg = {"ms_per_step": g_ms, "kernel_ms_per_step": gk["ms"] / args.steps,
                     "launches_per_step": gk["launches"] / args.steps,
                     "alg_bytes_per_step": gk["bytes"] / args.steps,
                     "achieved_gbs": gk["bytes"] / (gk["ms"] / 1e3) / 1e9 if gk["ms"] else None,
                     "ft_step_tokens_per_s": None}
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    sampler.join(timeout=2)
    clocks = summarize_clocks(samples)

    tokens = tokens_per_rank * (1 if tp_mode else world)
    value = tokens / (ms / 1e3)
    step_flops = flops_per_step(wl, specs)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("bf16_tflops_sustained", 1400.0))
    peak_burst = float(peaks.get("bf16_tflops", 1590.0))
    gemm_tflops = gemm["flops"] / (gemm["ms"] / 1e3) / 1e12 if gemm["ms"] else None
    # decode dispatches (a few rows per client) stream the weights: HBM roofline
    decode = args.workload.endswith("decode")
    gemm_gbs = gemm["bytes"] / (gemm["ms"] / 1e3) / 1e9 if gemm["ms"] else None
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tr_path) and args.workload == "13b":   # the capture is of the 13B step
        try:
            traffic = json.load(open(tr_path)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    dec_traffic = None
    dtr_path = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(dtr_path) and args.workload == "13b-decode":   # Q-shaped launches of this step
        try:
            dtr = json.load(open(dtr_path))
            dec_traffic = {"dram_bytes_per_launch": dtr["dram_bytes_per_launch"],
                           "algorithmic_bytes_per_launch": dtr["algorithmic_bytes_per_launch"],
                           "launch": "Q-shaped decode dispatch (ncu capture, profiles/r02/ncu_decode_gemm.md)"}
        except (OSError, ValueError, KeyError):
            dec_traffic = None

    if grads_leg is not None:
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        grads_leg["hbm_peak_gbs"] = hbm_peak
        grads_leg["hbm_peak_source"] = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"
        if grads_leg["achieved_gbs"]:
            grads_leg["frac"] = grads_leg["achieved_gbs"] / hbm_peak
        # the whole fine-tune step: executor fwd + bwd plus every FT client's adapter gradients
        grads_leg["ft_step_tokens_per_s"] = tokens / ((ms + grads_leg["ms_per_step"]) / 1e3)

    cublas = None
    if rank == 0 and world == 1 and not tp_mode and not args.workload.endswith("decode"):
        cublas = cublas_same_shapes(args.workload, specs, device)
        cublas["gemm_time_ratio"] = cublas["ms_per_step"] / (gemm["ms"] / prof_steps) if gemm["ms"] else None

    e2e = None
    if not args.skip_e2e and not tp_mode:
        e2e_steps = args.e2e_steps or (10 if args.workload.endswith("decode") else 3)
        dt, h2d, d2h = e2e_leg(ex, args.workload, specs, e2e_steps, device)
        if world > 1:
            t = torch.tensor([dt], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": tokens / dt, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3,
               "path": "GpuBaseExecutor.serve_forward / serve_backward, pinned host bf16 payloads + host reply buffers, "
                       f"{e2e_steps} timed step(s) after 1 warm-up"}
        if args.e2e_numpy_steps > 0:
            dt_n, h2d_n, d2h_n, (tb_n, th_n) = e2e_numpy_leg(ex, args.workload, specs, args.e2e_numpy_steps)
            if world > 1:
                t = torch.tensor([dt_n], device=device)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt_n = float(t.item())
            e2e["f32_numpy"] = {"value": tokens / dt_n, "unit": "tokens/s", "h2d_bytes_per_step": h2d_n,
                                "d2h_bytes_per_step": d2h_n, "ms_per_step": dt_n * 1e3,
                                "path": "GpuBaseExecutor.serve_forward / serve_backward, f32 numpy payloads "
                                        "(the reference channels' payload type), replies returned as f32 numpy "
                                        "views; native host pipeline, request rows converted to bf16 by host "
                                        "threads before the DMA (bytes: what crosses PCIe)",
                                "sample": f"block 0 ({tb_n * 1e3:.0f} ms) + LM_HEAD ({th_n * 1e3:.0f} ms), fwd all "
                                          f"clients + bwd FT clients, mean of {args.e2e_numpy_steps} after 1 "
                                          f"warm-up; step = L x block + head"}

    submit = None
    if args.submit_steps > 0 and not tp_mode:
        submit = {}
        for sched in ("native", "python"):
            try:
                dt_s, n_req, n_disp = submit_leg(ex, args.workload, specs, args.submit_steps, scheduler=sched)
                submit[sched] = {
                    "value": tokens_per_rank / dt_s, "unit": "tokens/s", "ms_per_step": dt_s * 1e3,
                    "requests_per_step": n_req, "requests_per_s": n_req / dt_s,
                    "dispatches_recorded": n_disp, "policy": "lockstep",
                    "path": f"{len(specs)} client threads, DeviceChannel.request -> "
                            + ("ss_sched_request (library scheduler thread: batch formation + dispatch)"
                               if sched == "native" else
                               "GpuBaseExecutor.submit -> Python scheduler thread batch formation")
                            + " -> one fused dispatch per layer and pass (no plans, no graph); wall clock, "
                            f"{args.submit_steps} step(s) after 1 warm-up"}
            except Exception as exc:   # noqa: BLE001 — the headline line must still print
                submit[sched] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    tp_info = None
    if world > 1 and not tp_mode and not args.no_tp_leg:
        try:
            tp_info = tp_leg(args.workload, device, rank, world, args.steps, args.warmup)
        except Exception as exc:   # the replicas line must still print
            tp_info = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu_ref = CpuReference(args.workload, args.cpu_tokens)
        lin = cpu_ref.linearity()
        tok_s, info = cpu_ref.sample()
        tok_s2, info = cpu_ref.sample()
        cpu_ref.close()
        cpu = {"value": 0.5 * (tok_s + tok_s2), "unit": "tokens/s", "cores": cpu_ref.n, "kind": "port",
               "sample": info + " (mean of 2 samples)", "cpu": cpu_model(), "linearity": lin}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if tp_mode else "weak", "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random-init weights/adapters/activations, per-layer seeds)",
            "config": config_dict(wl, tokens_per_rank, world, tp_mode, step_flops, ms),
            "achieved_step_tflops": step_flops * (1 if tp_mode else world) / (ms / 1e3) / 1e12,
            "roofline": ({"bound": "tensor", "kernel": "seg_gemm_kernel (fused base GEMM + LoRA/IA3 epilogue)",
                          "achieved": gemm_tflops, "peak": peak, "unit": "TFLOP/s",
                          "frac": (gemm_tflops / peak) if gemm_tflops else None, "traffic": traffic,
                          "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else "fallback",
                          # the GEMM runs inside a long power-capped step, so the sustained
                          # cuBLAS figure is the denominator; against the burst figure:
                          "peak_burst": peak_burst,
                          "frac_burst": (gemm_tflops / peak_burst) if gemm_tflops else None,
                          # cuBLAS on the same GEMM shapes, same box (ratio > 1: the fused kernel,
                          # which also does the adapters / IA3 / scatter, takes less time)
                          "cublas_same_shapes": cublas}
                         if not decode else
                         {"bound": "hbm", "kernel": "seg_gemm_dec_kernel + dec_fixup_kernel (decode class: split-K in the class order, 64-row decode tiles)",
                          "achieved": gemm_gbs, "peak": hbm_peak, "unit": "GB/s",
                          "frac": (gemm_gbs / hbm_peak) if gemm_gbs else None,
                          "traffic": dec_traffic["dram_bytes_per_launch"] if dec_traffic else None,
                          "traffic_detail": dec_traffic,
                          "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                          "tflops": gemm_tflops}) | {
                         "gemm_share_of_step": gemm["ms"] / (ms * prof_steps),
                         "gemm_launches": gemm["launches"],
                         "shrink_ms_per_step": shrink["ms"] / prof_steps,
                         "gather_ms_per_step": gather["ms"] / prof_steps,
                         "measured_on": ("eager event-bracketed pass of the same plans "
                                         f"({eager_ms:.1f} ms/step eager vs {ms:.1f} graph)") if graph is not None
                                        else "the timed steps",
                         "gather_gbs": (gather["bytes"] / (gather["ms"] / 1e3) / 1e9) if gather["ms"] else None},
            "adapter_grads": grads_leg,
            "submit_path": submit,
            "tensor_parallel": tp_info,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks,
            "launch_mode": "CUDA graph of prebuilt dispatch plans" if graph is not None else "eager prebuilt dispatch plans",
        }
        print(json.dumps(line), flush=True)
    if world > 1 or tp_mode:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
