"""Per-call cost of one decode-size zero-copy host dispatch (13B Q shape, 32 clients x 2 rows):
Python executor call vs bare C call vs the same dispatch's kernels replayed from a plan."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role  # noqa: E402
from paper_2507_03220_b200.device import Seg, SegmentTable  # noqa: E402
from paper_2507_03220_b200.protocol import Envelope  # noqa: E402

d, n_cli, t = 5120, 32, 2
W = (torch.randn(d, d) / d ** 0.5).numpy()
ex = GpuBaseExecutor({LayerAddress(0, Role.Q): AffineParams(W, None)})
hosts = [torch.randn(t, d).to(torch.bfloat16).pin_memory() for _ in range(n_cli)]
reps = [torch.empty(t, d, dtype=torch.bfloat16).pin_memory() for _ in range(n_cli)]
segs = [Seg(c, h, r, pinned=True) for c, (h, r) in enumerate(zip(hosts, reps))]
ctx = ex.ctx
N = 300
for cache in (1, 0):
    ctx.set_option("zc_cache", cache)
    for _ in range(20):
        ctx.compute_host(0, 0, int(Role.Q), segs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        ctx.compute_host(0, 0, int(Role.Q), segs)
    print(f"compute_host (zc_cache={cache}): {(time.perf_counter() - t0) / N * 1e6:.1f} us/call")
ctx.set_option("zc_cache", 1)
table = SegmentTable(segs, ctx._seg_cache)
import ctypes  # noqa: E402
s = torch.cuda.current_stream()
t0 = time.perf_counter()
for _ in range(N):
    ctx.lib.ss_compute_batch_host(ctx.h, 0, 0, int(Role.Q), table.n, table.arr, ctypes.c_void_p(s.cuda_stream), table.status)
print(f"bare C call: {(time.perf_counter() - t0) / N * 1e6:.1f} us/call")
rid = 0
t0 = time.perf_counter()
for _ in range(N):
    envs = []
    for c in range(n_cli):
        rid += 1
        envs.append(Envelope(c, rid, 0, int(Role.Q), 0, hosts[c], reply_to=reps[c]))
    ex.serve_forward(envs)
print(f"serve_forward: {(time.perf_counter() - t0) / N * 1e6:.1f} us/call")
dsegs = [Seg(c, h.cuda(), torch.empty(t, d, dtype=torch.bfloat16, device="cuda")) for c, h in enumerate(hosts)]
plan = ctx.plan(0, 0, int(Role.Q), dsegs)
for _ in range(10):
    plan.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    plan.launch()
e1.record()
torch.cuda.synchronize()
print(f"device plan, back to back: {e0.elapsed_time(e1) / N * 1e3:.1f} us/dispatch")
t0 = time.perf_counter()
for _ in range(N):
    plan.launch()
    torch.cuda.synchronize()
print(f"device plan + sync each: {(time.perf_counter() - t0) / N * 1e6:.1f} us/dispatch")
