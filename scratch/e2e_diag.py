"""Time single host-payload dispatches of 13B-shaped layers (pipelined path) to find the e2e limiter."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import AffineParams, Envelope, GpuBaseExecutor, LayerAddress, Role  # noqa

dev = torch.device("cuda:0")
shapes = {Role.Q: (5120, 5120), Role.FF_UP: (5120, 13824), Role.FF_DOWN: (13824, 5120)}
layers = {}
for r, (di, do) in shapes.items():
    layers[LayerAddress(0, r)] = AffineParams((torch.randn(di, do, device=dev) / math.sqrt(di)).to(torch.bfloat16),
                                              torch.zeros(do, device=dev))
layers[LayerAddress(40, Role.LM_HEAD)] = AffineParams((torch.randn(5120, 32000, device=dev) / 71.5).to(torch.bfloat16),
                                                      torch.zeros(32000, device=dev))
shapes[Role.LM_HEAD] = (5120, 32000)
ex = GpuBaseExecutor(layers, retain_layers=False)
if len(sys.argv) > 1:
    ex.pipeline_bytes = int(sys.argv[1]) << 20
if len(sys.argv) > 2:
    pass
t, n = 1024, 32
maxw = 32000
host = [torch.empty(t * maxw, dtype=torch.bfloat16).pin_memory() for _ in range(n)]
rid = [0]


def dispatch(block, role, pass_kind):
    di, do = shapes[role]
    wi, wo = (di, do) if pass_kind == 0 else (do, di)
    envs = []
    for c in range(n if pass_kind == 0 else n // 2):
        rid[0] += 1
        envs.append(Envelope(c, rid[0], block, role, pass_kind, host[c][: t * wi].view(t, wi),
                             reply_to=host[c][: t * wo].view(t, wo)))
    t0 = time.perf_counter()
    ex._compute_batch(pass_kind, envs)
    dt = time.perf_counter() - t0
    rows = len(envs) * t
    return dt, rows * wi * 2, rows * wo * 2


for role in (Role.Q, Role.FF_UP, Role.FF_DOWN, Role.LM_HEAD):
    block = 40 if role == Role.LM_HEAD else 0
    for pk in (0, 1):
        dispatch(block, role, pk)
        dts = [dispatch(block, role, pk) for _ in range(3)]
        dt = min(d[0] for d in dts)
        _, bi, bo = dts[0]
        floor = max(bi, bo) / 55.5e9
        print(f"{role.name:8s} pass {pk}: {dt*1e3:7.2f} ms  in {bi/1e9:5.2f} GB out {bo/1e9:5.2f} GB  "
              f"-> {(bi+bo)/dt/1e9:5.1f} GB/s  (one-direction floor {floor*1e3:6.2f} ms)")
