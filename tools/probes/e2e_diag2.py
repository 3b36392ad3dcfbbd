"""Split the host-dispatch time: Python executor overhead vs the native pipeline vs raw copies."""
import math, sys, time
import torch
sys.path.insert(0, ".")
from paper_2507_03220_b200 import AffineParams, Envelope, GpuBaseExecutor, LayerAddress, Role  # noqa
from paper_2507_03220_b200.device import Seg

dev = torch.device("cuda:0")
shapes = {Role.Q: (5120, 5120), Role.FF_DOWN: (13824, 5120), Role.LM_HEAD: (5120, 32000)}
layers = {LayerAddress(40 if r == Role.LM_HEAD else 0, r): AffineParams((torch.randn(di, do, device=dev) / math.sqrt(di)).to(torch.bfloat16), torch.zeros(do, device=dev)) for r, (di, do) in shapes.items()}
ex = GpuBaseExecutor(layers, retain_layers=False)
t, n = 1024, 32
host = [torch.empty(t * 32000, dtype=torch.bfloat16).pin_memory() for _ in range(n)]
for rows_min in (0, 1024, 2048):
    for pb in (24, 64):
        ex.ctx.set_option("pipeline_bytes", pb << 20)
        print(f"-- pipeline_bytes {pb} MB, min rows {rows_min}")
        for role, pk in ((Role.Q, 0), (Role.FF_DOWN, 0), (Role.LM_HEAD, 1), (Role.LM_HEAD, 0)):
            di, do = shapes[role]
            wi, wo = (di, do) if pk == 0 else (do, di)
            nc = n if pk == 0 else n // 2
            blk = 40 if role == Role.LM_HEAD else 0
            if rows_min:
                ex.ctx.set_option("pipeline_rows", 4096)
                ex.ctx.set_option("pipeline_bytes", max(pb << 20, rows_min * max(wi, wo) * 2))
            segs = [Seg(client_id=c, src=host[c][: t * wi].view(t, wi), dst=host[c][: t * wo].view(t, wo)) for c in range(nc)]
            ex.ctx.compute_host(pk, blk, int(role), segs)
            t0 = time.perf_counter()
            for _ in range(3):
                ex.ctx.compute_host(pk, blk, int(role), segs)
            dt = (time.perf_counter() - t0) / 3
            bi, bo = nc * t * wi * 2, nc * t * wo * 2
            print(f"{role.name:8s} pass {pk}: native {dt*1e3:7.2f} ms  ({(bi+bo)/dt/1e9:5.1f} GB/s)")
# raw copies, same pieces, two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d_in = torch.empty(64 << 20, dtype=torch.bfloat16, device=dev)
d_out = torch.empty(64 << 20, dtype=torch.bfloat16, device=dev)
for wi, wo, nc in ((5120, 5120, 32), (13824, 5120, 32), (32000, 5120, 16)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for c in range(nc):
        with torch.cuda.stream(s1):
            d_in[: t * wi].copy_(host[c][: t * wi], non_blocking=True)
        with torch.cuda.stream(s2):
            host[(c + 1) % n][: t * wo].copy_(d_out[: t * wo], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"raw copies in {wi} out {wo}: {dt*1e3:.2f} ms, H2D {nc*t*wi*2/dt/1e9:.1f} GB/s, D2H {nc*t*wo*2/dt/1e9:.1f} GB/s")
