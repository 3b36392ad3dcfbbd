"""Per-layer-shape e2e (pinned host payloads -> serve_forward / serve_backward -> pinned host
replies) at the 13B step's dispatch sizes, against the PCIe bound of each dispatch."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role  # noqa: E402
from paper_2507_03220_b200.protocol import Envelope  # noqa: E402

H2D, D2H, BIDIR = 55.6e9, 55.6e9, 95e9
shapes = [("Q", Role.Q, 5120, 5120), ("FF_UP", Role.FF_UP, 5120, 13824), ("FF_DOWN", Role.FF_DOWN, 13824, 5120)]
n_cli, t = 32, 1024
for name, role, din, dout in shapes:
    W = (torch.randn(din, dout) / din ** 0.5).numpy()
    ex = GpuBaseExecutor({LayerAddress(0, role): AffineParams(W, None)})
    for pass_kind, (wi, wo), ncl in ((0, (din, dout), n_cli), (1, (dout, din), n_cli // 2)):
        hosts = [torch.randn(t, wi).to(torch.bfloat16).pin_memory() for _ in range(ncl)]
        reps = [torch.empty(t, wo, dtype=torch.bfloat16).pin_memory() for _ in range(ncl)]
        rid = [0]

        def go():
            envs = []
            for c in range(ncl):
                rid[0] += 1
                envs.append(Envelope(c, rid[0], 0, int(role), pass_kind, hosts[c], reply_to=reps[c]))
            (ex.serve_forward if pass_kind == 0 else ex.serve_backward)(envs)
        go()
        torch.cuda.synchronize()
        n = 5
        t0 = time.perf_counter()
        for _ in range(n):
            go()
        dt = (time.perf_counter() - t0) / n
        bi, bo = ncl * t * wi * 2, ncl * t * wo * 2
        bound = max(bi / H2D, bo / D2H, (bi + bo) / BIDIR)
        print(f"{name:8s} pass {pass_kind}: {dt * 1e3:7.2f} ms  bound {bound * 1e3:6.2f} ms  "
              f"({bound / dt:.2f})  in {bi / 1e6:.0f} MB out {bo / 1e6:.0f} MB", flush=True)
    del ex
    torch.cuda.empty_cache()
