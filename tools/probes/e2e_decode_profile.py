"""cProfile of the decode e2e leg (13B shape, 32 clients x 2 rows, pinned host payloads through
GpuBaseExecutor.serve_forward): where the host time of a decode dispatch goes."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
ex, plan, specs, wl = bench.build_gpu_workload("13b-decode", dev, 0)
bench.e2e_leg(ex, "13b-decode", specs, 1, dev)
pr = cProfile.Profile()
pr.enable()
dt, h2d, d2h = bench.e2e_leg(ex, "13b-decode", specs, 3, dev)
pr.disable()
print(f"e2e {dt * 1e3:.1f} ms/step ({64 / dt:.0f} tokens/s)")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
