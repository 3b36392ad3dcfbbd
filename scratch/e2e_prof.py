"""cProfile of the decode e2e leg (host API overhead per dispatch)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "13b-decode"
dev = torch.device("cuda:0")
ex, plan, specs, _ = bench.build_gpu_workload(wl, dev, 0)
dt, _, _ = bench.e2e_leg(ex, wl, specs, 3, dev)
print(f"e2e {dt * 1e3:.2f} ms/step")
pr = cProfile.Profile()
pr.enable()
dt, _, _ = bench.e2e_leg(ex, wl, specs, 3, dev)
pr.disable()
print(f"e2e (profiled) {dt * 1e3:.2f} ms/step")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
