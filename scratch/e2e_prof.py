"""cProfile of the decode e2e leg (host clients through GpuBaseExecutor.serve_*)."""
import cProfile, pstats, sys, time
import torch
sys.path.insert(0, ".")
import bench
dev = torch.device("cuda", 0)
ex, plan, specs, wl = bench.build_gpu_workload("13b-decode", dev, 0)
bench.e2e_leg(ex, "13b-decode", specs, 1, dev)
pr = cProfile.Profile()
pr.enable()
dt, h2d, d2h = bench.e2e_leg(ex, "13b-decode", specs, 2, dev)
pr.disable()
print("e2e ms/step", dt * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
