"""Value statistics of the bench's client buffers after a few steps, in-place vs separate."""
import sys
import torch
sys.path.insert(0, ".")
import bench

for inplace in (True, False):
    bench.INPLACE = inplace
    dev = torch.device("cuda", 0)
    ex, plan, specs, wl = bench.build_gpu_workload("13b", dev, 0)
    s = torch.cuda.current_stream(dev)
    for step in range(3):
        bench.run_step(plan, s)
        torch.cuda.synchronize()
        for c in (0, 5, 30):
            src = plan[0].segments[c][1]
            dst = plan[0].segments[c][2]
            for name, t in (("src", src), ("dst", dst)):
                f = t.float()
                fin = torch.isfinite(f)
                print(f"inplace={inplace} step {step} client {c} {name}: finite {fin.float().mean().item():.4f} "
                      f"absmean {f[fin].abs().mean().item() if fin.any() else float('nan'):.3e} "
                      f"zeros {(f == 0).float().mean().item():.4f}", flush=True)
    ex.close()
    del ex, plan
    torch.cuda.empty_cache()
