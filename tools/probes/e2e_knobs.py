"""e2e leg of the 13B workload under different host-pipeline sub-batch sizes."""
import sys, torch
sys.path.insert(0, ".")
import bench
dev = torch.device("cuda", 0)
ex, plan, specs, wl = bench.build_gpu_workload("13b", dev, 0)
for rows, mb in ((4096, 24), (2048, 12), (8192, 48), (4096, 12), (1024, 8), (8192, 96)):
    ex.pipeline_rows, ex.pipeline_bytes = rows, mb << 20
    dt, h2d, d2h = bench.e2e_leg(ex, "13b", specs, 1, dev)
    print(f"rows {rows} bytes {mb} MB: {dt*1e3:.0f} ms/step  {32768/dt:.0f} tok/s", flush=True)
