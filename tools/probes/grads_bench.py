"""Time ss_adapter_grads at the 13B workload's shapes: 12 fine-tune LoRA clients (ranks
8/16/32/64, 1024 tokens) on a d5120 Q layer; 4 IA3 fine-tune clients on FF_UP (d_out 13824)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role, _lib
from paper_2507_03220_b200.device import GradSeg

dev = torch.device("cuda", 0)
d, f = 5120, 13824
layers = {LayerAddress(0, Role.Q): AffineParams((torch.randn(d, d, device=dev) / math.sqrt(d)).bfloat16(), torch.zeros(d, device=dev)),
          LayerAddress(0, Role.FF_UP): AffineParams((torch.randn(d, f, device=dev) / math.sqrt(d)).bfloat16(), torch.zeros(f, device=dev))}
ex = GpuBaseExecutor(layers, device=0)
class Ad:
    def __init__(s, **k): s.lora, s.ia3, s.alpha, s.rank = k.get("lora", {}), k.get("ia3", {}), k.get("alpha", 0.0), k.get("rank", 1)
t = 1024
lj, ij = [], []
for c in range(12):
    r = (8, 16, 32, 64)[c % 4]
    ex.register_adapter(c, Ad(lora={LayerAddress(0, Role.Q): (torch.randn(d, r, device=dev) / math.sqrt(d), 0.05 * torch.randn(r, d, device=dev))}, alpha=2.0 * r, rank=r))
    lj.append(GradSeg(c, dy=torch.randn(t, d, device=dev).bfloat16(), x=torch.randn(t, d, device=dev).bfloat16(),
                      grad_a=torch.zeros(d, r, device=dev), grad_b=torch.zeros(r, d, device=dev)))
for c in range(12, 16):
    ex.register_adapter(c, Ad(ia3={LayerAddress(0, Role.FF_UP): 1 + 0.1 * torch.randn(f, device=dev)}))
    ij.append(GradSeg(c, dy=torch.randn(t, f, device=dev).bfloat16(), y_base=torch.randn(t, f, device=dev).bfloat16(),
                      grad_l=torch.zeros(f, device=dev)))
for _ in range(3):
    ex.adapter_grads(0, Role.Q, lj); ex.adapter_grads(0, Role.FF_UP, ij)
torch.cuda.synchronize()
for name, role, jobs in (("lora Q x12", Role.Q, lj), ("ia3 FF_UP x4", Role.FF_UP, ij)):
    ex.ctx.profile(True)
    n = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        ex.adapter_grads(0, role, jobs)
    e1.record(); torch.cuda.synchronize()
    p = ex.ctx.profile_read(_lib.SS_KERNEL_GRAD)
    ex.ctx.profile(False)
    ms = e0.elapsed_time(e1) / n
    print(f"{name}: {ms:.3f} ms/call (events), kernels {p['ms']/n:.3f} ms, alg bytes {p['bytes']/n/1e6:.1f} MB -> "
          f"{p['bytes']/(p['ms']/1e3)/1e9:.0f} GB/s, {p['flops']/(p['ms']/1e3)/1e12:.1f} TFLOP/s")
