"""Adapter-gradient launches of one 13B-shape layer (d 5120 x 5120) for 16 LoRA clients of 1024
tokens (ranks 8..64) through the C ABI: kernel time per call (ss_profile) with the fused launch
(grad_fused 1, lag from argv) and the two-launch path. Run under ncu for per-kernel DRAM bytes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import splitserve_oracle as O  # noqa: E402  (parameter generator only)
from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role  # noqa: E402
from paper_2507_03220_b200.device import GradSeg  # noqa: E402


class _Adapter:
    def __init__(self, lora, alpha, rank):
        self.lora, self.ia3, self.alpha, self.rank = lora, {}, alpha, rank


d, t, n = 5120, 1024, 16
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
lags = [int(v) for v in sys.argv[2:]] or [2]
addr = LayerAddress(0, Role(O.Q))
w = (np.random.default_rng(0).standard_normal((d, d)) / d ** 0.5).astype(np.float32)
ex = GpuBaseExecutor({addr: AffineParams(w, np.zeros(d, np.float32))})
jobs = []
for c in range(n):
    r = (8, 16, 32, 64)[c % 4]
    a = (np.random.default_rng(c).standard_normal((d, r)) / d ** 0.5).astype(np.float32)
    b = (np.random.default_rng(c + 99).standard_normal((r, d)) / r ** 0.5).astype(np.float32)
    ex.register_adapter(c, _Adapter({addr: (a, b)}, 2.0 * r, r))
    jobs.append(GradSeg(client_id=c, x=torch.randn(t, d, device="cuda").bfloat16(),
                        dy=torch.randn(t, d, device="cuda").bfloat16(), accumulate=False,
                        grad_a=torch.zeros(d, r, device="cuda"), grad_b=torch.zeros(r, d, device="cuda")))
stream = torch.cuda.current_stream()
for fused, lag in [(0, 0)] + [(1, l) for l in lags]:
    ex.ctx.set_option("grad_fused", fused)
    ex.ctx.set_option("grad_fused_lag", lag)
    for _ in range(2):
        ex.adapter_grads(0, O.Q, jobs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ex.adapter_grads(0, O.Q, jobs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    alg = n * t * 2 * d * 2
    print(f"fused={fused} lag={lag}: {ms * 1e3:8.1f} us per call, {alg / (ms / 1e3) / 1e9:7.0f} GB/s of x+g", flush=True)
ex.close()
