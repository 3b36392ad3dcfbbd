import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
from tests.test_gpu_parity import _ex, _register_golden_adapters, _fused_run
from oracle import splitserve_oracle as O
g = np.load("tests/golden/fused_random_small.npz")
ex = _ex({(0, O.FF_UP): (g["W"], g["b"])})
for k, v in [kv.split("=") for kv in sys.argv[1:]]:
    ex.ctx.set_option(k, int(v))
_register_golden_adapters(ex, g)
ys, bases, dxs = _fused_run(ex, g, torch.bfloat16)
print([O.normwise_errors(ys[c], g[f"fwd/y{c}"]) for c in range(4)])
print("ok")
