"""Bitwise check of the cluster-of-4 GEMM against the pair kernel (mixed adapters, odd/even M tiles)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import splitserve_oracle as O
import test_gpu_parity as T

for d_in, d_out, counts in ((512, 1280, [700, 256, 3, 129, 512, 64, 1]), (5120, 1536, [1024, 512, 300, 2048, 77, 1, 700]),
                            (1024, 768, [300, 1, 200, 5, 1, 1, 90])):
    w, b = O.layer_params(13, 0, O.K, d_in, d_out)
    ex = T._ex({(0, O.K): (w, b)})
    T._mixed_clients(ex, d_in, d_out, seed=13)
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=ex.device).to(torch.bfloat16) for t in counts]
        outs = []
        for c4 in (0, 1):
            ex.ctx.set_option("gemm_2cta", 1)
            ex.ctx.set_option("pair_n", 256)
            ex.ctx.set_option("cluster4", c4)
            outs.append(ex._compute_batch(pass_kind, [T._env(c, 10 + 2 * pass_kind + c4, 0, O.K, pass_kind, x)
                                                      for c, x in enumerate(xs)]))
        torch.cuda.synchronize()
        ok = all(torch.equal(outs[0][c], outs[1][c]) for c in range(len(xs)))
        print(d_in, d_out, sum(counts), "pass", pass_kind, "bitwise", ok, flush=True)
    ex.close()
