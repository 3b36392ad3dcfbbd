"""Measure the normwise error of the fused executor against the f32 oracle (same bf16-rounded
inputs), per client kind, pass, output dtype and ``lora_hilo`` mode. Prints a markdown table
(profiles/r02_precision.md is this script's output on a B200).

    python tools/precision_probe.py [--shape 5120x13824]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import splitserve_oracle as O  # noqa: E402
from paper_2507_03220_b200 import AffineParams, Envelope, GpuBaseExecutor, LayerAddress, Role  # noqa: E402


class _Ad:
    def __init__(self, lora=None, ia3=None, alpha=0.0, rank=1):
        self.lora, self.ia3, self.alpha, self.rank = lora or {}, ia3 or {}, alpha, rank


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="5120x13824")
    ap.add_argument("--rows", type=int, default=300)
    args = ap.parse_args()
    d_in, d_out = (int(v) for v in args.shape.split("x"))
    role = O.FF_UP
    w, b = O.layer_params(1, 0, role, d_in, d_out)
    wr = O.bf16_round(w)
    ex = GpuBaseExecutor({LayerAddress(0, Role(role)): AffineParams(w, b)})
    la = LayerAddress(0, Role(role))
    kinds = [("plain", 0), ("lora", 8), ("lora", 64), ("ia3", 0), ("lora+ia3", 16)]
    ads = {}
    for cid, (kind, r) in enumerate(kinds):
        lo = O.lora_params(1, cid, 0, role, d_in, d_out, max(r, 1), 2.0 * max(r, 1)) if "lora" in kind else None
        ia = O.ia3_params(1, cid, 0, role, d_out).ia3 if "ia3" in kind else None
        if kind != "plain":
            ex.register_adapter(cid, _Ad(lora={la: (lo.a, lo.b)} if lo else None, ia3={la: ia} if ia is not None else None,
                                         alpha=2.0 * max(r, 1), rank=max(r, 1)))
        ads[cid] = O.OracleAdapter(a=O.bf16_round(lo.a) if lo else None, b=O.bf16_round(lo.b) if lo else None,
                                   alpha=2.0 * max(r, 1), rank=max(r, 1), ia3=ia)
    rng = np.random.default_rng(0)
    print(f"shape {d_in}x{d_out}, {args.rows} rows per client; normwise max|d|/max|ref| / mean|d|/mean|ref|"
          " vs the f32 oracle on the same bf16-rounded inputs (IA3 backward: g*l in f32)\n")
    print("| lora_hilo | out dtype | pass | " + " | ".join(k for k, _ in kinds) + " |")
    print("|---|---|---|" + "---|" * len(kinds))
    req = 1
    for hilo in (0, 1, 2):
        ex.ctx.set_option("lora_hilo", hilo)
        for dt in (torch.float32, torch.bfloat16):
            for pass_kind, width in ((0, d_in), (1, d_out)):
                xs = [O.bf16_round(rng.standard_normal((args.rows, width)).astype(np.float32)) for _ in kinds]
                envs = [Envelope(c, req, 0, role, pass_kind, torch.from_numpy(x).to(ex.device, dt)) for c, x in enumerate(xs)]
                req += 1
                res = ex._compute_batch(pass_kind, envs)
                cells = []
                for c, x in enumerate(xs):
                    if pass_kind == 0:
                        ref = O.apply_adapter(ads[c], x, O.affine_forward(x, wr, b))
                    else:
                        ref = O.layer_backward_dx(ads[c], wr, x)
                    mx, mn = O.normwise_errors(res[c].float().cpu().numpy(), ref)
                    cells.append(f"{mx:.1e} / {mn:.1e}")
                print(f"| {hilo} | {str(dt).split('.')[-1]} | {'fwd' if pass_kind == 0 else 'bwd'} | " + " | ".join(cells) + " |")
    ex.close()


if __name__ == "__main__":
    main()
