"""GEMM raster / L2-policy sweep at the 13B step's shapes (for timing and, under ncu, DRAM bytes).
Prints one line per (shape, config) in launch order; `--iters 1 --warm 0` under ncu."""
import argparse
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--configs", default="raster=0;raster=1;raster=0,hint_a=2,hint_out=1;raster=1,hint_b=2,hint_out=1;raster=1,l2_budget_mb=96")
ap.add_argument("--shapes", default="all")
args = ap.parse_args()

# (name, d_in, d_out, M, pass)
SHAPES = [
    ("Q_fwd", 5120, 5120, 32768, 0), ("FFUP_fwd", 5120, 13824, 32768, 0),
    ("FFDOWN_fwd", 13824, 5120, 32768, 0), ("HEAD_fwd", 5120, 32000, 32768, 0),
    ("Q_bwd", 5120, 5120, 16384, 1), ("FFUP_bwd", 5120, 13824, 16384, 1),
    ("FFDOWN_bwd", 13824, 5120, 16384, 1), ("HEAD_bwd", 5120, 32000, 16384, 1),
    ("Q_dec", 5120, 5120, 64, 0), ("FFUP_dec", 5120, 13824, 64, 0),
    ("FFDOWN_dec", 13824, 5120, 64, 0), ("HEAD_dec", 5120, 32000, 64, 0),
]
if args.shapes != "all":
    SHAPES = [s for s in SHAPES if s[0] in args.shapes.split(",")]
lib = L.load()
ctx = ctypes.c_void_p()
L.check(None, lib.ss_ctx_create(0, 0, 1, ctypes.byref(ctx)))
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream().cuda_stream
defaults = {"raster": 0, "group_n": 0, "l2_budget_mb": 48, "l2_hints": 1, "group_m": 16, "a_rows64": 1}
for li, (name, din, dout, M, pk) in enumerate(SHAPES):
    W = torch.randn(din, dout, device=dev, dtype=torch.bfloat16)
    L.check(ctx, lib.ss_load_layer(ctx, li, 4, din, dout, W.data_ptr(), dout, None, L.SS_MEM_DEVICE | L.SS_DT_BF16))
    K, N = (din, dout) if pk == 0 else (dout, din)
    x = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    arr = (L.SsSeg * 1)()
    s = arr[0]
    s.client_id, s.rows, s.width = 5, M, K
    s.flags = L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16
    s.src, s.src_ld, s.dst, s.dst_ld = x.data_ptr(), K, out.data_ptr(), N
    st = (ctypes.c_int32 * 1)()
    for cfg in args.configs.split(";"):
        opts = dict(defaults)
        for kv in filter(None, cfg.split(",")):
            k, v = kv.split("=")
            opts[k] = int(v)
        for k, v in opts.items():
            L.check(ctx, lib.ss_set_option(ctx, k.encode(), v))
        for _ in range(args.warm):
            L.check(ctx, lib.ss_compute_batch(ctx, pk, li, 4, 1, arr, stream, st))
        L.check(ctx, lib.ss_profile(ctx, 1))
        for _ in range(args.iters):
            L.check(ctx, lib.ss_compute_batch(ctx, pk, li, 4, 1, arr, stream, st))
        torch.cuda.synchronize()
        ms, n, fl, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        lib.ss_profile_read(ctx, 2, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl), ctypes.byref(by))
        L.check(ctx, lib.ss_profile(ctx, 0))
        t = ms.value / max(n.value, 1)
        print(f"{name:11s} {cfg:45s} {t:.3f} ms {fl.value / n.value / (t / 1e3) / 1e12:6.0f} TFLOP/s "
              f"alg {by.value / n.value / 1e6:.0f} MB", flush=True)
    lib.ss_unload_layer(ctx, li, 4)
    del W, x, out
lib.ss_ctx_destroy(ctx)
