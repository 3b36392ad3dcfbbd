"""Decode-size dispatches (32 clients x 2 rows) over 13B layer shapes through the C ABI: GEMM
kernel time per dispatch (ss_profile) and achieved W bytes/s, decode class (decode_rows 16,
K1d) against the single-chain kernels (decode_rows 0). args: [iters] [shapes...] [--lora]
Shapes: q ff_up ff_down lm_head (default all). SS_OPTS="key=value,..." sets context options."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import _lib as L  # noqa: E402

SHAPES = {"q": (5120, 5120), "ff_up": (5120, 13824), "ff_down": (13824, 5120), "lm_head": (5120, 32000)}
argv = sys.argv[1:]
if "--modes" in argv:
    del argv[argv.index("--modes") + 1]
args = [a for a in argv if not a.startswith("--")]
iters = int(args[0]) if args else 50
names = args[1:] or list(SHAPES)
lora = "--lora" in sys.argv
modes = [int(m) for m in (sys.argv[sys.argv.index("--modes") + 1].split(",") if "--modes" in sys.argv else ["16", "0"])]
lib = L.load()
dev = torch.device("cuda:0")
ctx = ctypes.c_void_p()
L.check(None, lib.ss_ctx_create(0, 0, 1, ctypes.byref(ctx)))
stream = torch.cuda.current_stream().cuda_stream
n_cl, rows = 32, 2
import os
for kv in os.environ.get("SS_OPTS", "").split(","):
    if kv:
        k, v = kv.split("=")
        L.check(ctx, lib.ss_set_option(ctx, k.encode(), int(v)))
for name in names:
    K, N = SHAPES[name]
    W = torch.randn(K, N, device=dev, dtype=torch.bfloat16) / K ** 0.5
    L.check(ctx, lib.ss_load_layer(ctx, 0, 4, K, N, W.data_ptr(), N, None, L.SS_MEM_DEVICE | L.SS_DT_BF16))
    if lora:
        for c in range(24):
            r = (8, 16, 32, 64)[c % 4]
            A = torch.randn(K, r, device=dev, dtype=torch.bfloat16) / K ** 0.5
            B = torch.randn(r, N, device=dev, dtype=torch.bfloat16) / r ** 0.5
            L.check(ctx, lib.ss_set_adapter(ctx, c, 0, 4, L.SS_ADAPTER_LORA, r, 2.0, A.data_ptr(),
                                            B.data_ptr(), None, L.SS_MEM_DEVICE | L.SS_DT_BF16))
    x = torch.randn(n_cl * rows, K, device=dev, dtype=torch.bfloat16)
    out = torch.empty(n_cl * rows, N, device=dev, dtype=torch.bfloat16)
    arr = (L.SsSeg * n_cl)()
    for c in range(n_cl):
        s = arr[c]
        s.client_id, s.rows, s.width = c, rows, K
        s.flags = L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16 | (L.SS_SEGF_ADAPTER if lora and c < 24 else 0)
        s.src, s.src_ld = x.data_ptr() + c * rows * K * 2, K
        s.dst, s.dst_ld = out.data_ptr() + c * rows * N * 2, N
    st = (ctypes.c_int32 * n_cl)()
    for mode in modes:
        L.check(ctx, lib.ss_set_option(ctx, b"decode_rows", mode))
        for _ in range(3):
            L.check(ctx, lib.ss_compute_batch(ctx, 0, 0, 4, n_cl, arr, stream, st))
        torch.cuda.synchronize()
        L.check(ctx, lib.ss_profile(ctx, 1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            L.check(ctx, lib.ss_compute_batch(ctx, 0, 0, 4, n_cl, arr, stream, st))
        e1.record()
        torch.cuda.synchronize()
        ms, n, fl, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        lib.ss_profile_read(ctx, 2, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl), ctypes.byref(by))
        L.check(ctx, lib.ss_profile(ctx, 0))
        g_us = ms.value / max(1, n.value) * 1e3
        if "--trace" in sys.argv and mode:
            tr = torch.zeros(4 * 148, dtype=torch.int64, device=dev)
            L.check(ctx, lib.ss_set_option(ctx, b"decode_trace", tr.data_ptr()))
            L.check(ctx, lib.ss_compute_batch(ctx, 0, 0, 4, n_cl, arr, stream, st))
            torch.cuda.synchronize()
            L.check(ctx, lib.ss_set_option(ctx, b"decode_trace", 0))
            t = tr.view(148, 4).cpu().tolist()
            t0 = min(r[0] for r in t if r[1])
            nn = (N + 63) // 64
            C = (K // 64 + 19) // 20
            durs = []
            for b, (s0, s1, u0, u1) in enumerate(t):
                if not s1:
                    continue
                ch = max(0, min(u1, C * nn) - u0)
                durs.append((s1 - s0) / 1e3)
                if b % 8 == 0 or (s1 - s0) / 1e3 > 1.3 * 0 + 0:
                    pass
            order = sorted(range(len(durs)), key=lambda i: -durs[i])
            print(f"   trace: start spread {(max(r[0] for r in t if r[1]) - t0)/1e3:.1f} us, "
                  f"end max {(max(r[1] for r in t) - t0)/1e3:.1f} us, dur min/med/max "
                  f"{min(durs):.1f}/{sorted(durs)[len(durs)//2]:.1f}/{max(durs):.1f} us")
            for b in order[:6] + order[-3:]:
                s0, s1, u0, u1 = t[b]
                ch = max(0, min(u1, C * nn) - u0)
                print(f"     cta {b:3d} start {(s0-t0)/1e3:6.1f} dur {(s1-s0)/1e3:6.1f} us groups {u0} units {u1}")
        print(f"{name:8s} K={K:6d} N={N:6d} decode_rows={mode:2d} lora={int(lora)}: gemm {g_us:7.2f} us "
              f"({K * N * 2 / (g_us * 1e-6) / 1e9:6.0f} GB/s of W), dispatch {e0.elapsed_time(e1) / iters * 1e3:7.2f} us",
              flush=True)
    L.check(ctx, lib.ss_unload_layer(ctx, 0, 4))
lib.ss_ctx_destroy(ctx)
