"""Quick GPU sanity check of the C ABI (development scratch)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import _lib as L  # noqa: E402

lib = L.load()
print(lib.ss_version().decode())
ctx = ctypes.c_void_p()
L.check(None, lib.ss_create if False else lib.ss_ctx_create(0, 0, 1, ctypes.byref(ctx)))
dev = torch.device("cuda:0")
rng = np.random.default_rng(0)


def run(pass_kind, block, role, segs_in, d_out_w, adapter=False, base=False, f32=True):
    arr = (L.SsSeg * len(segs_in))()
    outs = []
    keep = []
    for i, (cid, x) in enumerate(segs_in):
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        if not f32:
            xt = xt.to(torch.bfloat16)
        out = torch.zeros((x.shape[0], d_out_w), dtype=torch.float32 if f32 else torch.bfloat16, device=dev)
        bt = torch.zeros_like(out) if base else None
        keep += [xt, out, bt]
        s = arr[i]
        s.client_id = cid
        s.rows = x.shape[0]
        s.width = x.shape[1]
        s.flags = (0 if f32 else (L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16 | L.SS_SEGF_BASE_BF16)) | (L.SS_SEGF_ADAPTER if adapter else 0)
        s.src = xt.data_ptr()
        s.src_ld = x.shape[1]
        s.dst = out.data_ptr()
        s.dst_ld = d_out_w
        s.dst_base = bt.data_ptr() if base else None
        s.base_ld = d_out_w
        outs.append((out, bt))
    st = (ctypes.c_int32 * len(segs_in))()
    rc = lib.ss_compute_batch(ctx, pass_kind, block, role, len(segs_in), arr, None, st)
    L.check(ctx, rc)
    torch.cuda.synchronize()
    return [(o.float().cpu().numpy(), None if b is None else b.float().cpu().numpy()) for o, b in outs], list(st)


def load(block, role, W, b):
    W = np.ascontiguousarray(W, dtype=np.float32)
    rc = lib.ss_load_layer(ctx, block, role, W.shape[0], W.shape[1], W.ctypes.data, W.shape[1],
                           None if b is None else np.ascontiguousarray(b, np.float32).ctypes.data, 0)
    L.check(ctx, rc)


import os
L.check(ctx, lib.ss_set_option(ctx, b"gemm_2cta", int(os.environ.get("SS_2CTA", "1"))))
# ---- exact integer KAT
d_in, d_out = 320, 520
W = rng.integers(-2, 3, size=(d_in, d_out)).astype(np.float32)
b = rng.integers(-2, 3, size=d_out).astype(np.float32)
load(0, 0, W, b)
x1 = rng.integers(-2, 3, size=(100, d_in)).astype(np.float32)
x2 = rng.integers(-2, 3, size=(61, d_in)).astype(np.float32)
res, st = run(0, 0, 0, [(1, x1), (2, x2)], d_out)
print("fwd status", st)
for x, (o, _) in zip([x1, x2], res):
    ref = x.astype(np.float64) @ W + b
    print("fwd exact:", np.array_equal(o, ref), np.abs(o - ref).max())
g1 = rng.integers(-2, 3, size=(37, d_out)).astype(np.float32)
res, st = run(1, 0, 0, [(1, g1)], d_in)
ref = g1.astype(np.float64) @ W.T
print("bwd exact:", np.array_equal(res[0][0], ref), np.abs(res[0][0] - ref).max())
res, st = run(2, 0, 0, [(1, x1)], d_out)
print("noise exact:", np.array_equal(res[0][0], x1.astype(np.float64) @ W))

# ---- LoRA + IA3 KAT
r = 8
A = np.zeros((d_in, r), np.float32)
A[rng.integers(0, d_in, 12), rng.integers(0, r, 12)] = rng.integers(-2, 3, 12)
B = rng.integers(-2, 3, size=(r, d_out)).astype(np.float32)
rc = lib.ss_set_adapter(ctx, 1, 0, 0, L.SS_ADAPTER_LORA, r, ctypes.c_float(2.0), A.ctypes.data, B.ctypes.data, None, 0)
L.check(ctx, rc)
l = rng.integers(-2, 3, size=d_out).astype(np.float32)
rc = lib.ss_set_adapter(ctx, 2, 0, 0, L.SS_ADAPTER_IA3, 0, ctypes.c_float(0.0), None, None, l.ctypes.data, 0)
L.check(ctx, rc)
res, st = run(0, 0, 0, [(1, x1), (2, x2)], d_out, adapter=True, base=True)
ref1 = x1.astype(np.float64) @ W + b + 2.0 * ((x1 @ A) @ B)
ref2b = x2.astype(np.float64) @ W + b
ref2 = ref2b * l
print("lora fwd exact:", np.array_equal(res[0][0], ref1), np.abs(res[0][0] - ref1).max())
print("ia3 fwd exact:", np.array_equal(res[1][0], ref2), np.array_equal(res[1][1], ref2b))
res, st = run(1, 0, 0, [(2, g1), (1, g1[:20])], d_in, adapter=True)
refia = (g1 * l).astype(np.float64) @ W.T
refl = g1[:20].astype(np.float64) @ W.T + 2.0 * ((g1[:20] @ B.T) @ A.T)
print("ia3 bwd exact:", np.array_equal(res[0][0], refia), np.abs(res[0][0] - refia).max())
print("lora bwd exact:", np.array_equal(res[1][0], refl), np.abs(res[1][0] - refl).max())

# ---- large random bf16 perf probe
import os
mode = int(os.environ.get("SS_2CTA", "1"))
L.check(ctx, lib.ss_set_option(ctx, b"gemm_2cta", mode))
print("gemm_2cta =", mode)
for (K, N, M) in [(4096, 4096, 8192), (5120, 13824, 32768), (13824, 5120, 32768), (5120, 5120, 32768), (5120, 32000, 32768)]:
    W = (rng.standard_normal((K, N), dtype=np.float32) / np.sqrt(K))
    load(1, 4, W, np.zeros(N, np.float32))
    xt = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    arr = (L.SsSeg * 1)()
    s = arr[0]
    s.client_id, s.rows, s.width = 5, M, K
    s.flags = L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16
    s.src, s.src_ld, s.dst, s.dst_ld = xt.data_ptr(), K, out.data_ptr(), N
    st = (ctypes.c_int32 * 1)()
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        L.check(ctx, lib.ss_compute_batch(ctx, 0, 1, 4, 1, arr, stream, st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        L.check(ctx, lib.ss_compute_batch(ctx, 0, 1, 4, 1, arr, stream, st))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ref = (xt.float() @ torch.from_numpy(W).to(dev).to(torch.bfloat16).float())
    err = (out.float() - ref).abs().max().item() / ref.abs().max().item()
    print(f"fwd K={K} N={N} M={M}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TFLOP/s  normwise err {err:.2e}")
    gt = torch.randn(M, N, device=dev, dtype=torch.bfloat16)
    dx = torch.empty(M, K, device=dev, dtype=torch.bfloat16)
    s.rows, s.width, s.src, s.src_ld, s.dst, s.dst_ld = M, N, gt.data_ptr(), N, dx.data_ptr(), K
    for _ in range(3):
        L.check(ctx, lib.ss_compute_batch(ctx, 1, 1, 4, 1, arr, stream, st))
    e0.record()
    for _ in range(10):
        L.check(ctx, lib.ss_compute_batch(ctx, 1, 1, 4, 1, arr, stream, st))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ref = gt.float() @ torch.from_numpy(W).to(dev).to(torch.bfloat16).float().T
    err = (dx.float() - ref).abs().max().item() / ref.abs().max().item()
    print(f"bwd K={N} N={K} M={M}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TFLOP/s  normwise err {err:.2e}")
    a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    bm = torch.randn(K, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        a @ bm
    e0.record()
    for _ in range(10):
        a @ bm
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"  cuBLAS same shape: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s")
print("launches", lib.ss_kernel_launches(ctx))
lib.ss_ctx_destroy(ctx)
print("OK")
