"""One cuBLAS GEMM and one fused-kernel GEMM per shape (for an ncu comparison)."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_03220_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda:0")
lib = L.load()
ctx = ctypes.c_void_p()
L.check(None, lib.ss_ctx_create(0, 0, 1, ctypes.byref(ctx)))
stream = torch.cuda.current_stream().cuda_stream
for li, (K, N, M) in enumerate([(5120, 5120, 32768), (5120, 13824, 32768)]):
    W = (torch.randn(K, N, device=dev) / K ** 0.5).to(torch.bfloat16)
    x = torch.randn(M, K, device=dev).to(torch.bfloat16)
    y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(2):
        torch.matmul(x, W, out=y)
    L.check(ctx, lib.ss_load_layer(ctx, li, 4, K, N, W.data_ptr(), N, None, L.SS_MEM_DEVICE | L.SS_DT_BF16))
    arr = (L.SsSeg * 1)()
    s = arr[0]
    s.client_id, s.rows, s.width = 5, M, K
    s.flags = L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16
    s.src, s.src_ld, s.dst, s.dst_ld = x.data_ptr(), K, y.data_ptr(), N
    st = (ctypes.c_int32 * 1)()
    for _ in range(2):
        L.check(ctx, lib.ss_compute_batch(ctx, 0, li, 4, 1, arr, stream, st))
    torch.cuda.synchronize()
    # timing: 20 back-to-back each
    def ours(pn):
        L.check(ctx, lib.ss_set_option(ctx, b"pair_n", pn))
        L.check(ctx, lib.ss_compute_batch(ctx, 0, li, 4, 1, arr, stream, st))
    for name, fn in (("cublas", lambda: torch.matmul(x, W, out=y)),
                     ("ours256", lambda: ours(256)), ("ours512", lambda: ours(512))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(5):
            fn()
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"K={K} N={N} M={M} {name}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.0f} TFLOP/s", flush=True)
