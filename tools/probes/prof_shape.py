"""Run one GEMM shape a few times through the C ABI (for ncu). args: K N M pass 2cta group_m"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_03220_b200 import _lib as L  # noqa: E402

K, N, M, pk, mode, gm = (int(a) for a in sys.argv[1:7])
iters = int(sys.argv[7]) if len(sys.argv) > 7 else 3
lib = L.load()
ctx = ctypes.c_void_p()
L.check(None, lib.ss_ctx_create(0, 0, 1, ctypes.byref(ctx)))
L.check(ctx, lib.ss_set_option(ctx, b"gemm_2cta", mode))
L.check(ctx, lib.ss_set_option(ctx, b"group_m", gm))
import os
L.check(ctx, lib.ss_set_option(ctx, b"pair_n", int(os.environ.get("SS_PAIR_N", "256"))))
dev = torch.device("cuda:0")
W = torch.randn(K, N, device=dev, dtype=torch.bfloat16)
L.check(ctx, lib.ss_load_layer(ctx, 0, 4, K, N, W.data_ptr(), N, None, L.SS_MEM_DEVICE | L.SS_DT_BF16))
x = torch.randn(M, K if pk == 0 else N, device=dev, dtype=torch.bfloat16)
out = torch.empty(M, N if pk == 0 else K, device=dev, dtype=torch.bfloat16)
arr = (L.SsSeg * 1)()
s = arr[0]
s.client_id, s.rows, s.width = 5, M, x.shape[1]
s.flags = L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16
s.src, s.src_ld, s.dst, s.dst_ld = x.data_ptr(), x.shape[1], out.data_ptr(), out.shape[1]
st = (ctypes.c_int32 * 1)()
stream = torch.cuda.current_stream().cuda_stream
L.check(ctx, lib.ss_profile(ctx, 1))
for _ in range(iters):
    L.check(ctx, lib.ss_compute_batch(ctx, pk, 0, 4, 1, arr, stream, st))
torch.cuda.synchronize()
ms, n, fl, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
lib.ss_profile_read(ctx, 2, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl), ctypes.byref(by))
print(f"K={K} N={N} M={M} pass={pk} 2cta={mode} group_m={gm}: gemm {ms.value / n.value:.3f} ms "
      f"{fl.value / (ms.value / 1e3) / 1e12:.0f} TFLOP/s")
lib.ss_ctx_destroy(ctx)
