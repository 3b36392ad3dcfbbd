"""One 13B Q-shaped dispatch (32 clients x 1024 rows, d 5120) through GpuBaseExecutor.serve_forward
with f32 numpy payloads (the reference's channel payload) vs bf16 pinned payloads + pinned reply
buffers: wall ms per dispatch, host_convert on / off, and the host pool's conversion rate alone."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import splitserve_oracle as O  # noqa: E402  (parameter generator only)
from paper_2507_03220_b200 import AffineParams, Envelope, GpuBaseExecutor, LayerAddress, Role  # noqa: E402

d, t, n = 5120, 1024, 32
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
addr = LayerAddress(0, Role(O.Q))
w = (np.random.default_rng(0).standard_normal((d, d)) / d ** 0.5).astype(np.float32)
ex = GpuBaseExecutor({addr: AffineParams(w, np.zeros(d, np.float32))})
xs = [np.random.default_rng(c).standard_normal((t, d), dtype=np.float32) for c in range(n)]
rid = [0]


def envs(payloads, replies=None):
    out = []
    for c, p in enumerate(payloads):
        rid[0] += 1
        kw = {"reply_to": replies[c]} if replies is not None else {}
        out.append(Envelope(c, rid[0], 0, O.Q, 0, p, **kw))
    return out


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / iters * 1e3


mb = n * t * d * 4 / 1e6
for conv in (1, 0):
    ex.ctx.set_option("host_convert", conv)
    ms = timed(lambda: ex.serve_forward(envs(xs)))
    print(f"f32 numpy, host_convert={conv}: {ms:7.2f} ms per dispatch ({mb:.0f} MB f32 in, {mb:.0f} MB f32 out)", flush=True)
hb = [torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in xs]
rb = [torch.empty(t, d, dtype=torch.bfloat16).pin_memory() for _ in xs]
ms = timed(lambda: ex.serve_forward(envs(hb, rb)))
print(f"bf16 pinned in / out: {ms:7.2f} ms per dispatch ({mb / 2:.0f} MB in, {mb / 2:.0f} MB out)", flush=True)
# f32 numpy in, pinned f32 reply buffers (no reply-array allocation)
rf = [torch.empty(t, d, dtype=torch.float32).pin_memory() for _ in xs]
ms = timed(lambda: ex.serve_forward(envs(xs, [r.numpy() for r in rf])))
print(f"f32 numpy in, pinned f32 reply_to: {ms:7.2f} ms per dispatch", flush=True)
ex.close()
