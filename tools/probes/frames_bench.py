"""LSV1 frames served through ss_serve_frames at the 13B Q-layer shape: 32 clients x 1024 f32
tokens per call (one forward dispatch), timed end to end (parse + H2D + fused GEMM + D2H +
reply headers), from a pinned receive buffer into the pinned send buffer."""
import math, struct, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role
from paper_2507_03220_b200.frames import FrameServer

d = 5120
dev = torch.device("cuda", 0)
ex = GpuBaseExecutor({LayerAddress(0, Role.Q): AffineParams((torch.randn(d, d, device=dev) / math.sqrt(d)).bfloat16(),
                                                           torch.zeros(d, device=dev))})
hdr = struct.Struct("<4sHIQHBBII")
t, n = 1024, 32
payload = np.random.default_rng(0).standard_normal((t, d)).astype(np.float32).tobytes()
rid = [0]
def stream():
    parts = []
    for c in range(n):
        rid[0] += 1
        parts.append(hdr.pack(b"LSV1", 1, c, rid[0], 0, 0, 0, t, d) + payload)
    return b"".join(parts)
srv = FrameServer(ex)
reqs = [stream() for _ in range(4)]
buf = torch.empty(len(reqs[0]), dtype=torch.uint8, pin_memory=True)
srv.serve(reqs[0])
for k in (1, 2, 3):
    buf.numpy()[:] = np.frombuffer(reqs[k], dtype=np.uint8)
    t0 = time.perf_counter()
    out, used = srv.serve_pinned(buf, len(reqs[k]))
    dt = time.perf_counter() - t0
    print(f"serve_pinned: {len(reqs[k])/1e6:.0f} MB in, {out.numel()/1e6:.0f} MB out in {dt*1e3:.1f} ms -> "
          f"{(len(reqs[k]) + out.numel())/dt/1e9:.1f} GB/s, {n*t/dt:.0f} tokens/s for one Q layer")
# host codec cost of the reference path for the same stream (numpy frombuffer/astype + tobytes)
t0 = time.perf_counter()
pos, b = 0, reqs[1]
while pos < len(b):
    _, _, _, _, _, _, _, tt, w = hdr.unpack_from(b, pos)
    x = np.frombuffer(b, dtype="<f4", count=tt * w, offset=pos + 30).astype(np.float32, copy=False).reshape(tt, w)
    x = np.array(x)   # the reference's bytes(buf[...]) copy
    _ = hdr.pack(b"LSV1", 1, 0, 0, 0, 0, 0, tt, w) + np.ascontiguousarray(x, dtype="<f4").tobytes()
    pos += 30 + 4 * tt * w
print(f"numpy decode+encode of the same stream (reference codec work, no compute): {(time.perf_counter()-t0)*1e3:.1f} ms")
