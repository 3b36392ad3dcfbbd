import sys, struct, numpy as np
sys.path.insert(0, ".")
from oracle import splitserve_oracle as O
from tests.test_gpu_parity import _ex
from paper_2507_03220_b200.frames import FrameServer
g = np.load("tests/golden/frames.npz")
ex = _ex({(0, O.Q): (g["W_q"], g["b_q"]), (0, O.FF_UP): (g["W_up"], g["b_up"])})
srv = FrameServer(ex)
out, used = srv.serve(g["requests"].tobytes())
ref = g["replies"].tobytes()
print(len(out), len(ref), used, len(g["requests"]))
hdr = struct.Struct("<4sHIQHBBII")
for name, b in (("ours", out), ("ref", ref)):
    pos = 0
    while pos < len(b):
        m, v, c, r, bl, ro, pk, t, w = hdr.unpack(b[pos:pos+30])
        sz = t if pk == 255 else 4*t*w
        print(name, c, r, pk, t, w, b[pos+30:pos+30+sz].decode() if pk == 255 else np.frombuffer(b[pos+30:pos+30+sz], '<f4')[:4])
        pos += 30 + sz
