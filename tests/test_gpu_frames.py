"""LSV1 frames through the GPU without a host-side decode (ss_serve_frames / FrameServer) against
the reference's own codec + executor (tests/golden/frames.npz, made by make_golden.py
frames_golden): exact-integer payloads and weights, so the reply stream must be BITWISE the
reference's — headers, PASS_ERROR messages, f32 payloads, request order."""

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O

from .test_gpu_parity import _Adapter, _addr, _ex

pytestmark = pytest.mark.gpu


def _server(g, out_capacity=1 << 16):
    from paper_2507_03220_b200.frames import FrameServer
    ex = _ex({(0, O.Q): (g["W_q"], g["b_q"]), (0, O.FF_UP): (g["W_up"], g["b_up"])})
    return ex, FrameServer(ex, out_capacity=out_capacity)


def test_reply_stream_bitwise_equals_reference(golden):
    g = golden("frames")
    ex, srv = _server(g, out_capacity=64)      # forces the grow-and-retry path
    req = g["requests"].tobytes()
    out, used = srv.serve(req)
    assert used == len(req)
    assert out == g["replies"].tobytes()
    ex.close()


def test_partial_trailing_frame_and_request_ids_persist(golden):
    g = golden("frames")
    ex, srv = _server(g)
    req = g["requests"].tobytes()
    first = req[:30 + 5 * 16 * 4]                      # exactly frame 0
    out, used = srv.serve(first + req[:17])            # + a partial header of "another" frame
    assert used == len(first)
    assert out == g["replies"].tobytes()[:len(out)]
    # the intake remembers request ids across calls: replaying frame 0 is now rejected
    out2, _ = srv.serve(first)
    assert out2[21] == 255 and b"not increasing" in out2[30:]
    ex.close()


def test_corrupt_stream_is_a_connection_level_rejection(golden):
    from paper_2507_03220_b200 import _lib
    g = golden("frames")
    ex, srv = _server(g)
    bad = bytearray(g["requests"].tobytes())
    bad[0:4] = b"XSV1"
    with pytest.raises(_lib.SsError) as e:
        srv.serve(bytes(bad))
    assert e.value.code == _lib.SS_E_PROTOCOL
    bad = bytearray(g["requests"].tobytes())
    bad[4] = 2                                            # version 2
    with pytest.raises(_lib.SsError):
        srv.serve(bytes(bad))
    ex.close()


def test_fused_adapter_frames_match_oracle():
    """Random f32 payloads at a 13B-ish layer width through frames, with a fused LoRA client and
    an IA3 client; replies decoded here and compared with the oracle (bf16 operands)."""
    import struct
    from paper_2507_03220_b200.frames import FrameServer
    d_in, d_out = 1024, 1536
    w, b = O.layer_params(41, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    lo = O.lora_params(41, 1, 0, O.V, d_in, d_out, 32, 64.0)
    ia = O.ia3_params(41, 2, 0, O.V, d_out)
    ex.register_adapter(1, _Adapter(lora={_addr(0, O.V): (lo.a, lo.b)}, alpha=64.0, rank=32))
    ex.register_adapter(2, _Adapter(ia3={_addr(0, O.V): ia.ia3}))
    ads = {1: O.OracleAdapter(a=O.bf16_round(lo.a), b=O.bf16_round(lo.b), alpha=64.0, rank=32), 2: ia, 3: None}
    rng = np.random.default_rng(41)
    hdr = struct.Struct("<4sHIQHBBII")
    xs, req = {}, b""
    for i, (cid, t) in enumerate(((1, 300), (2, 129), (3, 1000), (1, 7))):
        x = rng.standard_normal((t, d_in)).astype(np.float32)
        xs[i] = (cid, x)
        req += hdr.pack(b"LSV1", 1, cid, 10 + i, 0, O.V, 0, t, d_in) + x.tobytes()
    srv = FrameServer(ex)
    out, used = srv.serve(req)
    assert used == len(req)
    pos, wr = 0, O.bf16_round(w)
    for i in range(4):
        magic, ver, cid, rid, blk, role, pk, t, wd = hdr.unpack(out[pos:pos + 30])
        assert (magic, cid, rid, pk, wd) == (b"LSV1", xs[i][0], 10 + i, 0, d_out)
        y = np.frombuffer(out[pos + 30:pos + 30 + 4 * t * wd], dtype="<f4").reshape(t, wd)
        pos += 30 + 4 * t * wd
        x = O.bf16_round(xs[i][1])
        ref = O.apply_adapter(ads[cid], x, O.affine_forward(x, wr, b))
        mx, mn = O.normwise_errors(y, ref)
        assert mx <= 1e-2 and mn <= 1.5e-3, (i, mx, mn)   # f32 outputs tier
    assert pos == len(out)
    ex.close()
