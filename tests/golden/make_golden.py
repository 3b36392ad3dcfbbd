"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container, where the reference is importable read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``splitserve`` from /root/reference/pkg/src (never copied), drives the reference's
own public functions — BaseExecutor.serve_forward / serve_backward / serve_noise_effect
(executor.py:182-189), apply_adapter (adapters.py:127-145), lora_forward / lora_backward
(adapters.py:19-41), build_model (model.py:65-85) — on seeded inputs, and writes the inputs and
outputs as .npz fixtures next to this script. The fixtures travel with the repo; the GPU box
never needs the reference.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("SPLITSERVE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from splitserve.adapters import (AdapterState, apply_adapter, lora_backward,  # noqa: E402
                                 lora_forward)
from splitserve.config import LayerAddress, ModelConfig, Role, base_addresses  # noqa: E402
from splitserve.errors import ProtocolError  # noqa: E402
from splitserve.executor import BaseExecutor  # noqa: E402
from splitserve.model import build_model  # noqa: E402
from splitserve.protocol import (PASS_BACKWARD, PASS_FORWARD,  # noqa: E402
                                 PASS_NOISE_EFFECT, Envelope)
from splitserve.tensor_ops import AffineParams  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_round(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32).reshape(x.shape)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def model_checksums():
    """build_model layer bytes for the configs the reference tests and BASELINE config 1 use."""
    out = {}
    cfgs = {
        "executor_cfg": ModelConfig(1, 8, 2, 16, 16, 32, 0),      # test_executor.py:19-20
        "client_cfg": ModelConfig(2, 16, 4, 32, 32, 64, 2),       # test_client.py:21-22
        "tiny_cfg": ModelConfig(2, 256, 4, 512, 512, 128, 0),     # BASELINE configs[0]
    }
    for name, cfg in cfgs.items():
        model = build_model(cfg)
        layer_bytes = []
        for addr in base_addresses(cfg):
            p = model.layers[addr]
            layer_bytes += [p.weight, p.bias]
            out[f"{name}/{addr.block}/{int(addr.role)}"] = np.frombuffer(
                sha(p.weight, p.bias).encode(), dtype=np.uint8)
        out[f"{name}/all"] = np.frombuffer(sha(*layer_bytes).encode(), dtype=np.uint8)
        out[f"{name}/embedding"] = np.frombuffer(sha(model.embedding).encode(), dtype=np.uint8)
        out[f"{name}/dims"] = np.array([cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.d_ff,
                                        cfg.vocab_size, cfg.max_seq, cfg.seed], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "model_checksums.npz"), **out)


def executor_kat():
    """test_executor.py fixtures: serve_forward/backward/noise on build_model(CFG) (0, Q)."""
    cfg = ModelConfig(1, 8, 2, 16, 16, 32, 0)
    model = build_model(cfg)
    ex = BaseExecutor(model.layers)
    addr = LayerAddress(0, Role.Q)

    def env(client, req, rows, pass_kind=PASS_FORWARD, width=8, seed=None):
        rng = np.random.default_rng(seed if seed is not None else client * 100 + req)
        return Envelope(client, req, addr.block, int(addr.role), pass_kind,
                        rng.standard_normal((rows, width)).astype(np.float32))

    d = {}
    p = model.layers[addr]
    d["W"], d["b"] = p.weight, p.bias
    fw = [env(1, 1, 3), env(2, 1, 5), env(3, 1, 0), env(4, 1, 7)]
    res = ex.serve_forward(fw)
    for i, (e, r) in enumerate(zip(fw, res)):
        d[f"fwd/x{i}"], d[f"fwd/y{i}"] = e.payload, r
    bw = [env(1, 2, 2, PASS_BACKWARD), env(2, 2, 4, PASS_BACKWARD)]
    for i, (e, r) in enumerate(zip(bw, ex.serve_backward(bw))):
        d[f"bwd/g{i}"], d[f"bwd/dx{i}"] = e.payload, r
    ne = env(1, 3, 4, PASS_NOISE_EFFECT)
    d["noise/x"], d["noise/y"] = ne.payload, ex.serve_noise_effect(ne)
    # malformed envelope fails alone (test_executor.py:66-72); plus layer/pass mismatches
    good, bad = env(1, 4, 3), env(2, 4, 3, width=5)
    wrong_pass = env(5, 4, 2, PASS_BACKWARD)
    res = ex.serve_forward([good, bad, wrong_pass])
    d["bad/x_good"], d["bad/x_bad"], d["bad/x_wrong_pass"] = good.payload, bad.payload, wrong_pass.payload
    d["bad/y_good"] = res[0]
    d["bad/kinds"] = np.array([0 if isinstance(r, np.ndarray) else 1 for r in res])
    d["bad/msgs"] = np.array([str(r) if isinstance(r, ProtocolError) else "" for r in res])
    np.savez_compressed(os.path.join(HERE, "executor_kat.npz"), **d)


def adapters_golden():
    rng = np.random.default_rng(11)
    d = {}
    x = rng.standard_normal((5, 24)).astype(np.float32)
    a = rng.standard_normal((24, 4)).astype(np.float32)
    b = rng.standard_normal((4, 40)).astype(np.float32)
    gy = rng.standard_normal((5, 40)).astype(np.float32)
    d["x"], d["a"], d["b"], d["gy"] = x, a, b, gy
    d["lora_fwd"] = lora_forward(x, a, b, 8.0, 4)
    ga, gb, gx = lora_backward(x, gy, a, b, 8.0, 4)
    d["lora_ga"], d["lora_gb"], d["lora_gx"] = ga, gb, gx
    cfg = ModelConfig(1, 24, 2, 40, 16, 32, 0)
    st = AdapterState.init_lora(cfg, rank=4, alpha=8.0, targets=[Role.FF_UP], seed=3)
    addr = LayerAddress(0, Role.FF_UP)
    st.lora[addr] = (a, b)
    yb = rng.standard_normal((5, 40)).astype(np.float32)
    d["y_base"] = yb
    d["apply_lora"] = apply_adapter(st, addr, x, yb)
    ia = AdapterState.init_ia3(cfg, targets=[Role.FF_UP])
    l = (1 + 0.1 * rng.standard_normal(40)).astype(np.float32)
    ia.ia3[addr] = l
    d["l"] = l
    d["apply_ia3"] = apply_adapter(ia, addr, x, yb)
    d["apply_ia3_other"] = apply_adapter(ia, LayerAddress(0, Role.Q), x, yb)
    # init_lora stream (adapters.py:62-73) for the tiny config, first target A
    tcfg = ModelConfig(2, 256, 4, 512, 512, 128, 0)
    st2 = AdapterState.init_lora(tcfg, rank=8, alpha=16.0, targets=[Role.Q, Role.K, Role.V, Role.O], seed=1)
    d["init_lora_sha"] = np.frombuffer(
        sha(*[st2.lora[k][0] for k in sorted(st2.lora)], *[st2.lora[k][1] for k in sorted(st2.lora)]).encode(),
        dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "adapters.npz"), **d)


def fused_batch(name, d_in, d_out, seed, integer=False, rows=(37, 130, 5, 64), ranks=(8, 16)):
    """A mixed batch through the reference executor + each client's adapter step.

    Clients: 0 LoRA rank ranks[0], 1 IA3, 2 plain, 3 LoRA rank ranks[1]. Forward: serve_forward
    then apply_adapter per client (client.py:206-209). Backward: IA3 g = dy*l (client.py:291-294),
    serve_backward on g, plus lora_backward's grad_x (client.py:296-304)."""
    rng = np.random.default_rng(seed)

    def draw(shape, scale=1.0):
        if integer:
            return rng.integers(-2, 3, size=shape).astype(np.float32)
        return bf16_round((rng.standard_normal(shape) * scale).astype(np.float32))

    W = draw((d_in, d_out), 1.0 / np.sqrt(d_in))
    b = draw((d_out,), 0.05)
    addr = LayerAddress(0, Role.FF_UP)
    ex = BaseExecutor({addr: AffineParams(W, b)})
    cfg = ModelConfig(1, d_in, 1, d_out, 16, 32, 0)
    d = {"W": W, "b": b, "rows": np.array(rows), "ranks": np.array(ranks)}
    adapters = {}
    for cid, rank in ((0, ranks[0]), (3, ranks[1])):
        st = AdapterState.init_lora(cfg, rank=rank, alpha=2.0 * rank, targets=[Role.FF_UP], seed=cid)
        if integer:
            a = np.zeros((d_in, rank), np.float32)
            idx = rng.integers(0, d_in, size=2 * rank)
            a[idx, rng.integers(0, rank, size=2 * rank)] = rng.integers(-1, 2, size=2 * rank)
            # sparse B keeps the backward shrink s*g.B^T within +-256 (exact in bf16)
            bb = rng.integers(-2, 3, size=(rank, d_out)).astype(np.float32)
            bb *= rng.random((rank, d_out)) < 0.08
        else:
            a = bf16_round(rng.standard_normal((d_in, rank)).astype(np.float32) / np.sqrt(d_in))
            bb = bf16_round((0.05 * rng.standard_normal((rank, d_out))).astype(np.float32))
        st.lora[addr] = (a, bb)
        adapters[cid] = st
        d[f"A{cid}"], d[f"B{cid}"], d[f"alpha{cid}"] = a, bb, np.float32(2.0 * rank)
    ia = AdapterState.init_ia3(cfg, targets=[Role.FF_UP])
    l = (rng.integers(-2, 3, size=d_out).astype(np.float32) if integer
         else bf16_round((1 + 0.1 * rng.standard_normal(d_out)).astype(np.float32)))
    ia.ia3[addr] = l
    adapters[1] = ia
    d["l1"] = l
    xs = [draw((r, d_in)) for r in rows]
    envs = [Envelope(c, 1, 0, int(Role.FF_UP), PASS_FORWARD, x) for c, x in enumerate(xs)]
    base = ex.serve_forward(envs)
    for c, (x, yb) in enumerate(zip(xs, base)):
        d[f"fwd/x{c}"] = x
        d[f"fwd/ybase{c}"] = yb
        d[f"fwd/y{c}"] = apply_adapter(adapters.get(c), addr, x, yb)
    gs = [draw((r, d_out)) for r in rows]
    gin = []
    for c, g in enumerate(gs):
        st = adapters.get(c)
        gin.append(g * st.ia3[addr] if (st is not None and addr in st.ia3) else g)
    benv = [Envelope(c, 2, 0, int(Role.FF_UP), PASS_BACKWARD, g) for c, g in enumerate(gin)]
    bres = ex.serve_backward(benv)
    for c, (g, dx) in enumerate(zip(gs, bres)):
        st = adapters.get(c)
        if st is not None and addr in st.lora:
            a, bb = st.lora[addr]
            _, _, gx = lora_backward(xs[c], gin[c], a, bb, st.alpha, st.rank)
            dx = dx + gx
        d[f"bwd/g{c}"] = g
        d[f"bwd/dx{c}"] = dx
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)


def row_independence():
    """tensor_ops.py:1-8 / test_tensor_ops.py:62-75: batched == solo bitwise in the reference."""
    cfg = ModelConfig(1, 64, 2, 96, 16, 32, 0)
    model = build_model(cfg)
    addr = LayerAddress(0, Role.FF_UP)
    ex = BaseExecutor(model.layers)
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal((r, 64)).astype(np.float32) for r in (1, 9, 33)]
    batched = ex.serve_forward([Envelope(i, 1, 0, int(Role.FF_UP), 0, x) for i, x in enumerate(xs)])
    solo = [ex.serve_forward([Envelope(i, 2, 0, int(Role.FF_UP), 0, x)])[0] for i, x in enumerate(xs)]
    assert all(np.array_equal(a, b) for a, b in zip(batched, solo))
    d = {"W": model.layers[addr].weight, "b": model.layers[addr].bias}
    for i, (x, y) in enumerate(zip(xs, batched)):
        d[f"x{i}"], d[f"y{i}"] = x, y
    np.savez_compressed(os.path.join(HERE, "row_independence.npz"), **d)


def privacy_golden():
    """privacy.py:33-106 — rotate indices, draw_noise samples and a blind -> serve_forward ->
    unblind round trip through the reference's own NoiseSet / LocalChannel / BaseExecutor."""
    from splitserve.privacy import NoiseSet, draw_noise, precompute_noise, rotate
    from splitserve.transport import LocalChannel
    d = {}
    addrs = [LayerAddress(0, Role.Q), LayerAddress(3, Role.FF_UP), LayerAddress(2, Role.LM_HEAD)]
    d["rotate"] = np.array([[rotate(s, a, it, k) for a in addrs for it in range(6) for k in (2, 3, 5)]
                            for s in (0, 7)], dtype=np.int64)
    d["noise_q"] = draw_noise(4, addrs[0], 1, 5, 16, 1.0)
    d["noise_up"] = draw_noise(9, addrs[1], 0, 3, 24, 0.25)
    cfg = ModelConfig(1, 16, 2, 32, 32, 16, 0)
    layers = build_model(cfg).layers
    addr = LayerAddress(0, Role.FF_UP)
    ex = BaseExecutor({addr: layers[addr]})
    ex.start()
    try:
        ch = LocalChannel(ex, 1, 1, 8, 32)
        ch.register(sends_backward=False)
        ns = precompute_noise(ch, cfg, k=2, scale=1.0, seed=3, t_max=8, layers=[addr])
        x = np.random.default_rng(5).standard_normal((8, 16)).astype(np.float32)
        payload, idx = ns.blind(addr, x, 4)
        y_noisy = np.array(ch.request(0, int(Role.FF_UP), PASS_FORWARD, payload), copy=True)
        d["rt_x"], d["rt_idx"] = x, np.int64(idx)
        d["rt_y"] = ns.unblind(addr, y_noisy, idx)
        d["rt_effect"] = ns.effects[addr][idx]
        d["rt_W"], d["rt_b"] = layers[addr].weight, layers[addr].bias
    finally:
        ex.stop()
    np.savez_compressed(os.path.join(HERE, "privacy.npz"), **d)


def frames_golden():
    """protocol.py:96-153 + executor.py:162-231, 295-300 — a run of LSV1 request frames (valid
    forward / backward / noise frames of two layers, exact-integer payloads, plus frames the
    intake rejects) encoded by the reference, and the reply frames the reference executor
    produces for them (submit's error replies; serve_* results wrapped as replies), encoded by
    the reference codec."""
    from splitserve.protocol import (PASS_ERROR, encode, error_envelope, try_decode)  # noqa: F401
    cfg = ModelConfig(1, 16, 2, 32, 32, 16, 0)
    model = build_model(cfg)
    q, up = LayerAddress(0, Role.Q), LayerAddress(0, Role.FF_UP)
    # exact-integer weights so f32 replies are exact regardless of accumulation order
    rng = np.random.default_rng(31)
    layers = {}
    for a in (q, up):
        p = model.layers[a]
        w = rng.integers(-2, 3, p.weight.shape).astype(np.float32)
        b = rng.integers(-2, 3, p.bias.shape).astype(np.float32)
        layers[a] = AffineParams(w, b)
    ex = BaseExecutor(layers)
    def pay(t, w):
        return rng.integers(-3, 4, (t, w)).astype(np.float32)
    reqs = [
        Envelope(1, 1, 0, int(Role.Q), PASS_FORWARD, pay(5, 16)),
        Envelope(2, 1, 0, int(Role.Q), PASS_FORWARD, pay(3, 16)),
        Envelope(1, 2, 0, int(Role.FF_UP), PASS_FORWARD, pay(4, 16)),
        Envelope(3, 7, 0, int(Role.Q), 9, pay(1, 16)),               # unknown pass
        Envelope(2, 1, 0, int(Role.Q), PASS_FORWARD, pay(2, 16)),     # request id not increasing
        Envelope(4, 1, 5, int(Role.Q), PASS_FORWARD, pay(2, 16)),     # unknown layer
        Envelope(5, 1, 0, int(Role.Q), PASS_FORWARD, pay(2, 12)),     # width mismatch
        Envelope(1, 3, 0, int(Role.FF_UP), PASS_BACKWARD, pay(6, 32)),
        Envelope(2, 2, 0, int(Role.Q), PASS_NOISE_EFFECT, pay(3, 16)),
        Envelope(6, 1, 0, int(Role.Q), PASS_FORWARD, pay(0, 16)),     # zero tokens
        Envelope(2, 3, 0, int(Role.Q), PASS_FORWARD, pay(7, 16)),
    ]
    stream = b"".join(encode(e) for e in reqs)
    # the reference server path: decode, submit (intake errors reply at once), then each
    # (layer, pass) queue in FIFO order through _compute_batch, replies wrapped per envelope
    replies = {}
    queues = {}
    buf = memoryview(stream)
    pos = 0
    order = []
    while pos < len(stream):
        env, used = try_decode(buf[pos:])
        pos += used
        order.append((env.client_id, env.request_id, env.pass_kind, len(order)))
        idx = len(order) - 1
        def reply_fn(r, idx=idx):
            replies[idx] = r
        before = len(replies)
        ex.submit(env, reply_fn)
        if len(replies) == before:   # queued, not rejected
            queues.setdefault((env.block, env.role, env.pass_kind), []).append((idx, env))
    for key, items in queues.items():
        envs = [e for _, e in items]
        res = ex._compute_batch(key[2], envs)
        for (idx, env), r in zip(items, res):
            if isinstance(r, ProtocolError):
                replies[idx] = error_envelope(env, str(r))
            else:
                replies[idx] = Envelope(env.client_id, env.request_id, env.block, env.role, env.pass_kind, r)
    out = b"".join(encode(replies[i]) for i in range(len(order)))
    d = {"requests": np.frombuffer(stream, dtype=np.uint8), "replies": np.frombuffer(out, dtype=np.uint8)}
    for a, name in ((q, "q"), (up, "up")):
        d[f"W_{name}"], d[f"b_{name}"] = layers[a].weight, layers[a].bias
    np.savez_compressed(os.path.join(HERE, "frames.npz"), **d)


if __name__ == "__main__" and len(sys.argv) > 1:
    globals()[sys.argv[1]]()
elif __name__ == "__main__":
    model_checksums()
    executor_kat()
    adapters_golden()
    fused_batch("fused_int_kat", 136, 200, seed=21, integer=True)
    fused_batch("fused_random_small", 256, 512, seed=22)
    fused_batch("fused_random_ragged", 200, 328, seed=23, rows=(1, 127, 129, 3), ranks=(24, 64))
    row_independence()
    privacy_golden()
    frames_golden()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
