"""GPU parity: the CUDA path (through the C ABI via GpuBaseExecutor) against the oracle and
the reference's golden vectors. Run on a B200: ``python -m pytest tests -m gpu``.

Tolerances (stated once, oracle/splitserve_oracle.py TOL_*): against the f32
oracle fed the same bf16-rounded inputs, normwise max|d|/max|ref| and mean|d|/mean|ref|:
bf16 activations in/out <= 2e-2 / 3e-3; fp32 outputs <= 1e-2 / 1.5e-3. fp32 outputs of exactly
representable integer inputs: bitwise. Routing: bit-exact. Batched == solo: bitwise.
"""

import threading

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O

pytestmark = pytest.mark.gpu

MAX_REL, MEAN_REL = O.TOL_MAX_REL, O.TOL_MEAN_REL


def _ex(layers, **kw):
    from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role
    return GpuBaseExecutor({LayerAddress(b, Role(r)): AffineParams(w, bias)
                            for (b, r), (w, bias) in layers.items()}, **kw)


def _env(cid, req, block, role, pass_kind, payload, **kw):
    from paper_2507_03220_b200 import Envelope
    return Envelope(cid, req, block, role, pass_kind, payload, **kw)


class _Adapter:
    """AdapterState-like record for register_adapter (adapters.py:44-60 fields)."""

    def __init__(self, lora=None, ia3=None, alpha=0.0, rank=1):
        self.lora, self.ia3, self.alpha, self.rank = lora or {}, ia3 or {}, alpha, rank


def _addr(block, role):
    from paper_2507_03220_b200 import LayerAddress, Role
    return LayerAddress(block, Role(role))


def _close(got, ref, max_rel=MAX_REL, mean_rel=MEAN_REL, what=""):
    mx, mn = O.normwise_errors(np.asarray(got, np.float64), np.asarray(ref, np.float64))
    assert mx <= max_rel and mn <= mean_rel, f"{what}: normwise max {mx:.3e} mean {mn:.3e}"


def _register_golden_adapters(ex, g, block=0, role=O.FF_UP):
    for cid in (0, 3):
        a, b = g[f"A{cid}"], g[f"B{cid}"]
        ex.register_adapter(cid, _Adapter(lora={_addr(block, role): (a, b)},
                                          alpha=float(g[f"alpha{cid}"]), rank=a.shape[1]))
    ex.register_adapter(1, _Adapter(ia3={_addr(block, role): g["l1"]}))


# ----------------------------------------------------------------------- golden: executor

def test_executor_golden_fwd_bwd_noise(golden):
    g = golden("executor_kat")
    W, b = g["W"], g["b"]
    ex = _ex({(0, O.Q): (W, b)})
    Wr, br = O.bf16_round(W), b
    fw = [_env(i + 1, 1, 0, O.Q, 0, g[f"fwd/x{i}"]) for i in range(4)]
    for i, r in enumerate(ex.serve_forward(fw)):
        assert isinstance(r, np.ndarray) and r.dtype == np.float32
        assert r.shape == g[f"fwd/y{i}"].shape
        # same bf16-rounded operands -> tight; vs the reference's un-rounded f32 -> bf16 level
        ref = O.affine_forward(O.bf16_round(g[f"fwd/x{i}"]), Wr, br)
        if r.size:
            _close(r, ref, 1e-5, 1e-5, "fwd vs oracle(bf16 inputs)")
            _close(r, g[f"fwd/y{i}"], 2e-2, 1e-2, "fwd vs reference golden")
    bw = [_env(i + 1, 2, 0, O.Q, 1, g[f"bwd/g{i}"]) for i in range(2)]
    for i, r in enumerate(ex.serve_backward(bw)):
        _close(r, O.affine_backward_input(O.bf16_round(g[f"bwd/g{i}"]), Wr), 1e-5, 1e-5, "bwd")
        _close(r, g[f"bwd/dx{i}"], 2e-2, 1e-2, "bwd vs golden")
    out = ex.serve_noise_effect(_env(1, 3, 0, O.Q, 2, g["noise/x"]))
    _close(out, O.matmul(O.bf16_round(g["noise/x"]), Wr), 1e-5, 1e-5, "noise")
    assert np.any(np.abs(out - ex.serve_forward([_env(1, 4, 0, O.Q, 0, g["noise/x"])])[0]) > 1e-3)


def test_malformed_envelope_fails_alone_same_messages(golden):
    from paper_2507_03220_b200 import ProtocolError
    g = golden("executor_kat")
    ex = _ex({(0, O.Q): (g["W"], g["b"])})
    res = ex.serve_forward([_env(1, 4, 0, O.Q, 0, g["bad/x_good"]),
                            _env(2, 4, 0, O.Q, 0, g["bad/x_bad"]),
                            _env(5, 4, 0, O.Q, 1, g["bad/x_wrong_pass"])])
    assert isinstance(res[0], np.ndarray)
    assert all(isinstance(r, ProtocolError) for r in res[1:])
    assert [str(r) for r in res[1:]] == [str(m) for m in g["bad/msgs"][1:]]


# ----------------------------------------------------------------------- golden: fused adapters

def _fused_run(ex, g, dtype, want_base=True):
    rows = [int(r) for r in g["rows"]]
    dev = ex.device
    xs = [torch.from_numpy(g[f"fwd/x{c}"]).to(dev, dtype) for c in range(len(rows))]
    d_out = g["W"].shape[1]
    outs = [torch.empty(r, d_out, dtype=dtype, device=dev) for r in rows]
    bases = [torch.empty(r, d_out, dtype=dtype, device=dev) for r in rows]
    envs = [_env(c, 1, 0, O.FF_UP, 0, xs[c], reply_to=outs[c],
                 base_to=bases[c] if (want_base and c == 1) else None) for c in range(len(rows))]
    res = ex.serve_forward(envs)
    assert all(r is outs[c] for c, r in enumerate(res))
    gs = [torch.from_numpy(g[f"bwd/g{c}"]).to(dev, dtype) for c in range(len(rows))]
    dxs = ex.serve_backward([_env(c, 2, 0, O.FF_UP, 1, gs[c]) for c in range(len(rows))])
    torch.cuda.synchronize()
    return ([o.float().cpu().numpy() for o in outs], [b.float().cpu().numpy() for b in bases],
            [d.float().cpu().numpy() for d in dxs])


def test_fused_integer_kat_bitwise(golden):
    """Exact-integer KAT: fp32 outputs equal the reference bitwise."""
    g = golden("fused_int_kat")
    ex = _ex({(0, O.FF_UP): (g["W"], g["b"])})
    _register_golden_adapters(ex, g)
    ys, bases, dxs = _fused_run(ex, g, torch.float32)
    for c in range(len(ys)):
        assert np.array_equal(ys[c], g[f"fwd/y{c}"]), f"fwd client {c}"
        assert np.array_equal(dxs[c], g[f"bwd/dx{c}"]), f"bwd client {c}"
    assert np.array_equal(bases[1], g["fwd/ybase1"])


@pytest.mark.parametrize("name", ["fused_random_small", "fused_random_ragged"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fused_random_parity(golden, name, dtype):
    g = golden(name)
    ex = _ex({(0, O.FF_UP): (g["W"], g["b"])})
    _register_golden_adapters(ex, g)
    ys, bases, dxs = _fused_run(ex, g, dtype)
    tol = (MAX_REL, MEAN_REL) if dtype == torch.bfloat16 else (O.TOL_F32_MAX_REL, O.TOL_F32_MEAN_REL)
    for c in range(len(ys)):
        _close(ys[c], g[f"fwd/y{c}"], *tol, what=f"{name} fwd client {c}")
        if c == 1:
            # IA3 backward: the GEMM operand is g*l (client.py:291-294 computes it in f32). f32
            # outputs carry it as hi + lo (second K pass): the golden at the f32 tier; bf16
            # outputs round it to bf16 once: the golden at the IA3-backward bf16 tier.
            if dtype == torch.float32:
                _close(dxs[c], g[f"bwd/dx{c}"], *tol, what="IA3 bwd (hi+lo) vs golden")
            else:
                _close(dxs[c], g[f"bwd/dx{c}"], MAX_REL, O.TOL_IA3_BWD_MEAN_REL, what="IA3 bwd vs golden")
        else:
            _close(dxs[c], g[f"bwd/dx{c}"], *tol, what=f"{name} bwd client {c}")
    _close(bases[1], g["fwd/ybase1"], *tol, what="IA3 y_base")


# ----------------------------------------------------------------------- routing & invisibility

def test_routing_bit_exact_with_identity_weight():
    """W = I, b = 0, integer rows tagging (segment, row): every output row is its own input row
    (split_rows offsets, tensor_ops.py:149-156), including around a rejected envelope."""
    from paper_2507_03220_b200 import ProtocolError
    d = 256
    ex = _ex({(0, O.Q): (np.eye(d, dtype=np.float32), np.zeros(d, np.float32))})
    rows = [1, 127, 0, 129, 5, 300, 2]
    xs = []
    for s, t in enumerate(rows):
        x = np.zeros((t, d), np.float32)
        x[:, 0] = s
        x[:, 1] = np.arange(t) % 256
        x[:, 2] = np.arange(t) // 256
        x[:, 3:] = np.random.default_rng(s).integers(-100, 100, size=(t, d - 3))
        xs.append(x)
    envs = [_env(s, 1, 0, O.Q, 0, x) for s, x in enumerate(xs)]
    envs.insert(3, _env(99, 1, 0, O.Q, 0, np.zeros((4, d - 1), np.float32)))
    res = ex.serve_forward(envs)
    assert isinstance(res[3], ProtocolError)
    for x, r in zip(xs, [r for i, r in enumerate(res) if i != 3]):
        assert np.array_equal(r, x)


def _mixed_clients(ex, d_in, d_out, seed, block=0, role=O.K):
    rng = np.random.default_rng(seed)
    specs = [("lora", 8), ("plain", 0), ("lora", 64), ("ia3", 0), ("lora", 16), ("lora", 32), ("plain", 0)]
    for cid, (kind, r) in enumerate(specs):
        if kind == "lora":
            ad = O.lora_params(seed, cid, block, role, d_in, d_out, r, 2.0 * r)
            ex.register_adapter(cid, _Adapter(lora={_addr(block, role): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
        elif kind == "ia3":
            ex.register_adapter(cid, _Adapter(ia3={_addr(block, role): O.ia3_params(seed, cid, block, role, d_out).ia3}))
    counts = [int(t) for t in rng.integers(1, 300, size=len(specs))]
    return specs, counts


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_batched_equals_solo_bitwise(dtype):
    """GPU analogue of acceptance C5 / test_executor.py:36-45: batching is invisible, bitwise,
    for every client and adapter kind, forward and backward."""
    d_in, d_out = 384, 640
    w, b = O.layer_params(3, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    specs, counts = _mixed_clients(ex, d_in, d_out, seed=5)
    dev = ex.device
    gen = torch.Generator(device=dev).manual_seed(0)
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, generator=gen, device=dev).to(dtype) for t in counts]
        batched = ex._compute_batch(pass_kind, [_env(c, 10 + pass_kind, 0, O.K, pass_kind, x) for c, x in enumerate(xs)])
        for c, x in enumerate(xs):
            solo = ex._compute_batch(pass_kind, [_env(c, 20 + pass_kind, 0, O.K, pass_kind, x)])[0]
            assert torch.equal(batched[c], solo), (pass_kind, c, specs[c])
        # and in a different batch order / company
        perm = list(reversed(range(len(xs))))
        again = ex._compute_batch(pass_kind, [_env(c, 30 + pass_kind, 0, O.K, pass_kind, xs[c]) for c in perm])
        for j, c in enumerate(perm):
            assert torch.equal(again[j], batched[c])


@pytest.mark.parametrize("shape", [("7b_q", 4096, 4096), ("13b_ff_up", 5120, 13824),
                                   ("13b_ff_down", 13824, 5120), ("13b_lm_head", 5120, 32000),
                                   # Granite-20B shape (BASELINE configs[4]): K up to 24576, V 49152
                                   ("g20_q", 6144, 6144), ("g20_ff_up", 6144, 24576),
                                   ("g20_ff_down", 24576, 6144), ("g20_lm_head", 6144, 49152)])
def test_large_layer_parity_vs_fp32(shape):
    """Llama2-7B/13B layer shapes, mixed LoRA ranks 8..64 + IA3 + plain, bf16 in/out, against
    an fp32 torch evaluation of the same math on the same bf16 operands."""
    name, d_in, d_out = shape
    role = O.FF_UP if "ff_up" in name else (O.FF_DOWN if "ff_down" in name else (O.LM_HEAD if "head" in name else O.Q))
    block = (52 if name.startswith("g20") else 40) if role == O.LM_HEAD else 0
    w, b = O.layer_params(7, block, role, d_in, d_out)
    ex = _ex({(block, role): (w, b)})
    rng = np.random.default_rng(1)
    dev = ex.device
    kinds = [("lora", 8), ("lora", 16), ("lora", 32), ("lora", 64), ("plain", 0)]
    if role in O.IA3_ROLES:
        kinds.append(("ia3", 0))
    ads = {}
    for cid, (kind, r) in enumerate(kinds):
        if kind == "lora":
            ad = O.lora_params(7, cid, block, role, d_in, d_out, r, 2.0 * r)
            ads[cid] = ad
            ex.register_adapter(cid, _Adapter(lora={_addr(block, role): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
        elif kind == "ia3":
            ad = O.ia3_params(7, cid, block, role, d_out)
            ads[cid] = ad
            ex.register_adapter(cid, _Adapter(ia3={_addr(block, role): ad.ia3}))
    counts = [int(t) for t in rng.integers(64, 700, size=len(kinds))]
    Wt = torch.from_numpy(w).to(dev).to(torch.bfloat16).float()
    bt = torch.from_numpy(b).to(dev)
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]
        res = ex._compute_batch(pass_kind, [_env(c, 1 + pass_kind, block, role, pass_kind, x) for c, x in enumerate(xs)])
        for c, (x, y) in enumerate(zip(xs, res)):
            xf = x.float()
            ad = ads.get(c)
            if pass_kind == 0:
                ref = xf @ Wt + bt
                if ad is not None and ad.a is not None:
                    A = torch.from_numpy(ad.a).to(dev).to(torch.bfloat16).float()
                    B = torch.from_numpy(ad.b).to(dev).to(torch.bfloat16).float()
                    ref = ref + ((xf @ A) @ B) * ad.scale
                if ad is not None and ad.ia3 is not None:
                    ref = ref * torch.from_numpy(ad.ia3).to(dev)
            else:
                gf = xf
                if ad is not None and ad.ia3 is not None:
                    gf = gf * torch.from_numpy(ad.ia3).to(dev)
                ref = gf @ Wt.T
                if ad is not None and ad.a is not None:
                    A = torch.from_numpy(ad.a).to(dev).to(torch.bfloat16).float()
                    B = torch.from_numpy(ad.b).to(dev).to(torch.bfloat16).float()
                    ref = ref + ((gf @ B.T) @ A.T) * ad.scale
            ia3_bwd = pass_kind == 1 and ad is not None and ad.ia3 is not None
            _close(y.float().cpu().numpy(), ref.cpu().numpy(),
                   mean_rel=O.TOL_IA3_BWD_MEAN_REL if ia3_bwd else MEAN_REL,
                   what=f"{name} pass {pass_kind} client {c}")


# ----------------------------------------------------------------------- statelessness / edges

def test_executor_retains_nothing_between_requests():
    from paper_2507_03220_b200 import ledger as L
    w, b = O.layer_params(0, 0, O.Q, 64, 64)
    ex = _ex({(0, O.Q): (w, b)})
    weights = ex.ledger.get(L.WEIGHTS)
    rng = np.random.default_rng(0)
    for i in range(5):
        ex.serve_forward([_env(1, i + 1, 0, O.Q, 0, rng.standard_normal((4, 64)).astype(np.float32))])
        ex.serve_backward([_env(2, i + 1, 0, O.Q, 1, rng.standard_normal((4, 64)).astype(np.float32))])
    assert ex.ledger.get(L.SAVED_ACTIVATIONS) == 0
    assert ex.ledger.get(L.TRANSIENT_BUFFER) == 0
    assert ex.ledger.get(L.WEIGHTS) == weights > 0
    assert ex.ledger.transient_high_water > 0


def test_save_activations_negative_control():
    from paper_2507_03220_b200 import ledger as L
    w, b = O.layer_params(0, 0, O.Q, 64, 64)
    ex = _ex({(0, O.Q): (w, b)}, save_activations=True)
    x = np.ones((4, 64), np.float32)
    ex.serve_forward([_env(1, 1, 0, O.Q, 0, x)])
    first = ex.ledger.get(L.SAVED_ACTIVATIONS)
    ex.serve_forward([_env(1, 2, 0, O.Q, 0, x)])
    assert first > 0 and ex.ledger.get(L.SAVED_ACTIVATIONS) == 2 * first


def test_edge_cases_empty_and_zero_rows():
    w, b = O.layer_params(0, 0, O.Q, 64, 96)
    ex = _ex({(0, O.Q): (w, b)})
    assert ex.serve_forward([]) == []
    res = ex.serve_forward([_env(1, 1, 0, O.Q, 0, np.zeros((0, 64), np.float32)),
                            _env(2, 1, 0, O.Q, 0, np.ones((3, 64), np.float32))])
    assert res[0].shape == (0, 96) and res[1].shape == (3, 96)
    res = ex.serve_backward([_env(3, 1, 0, O.Q, 1, np.zeros((0, 96), np.float32))])
    assert res[0].shape == (0, 64)


def test_large_batch_many_small_segments():
    """Decode-like dispatch: 200 clients x 1-3 tokens, all with LoRA (many rank blocks per tile)."""
    d = 512
    w, b = O.layer_params(1, 0, O.V, d, d)
    ex = _ex({(0, O.V): (w, b)})
    n = 200
    rng = np.random.default_rng(3)
    for cid in range(n):
        r = [8, 16, 32, 64][cid % 4]
        ad = O.lora_params(1, cid, 0, O.V, d, d, r, 2.0 * r)
        ex.register_adapter(cid, _Adapter(lora={_addr(0, O.V): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
    xs = [O.bf16_round(rng.standard_normal((int(rng.integers(1, 4)), d)).astype(np.float32)) for _ in range(n)]
    res = ex.serve_forward([_env(c, 1, 0, O.V, 0, x) for c, x in enumerate(xs)])
    wr, br = O.bf16_round(w), b
    for c, (x, y) in enumerate(zip(xs, res)):
        r = [8, 16, 32, 64][c % 4]
        ad = O.lora_params(1, c, 0, O.V, d, d, r, 2.0 * r)
        ref = O.apply_adapter(O.OracleAdapter(a=O.bf16_round(ad.a), b=O.bf16_round(ad.b), alpha=ad.alpha, rank=r),
                              x, O.affine_forward(x, wr, br))
        _close(y, ref, what=f"client {c}")


def test_adapter_refresh_and_rank_change():
    d_in, d_out = 256, 256
    w, b = O.layer_params(2, 0, O.O, d_in, d_out)
    ex = _ex({(0, O.O): (w, b)})
    x = O.bf16_round(np.random.default_rng(0).standard_normal((50, d_in)).astype(np.float32))
    base = O.affine_forward(x, O.bf16_round(w), b)
    for step, r in enumerate([8, 8, 32, 16]):
        ad = O.lora_params(10 + step, 0, 0, O.O, d_in, d_out, r, 2.0 * r)
        ad = O.OracleAdapter(a=O.bf16_round(ad.a), b=O.bf16_round(ad.b), alpha=ad.alpha, rank=r)
        ex.refresh_adapter(0, _Adapter(lora={_addr(0, O.O): (ad.a, ad.b)}, alpha=ad.alpha, rank=r))
        y = ex.serve_forward([_env(0, step + 1, 0, O.O, 0, x)])[0]
        _close(y, O.apply_adapter(ad, x, base), what=f"refresh {step}")
    ex.deregister_adapter(0)
    y = ex.serve_forward([_env(0, 9, 0, O.O, 0, x)])[0]
    _close(y, base, 1e-5, 1e-5, "after deregister_adapter")


# ----------------------------------------------------------------------- channel / scheduler

def test_device_channel_virtlayer_roundtrip():
    from paper_2507_03220_b200 import DeviceChannel, VirtLayer
    d_in, d_out = 256, 512
    w, b = O.layer_params(4, 0, O.FF_UP, d_in, d_out)
    ex = _ex({(0, O.FF_UP): (w, b)})
    with ex:
        ch = DeviceChannel(ex, 7, batch_size=2, seq_len=16, max_width=512)
        ch.register(sends_backward=True)
        layer = VirtLayer(_addr(0, O.FF_UP), d_in, d_out, ch)
        x = torch.randn(32, d_in, device=ex.device).to(torch.bfloat16)
        y = layer.forward(x)
        g = torch.randn(32, d_out, device=ex.device).to(torch.bfloat16)
        dx = layer.backward(g)
    ref_y = ex._compute_batch(0, [_env(7, 100, 0, O.FF_UP, 0, x)])[0]
    ref_dx = ex._compute_batch(1, [_env(7, 101, 0, O.FF_UP, 1, g)])[0]
    assert torch.equal(y, ref_y) and torch.equal(dx, ref_dx)
    assert ch.buffer.resizes == 0


def test_lockstep_eight_clients_one_batch_over_device_channels():
    from paper_2507_03220_b200 import BatchPolicy, DeviceChannel
    w, b = O.layer_params(5, 0, O.Q, 128, 128)
    ex = _ex({(0, O.Q): (w, b)}, policy=BatchPolicy(mode="lockstep"))
    results = {}
    with ex:
        chans = [DeviceChannel(ex, c, 1, 8, 128) for c in range(8)]
        for ch in chans:
            ch.register()
        xs = [torch.randn(4, 128, device=ex.device).to(torch.bfloat16) for _ in range(8)]

        def one(c):
            torch.cuda.set_device(ex.device)
            results[c] = chans[c].request(0, O.Q, 0, xs[c]).clone()

        ts = [threading.Thread(target=one, args=(c,)) for c in range(8)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(30)
    assert ex.metrics.mean_batch_size() == 8.0
    torch.cuda.synchronize()
    for c in range(8):
        solo = ex._compute_batch(0, [_env(c, 50, 0, O.Q, 0, xs[c])])[0]
        assert torch.equal(results[c], solo)


def test_submit_rejections_match_reference_messages():
    from paper_2507_03220_b200 import PASS_ERROR, error_message
    w, b = O.layer_params(0, 0, O.Q, 64, 64)
    ex = _ex({(0, O.Q): (w, b)})
    got = []
    with ex:
        ex.register(1)
        done = threading.Event()

        def reply(e):
            got.append(e)
            done.set()
        x = np.ones((2, 64), np.float32)
        ex.submit(_env(1, 5, 0, O.Q, 0, x), reply)
        assert done.wait(10)
        done.clear()
        ex.submit(_env(1, 5, 0, O.Q, 0, x), reply)
        assert done.wait(10)
        done.clear()
        ex.submit(_env(1, 6, 3, O.Q, 0, x), reply)
        assert done.wait(10)
    assert got[0].pass_kind == 0
    assert got[1].pass_kind == PASS_ERROR and "not increasing" in error_message(got[1])
    assert got[2].pass_kind == PASS_ERROR and "unknown layer" in error_message(got[2])


@pytest.mark.parametrize("zero_copy", [0, 1 << 30])
def test_pipelined_host_dispatch_bitwise_equals_device_dispatch(zero_copy):
    """Pinned-host clients take the pipelined path (row sub-batches, H2D/GEMM/D2H overlapped)
    or, for small dispatches, the zero-copy path (kernels read / write the pinned host rows
    directly); either result must be bitwise the device-resident single-batch result."""
    d_in, d_out = 512, 768
    w, b = O.layer_params(6, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ex.ctx.set_option("zero_copy_bytes", zero_copy)
    ex.pipeline_rows = 200   # force several sub-batches and ring reuse
    specs, counts = _mixed_clients(ex, d_in, d_out, seed=9, role=O.V)
    for pass_kind, (wi, wo) in ((0, (d_in, d_out)), (1, (d_out, d_in))):
        hosts = [torch.randn(t, wi).to(torch.bfloat16).pin_memory() for t in counts]
        replies = [torch.empty(t, wo, dtype=torch.bfloat16).pin_memory() for t in counts]
        res = ex._compute_batch(pass_kind, [_env(c, 40 + pass_kind, 0, O.V, pass_kind, h, reply_to=r)
                                            for c, (h, r) in enumerate(zip(hosts, replies))])
        assert all(r is replies[c] for c, r in enumerate(res))
        dev = ex._compute_batch(pass_kind, [_env(c, 50 + pass_kind, 0, O.V, pass_kind, h.to(ex.device))
                                            for c, h in enumerate(hosts)])
        for c in range(len(counts)):
            assert torch.equal(replies[c], dev[c].cpu()), (pass_kind, c)


@pytest.mark.parametrize("shape", [(384, 640), (13824, 512)])   # pair kernel / single-CTA kernel
def test_direct_tiles_bitwise_equal_packed_path(shape):
    """Segment-aligned tiles TMA-loaded in place from the client buffers must give exactly the
    rows the gather -> packed-operand path gives (block-diagonal LoRA adds exact zeros)."""
    d_in, d_out = shape
    w, b = O.layer_params(8, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    specs, _ = _mixed_clients(ex, d_in, d_out, seed=11)
    counts = [512, 300, 1, 256, 700, 129, 1024][: len(specs)]
    dev = ex.device
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]
        xs[1] = xs[1].float()   # an f32 source always takes the packed path
        outs = {}
        for direct in (1, 0):
            ex.ctx.set_option("direct_tiles", direct)
            outs[direct] = ex._compute_batch(pass_kind, [_env(c, 60 + 2 * pass_kind + direct, 0, O.K, pass_kind, x)
                                                         for c, x in enumerate(xs)])
        ex.ctx.set_option("direct_tiles", 1)
        for c in range(len(xs)):
            assert torch.equal(outs[1][c], outs[0][c]), (pass_kind, c, counts[c])


@pytest.mark.parametrize("world", [2, 4])
def test_tensor_parallel_shards_through_cuda_path(world):
    """Every TP rank's shard runs through the real C-ABI path (strided column views in, local
    outputs); the collective is emulated in-process. Column-split forward / row-split backward
    (all-gather) must equal the single-GPU executor bitwise; the all-reduce kinds (fp32 partial
    sums) within the fp32-output tier."""
    from paper_2507_03220_b200.tp import TensorParallelExecutor, combine_local
    d, f, v = 512, 768, 1024
    roles = [(O.Q, d, d), (O.O, d, d), (O.FF_UP, d, f), (O.FF_DOWN, f, d), (O.LM_HEAD, d, v), (O.K, d, d)]
    layers = {}
    for role, di, do in roles:
        blk = 1 if role == O.LM_HEAD else 0
        layers[(blk, role)] = O.layer_params(12, blk, role, di, do)
    full = _ex(layers)
    ranks = [TensorParallelExecutor({_addr(b, r): _params(w, bb) for (b, r), (w, bb) in layers.items()},
                                    rk, world) for rk in range(world)]
    ads = {}
    for cid, (kind, r) in enumerate([("lora", 16), ("ia3", 0), ("plain", 0), ("lora", 64)]):
        if kind == "lora":
            lo = {}
            for role, di, do in roles:
                blk = 1 if role == O.LM_HEAD else 0
                ad = O.lora_params(3, cid, blk, role, di, do, r, 2.0 * r)
                lo[_addr(blk, role)] = (ad.a, ad.b)
            ads[cid] = _Adapter(lora=lo, alpha=2.0 * r, rank=r)
        elif kind == "ia3":
            ads[cid] = _Adapter(ia3={_addr(0, role): O.ia3_params(3, cid, 0, role, do).ia3
                                     for role, di, do in roles if role in O.IA3_ROLES})
    for cid, ad in ads.items():
        full.register_adapter(cid, ad)
        for rk in ranks:
            rk.register_adapter(cid, ad)
    counts = [300, 64, 513, 256]
    for role, di, do in roles:
        blk = 1 if role == O.LM_HEAD else 0
        for pass_kind, width in ((0, di), (1, do)):
            xs = [torch.randn(t, width, device=full.device).to(torch.bfloat16) for t in counts]
            ref = full._compute_batch(pass_kind, [_env(c, 900 + pass_kind, blk, role, pass_kind, x)
                                                  for c, x in enumerate(xs)])
            parts = [rk.dispatch_local(pass_kind, blk, role, xs, list(range(len(xs)))) for rk in ranks]
            combined = combine_local([(s, loc) for s, loc, _ in parts], pass_kind)
            got = combined.to(torch.bfloat16)
            pos = 0
            for c, t in enumerate(counts):
                g, rf = got[pos:pos + t], ref[c]
                pos += t
                if parts[0][0].collective(pass_kind) == "all_gather":
                    assert torch.equal(g, rf), (role, pass_kind, c)
                else:
                    _close(g.float().cpu().numpy(), rf.float().cpu().numpy(), MAX_REL, MEAN_REL,
                           what=f"TP{world} {role} pass {pass_kind} client {c}")


def _params(w, b):
    from paper_2507_03220_b200 import AffineParams
    return AffineParams(w, b)


@pytest.mark.parametrize("shape", [(512, 1280), (5120, 1536)])
def test_every_kernel_and_tile_width_gives_identical_rows(shape):
    """The dispatch picks the CTA-pair kernel or the single-CTA kernel with 256/128/64-wide tiles
    from the dispatch size; all of them must produce bitwise the same rows (the per-element K
    order is the same), otherwise batching would become visible (acceptance C5)."""
    d_in, d_out = shape
    w, b = O.layer_params(13, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    _mixed_clients(ex, d_in, d_out, seed=13)
    counts = [700, 256, 3, 129, 512, 64, 1]
    dev = ex.device
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]
        outs = []
        for pair, tn, pn, c4 in ((1, 0, 256, 0), (1, 0, 512, 0), (1, 0, 256, 1), (0, 256, 256, 0),
                                 (0, 128, 256, 0), (0, 64, 256, 0)):
            ex.ctx.set_option("gemm_2cta", pair)
            ex.ctx.set_option("tile_n", tn)
            ex.ctx.set_option("pair_n", pn)
            ex.ctx.set_option("cluster4", c4)
            outs.append(ex._compute_batch(pass_kind, [_env(c, 70 + 10 * pass_kind + len(outs), 0, O.K, pass_kind, x)
                                                      for c, x in enumerate(xs)]))
        ex.ctx.set_option("gemm_2cta", -1)
        ex.ctx.set_option("tile_n", 0)
        ex.ctx.set_option("pair_n", 0)
        ex.ctx.set_option("cluster4", 0)
        for k in range(1, len(outs)):
            for c in range(len(xs)):
                assert torch.equal(outs[0][c], outs[k][c]), (pass_kind, k, c)


@pytest.mark.parametrize("pair", [1, 0])
def test_tma_store_epilogue_bitwise_equals_direct_stores(pair):
    """bf16 outputs leave through swizzled smem + TMA bulk stores (clipped per destination
    segment) or through per-thread global stores; both must write identical bytes, including
    packed tiles shared by several clients and partial last tiles."""
    d_in, d_out = 512, 1088
    w, b = O.layer_params(14, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    _mixed_clients(ex, d_in, d_out, seed=14, role=O.V)
    counts = [300, 1, 700, 130, 5, 256, 77]
    ex.ctx.set_option("gemm_2cta", pair)
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=ex.device).to(torch.bfloat16) for t in counts]
        outs = []
        for ts in (1, 0):
            ex.ctx.set_option("tma_store", ts)
            outs.append(ex._compute_batch(pass_kind, [_env(c, 80 + 4 * pass_kind + 2 * ts, 0, O.V, pass_kind, x)
                                                      for c, x in enumerate(xs)]))
        for c in range(len(xs)):
            assert torch.equal(outs[0][c], outs[1][c]), (pass_kind, c)
    ex.ctx.set_option("tma_store", 1)
    ex.ctx.set_option("gemm_2cta", -1)


@pytest.mark.parametrize("d_in", [5120, 13824])
def test_shrink_whole_and_split_modes_bitwise_equal(d_in):
    """The LoRA shrink splits K into fixed chunks (kernels.cuh SHRINK_KB_CHUNK) and sums the chunk
    partials in chunk order — either in one CTA per slab (large dispatches) or across CTAs via
    the workspace (decode-size dispatches). Both must give the same bits, and a decode-size
    client must get the same rows alone as inside a prefill-size dispatch."""
    d_out = 512
    w, b = O.layer_params(15, 0, O.Q, d_in, d_out)
    ex = _ex({(0, O.Q): (w, b)})
    _mixed_clients(ex, d_in, d_out, seed=15, role=O.Q)
    counts = [2, 1, 2000, 3, 700, 1, 2]      # decode-size LoRA clients next to prefill-size ones
    xs = [torch.randn(t, d_in, device=ex.device).to(torch.bfloat16) for t in counts]
    outs = {}
    for mode in (1, 2):
        ex.ctx.set_option("shrink_mode", mode)
        outs[mode] = ex._compute_batch(0, [_env(c, 80 + mode, 0, O.Q, 0, x) for c, x in enumerate(xs)])
    ex.ctx.set_option("shrink_mode", 0)
    for c in range(len(xs)):
        assert torch.equal(outs[1][c], outs[2][c]), c
    big = ex._compute_batch(0, [_env(c, 90, 0, O.Q, 0, x) for c, x in enumerate(xs)])
    for c in (0, 2):                         # LoRA r8 (decode rows) and LoRA r64 (prefill rows)
        solo = ex._compute_batch(0, [_env(c, 91 + c, 0, O.Q, 0, xs[c])])[0]
        assert torch.equal(solo, big[c]), c


def test_peer_gpu_routing_bitwise_equals_local():
    """Segments whose buffers live on another GPU (clients reached over
    NVLink) are gathered with plain loads and written with plain stores, never through TMA
    tensor maps. `force_remote` routes every segment that way on one GPU: the rows (and the
    IA3 client's pre-IA3 y_base) must be bitwise those of the local path."""
    d_in, d_out = 512, 1088
    w, b = O.layer_params(16, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    _mixed_clients(ex, d_in, d_out, seed=16, role=O.V)
    counts = [300, 1, 700, 130, 5, 256, 77]
    dev = ex.device
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]
        outs, bases = {}, {}
        for remote in (0, 1):
            ex.ctx.set_option("force_remote", remote)
            bs = [torch.full((t, d_out), 7.0, dtype=torch.bfloat16, device=dev) for t in counts]
            envs = [_env(c, 100 + 2 * pass_kind + remote, 0, O.V, pass_kind, x,
                         base_to=bs[c] if (pass_kind == 0 and c == 3) else None) for c, x in enumerate(xs)]
            outs[remote] = ex._compute_batch(pass_kind, envs)
            bases[remote] = bs[3]
        ex.ctx.set_option("force_remote", 0)
        for c in range(len(xs)):
            assert torch.equal(outs[0][c], outs[1][c]), (pass_kind, c)
        if pass_kind == 0:
            assert torch.equal(bases[0], bases[1])


@pytest.mark.parametrize("decode_rows", [16, 0])
def test_decode_size_dispatch_64_row_box_bitwise(decode_rows):
    """A dispatch of <= 64 packed rows runs the weight-streaming kernel (4 k-blocks of A and W
    per TMA operation, 64-row A boxes whose MMA rows 64-127 are never stored) or, with it off,
    the single-CTA kernel with a 64- or 128-row A box; the streaming kernel either overlaps the
    side-stream LoRA shrink (waiting on its completion counter) or starts after it, and is
    launched early behind the gather (W streaming before griddepcontrol.wait) or not. All must
    give the same bits, equal to
    the same clients' rows inside a prefill-size dispatch (batching invisibility at decode
    sizes), forward and backward, every adapter kind."""
    d_in, d_out = 5120, 1024
    w, b = O.layer_params(17, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    ex.ctx.set_option("decode_rows", decode_rows)   # 0: these rows take the single-chain kernels
    _mixed_clients(ex, d_in, d_out, seed=17)
    counts = [2, 2, 1, 2, 2, 3, 2]                      # 14 decode rows, every adapter kind
    dev = ex.device
    for pass_kind, width in ((0, d_in), (1, d_out)):
        xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]
        outs = []
        for stream, box64, overlap, pdl in ((1, 1, 1, 1), (1, 1, 0, 1), (1, 1, 1, 0), (0, 1, 1, 1), (0, 0, 1, 1)):
            ex.ctx.set_option("stream_gemm", stream)
            ex.ctx.set_option("a_rows64", box64)
            ex.ctx.set_option("lora_overlap", overlap)
            ex.ctx.set_option("stream_pdl", pdl)
            outs.append(ex._compute_batch(pass_kind, [_env(c, 110 + 4 * pass_kind + len(outs), 0, O.K, pass_kind, x)
                                                      for c, x in enumerate(xs)]))
        ex.ctx.set_option("stream_gemm", 1)
        ex.ctx.set_option("a_rows64", 1)
        filler = torch.randn(3000, width, device=dev).to(torch.bfloat16)
        big = ex._compute_batch(pass_kind, [_env(c, 120 + pass_kind, 0, O.K, pass_kind, x) for c, x in enumerate(xs)] +
                                [_env(1, 122 + pass_kind, 0, O.K, pass_kind, filler)])
        for c in range(len(xs)):
            for k in (1, 2, 3, 4):
                assert torch.equal(outs[0][c], outs[k][c]), (pass_kind, k, c)
            assert torch.equal(outs[0][c], big[c]), (pass_kind, c)


@pytest.mark.parametrize("decode_rows", [16, 0])
def test_decode_wide_layer_128_tiles_bitwise(decode_rows):
    """A decode-size dispatch over a layer whose 64-wide tiles would need more than one wave
    (N = 10240: 160 tiles on 148 SMs) runs 128-wide single-CTA tiles instead of the streaming
    kernel; rows must be bitwise those of the streaming kernel and of a prefill-size dispatch."""
    d_in, d_out = 512, 10240
    w, b = O.layer_params(23, 0, O.FF_UP, d_in, d_out)
    ex = _ex({(0, O.FF_UP): (w, b)})
    ex.ctx.set_option("decode_rows", decode_rows)
    rng = np.random.default_rng(23)
    ex.register_adapter(3, _Adapter(ia3={_addr(0, O.FF_UP): O.ia3_params(23, 3, 0, O.FF_UP, d_out).ia3}))
    counts = [2, 1, 2, 2]
    dev = ex.device
    xs = [torch.from_numpy(rng.standard_normal((t, d_in), dtype=np.float32)).to(dev).to(torch.bfloat16) for t in counts]
    outs = []
    for wide in (1, 0):
        ex.ctx.set_option("wide_decode", wide)
        outs.append(ex._compute_batch(0, [_env(c, 10 + wide * 10 + c, 0, O.FF_UP, 0, x) for c, x in enumerate(xs)]))
    ex.ctx.set_option("wide_decode", 1)
    filler = torch.randn(700, d_in, device=dev).to(torch.bfloat16)
    big = ex._compute_batch(0, [_env(c, 40 + c, 0, O.FF_UP, 0, x) for c, x in enumerate(xs)] +
                            [_env(9, 50, 0, O.FF_UP, 0, filler)])
    for c in range(len(xs)):
        assert torch.equal(outs[0][c], outs[1][c]), c
        assert torch.equal(outs[0][c], big[c]), c


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (client buffers on a peer GPU)")
def test_client_buffers_on_peer_gpu():
    """the executor on cuda:0 serves a client whose exchange buffers live on
    cuda:1 (NVLink peer loads / stores); rows must equal the co-located client's."""
    from paper_2507_03220_b200.channel import enable_peer_access
    assert enable_peer_access(0, 1)
    d_in, d_out = 512, 1088
    w, b = O.layer_params(18, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)}, device=0)
    _mixed_clients(ex, d_in, d_out, seed=18, role=O.V)
    counts = [300, 1, 700, 130, 5, 256, 77]
    xs = [torch.randn(t, d_in, device="cuda:0").to(torch.bfloat16) for t in counts]
    local = ex._compute_batch(0, [_env(c, 130, 0, O.V, 0, x) for c, x in enumerate(xs)])
    xr = [x.to("cuda:1") for x in xs]
    outr = [torch.empty(t, d_out, dtype=torch.bfloat16, device="cuda:1") for t in counts]
    torch.cuda.synchronize(1)
    ex._compute_batch(0, [_env(c, 131, 0, O.V, 0, x, reply_to=outr[c]) for c, x in enumerate(xr)])
    torch.cuda.synchronize(0)
    for c in range(len(xs)):
        assert torch.equal(local[c], outr[c].to("cuda:0")), c


@pytest.mark.parametrize("dims", [(1024, 2048), (2048, 1024), (1536, 1536)])
def test_in_place_device_handoff_bitwise(dims):
    """The reference hands the reply back in the request's own buffer (SharedBuffer,
    transport.py:76-97). With the reply written over the request rows of a multi-wave dispatch,
    every row must still equal the separate-buffer result (aliased sources are gathered
    before the GEMM writes)."""
    d_in, d_out = dims
    w, b = O.layer_params(19, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    _mixed_clients(ex, d_in, d_out, seed=19, role=O.V)
    counts = [3000, 1, 2500, 130, 5, 2048, 77]
    dev = ex.device
    for pass_kind, (wi, wo) in ((0, (d_in, d_out)), (1, (d_out, d_in))):
        xs = [torch.randn(t, wi, device=dev).to(torch.bfloat16) for t in counts]
        ref = ex._compute_batch(pass_kind, [_env(c, 140 + pass_kind, 0, O.V, pass_kind, x) for c, x in enumerate(xs)])
        bufs = [torch.empty(t * max(wi, wo), dtype=torch.bfloat16, device=dev) for t in counts]
        for x, buf in zip(xs, bufs):
            buf[: x.numel()].copy_(x.reshape(-1))
        got = ex._compute_batch(pass_kind, [_env(c, 150 + pass_kind, 0, O.V, pass_kind, bufs[c][: t * wi].view(t, wi),
                                                 reply_to=bufs[c][: t * wo].view(t, wo))
                                            for c, t in enumerate(counts)])
        for c in range(len(counts)):
            assert torch.equal(got[c], ref[c]), (pass_kind, c)


@pytest.mark.parametrize("zero_copy", [0, 1 << 30])
def test_in_place_host_handoff_bitwise(zero_copy):
    """Pinned-host clients whose reply buffer IS the request buffer (the reference's in-place
    hand-off) through the pipelined host path: a sub-batch's reply must never land on request
    rows a later sub-batch has not uploaded yet."""
    d_in, d_out = 512, 1408
    w, b = O.layer_params(20, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ex.pipeline_rows = 128   # many sub-batches
    ex.ctx.set_option("zero_copy_bytes", zero_copy)
    _mixed_clients(ex, d_in, d_out, seed=20, role=O.V)
    counts = [900, 1, 700, 130, 5, 1024, 77]
    for pass_kind, (wi, wo) in ((0, (d_in, d_out)), (1, (d_out, d_in))):
        xs = [torch.randn(t, wi).to(torch.bfloat16) for t in counts]
        dev = ex._compute_batch(pass_kind, [_env(c, 160 + pass_kind, 0, O.V, pass_kind, x.to(ex.device))
                                            for c, x in enumerate(xs)])
        bufs = [torch.empty(t * max(wi, wo), dtype=torch.bfloat16).pin_memory() for t in counts]
        for x, buf in zip(xs, bufs):
            buf[: x.numel()].copy_(x.reshape(-1))
        got = ex._compute_batch(pass_kind, [_env(c, 170 + pass_kind, 0, O.V, pass_kind, bufs[c][: t * wi].view(t, wi),
                                                 reply_to=bufs[c][: t * wo].view(t, wo))
                                            for c, t in enumerate(counts)])
        for c in range(len(counts)):
            assert torch.equal(got[c], dev[c].cpu()), (pass_kind, c)


def test_zero_copy_dispatch_cache_follows_data_and_adapters():
    """A zero-copy host dispatch that recurs (same client buffers and rows, as in decode) reuses
    its packed segment table (executor memo) and its routing tables (library dispatch cache);
    it must still read each call's new request rows, follow an adapter refresh (new values,
    new rank) and a client gaining an adapter, and equal the uncached result bitwise."""
    d_in, d_out = 512, 768
    w, b = O.layer_params(8, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ex.ctx.set_option("zero_copy_bytes", 1 << 30)
    _mixed_clients(ex, d_in, d_out, seed=8, role=O.V)
    counts = [2, 1, 2, 2, 3, 2, 1]
    hosts = [torch.empty(t, d_in, dtype=torch.bfloat16).pin_memory() for t in counts]
    replies = [torch.empty(t, d_out, dtype=torch.bfloat16).pin_memory() for t in counts]
    gen = torch.Generator().manual_seed(3)
    rid = [300]

    def run():
        out = []
        for cache in (1, 0):
            ex.ctx.set_option("zc_cache", cache)
            for _ in range(2):                        # the second call of each is a cache hit
                rid[0] += 1
                ex._compute_batch(0, [_env(c, rid[0], 0, O.V, 0, h, reply_to=r)
                                      for c, (h, r) in enumerate(zip(hosts, replies))])
            out.append([r.clone() for r in replies])
        for c in range(len(counts)):
            assert torch.equal(out[0][c], out[1][c]), c
        return out[0]

    ex.ctx.set_option("zc_cache", 1)
    seen = []
    for step in range(3):
        for h in hosts:
            h.copy_(torch.randn(h.shape, generator=gen).to(torch.bfloat16))
        if step == 2:     # refresh client 0's LoRA (new values and rank); client 1 gains an IA3
            ad = O.lora_params(99, 0, 0, O.V, d_in, d_out, 32, 64.0)
            ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad.a, ad.b)}, alpha=64.0, rank=32))
            ex.register_adapter(1, _Adapter(ia3={_addr(0, O.V): O.ia3_params(99, 1, 0, O.V, d_out).ia3}))
        got = run()
        dev = ex._compute_batch(0, [_env(c, 900 + 10 * step + c, 0, O.V, 0, h.to(ex.device))
                                    for c, h in enumerate(hosts)])
        for c in range(len(counts)):
            assert torch.equal(got[c], dev[c].cpu()), (step, c)
        seen.append(got[0])
    assert not torch.equal(seen[0], seen[1])
    assert len(ex._host_memo) >= 1


@pytest.mark.parametrize("zero_copy", [0, 1 << 30])
def test_host_dispatch_rejected_segment_untouched(zero_copy):
    """ss_compute_batch_host (both the pipelined and the zero-copy path): a segment the library
    rejects (wrong width) gets a nonzero status and its host reply buffer is not written; the
    other segments' replies equal the device path bitwise (executor.py:192-215: a malformed
    envelope fails alone)."""
    from paper_2507_03220_b200 import _lib
    from paper_2507_03220_b200.device import Seg
    d_in, d_out = 512, 768
    w, b = O.layer_params(21, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ex.ctx.set_option("zero_copy_bytes", zero_copy)
    _mixed_clients(ex, d_in, d_out, seed=21, role=O.V)
    counts = [300, 2, 129, 64]
    xs = [torch.randn(t, d_in).to(torch.bfloat16).pin_memory() for t in counts]
    xs[2] = torch.randn(counts[2], d_in + 64).to(torch.bfloat16).pin_memory()   # malformed width
    outs = [torch.full((t, d_out), 3.0, dtype=torch.bfloat16).pin_memory() for t in counts]
    segs = [Seg(c, x, o, adapter=(0, O.V) in ex._fused.get(c, ())) for c, (x, o) in enumerate(zip(xs, outs))]
    status = ex.ctx.compute_host(0, 0, O.V, segs)
    assert status[2] == _lib.SS_SEG_BAD_WIDTH and [status[i] for i in (0, 1, 3)] == [0, 0, 0]
    assert torch.equal(outs[2], torch.full((counts[2], d_out), 3.0, dtype=torch.bfloat16))
    dev = ex._compute_batch(0, [_env(c, 200 + c, 0, O.V, 0, xs[c].to(ex.device)) for c in (0, 1, 3)])
    for j, c in enumerate((0, 1, 3)):
        assert torch.equal(outs[c], dev[j].cpu()), c


def test_full_size_batched_equals_solo_13b_ff_up():
    """BASELINE configs[2] size: a 13B FF_UP forward over 32 clients x 1024 rows (M = 32768,
    the 256x512 CTA-pair kernel) against three of the clients alone (1024 rows: the 256x256
    pair kernel) — a size-independent property (batching invisibility, acceptance C5), bitwise,
    with LoRA r8 / r64 and IA3 y_base outputs."""
    d_in, d_out = 5120, 13824
    w, b = O.layer_params(30, 0, O.FF_UP, d_in, d_out)
    ex = _ex({(0, O.FF_UP): (w, b)})
    for cid, r in ((0, 8), (1, 64)):
        ad = O.lora_params(30, cid, 0, O.FF_UP, d_in, d_out, r, 2.0 * r)
        ex.register_adapter(cid, _Adapter(lora={_addr(0, O.FF_UP): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
    ex.register_adapter(2, _Adapter(ia3={_addr(0, O.FF_UP): O.ia3_params(30, 2, 0, O.FF_UP, d_out).ia3}))
    dev = ex.device
    gen = torch.Generator(device=dev).manual_seed(30)
    xs = [torch.randn(1024, d_in, generator=gen, device=dev).to(torch.bfloat16) for _ in range(32)]
    base_b = torch.empty(1024, d_out, dtype=torch.bfloat16, device=dev)
    batched = ex._compute_batch(0, [_env(c, 1, 0, O.FF_UP, 0, x, base_to=base_b if c == 2 else None)
                                    for c, x in enumerate(xs)])
    base_batched = base_b.clone()
    for c in (0, 1, 2):
        base_s = torch.empty(1024, d_out, dtype=torch.bfloat16, device=dev)
        solo = ex._compute_batch(0, [_env(c, 2 + c, 0, O.FF_UP, 0, xs[c], base_to=base_s if c == 2 else None)])[0]
        assert torch.equal(solo, batched[c]), c
        if c == 2:
            assert torch.equal(base_s, base_batched)


@pytest.mark.parametrize("pass_kind,role,d_in,d_out", [(0, O.K, 5120, 5120), (1, O.K, 5120, 5120),
                                                       (1, O.FF_DOWN, 13824, 5120)])
def test_tail_split_bitwise(pass_kind, role, d_in, d_out):
    """tail_split: a 13B K-projection forward of 32 clients x 1024 rows (1280 tiles of 256 x 512
    = 17 waves of 74 CTA pairs + 22: the last 96 raster tiles run as 192 tiles of 256 x 256 in a
    second launch), its backward at 16 x 1024 rows (640 tiles: not split) and an FF_DOWN backward
    (N = 13824: 1728 tiles, 23 waves + 26: split, backward kernels) give the same bits as one
    256 x 512 launch, and as a client alone; LoRA r16 / r64 and IA3 (forward: with y_base)."""
    w, b = O.layer_params(31, 0, role, d_in, d_out)
    ex = _ex({(0, role): (w, b)})
    for cid, r in ((0, 16), (5, 64)):
        ad = O.lora_params(31, cid, 0, role, d_in, d_out, r, 2.0 * r)
        ex.register_adapter(cid, _Adapter(lora={_addr(0, role): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
    if role in O.IA3_ROLES:
        ex.register_adapter(2, _Adapter(ia3={_addr(0, role): O.ia3_params(31, 2, 0, role, d_out).ia3}))
    dev = ex.device
    gen = torch.Generator(device=dev).manual_seed(31)
    n = 32 if pass_kind == 0 else 16
    width = d_out if pass_kind == 1 else d_in
    xs = [torch.randn(1024, width, generator=gen, device=dev).to(torch.bfloat16) for _ in range(n)]
    base = {}

    def run(rid, idx):
        envs = []
        for c in idx:
            kw = {}
            if c == 2 and pass_kind == 0 and role in O.IA3_ROLES:
                base[rid] = torch.empty(1024, d_out, dtype=torch.bfloat16, device=dev)
                kw["base_to"] = base[rid]
            envs.append(_env(c, rid, 0, role, pass_kind, xs[c], **kw))
        return ex._compute_batch(pass_kind, envs)

    ex.ctx.set_option("tail_split", 0)
    ref = run(1, range(n))
    ex.ctx.set_option("tail_split", 1)
    got = run(2, range(n))
    for c in range(n):
        assert torch.equal(got[c], ref[c]), c
    if base:
        assert torch.equal(base[1], base[2])
    for c in (0, 2, n - 1):
        solo = run(10 + c, [c])[0]
        assert torch.equal(solo, got[c]), c


@pytest.mark.parametrize("rows", [[2, 3], [200, 7], [128 + 5]])
def test_backward_lora_plus_ia3_short_pieces(rows):
    """a client with LoRA AND IA3 on one layer, backward, with LoRA pieces of <= 16
    rows (decode rows and short tails of larger segments). The shrink must read the IA3-scaled
    g = dy*l (client.py:291-294 -> adapters.py:37), not dy."""
    d_in, d_out = 512, 1024
    w, b = O.layer_params(41, 0, O.FF_UP, d_in, d_out)
    ex = _ex({(0, O.FF_UP): (w, b)})
    lo = O.lora_params(41, 0, 0, O.FF_UP, d_in, d_out, 16, 32.0)
    ia = O.ia3_params(41, 0, 0, O.FF_UP, d_out)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.FF_UP): (lo.a, lo.b)}, ia3={_addr(0, O.FF_UP): ia.ia3},
                                    alpha=32.0, rank=16))
    ad = O.OracleAdapter(a=O.bf16_round(lo.a), b=O.bf16_round(lo.b), alpha=32.0, rank=16, ia3=ia.ia3)
    wr = O.bf16_round(w)
    for dtype in (torch.bfloat16, torch.float32):
        gs = [torch.randn(t, d_out, device=ex.device).to(torch.bfloat16).to(dtype) for t in rows]
        res = ex._compute_batch(1, [_env(0 if c == 0 else 1, 1, 0, O.FF_UP, 1, g) for c, g in enumerate(gs)])
        g0 = gs[0].float().cpu().numpy()
        _close(res[0].float().cpu().numpy(), O.layer_backward_dx(ad, wr, g0), mean_rel=O.TOL_IA3_BWD_MEAN_REL,
               what=f"bwd LoRA+IA3 rows={rows} {dtype}")


def test_host_batch_with_mixed_dtypes_computes_every_envelope():
    """pinned-host clients sending bf16 and f32 in one dispatch must all compute
    (the native host pipeline needs one dtype; mixed batches take the staged path)."""
    d_in, d_out = 256, 512
    w, b = O.layer_params(42, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    dts = (torch.bfloat16, torch.float32, torch.bfloat16)
    hosts = [torch.randn(t, d_in).to(torch.bfloat16).to(dt).pin_memory() for t, dt in zip((9, 40, 3), dts)]
    replies = [torch.empty(h.shape[0], d_out, dtype=dt).pin_memory() for h, dt in zip(hosts, dts)]
    res = ex._compute_batch(0, [_env(c, 1, 0, O.V, 0, h, reply_to=r) for c, (h, r) in enumerate(zip(hosts, replies))])
    wr = O.bf16_round(w)
    for c, r in enumerate(res):
        assert isinstance(r, torch.Tensor), r
        ref = O.affine_forward(hosts[c].float().numpy(), wr, b)
        _close(r.float().cpu().numpy(), ref, what=f"mixed host client {c}")


def test_dispatches_on_two_streams_are_ordered():
    """One context, consecutive dispatches on two different streams with no synchronisation in
    between: the second is ordered after the first (they share the context's workspace), so both
    give their solo results bitwise."""
    d_in, d_out = 2048, 3072
    w, b = O.layer_params(61, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    dev = ex.device
    xa = [torch.randn(t, d_in, device=dev).to(torch.bfloat16) for t in (3000, 700, 5)]
    xb = [torch.randn(t, d_in, device=dev).to(torch.bfloat16) for t in (2500, 2, 900)]
    solo_a = ex._compute_batch(0, [_env(c, 1, 0, O.V, 0, x) for c, x in enumerate(xa)])
    solo_b = ex._compute_batch(0, [_env(c, 2, 0, O.V, 0, x) for c, x in enumerate(xb)])
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        outs_a = [torch.empty(x.shape[0], d_out, device=dev, dtype=torch.bfloat16) for x in xa]
        outs_b = [torch.empty(x.shape[0], d_out, device=dev, dtype=torch.bfloat16) for x in xb]
        segs_a = [(c, x, outs_a[c], None) for c, x in enumerate(xa)]
        segs_b = [(c, x, outs_b[c], None) for c, x in enumerate(xb)]
        da = ex.compile_dispatch(0, 0, O.V, segs_a)
        db = ex.compile_dispatch(0, 0, O.V, segs_b)
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            da.run()
        with torch.cuda.stream(s2):
            db.run()
        torch.cuda.synchronize()
        for c in range(len(xa)):
            assert torch.equal(outs_a[c], solo_a[c]), ("a", c)
        for c in range(len(xb)):
            assert torch.equal(outs_b[c], solo_b[c]), ("b", c)


def test_long_k_raster_group_bitwise():
    """group_m_longk (raster group size of K >= longk dispatches) only reorders tiles: a K = 13824
    forward of 8 x 1024 rows gives the same bits with groups of 16, 6 and 1 pair M-tiles."""
    d_in, d_out = 13824, 1536
    w, b = O.layer_params(43, 0, O.FF_DOWN, d_in, d_out)
    ex = _ex({(0, O.FF_DOWN): (w, b)})
    ad = O.lora_params(43, 1, 0, O.FF_DOWN, d_in, d_out, 32, 64.0)
    ex.register_adapter(1, _Adapter(lora={_addr(0, O.FF_DOWN): (ad.a, ad.b)}, alpha=64.0, rank=32))
    gen = torch.Generator(device=ex.device).manual_seed(43)
    xs = [torch.randn(1024, d_in, generator=gen, device=ex.device).to(torch.bfloat16) for _ in range(8)]
    outs = []
    for g in (0, 6, 1):
        ex.ctx.set_option("group_m_longk", g)
        outs.append(ex._compute_batch(0, [_env(c, 1 + g, 0, O.FF_DOWN, 0, x) for c, x in enumerate(xs)]))
    ex.ctx.set_option("group_m_longk", 0)
    for o in outs[1:]:
        for c in range(len(xs)):
            assert torch.equal(o[c], outs[0][c]), c
