"""Prebuilt dispatch plans (ss_plan_*) and CUDA-graph capture of a plan sequence: same kernels,
same tables, so every result must be BITWISE the per-call ss_compute_batch result."""

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O

from .test_gpu_parity import _Adapter, _addr, _env, _ex, _mixed_clients

pytestmark = pytest.mark.gpu


def _buffers(ex, counts, width_in, width_out, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device=ex.device).manual_seed(seed)
    xs = [torch.randn(t, width_in, generator=g, device=ex.device).to(dtype) for t in counts]
    ys = [torch.empty(t, width_out, dtype=dtype, device=ex.device) for t in counts]
    return xs, ys


@pytest.mark.parametrize("shape", [(384, 640), (5120, 1536)])
def test_plan_launch_bitwise_equals_compute_batch(shape):
    d_in, d_out = shape
    w, b = O.layer_params(21, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    _, counts = _mixed_clients(ex, d_in, d_out, seed=21)
    counts[2] = 1024   # a whole-tile client (direct TMA tiles) next to ragged ones
    for pass_kind, (wi, wo) in ((0, (d_in, d_out)), (1, (d_out, d_in))):
        xs, ys = _buffers(ex, counts, wi, wo, seed=pass_kind)
        ref = ex._compute_batch(pass_kind, [_env(c, 10 + pass_kind, 0, O.K, pass_kind, x) for c, x in enumerate(xs)])
        d = ex.compile_dispatch(pass_kind, 0, O.K, [(c, x, y, None) for c, (x, y) in enumerate(zip(xs, ys))])
        for _ in range(2):       # relaunch: tables are reused, result unchanged
            d.run()
            torch.cuda.synchronize()
            for c in range(len(xs)):
                assert torch.equal(ys[c], ref[c]), (pass_kind, c)


def test_plan_rebuilds_after_workspace_growth_and_rank_change():
    d_in, d_out = 512, 768
    w, b = O.layer_params(22, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ad = O.lora_params(22, 0, 0, O.V, d_in, d_out, 8, 16.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad.a, ad.b)}, alpha=16.0, rank=8))
    xs, ys = _buffers(ex, [37, 5], d_in, d_out)
    d = ex.compile_dispatch(0, 0, O.V, [(0, xs[0], ys[0], None), (1, xs[1], ys[1], None)])
    d.run()
    # a much larger dispatch grows the shared workspace (X / LoRA operand are reallocated)
    big = [torch.randn(3000, d_in, device=ex.device).to(torch.bfloat16) for _ in range(3)]
    ex._compute_batch(0, [_env(c, 5, 0, O.V, 0, x) for c, x in enumerate(big)])
    d.run()
    torch.cuda.synchronize()
    ref = ex._compute_batch(0, [_env(0, 6, 0, O.V, 0, xs[0]), _env(1, 6, 0, O.V, 0, xs[1])])
    assert torch.equal(ys[0], ref[0]) and torch.equal(ys[1], ref[1])
    # rank change moves the client's pack block: the plan must pick up the new adapter
    ad2 = O.lora_params(23, 0, 0, O.V, d_in, d_out, 32, 64.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad2.a, ad2.b)}, alpha=64.0, rank=32))
    d.run()
    torch.cuda.synchronize()
    ref = ex._compute_batch(0, [_env(0, 7, 0, O.V, 0, xs[0])])
    assert torch.equal(ys[0], ref[0])
    wr = O.bf16_round(w)
    x0 = xs[0].float().cpu().numpy()
    oracle = O.apply_adapter(O.OracleAdapter(a=O.bf16_round(ad2.a), b=O.bf16_round(ad2.b), alpha=64.0, rank=32),
                             x0, O.affine_forward(x0, wr, b))
    mx, mn = O.normwise_errors(ys[0].float().cpu().numpy(), oracle)
    assert mx <= O.TOL_MAX_REL and mn <= O.TOL_MEAN_REL


@pytest.mark.parametrize("decode", [False, True])
def test_cuda_graph_of_plans_bitwise_equals_eager(decode):
    """A whole executor step (forward over several layers, then backward in reverse) captured in
    one CUDA graph gives the eager results bitwise, and replays deterministically. `decode`:
    two-row clients, so the weight-streaming kernel runs and the LoRA shrink reads the client
    rows in place on the side stream (a parallel branch of the captured graph)."""
    layers = {}
    dims = {O.Q: (256, 256), O.FF_UP: (256, 512), O.FF_DOWN: (512, 256)}
    for role, (di, do) in dims.items():
        layers[(0, role)] = O.layer_params(24, 0, role, di, do)
    ex = _ex(layers)
    rng = np.random.default_rng(24)
    for cid, r in enumerate((8, 16, 64)):
        lo = {}
        for role, (di, do) in dims.items():
            ad = O.lora_params(24, cid, 0, role, di, do, r, 2.0 * r)
            lo[_addr(0, role)] = (ad.a, ad.b)
        ex.register_adapter(cid, _Adapter(lora=lo, alpha=2.0 * r, rank=r))
    counts = [2, 2, 1, 2] if decode else [int(t) for t in rng.integers(1, 400, size=4)]
    bufs = [torch.randn(t * 512, device=ex.device).to(torch.bfloat16) for t in counts]
    outs = [torch.empty(t * 512, device=ex.device, dtype=torch.bfloat16) for t in counts]
    plan = []
    order = [O.Q, O.FF_UP, O.FF_DOWN]
    for role in order:
        di, do = dims[role]
        plan.append(ex.compile_dispatch(0, 0, role, [(c, bufs[c][: t * di].view(t, di), outs[c][: t * do].view(t, do), None)
                                                     for c, t in enumerate(counts)]))
    for role in reversed(order):
        di, do = dims[role]
        plan.append(ex.compile_dispatch(1, 0, role, [(c, bufs[c][: t * do].view(t, do), outs[c][: t * di].view(t, di), None)
                                                     for c, t in enumerate(counts)]))
    # eager reference: each dispatch alone, snapshot its outputs
    eager = []
    for d in plan:
        d.run()
        torch.cuda.synchronize()
        eager.append([o.clone() for o in outs])
    g = ex.capture(plan)
    for _ in range(2):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        # outputs of the last dispatch (and of every earlier one whose columns it did not
        # overwrite) match the eager sequence
        for c in range(len(counts)):
            assert torch.equal(outs[c], eager[-1][c]), c


def test_captured_graph_recaptures_after_workspace_growth_and_rank_change():
    """VERDICT r1 'stale CUDA graphs': a graph bakes workspace / pack addresses. After a
    larger eager dispatch grows (frees + reallocates) the workspace, or a rank change moves a
    client's pack block, ``CapturedStep.replay`` must re-capture instead of replaying freed
    memory — and the replayed results must equal a fresh eager dispatch bitwise."""
    d_in, d_out = 512, 768
    w, b = O.layer_params(31, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ad = O.lora_params(31, 0, 0, O.V, d_in, d_out, 8, 16.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad.a, ad.b)}, alpha=16.0, rank=8))
    xs, ys = _buffers(ex, [37, 5], d_in, d_out)
    d = ex.compile_dispatch(0, 0, O.V, [(0, xs[0], ys[0], None), (1, xs[1], ys[1], None)])
    g = ex.capture([d])
    assert g.recaptures == 0 and not g.stale
    e0 = ex.ctx.epoch()
    big = [torch.randn(3000, d_in, device=ex.device).to(torch.bfloat16) for _ in range(3)]
    ex._compute_batch(0, [_env(c, 5, 0, O.V, 0, x) for c, x in enumerate(big)])
    assert ex.ctx.epoch() != e0 and g.stale
    for o in ys:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert g.recaptures == 1
    ref = ex._compute_batch(0, [_env(0, 6, 0, O.V, 0, xs[0]), _env(1, 6, 0, O.V, 0, xs[1])])
    assert torch.equal(ys[0], ref[0]) and torch.equal(ys[1], ref[1])
    # a same-rank value refresh writes the pack in place: no re-capture, new values seen
    ad_v = O.lora_params(32, 0, 0, O.V, d_in, d_out, 8, 16.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad_v.a, ad_v.b)}, alpha=16.0, rank=8))
    assert not g.stale
    g.replay()
    torch.cuda.synchronize()
    ref = ex._compute_batch(0, [_env(0, 7, 0, O.V, 0, xs[0])])
    assert torch.equal(ys[0], ref[0]) and g.recaptures == 1
    # a scale change at the same padded rank (alpha) and a rank change both invalidate
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad_v.a, ad_v.b)}, alpha=32.0, rank=8))
    assert g.stale
    g.replay()
    torch.cuda.synchronize()
    ref = ex._compute_batch(0, [_env(0, 8, 0, O.V, 0, xs[0])])
    assert torch.equal(ys[0], ref[0]) and g.recaptures == 2
    ad2 = O.lora_params(33, 0, 0, O.V, d_in, d_out, 32, 64.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.V): (ad2.a, ad2.b)}, alpha=64.0, rank=32))
    g.replay()
    torch.cuda.synchronize()
    ref = ex._compute_batch(0, [_env(0, 9, 0, O.V, 0, xs[0])])
    assert torch.equal(ys[0], ref[0]) and g.recaptures == 3


def test_plan_sees_alpha_change_at_same_rank():
    """re-registering with a different alpha (same padded rank) must reach prebuilt
    plans (the scale is baked into their segment tables)."""
    d_in, d_out = 256, 512
    w, b = O.layer_params(34, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    ad = O.lora_params(34, 0, 0, O.K, d_in, d_out, 16, 32.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.K): (ad.a, ad.b)}, alpha=32.0, rank=16))
    xs, ys = _buffers(ex, [40], d_in, d_out)
    d = ex.compile_dispatch(0, 0, O.K, [(0, xs[0], ys[0], None)])
    d.run()
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.K): (ad.a, ad.b)}, alpha=128.0, rank=16))
    d.run()
    torch.cuda.synchronize()
    ref = ex._compute_batch(0, [_env(0, 2, 0, O.K, 0, xs[0])])
    assert torch.equal(ys[0], ref[0])
    x0 = xs[0].float().cpu().numpy()
    oracle = O.apply_adapter(O.OracleAdapter(a=O.bf16_round(ad.a), b=O.bf16_round(ad.b), alpha=128.0, rank=16),
                             x0, O.affine_forward(x0, O.bf16_round(w), b))
    mx, mn = O.normwise_errors(ys[0].float().cpu().numpy(), oracle)
    assert mx <= O.TOL_MAX_REL and mn <= O.TOL_MEAN_REL


def test_concurrent_adapter_refresh_during_dispatch():
    """VERDICT r1 'adapter refresh races dispatch': client threads refresh their adapters
    (values every time, the rank now and then, which grows / moves the packs) while the
    scheduler thread dispatches. Every call into the library is serialised by the executor's
    lock: no error, and once the refreshes stop the next dispatch equals the oracle with the
    final adapters."""
    import threading
    d_in, d_out = 512, 1024
    w, b = O.layer_params(35, 0, O.Q, d_in, d_out)
    ex = _ex({(0, O.Q): (w, b)})
    finals = {}
    for cid in range(4):
        ad = O.lora_params(35, cid, 0, O.Q, d_in, d_out, 8, 16.0)
        ex.register_adapter(cid, _Adapter(lora={_addr(0, O.Q): (ad.a, ad.b)}, alpha=16.0, rank=8))
    xs = [torch.randn(t, d_in, device=ex.device).to(torch.bfloat16) for t in (50, 3, 130, 17)]
    stop = threading.Event()
    errors = []

    def refresher(cid):
        k = 0
        try:
            while not stop.is_set() or k < 3:
                r = (8, 16, 8, 32)[k % 4]
                ad = O.lora_params(100 + k, cid, 0, O.Q, d_in, d_out, r, 2.0 * r)
                ex.register_adapter(cid, _Adapter(lora={_addr(0, O.Q): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
                finals[cid] = ad
                k += 1
        except Exception as exc:        # pragma: no cover - reported below
            errors.append(exc)

    ts = [threading.Thread(target=refresher, args=(c,)) for c in range(4)]
    for t in ts:
        t.start()
    req = 1
    for _ in range(40):
        out = ex._compute_batch(0, [_env(c, req, 0, O.Q, 0, x) for c, x in enumerate(xs)])
        assert all(isinstance(o, torch.Tensor) for o in out), out
        req += 1
    stop.set()
    for t in ts:
        t.join(60)
    assert not errors, errors
    out = ex._compute_batch(0, [_env(c, req, 0, O.Q, 0, x) for c, x in enumerate(xs)])
    torch.cuda.synchronize()
    wr = O.bf16_round(w)
    for c, x in enumerate(xs):
        ad = finals[c]
        x0 = x.float().cpu().numpy()
        oracle = O.apply_adapter(O.OracleAdapter(a=O.bf16_round(ad.a), b=O.bf16_round(ad.b), alpha=ad.alpha,
                                                 rank=ad.rank), x0, O.affine_forward(x0, wr, b))
        mx, mn = O.normwise_errors(out[c].float().cpu().numpy(), oracle)
        assert mx <= O.TOL_MAX_REL and mn <= O.TOL_MEAN_REL, (c, mx, mn)


def test_cuda_graph_of_tail_split_dispatches_bitwise():
    """The bench's path for split dispatches: two consecutive 13B K-projection forwards of
    32 x 1024 rows (each a 256 x 512 launch + the programmatically launched 256 x 256 tail, the
    second reading the first's output) captured as one graph equal the eager plans and the
    unsplit launch, replay after replay."""
    d = 5120
    w, b = O.layer_params(23, 0, O.K, d, d)
    w2, b2 = O.layer_params(23, 0, O.V, d, d)
    ex = _ex({(0, O.K): (w, b), (0, O.V): (w2, b2)})
    for cid, r in ((0, 16), (7, 64)):
        for role in (O.K, O.V):
            ad = O.lora_params(23, cid, 0, role, d, d, r, 2.0 * r)
            ex.register_adapter(cid, _Adapter(lora={_addr(0, role): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
    n = 32
    xs, mid = _buffers(ex, [1024] * n, d, d, seed=23)
    out = [torch.empty_like(m) for m in mid]
    plan = [ex.compile_dispatch(0, 0, O.K, [(c, xs[c], mid[c], None) for c in range(n)]),
            ex.compile_dispatch(0, 0, O.V, [(c, mid[c], out[c], None) for c in range(n)])]
    ex.ctx.set_option("tail_split", 0)
    ref_mid = ex._compute_batch(0, [_env(c, 1, 0, O.K, 0, xs[c]) for c in range(n)])
    ref_out = ex._compute_batch(0, [_env(c, 2, 0, O.V, 0, ref_mid[c]) for c in range(n)])
    ex.ctx.set_option("tail_split", 1)
    g = ex.capture(plan)
    for _ in range(3):
        for t in mid + out:
            t.zero_()
        g.replay()
        torch.cuda.synchronize()
        for c in range(n):
            assert torch.equal(mid[c], ref_mid[c]), c
            assert torch.equal(out[c], ref_out[c]), c
