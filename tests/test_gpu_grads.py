"""GPU parity of the adapter weight-gradient path (ss_adapter_grads: K3 shrinks + K6 token
contraction for LoRA, K7 column reduction for IA3) against the oracle / the reference's golden
``lora_backward`` outputs (adapters.py:26-41) and ``_layer_backward``'s IA3 term
(client.py:291-293).

Tolerances: exact-integer inputs -> bitwise; random inputs -> normwise against the f32 oracle
fed the same bf16-rounded x / dy: max|d|/max|ref| <= 2e-2, mean|d|/mean|ref| <= 3e-3 (the
s*x.A and s*g.B^T intermediates are rounded to bf16 once, like the forward's shrink).
"""

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O

pytestmark = pytest.mark.gpu

MAX_REL, MEAN_REL = O.TOL_MAX_REL, O.TOL_GRAD_MEAN_REL


class _Adapter:
    def __init__(self, lora=None, ia3=None, alpha=0.0, rank=1):
        self.lora, self.ia3, self.alpha, self.rank = lora or {}, ia3 or {}, alpha, rank


def _addr(block, role):
    from paper_2507_03220_b200 import LayerAddress, Role
    return LayerAddress(block, Role(role))


def _ex(d_in, d_out, role=O.Q, seed=0):
    from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor
    w, b = O.layer_params(seed, 0, role, d_in, d_out)
    return GpuBaseExecutor({_addr(0, role): AffineParams(w, b)}), w


def _dev(a, dtype=torch.bfloat16):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _close(got, ref, max_rel=MAX_REL, mean_rel=MEAN_REL, what=""):
    mx, mn = O.normwise_errors(np.asarray(got, np.float64), np.asarray(ref, np.float64))
    assert mx <= max_rel and mn <= mean_rel, f"{what}: normwise max {mx:.3e} mean {mn:.3e}"


def _lora_job(cid, x, dy, rank, d_in, d_out, accumulate=False):
    from paper_2507_03220_b200.device import GradSeg
    return GradSeg(client_id=cid, x=x, dy=dy, accumulate=accumulate,
                   grad_a=torch.zeros(d_in, rank, device="cuda"),
                   grad_b=torch.zeros(rank, d_out, device="cuda"))


def test_lora_grads_golden():
    """The reference's own lora_backward outputs (tests/golden/adapters.npz, x 5x24, r 4)."""
    g = np.load("tests/golden/adapters.npz")
    x, a, b, gy = g["x"], g["a"], g["b"], g["gy"]
    d_in, r = a.shape
    d_out = b.shape[1]
    ex, _ = _ex(d_in, d_out)
    ex.register_adapter(7, _Adapter(lora={_addr(0, O.Q): (a, b)}, alpha=2.0 * r, rank=r))
    job = _lora_job(7, _dev(x), _dev(gy), r, d_in, d_out)
    assert ex.adapter_grads(0, O.Q, [job]) == [0]
    torch.cuda.synchronize()
    ar, br = O.bf16_round(a), O.bf16_round(b)
    ga, gb, _ = O.lora_backward(O.bf16_round(x), O.bf16_round(gy), ar, br, 2.0 * r, r)
    _close(job.grad_a.cpu().numpy(), ga, what="grad_a vs oracle(bf16 inputs)")
    _close(job.grad_b.cpu().numpy(), gb, what="grad_b vs oracle(bf16 inputs)")
    _close(job.grad_a.cpu().numpy(), g["lora_ga"], 3e-2, 1e-2, "grad_a vs reference golden")
    _close(job.grad_b.cpu().numpy(), g["lora_gb"], 3e-2, 1e-2, "grad_b vs reference golden")
    ex.close()


def test_lora_grads_exact_integer_bitwise():
    """Small-integer x, dy, A, B and s = 1/2: every product and partial sum is exact in fp32 and
    the bf16 intermediates s*x.A, s*g.B^T stay exact integers/halves (|v| <= 256) -> bitwise."""
    rng = np.random.default_rng(3)
    d_in, d_out, t = 320, 192, 200
    for rank in (8, 16, 40, 64, 96):
        ex, _ = _ex(d_in, d_out, seed=rank)
        x = (rng.integers(-1, 2, (t, d_in)) * (rng.random((t, d_in)) < 0.1)).astype(np.float32)
        dy = (rng.integers(-1, 2, (t, d_out)) * (rng.random((t, d_out)) < 0.1)).astype(np.float32)
        a = rng.integers(-2, 3, (d_in, rank)).astype(np.float32)
        b = rng.integers(-2, 3, (rank, d_out)).astype(np.float32)
        alpha = rank / 2.0
        ex.register_adapter(1, _Adapter(lora={_addr(0, O.Q): (a, b)}, alpha=alpha, rank=rank))
        job = _lora_job(1, _dev(x), _dev(dy), rank, d_in, d_out)
        assert ex.adapter_grads(0, O.Q, [job]) == [0]
        torch.cuda.synchronize()
        ga, gb, _ = O.lora_backward(x, dy, a, b, alpha, rank)
        assert np.array_equal(job.grad_a.cpu().numpy(), ga), f"grad_a rank {rank}"
        assert np.array_equal(job.grad_b.cpu().numpy(), gb), f"grad_b rank {rank}"
        ex.close()


@pytest.mark.parametrize("d_in,d_out,role", [(256, 512, O.FF_UP), (4096, 4096, O.Q), (5120, 5120, O.V)])
def test_lora_grads_random_mixed_ranks_ragged(d_in, d_out, role):
    """Several clients of one layer in one call: mixed ranks (8..64 and 100 -> two 64-column
    UMMA chunks), ragged token counts (1, 37, 130, 512, 1024), random-normal parity; then the
    batched call equals per-client calls bitwise (batching invisibility for gradients)."""
    rng = np.random.default_rng(d_in + role)
    ex, _ = _ex(d_in, d_out, role, seed=role)
    specs = [(0, 8, 37), (1, 16, 1), (2, 32, 130), (3, 64, 512), (4, 100, 1024)]
    jobs, refs = [], []
    for cid, rank, t in specs:
        ad = O.lora_params(5, cid, 0, role, d_in, d_out, rank, 2.0 * rank)
        ex.register_adapter(cid, _Adapter(lora={_addr(0, role): (ad.a, ad.b)}, alpha=2.0 * rank, rank=rank))
        x = O.bf16_round(rng.standard_normal((t, d_in)).astype(np.float32))
        dy = O.bf16_round(rng.standard_normal((t, d_out)).astype(np.float32))
        jobs.append(_lora_job(cid, _dev(x), _dev(dy), rank, d_in, d_out))
        refs.append(O.lora_backward(x, dy, O.bf16_round(ad.a), O.bf16_round(ad.b), 2.0 * rank, rank))
    assert ex.adapter_grads(0, role, jobs) == [0] * len(jobs)
    torch.cuda.synchronize()
    for (cid, rank, t), job, (ga, gb, _) in zip(specs, jobs, refs):
        _close(job.grad_a.cpu().numpy(), ga, what=f"grad_a client {cid} r{rank} t{t}")
        _close(job.grad_b.cpu().numpy(), gb, what=f"grad_b client {cid} r{rank} t{t}")
    for (cid, rank, t), job in zip(specs, jobs):
        solo = _lora_job(cid, job.x, job.dy, rank, d_in, d_out)
        assert ex.adapter_grads(0, role, [solo]) == [0]
        torch.cuda.synchronize()
        assert torch.equal(solo.grad_a, job.grad_a) and torch.equal(solo.grad_b, job.grad_b), cid
    ex.close()


@pytest.mark.parametrize("lag", [0, 1, 2, 5])
def test_lora_grads_fused_launch_bitwise(lag):
    """grad_fused (one launch: each client's shrinks, then its token contractions `lag` clients
    later, picked up through an atomic work ticket) equals the two-launch path bitwise, for more
    clients than the lag, mixed ranks 8..64, ragged token counts."""
    d_in, d_out, role = 1024, 1536, O.V
    rng = np.random.default_rng(41 + lag)
    ex, _ = _ex(d_in, d_out, role, seed=41)
    specs = [(c, (8, 16, 32, 64)[c % 4], t) for c, t in enumerate((1, 37, 130, 512, 64, 300, 17, 256))]
    xs = []
    for cid, rank, t in specs:
        ad = O.lora_params(7, cid, 0, role, d_in, d_out, rank, 2.0 * rank)
        ex.register_adapter(cid, _Adapter(lora={_addr(0, role): (ad.a, ad.b)}, alpha=2.0 * rank, rank=rank))
        xs.append((_dev(rng.standard_normal((t, d_in))), _dev(rng.standard_normal((t, d_out)))))

    def run(fused):
        ex.ctx.set_option("grad_fused", fused)
        ex.ctx.set_option("grad_fused_lag", lag)
        jobs = [_lora_job(cid, x, dy, rank, d_in, d_out) for (cid, rank, _), (x, dy) in zip(specs, xs)]
        assert ex.adapter_grads(0, role, jobs) == [0] * len(jobs)
        torch.cuda.synchronize()
        return jobs

    two, one = run(0), run(1)
    for (cid, _, _), a, b in zip(specs, two, one):
        assert torch.equal(a.grad_a, b.grad_a) and torch.equal(a.grad_b, b.grad_b), cid
    ex.close()


def test_lora_grads_accumulate():
    rng = np.random.default_rng(11)
    d_in, d_out, r = 256, 384, 16
    ex, _ = _ex(d_in, d_out)
    ad = O.lora_params(1, 0, 0, O.Q, d_in, d_out, r, 32.0)
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.Q): (ad.a, ad.b)}, alpha=32.0, rank=r))
    x = _dev(rng.standard_normal((64, d_in)))
    dy = _dev(rng.standard_normal((64, d_out)))
    job = _lora_job(0, x, dy, r, d_in, d_out)
    ex.adapter_grads(0, O.Q, [job])
    first_a, first_b = job.grad_a.clone(), job.grad_b.clone()
    job.accumulate = True
    ex.adapter_grads(0, O.Q, [job])
    torch.cuda.synchronize()
    assert torch.equal(job.grad_a, 2 * first_a) and torch.equal(job.grad_b, 2 * first_b)
    ex.close()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_ia3_grad(dtype):
    """grad_l = sum_rows(dy * y_base) (client.py:291-293), ragged width (d_out = 300) and rows."""
    from paper_2507_03220_b200.device import GradSeg
    rng = np.random.default_rng(2)
    d_in, d_out = 128, 300
    ex, _ = _ex(d_in, d_out, O.K)
    jobs, refs = [], []
    for cid, t in ((0, 1), (1, 77), (2, 1024)):
        ex.register_adapter(cid, _Adapter(ia3={_addr(0, O.K): O.ia3_params(0, cid, 0, O.K, d_out).ia3}))
        dy = rng.standard_normal((t, d_out)).astype(np.float32)
        yb = rng.standard_normal((t, d_out)).astype(np.float32)
        if dtype == torch.bfloat16:
            dy, yb = O.bf16_round(dy), O.bf16_round(yb)
        jobs.append(GradSeg(client_id=cid, dy=_dev(dy, dtype), y_base=_dev(yb, dtype),
                            grad_l=torch.zeros(d_out, device="cuda")))
        refs.append(np.sum(dy.astype(np.float64) * yb, axis=0))
    assert ex.adapter_grads(0, O.K, jobs) == [0, 0, 0]
    torch.cuda.synchronize()
    for job, ref in zip(jobs, refs):
        got = job.grad_l.cpu().numpy()
        assert np.max(np.abs(got - ref)) <= 1e-4 * max(1.0, np.max(np.abs(ref))) + 1e-4
    ex.close()


def test_grad_job_rejections():
    from paper_2507_03220_b200 import _lib
    from paper_2507_03220_b200.device import GradSeg
    d_in, d_out = 128, 128
    ex, _ = _ex(d_in, d_out)
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((d_in, 8)), rng.standard_normal((8, d_out))
    ex.register_adapter(0, _Adapter(lora={_addr(0, O.Q): (a, b)}, alpha=8.0, rank=8))
    ex.register_adapter(1, _Adapter(lora={_addr(0, O.Q): (a, b)}, ia3={_addr(0, O.Q): np.ones(d_out)},
                                    alpha=8.0, rank=8))
    x = _dev(rng.standard_normal((16, d_in)))
    dy = _dev(rng.standard_normal((16, d_out)))
    jobs = [
        _lora_job(0, x.float(), dy, 8, d_in, d_out),        # f32 x: LoRA needs bf16 TMA rows
        _lora_job(1, x, dy, 8, d_in, d_out),                # LoRA + IA3 on one layer
        _lora_job(9, x, dy, 8, d_in, d_out),                # no adapter registered
        _lora_job(0, x, dy, 8, d_in, d_out),                # fine
    ]
    st = ex.adapter_grads(0, O.Q, jobs)
    assert st == [_lib.SS_SEG_BAD_PTR, _lib.SS_SEG_UNSUPPORTED, _lib.SS_SEG_NO_ADAPTER, 0]
    torch.cuda.synchronize()
    assert float(jobs[0].grad_a.abs().sum()) == 0.0     # rejected: untouched
    assert float(jobs[3].grad_a.abs().sum()) > 0.0
    ex.close()


def test_client_layer_backward_matches_reference_layer_backward():
    """client.client_layer_backward == ClientModel._layer_backward (client.py:286-305): grad_x
    from one fused backward dispatch, grads dict accumulated under (addr, 'a'|'b'|'l')."""
    from paper_2507_03220_b200 import DeviceChannel, VirtLayer
    from paper_2507_03220_b200.client import client_forward, client_layer_backward
    rng = np.random.default_rng(4)
    d_in, d_out, t = 256, 512, 96
    ex, w = _ex(d_in, d_out, O.FF_UP)
    wr = O.bf16_round(w)
    addr = _addr(0, O.FF_UP)
    lo = O.lora_params(2, 0, 0, O.FF_UP, d_in, d_out, 16, 32.0)
    ia = O.ia3_params(2, 1, 0, O.FF_UP, d_out)
    ads = {0: _Adapter(lora={addr: (lo.a, lo.b)}, alpha=32.0, rank=16), 1: _Adapter(ia3={addr: ia.ia3})}
    for cid, ad in ads.items():
        ex.register_adapter(cid, ad)
    ex.start()
    for cid, ad in ads.items():
        ch = DeviceChannel(ex, cid, 1, t, max(d_in, d_out))
        ch.register(sends_backward=True)
        layer = VirtLayer(addr, d_in, d_out, ch)
        fused = ex.fused_addresses(cid)
        x = _dev(O.bf16_round(rng.standard_normal((t, d_in)).astype(np.float32)))
        _, y_base = client_forward(layer, fused, ad, x)
        dy = _dev(O.bf16_round(rng.standard_normal((t, d_out)).astype(np.float32)))
        grads = {}
        gx = client_layer_backward(layer, fused, ex, cid, ad, x, dy, grads, y_base=y_base)
        gx = client_layer_backward(layer, fused, ex, cid, ad, x, dy, grads, y_base=y_base)
        torch.cuda.synchronize()
        xn, dyn = x.float().cpu().numpy(), dy.float().cpu().numpy()
        if cid == 0:
            ga, gb, _ = O.lora_backward(xn, dyn, O.bf16_round(lo.a), O.bf16_round(lo.b), 32.0, 16)
            _close(grads[(addr, "a")].cpu().numpy(), 2 * ga, what="grads a (2 accumulations)")
            _close(grads[(addr, "b")].cpu().numpy(), 2 * gb, what="grads b")
            ref_dx = O.layer_backward_dx(O.OracleAdapter(a=O.bf16_round(lo.a), b=O.bf16_round(lo.b),
                                                         alpha=32.0, rank=16), wr, dyn)
        else:
            ybn = y_base.float().cpu().numpy()
            _close(grads[(addr, "l")].cpu().numpy(), 2 * np.sum(dyn * ybn, axis=0), 1e-4, 1e-4, "grads l")
            ref_dx = O.layer_backward_dx(ia, wr, dyn)
        _close(gx.float().cpu().numpy(), ref_dx, what=f"grad_x client {cid}")
        ch.deregister()
    ex.close()
