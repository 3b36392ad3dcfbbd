"""Native batch formation (ss_sched_*, sched.py, GpuBaseExecutor(scheduler="native")).

The reference's scheduler contract (executor.py:162-178 submit, 235-300 _loop / _pick_ready /
_dispatch; tests mirrored in test_gpu_dropin.py for both loops) driven by many device clients:
* every client's replies are bitwise what the Python scheduler loop gives (rows are
  independent: batch composition is invisible, acceptance C5), and lockstep forms one batch of
  all registered clients per layer and pass;
* intake rejections carry the reference's messages on the DeviceChannel fast path;
* adapter refreshes from client threads while the native thread dispatches are serialised by
  the context lock (the library's pack growth frees what a concurrent table build would read).
"""

from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

D, F = 512, 1024
N_CLIENTS = 12


def _layers():
    from paper_2507_03220_b200 import AffineParams, LayerAddress, Role
    rng = np.random.default_rng(11)
    out = {}
    for role, (di, do) in ((Role.Q, (D, D)), (Role.FF_UP, (D, F)), (Role.FF_DOWN, (F, D))):
        w = (rng.standard_normal((di, do)) / np.sqrt(di)).astype(np.float32)
        out[LayerAddress(0, role)] = AffineParams(w, (rng.standard_normal(do) * 0.1).astype(np.float32))
    return out


class _Ad:
    def __init__(self, lora=None, ia3=None, alpha=0.0, rank=1):
        self.lora, self.ia3, self.alpha, self.rank = lora or {}, ia3 or {}, alpha, rank


def _adapter(c):
    from paper_2507_03220_b200 import LayerAddress, Role
    rng = np.random.default_rng(100 + c)
    if c % 3 == 2:
        return _Ad(ia3={LayerAddress(0, Role.FF_UP): (1 + 0.1 * rng.standard_normal(F)).astype(np.float32)})
    r = (8, 16, 32)[c % 3]
    lora = {}
    for role, (di, do) in ((Role.Q, (D, D)), (Role.FF_UP, (D, F))):
        lora[LayerAddress(0, role)] = ((rng.standard_normal((di, r)) / np.sqrt(di)).astype(np.float32),
                                       (rng.standard_normal((r, do)) * 0.05).astype(np.float32))
    return _Ad(lora=lora, alpha=2.0 * r, rank=r)


def _executor(scheduler, policy="lockstep", **kw):
    from paper_2507_03220_b200 import BatchPolicy, GpuBaseExecutor
    ex = GpuBaseExecutor(_layers(), BatchPolicy(mode=policy, **kw), scheduler=scheduler)
    for c in range(N_CLIENTS):
        ex.register_adapter(c, _adapter(c))
    return ex


def _client_run(ex, c, rows, steps=2):
    """fwd Q -> FF_UP (IA3 clients ask for y_base) -> FF_DOWN, then bwd in reverse (fine-tune
    clients = even ids); returns host copies of every reply."""
    from paper_2507_03220_b200 import PASS_BACKWARD, PASS_FORWARD, DeviceChannel, Role
    ch = DeviceChannel(ex, c, 1, rows, F)
    ft = c % 2 == 0
    ch.register(sends_backward=ft)
    g = torch.Generator(device="cuda").manual_seed(1000 + c)
    out = []
    for _ in range(steps):
        ch.buffer.buf.copy_(torch.randn(ch.buffer.capacity, generator=g, device="cuda"))
        for role, di in ((Role.Q, D), (Role.FF_UP, D), (Role.FF_DOWN, F)):
            want = c % 3 == 2 and role == Role.FF_UP
            y = ch.request(0, int(role), PASS_FORWARD, ch.buffer.view(rows, di), want_base=want)
            out.append(y.cpu().clone())
            if want:
                out.append(ch.last_base.cpu().clone())
        if ft:
            for role, do in ((Role.FF_DOWN, D), (Role.FF_UP, F), (Role.Q, D)):
                out.append(ch.request(0, int(role), PASS_BACKWARD, ch.buffer.view(rows, do)).cpu().clone())
    return ch, out


def _run_all(ex, rows_of):
    results, errors = {}, []
    chans = {}
    barrier = threading.Barrier(N_CLIENTS)

    def one(c):
        try:
            barrier.wait()
            chans[c], results[c] = _client_run(ex, c, rows_of(c))
        except Exception as exc:   # noqa: BLE001
            errors.append(repr(exc))
            barrier.abort()

    ts = [threading.Thread(target=one, args=(c,), daemon=True) for c in range(N_CLIENTS)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not errors, errors[0]
    for ch in chans.values():
        ch.deregister()
    return results


def test_native_scheduler_bitwise_equals_python_scheduler_lockstep():
    rows_of = lambda c: 16 + 9 * c      # noqa: E731 — ragged segments
    out = {}
    for scheduler in ("python", "native"):
        ex = _executor(scheduler)
        try:
            with ex:
                out[scheduler] = _run_all(ex, rows_of)
                m = ex.metrics
            fwd_sizes = [s for (b, r, p), v in m.batch_sizes.items() if p == 0 for s in v]
            bwd_sizes = [s for (b, r, p), v in m.batch_sizes.items() if p == 1 for s in v]
            # lockstep: one batch of every registered client per layer (backward: the senders)
            assert set(fwd_sizes) == {N_CLIENTS}, (scheduler, fwd_sizes)
            assert set(bwd_sizes) == {N_CLIENTS // 2}, (scheduler, bwd_sizes)
        finally:
            ex.close()
    for c in range(N_CLIENTS):
        a, b = out["python"][c], out["native"][c]
        assert len(a) == len(b)
        for i, (x, y) in enumerate(zip(a, b)):
            assert torch.equal(x, y), f"client {c} reply {i}"


@pytest.mark.parametrize("policy", ["nolockstep", "opportunistic"])
def test_native_scheduler_other_policies_bitwise(policy):
    """Batch composition differs run to run under these policies; every reply must not."""
    rows_of = lambda c: 8 + 5 * c      # noqa: E731
    ref = _executor("python", "nolockstep")
    ex = _executor("native", policy, wait_per_token=0.001, wait_cap=0.01)
    try:
        with ref:
            want = _run_all(ref, rows_of)
        with ex:
            got = _run_all(ex, rows_of)
            sizes = [s for v in ex.metrics.batch_sizes.values() for s in v]
        if policy == "nolockstep":
            assert set(sizes) == {1}
        for c in range(N_CLIENTS):
            for i, (x, y) in enumerate(zip(want[c], got[c])):
                assert torch.equal(x, y), f"client {c} reply {i}"
    finally:
        ref.close()
        ex.close()


def test_native_rejections_on_device_fast_path():
    from paper_2507_03220_b200 import (PASS_FORWARD, DeviceChannel, Envelope, ProtocolError, Role,
                                       error_message)
    ex = _executor("native", "nolockstep")
    try:
        with ex:
            ch = DeviceChannel(ex, 1, 1, 8, F)
            ch.register()
            with pytest.raises(ProtocolError, match=r"row width 520 does not match layer .* expected 512"):
                ch.request(0, int(Role.Q), PASS_FORWARD, torch.zeros(4, D + 8, device="cuda", dtype=torch.bfloat16))
            with pytest.raises(ProtocolError, match="unknown layer"):
                ch.request(3, int(Role.Q), PASS_FORWARD, torch.zeros(4, D, device="cuda", dtype=torch.bfloat16))
            y = ch.request(0, int(Role.Q), PASS_FORWARD, torch.ones(4, D, device="cuda", dtype=torch.bfloat16))
            assert y.shape == (4, D) and torch.isfinite(y.float()).all()
            # a stale request id through submit(): the reference's message
            box, done = {}, threading.Event()

            def reply(e):
                box["e"] = e
                done.set()
            ex.submit(Envelope(1, 2, 0, int(Role.Q), PASS_FORWARD,
                               torch.ones(2, D, device="cuda", dtype=torch.bfloat16)), reply)
            assert done.wait(10)
            assert error_message(box["e"]) == "request_id 2 not increasing (last 3)"
            ch.deregister()
    finally:
        ex.close()


def test_adapter_refresh_while_native_thread_dispatches():
    """Client threads refresh their adapters (same values: the math must not move) while the
    native thread dispatches other clients' requests; every reply equals the quiet run's."""
    rows_of = lambda c: 24      # noqa: E731
    quiet = _executor("native", "nolockstep")
    busy = _executor("native", "nolockstep")
    stop = threading.Event()
    try:
        with quiet:
            want = _run_all(quiet, rows_of)

        def refresher():
            while not stop.is_set():
                for c in range(N_CLIENTS):
                    busy.refresh_adapter(c, _adapter(c))

        with busy:
            t = threading.Thread(target=refresher, daemon=True)
            t.start()
            got = _run_all(busy, rows_of)
            stop.set()
            t.join(30)
        for c in range(N_CLIENTS):
            for i, (x, y) in enumerate(zip(want[c], got[c])):
                assert torch.equal(x, y), f"client {c} reply {i}"
    finally:
        stop.set()
        quiet.close()
        busy.close()
