"""Client processes hand activations to the executor process through CUDA IPC (ipc.py).

The paper's local mode shares the exchange tensor between processes; the
reference's process mode (harness.py:243-260, 367-394) is the topology. Checks:
* a GPU client in another OS process gets bitwise the results an in-process DeviceChannel
  client gets for the same inputs and adapter (rows are independent, so the executor's batch
  composition does not matter), with every payload served from the client's own device memory
  (no host staging) and buffer growth re-exported;
* the reference harness in process mode, with its ``RemoteChannel`` / ``ExecutorServer`` pair
  replaced by ``IpcChannel`` / ``IpcExecutorServer``, produces bitwise the thread-mode
  (in-process channels) results.
"""

from __future__ import annotations

import concurrent.futures
import dataclasses
import multiprocessing
import os
import tempfile

import numpy as np
import pytest
import torch

from tests import ipc_worker as W

pytestmark = pytest.mark.gpu

D_IN, D_OUT = 512, 768


def _executor(scheduler=None):
    from paper_2507_03220_b200 import AffineParams, GpuBaseExecutor, LayerAddress, Role
    rng = np.random.default_rng(7)
    layers = {}
    for role, (di, do) in ((Role.Q, (D_IN, D_IN)), (Role.FF_UP, (D_IN, D_OUT))):
        w = (rng.standard_normal((di, do)) / np.sqrt(di)).astype(np.float32)
        b = (rng.standard_normal(do) * 0.1).astype(np.float32)
        layers[LayerAddress(0, role)] = AffineParams(w, b)
    return GpuBaseExecutor(layers, scheduler=scheduler).start()


def _plan():
    from paper_2507_03220_b200 import PASS_BACKWARD, PASS_FORWARD, Role
    q, up = int(Role.Q), int(Role.FF_UP)
    # (block, role, pass, input, want_base); input 3 is larger than the first request, so the
    # client's buffers grow (and are re-exported) mid-sequence
    return [(0, up, PASS_FORWARD, 0, False), (0, up, PASS_BACKWARD, 1, False),
            (0, q, PASS_FORWARD, 2, False), (0, up, PASS_FORWARD, 3, True),
            (0, up, PASS_BACKWARD, 4, False)]


SHAPES = [(37, D_IN), (37, D_OUT), (5, D_IN), (300, D_IN), (300, D_OUT)]


def _adapter_spec():
    from paper_2507_03220_b200 import Role
    up = (0, int(Role.FF_UP))
    rng = np.random.default_rng(3)
    return {"lora": {up: (11, D_IN, D_OUT, 16)},
            "ia3": {up: (1.0 + 0.1 * rng.standard_normal(D_OUT)).astype(np.float32)},
            "alpha": 32.0, "rank": 16}


def _in_process(ex, client_id, spec):
    from paper_2507_03220_b200 import DeviceChannel
    ch = DeviceChannel(ex, client_id, 1, 1, max(D_IN, D_OUT))
    ch.register(sends_backward=True)
    lora = {k: W.make_lora(*v) for k, v in spec["lora"].items()}
    ch.register_adapter(W.Adapter(lora, spec["ia3"], spec["alpha"], spec["rank"]))
    out = W.run_sequence(ch, _plan(), W.make_inputs(1234, SHAPES))
    ch.deregister()
    return out


@pytest.mark.parametrize("scheduler", ["python", "native"])
def test_device_client_process_bitwise_equals_in_process_channel(scheduler):
    from paper_2507_03220_b200.executor import _is_device
    from paper_2507_03220_b200.ipc import IpcExecutorServer
    ex = _executor(scheduler)
    seen = []
    orig_submit = ex.submit

    def submit(env, reply_fn):
        seen.append((_is_device(env.payload), env.reply_to is not None and _is_device(env.reply_to)))
        orig_submit(env, reply_fn)
    ex.submit = submit
    try:
        spec = _adapter_spec()
        with IpcExecutorServer(ex) as server:
            ctx = multiprocessing.get_context("spawn")
            q = ctx.Queue()
            p = ctx.Process(target=W.device_client,
                            args=((server.host, server.port), server.authkey, 5, 0, 1234, SHAPES,
                                  _plan(), spec, q))
            p.start()
            status, out, resizes = q.get(timeout=150)
            p.join(60)
            assert status == "ok", out
            out = [W.from_wire(w) for w in out]
            assert server.requests_served == len(_plan())
        assert resizes[0] >= 1 and resizes[1] >= 1          # grew and was re-exported mid-run
        assert seen and all(a and b for a, b in seen)         # served from device memory only
        ref = _in_process(ex, 6, spec)
        assert len(out) == len(ref)
        for i, (a, b) in enumerate(zip(out, ref)):
            assert a.dtype == b.dtype and a.shape == b.shape, i
            assert torch.equal(a, b), f"reply {i} differs"
    finally:
        ex.close()


def test_rejected_request_fails_only_that_request_and_wrong_key_is_refused():
    """A malformed request (wrong row width) and an unknown layer are answered with the
    executor's ProtocolError messages (executor.py:172-174, 208-211) and the channel keeps
    working (test_executor.py:66-72); a connection without the server's authkey is refused."""
    from paper_2507_03220_b200.ipc import IpcChannel, IpcExecutorServer
    ex = _executor()
    try:
        with IpcExecutorServer(ex) as server:
            ctx = multiprocessing.get_context("spawn")
            q = ctx.Queue()
            p = ctx.Process(target=W.rejection_client, args=((server.host, server.port), server.authkey, q))
            p.start()
            status, out = q.get(timeout=150)
            p.join(60)
            assert status == "ok", out
            with pytest.raises(Exception, match="another process"):   # same-process client
                IpcChannel(server.host, server.port, 9, authkey=server.authkey, device=0)
        assert out[0][0] == "refused"
        assert out[1][0] == "ProtocolError" and "row width" in out[1][1]
        assert out[2] == ("ok", (4, D_OUT), True)
        assert out[3][0] == "ProtocolError" and "unknown layer" in out[3][1]
    finally:
        ex.close()


# ------------------------------------------------------- the reference harness, process mode

def _reference():
    from tests import test_gpu_dropin as D     # puts baseline/_ref (or the mounted reference) on sys.path
    return D


@pytest.mark.parametrize("fused", [False, True])
def test_reference_harness_process_mode_over_ipc(monkeypatch, fused):
    """harness.run(mode="process") with the executor built by the harness (GpuBaseExecutor
    through the monkeypatched BaseExecutor name) and _run_processes' RemoteChannel /
    ExecutorServer replaced by IpcChannel / IpcExecutorServer: results equal the thread-mode
    run bitwise (test_acceptance.py:394-417 shape), and no client payload crosses the host on
    the executor side."""
    D = _reference()
    H = D.H
    from splitserve.model import build_model, save_checkpoint

    from paper_2507_03220_b200.ipc import IpcExecutorServer
    monkeypatch.setattr(H, "BaseExecutor", D.gpu_executor)
    served = {}

    def run_processes_ipc(scenario, executor):          # harness._run_processes, harness.py:367-394
        model = build_model(scenario.model)
        results = {}
        with tempfile.TemporaryDirectory() as tmp:
            checkpoint = os.path.join(tmp, "model.ckpt")
            save_checkpoint(model, checkpoint)
            with IpcExecutorServer(executor) as server:
                ctx = multiprocessing.get_context("spawn")
                with concurrent.futures.ProcessPoolExecutor(max_workers=len(scenario.jobs), mp_context=ctx) as pool:
                    futs = {pool.submit(W.harness_worker, i, j.to_dict(), checkpoint, server.host,
                                        server.port, server.authkey, fused): i
                            for i, j in enumerate(scenario.jobs)}
                    for f in concurrent.futures.as_completed(futs, timeout=600):
                        results[futs[f]] = f.result()
                served["n"] = server.requests_served
        return results

    base = H.named_scenario("remote-ft")
    monkeypatch.setattr(H, "_run_processes", run_processes_ipc)
    proc = H.run(dataclasses.replace(base, mode="process"))
    assert proc.ok, proc.errors()
    assert served["n"] > 0
    if fused:
        # the threaded reference run with the same fusion (the adapter applied executor-side)
        orig = H._build_job

        def build(job_id, jcfg, config, channel, client_parts=None, base_model=None):
            from paper_2507_03220_b200.fusion import fuse_client_model
            job = orig(job_id, jcfg, config, channel, client_parts=client_parts, base_model=base_model)
            if job.adapter is not None:
                fuse_client_model(job.model, job_id, job.adapter)
            return job
        monkeypatch.setattr(H, "_build_job", build)
    thr = H.run(dataclasses.replace(base, jobs=[dataclasses.replace(j, endpoint="local") for j in base.jobs]))
    assert thr.ok, thr.errors()
    for i in proc.jobs:
        assert len(proc.jobs[i].logits) == len(thr.jobs[i].logits)
        for a, b in zip(proc.jobs[i].logits, thr.jobs[i].logits):
            assert np.array_equal(a, b), f"job {i}"
