"""Client-process entry points for tests/test_gpu_ipc.py (spawned: importable by module name).

``device_client`` is a GPU client (torch activations on the device) talking to the executor
process through ``IpcChannel``. ``harness_worker`` mirrors the reference's
``_process_worker`` (harness.py:243-260) with ``IpcChannel`` in place of ``RemoteChannel``:
only the client half of the checkpoint is loaded, the reference ClientModel drives the job.
"""

from __future__ import annotations


def make_inputs(seed: int, shapes):
    import torch
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(s, generator=g).to(torch.bfloat16) for s in shapes]


def make_lora(seed: int, d_in: int, d_out: int, rank: int):
    import numpy as np
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal((d_in, rank)) * 0.05).astype(np.float32)
    b = (rng.standard_normal((rank, d_out)) * 0.05).astype(np.float32)
    return a, b


class Adapter:
    def __init__(self, lora=None, ia3=None, alpha=16.0, rank=8):
        self.lora, self.ia3, self.alpha, self.rank = lora or {}, ia3 or {}, alpha, rank


def to_wire(t):
    """CPU tensor -> picklable numpy (bf16 as its int16 bits): torch's shared-memory tensor
    pickling would outlive this process's exit."""
    import torch
    return (t.dtype == torch.bfloat16, t.view(torch.int16).numpy() if t.dtype == torch.bfloat16 else t.numpy())


def from_wire(w):
    import torch
    bf16, a = w
    t = torch.from_numpy(a)
    return t.view(torch.bfloat16) if bf16 else t


def run_sequence(channel, plan, inputs):
    """plan: [(block, role, pass_kind, input index, want_base)] -> host copies of the replies."""
    out = []
    for block, role, pass_kind, idx, want_base in plan:
        x = inputs[idx].to(f"cuda:{channel.device}" if hasattr(channel, "device") else "cuda")
        y = channel.request(block, role, pass_kind, x, want_base=want_base)
        out.append(y.cpu().clone())
        if want_base:
            out.append(channel.last_base.cpu().clone())
    return out


def device_client(address, authkey, client_id, device, seed, shapes, plan, adapter_spec, q):
    import torch
    torch.cuda.set_device(device)
    from paper_2507_03220_b200.ipc import IpcChannel
    try:
        ch = IpcChannel(address[0], address[1], client_id, authkey=authkey, device=device)
        ch.register(sends_backward=True)
        if adapter_spec is not None:
            lora = {k: make_lora(*v) for k, v in adapter_spec.get("lora", {}).items()}
            ia3 = {k: v for k, v in adapter_spec.get("ia3", {}).items()}
            ch.register_adapter(Adapter(lora, ia3, adapter_spec["alpha"], adapter_spec["rank"]))
        inputs = make_inputs(seed, shapes)
        out = run_sequence(ch, plan, inputs)
        resizes = (ch.buffer.resizes, ch.reply_buffer.resizes)
        ch.deregister()
        ch.close()
        q.put(("ok", [to_wire(t) for t in out], resizes))
    except Exception as exc:   # reported to the parent
        import traceback
        q.put(("error", f"{type(exc).__name__}: {exc}\n{traceback.format_exc()}", None))


def harness_worker(job_id, job_dict, checkpoint, host, port, authkey, fused):
    """harness._process_worker (harness.py:243-260) over IpcChannel."""
    from splitserve import harness as H
    from splitserve.model import load_client_half

    from paper_2507_03220_b200.fusion import fuse_client_model
    from paper_2507_03220_b200.ipc import IpcChannel
    jcfg = H.JobConfig.from_dict(job_dict)
    config, *client_parts = load_client_half(checkpoint)
    import torch
    # f32 exchange buffers: the reference client's payloads are f32 (transport.py:36), and the
    # reply keeps the f32 the in-process LocalChannel path returns
    channel = IpcChannel(host, port, client_id=job_id, authkey=authkey, device=0, dtype=torch.float32)
    try:
        channel.register(sends_backward=(jcfg.kind == "finetune"))
        job = H._build_job(job_id, jcfg, config, channel, client_parts=tuple(client_parts))
        if fused and job.adapter is not None:
            fuse_client_model(job.model, job_id, job.adapter)
        result = H._drive_job(job, config)
        channel.deregister()
        return result
    except Exception as exc:
        return H.JobResult(job_id, jcfg.kind, error=f"{type(exc).__name__}: {exc}")
    finally:
        channel.close()


def rejection_client(address, authkey, q):
    """A malformed request, a good one, an unknown layer: (kind, message / shape) per request."""
    import torch
    from paper_2507_03220_b200 import PASS_FORWARD, Role
    from paper_2507_03220_b200.ipc import IpcChannel
    out = []
    try:
        try:
            IpcChannel(address[0], address[1], 1, authkey=b"not-the-key", device=0)
            out.append(("connected", ""))
        except Exception as exc:   # the HMAC handshake refuses the wrong key
            out.append(("refused", type(exc).__name__))
        ch = IpcChannel(address[0], address[1], 3, authkey=authkey, device=0)
        ch.register()
        up = int(Role.FF_UP)
        d_in = ch.executor.layer_dims(0, up)[0]
        for block, width in ((0, d_in + 8), (0, d_in), (7, d_in)):
            try:
                y = ch.request(block, up, PASS_FORWARD,
                               torch.ones(4, width, device="cuda", dtype=torch.bfloat16))
                out.append(("ok", tuple(y.shape), bool(torch.isfinite(y.float()).all())))
            except Exception as exc:
                out.append((type(exc).__name__, str(exc)))
        ch.deregister()
        ch.close()
        q.put(("ok", out))
    except Exception as exc:
        import traceback
        q.put(("error", f"{type(exc).__name__}: {exc}\n{traceback.format_exc()}"))
