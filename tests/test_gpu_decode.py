"""Decode-class rows (segments of <= decode_rows rows): the split-K kernel K1d + its fixup
(csrc/decode.cuh). Their K reduction is C = ceil(K / (64 * decode_chunk_kb)) fixed chunks folded
left to right, then the row's own LoRA chain, a property of the request and the layer alone, so

* parity: against an fp32 evaluation of the reference math (tensor_ops.py:71-89,
  adapters.py:19-40, 127-145, client.py:291-294) at the same tolerances as every other row;
* batching invisibility (acceptance C5): a decode-class request gives the same bits solo, with
  other decode requests (several 64-row decode tiles, LoRA pieces cut differently), and beside
  prefill-class requests;
* pieces keep their request's class: the host pipelines split requests into sub-batches, and a
  piece of a decode (prefill) request reduces K as the whole request would.
"""

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O
from tests.test_gpu_parity import _Adapter, _addr, _close, _env
from tests.test_gpu_parity import _ex as _ex0

pytestmark = pytest.mark.gpu


def _ex(layers):
    """An executor with the decode class on (requests of <= 16 rows)."""
    ex = _ex0(layers)
    ex.ctx.set_option("decode_rows", 16)
    return ex

KINDS = [("lora", 8), ("lora", 16), ("lora", 32), ("lora", 64), ("plain", 0), ("ia3", 0), ("both", 16)]


def _clients(ex, seed, block, role, d_in, d_out, n):
    """n clients cycling through KINDS; returns {cid: (lora adapter | None, ia3 vector | None)}."""
    ads = {}
    for cid in range(n):
        kind, r = KINDS[cid % len(KINDS)]
        lora = ia3 = None
        kw = {}
        if kind in ("lora", "both"):
            lora = O.lora_params(seed, cid, block, role, d_in, d_out, r, 2.0 * r)
            kw.update(lora={_addr(block, role): (lora.a, lora.b)}, alpha=2.0 * r, rank=r)
        if kind in ("ia3", "both") and role in O.IA3_ROLES:
            ia3 = O.ia3_params(seed, cid, block, role, d_out).ia3
            kw.update(ia3={_addr(block, role): ia3})
        if kw:
            ex.register_adapter(cid, _Adapter(**kw))
        ads[cid] = (lora, ia3)
    return ads


def _ref(dev, pass_kind, x, Wt, bt, lora, ia3):
    xf = x.float()
    if pass_kind == 0:
        y = xf @ Wt + bt
        if lora is not None:
            A = torch.from_numpy(lora.a).to(dev).to(torch.bfloat16).float()
            B = torch.from_numpy(lora.b).to(dev).to(torch.bfloat16).float()
            y = y + ((xf @ A) @ B) * lora.scale
        if ia3 is not None:
            y = y * torch.from_numpy(ia3).to(dev)
        return y
    g = xf if ia3 is None else xf * torch.from_numpy(ia3).to(dev)
    y = g @ Wt.T
    if lora is not None:
        A = torch.from_numpy(lora.a).to(dev).to(torch.bfloat16).float()
        B = torch.from_numpy(lora.b).to(dev).to(torch.bfloat16).float()
        y = y + ((g @ B.T) @ A.T) * lora.scale
    return y


@pytest.mark.parametrize("shape", [("13b_q", 5120, 5120, O.Q), ("13b_ff_up", 5120, 13824, O.FF_UP),
                                   ("13b_ff_down", 13824, 5120, O.FF_DOWN), ("13b_lm_head", 5120, 32000, O.LM_HEAD),
                                   ("g20_ff_down", 24576, 6144, O.FF_DOWN), ("small_k", 320, 1000, O.V)])
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_decode_class_parity_vs_fp32(shape, out_dtype):
    """Decode-size requests (1..16 rows) of mixed LoRA ranks 8..64 / IA3 / LoRA+IA3 / plain
    clients, forward and backward, against fp32 torch on the same bf16 operands."""
    name, d_in, d_out, role = shape
    block = 40 if role == O.LM_HEAD else 0
    w, b = O.layer_params(31, block, role, d_in, d_out)
    ex = _ex({(block, role): (w, b)})
    dev = ex.device
    n = 20
    ads = _clients(ex, 31, block, role, d_in, d_out, n)
    rng = np.random.default_rng(31)
    counts = [int(t) for t in rng.integers(1, 17, size=n)]
    Wt = torch.from_numpy(w).to(dev).to(torch.bfloat16).float()
    bt = torch.from_numpy(b).to(dev)
    f32 = out_dtype == torch.float32
    for pass_kind, (wi, wo) in ((0, (d_in, d_out)), (1, (d_out, d_in))):
        xs = [torch.randn(t, wi, device=dev).to(torch.bfloat16) for t in counts]
        outs = [torch.empty(t, wo, device=dev, dtype=out_dtype) for t in counts]
        res = ex._compute_batch(pass_kind, [_env(c, 1 + pass_kind, block, role, pass_kind, x, reply_to=outs[c])
                                            for c, x in enumerate(xs)])
        for c, (x, y) in enumerate(zip(xs, res)):
            lora, ia3 = ads[c]
            ref = _ref(dev, pass_kind, x, Wt, bt, lora, ia3)
            if f32:
                mx, mn = O.TOL_F32_MAX_REL, O.TOL_F32_MEAN_REL
            else:
                mx = O.TOL_MAX_REL
                mn = O.TOL_IA3_BWD_MEAN_REL if (pass_kind == 1 and ia3 is not None) else O.TOL_MEAN_REL
            _close(y.float().cpu().numpy(), ref.cpu().numpy(), mx, mn, f"{name} pass {pass_kind} client {c} {KINDS[c % len(KINDS)]}")


@pytest.mark.parametrize("pass_kind", [0, 1, 2])
def test_decode_class_batched_equals_solo_bitwise(pass_kind):
    """A decode-class request's rows are the same bits solo, among ~40 decode requests (several
    64-row decode tiles, LoRA segments spread over the cluster's CTAs), and beside prefill-class
    requests of the same dispatch."""
    d_in, d_out = 4096, 1408
    role = O.K
    w, b = O.layer_params(33, 0, role, d_in, d_out)
    ex = _ex({(0, role): (w, b)})
    dev = ex.device
    n = 40
    _clients(ex, 33, 0, role, d_in, d_out, n)
    rng = np.random.default_rng(33)
    counts = [int(t) for t in rng.integers(1, 17, size=n)]
    width = d_out if pass_kind == 1 else d_in
    xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]

    def run(idx, extra=()):
        envs = [_env(c, 1000 + len(idx), 0, role, pass_kind, xs[c]) for c in idx]
        envs += [_env(c, 2000, 0, role, pass_kind, x) for c, x in extra]
        return ex._compute_batch(pass_kind, envs)

    batched = run(range(n))
    assert sum(counts) > 2 * 64        # more than two decode tiles
    for c in (0, 3, 6, 11, 25, 39):
        solo = run([c])[0]
        assert torch.equal(solo, batched[c]), c
    perm = list(reversed(range(n)))
    again = run(perm)
    for j, c in enumerate(perm):
        assert torch.equal(again[j], batched[c]), c
    big = [(n + 1, torch.randn(700, width, device=dev).to(torch.bfloat16)),
           (n + 2, torch.randn(33, width, device=dev).to(torch.bfloat16))]
    mixed = run(range(n), big)
    for c in range(n):
        assert torch.equal(mixed[c], batched[c]), c
    # the prefill-class requests are unaffected by the decode rows beside them
    alone = ex._compute_batch(pass_kind, [_env(c, 3000, 0, role, pass_kind, x) for c, x in big])
    for j in range(len(big)):
        assert torch.equal(mixed[n + j], alone[j]), j


@pytest.mark.parametrize("pass_kind", [0, 1, 2])
def test_fused_fixup_equals_fixup_launch_bitwise(pass_kind):
    """decode_fixup_fused (the fold + epilogue run by K1d's idle warps behind per-tile completion
    counters) gives the same bits as the separate fixup launch, for ~40 mixed decode requests
    (several tiles, LoRA pieces, IA3, hi/lo rows), repeated launches (self-resetting counters and
    ticket) and f32 outputs."""
    d_in, d_out = 4096, 1408
    role = O.K
    w, b = O.layer_params(37, 0, role, d_in, d_out)
    ex = _ex({(0, role): (w, b)})
    dev = ex.device
    n = 40
    _clients(ex, 37, 0, role, d_in, d_out, n)
    rng = np.random.default_rng(37)
    counts = [int(t) for t in rng.integers(1, 17, size=n)]
    width = d_out if pass_kind == 1 else d_in
    xs = [torch.randn(t, width, device=dev).to(torch.bfloat16) for t in counts]
    xf = [torch.randn(t, width, device=dev) for t in counts[:9]]

    def run(rid):
        envs = [_env(c, rid, 0, role, pass_kind, xs[c]) for c in range(n)]
        envs += [_env(n + c, rid, 0, role, pass_kind, x) for c, x in enumerate(xf)]
        return ex._compute_batch(pass_kind, envs)

    ex.ctx.set_option("decode_fixup_fused", 0)
    ref = run(1)
    ex.ctx.set_option("decode_fixup_fused", 1)
    for rep in range(3):
        got = run(2 + rep)
        for c in range(len(ref)):
            assert torch.equal(got[c], ref[c]), (rep, c)


def test_decode_rows_option_zero_restores_single_chain():
    """decode_rows = 0: no decode class, a 2-row request equals its rows inside a prefill-size
    dispatch of the single-chain kernels (the round-1 invariant)."""
    d_in, d_out = 5120, 1024
    w, b = O.layer_params(35, 0, O.K, d_in, d_out)
    ex = _ex({(0, O.K): (w, b)})
    ex.ctx.set_option("decode_rows", 0)
    dev = ex.device
    _clients(ex, 35, 0, O.K, d_in, d_out, 7)
    x = torch.randn(2, d_in, device=dev).to(torch.bfloat16)
    filler = torch.randn(3000, d_in, device=dev).to(torch.bfloat16)
    solo = ex._compute_batch(0, [_env(0, 1, 0, O.K, 0, x)])[0]
    big = ex._compute_batch(0, [_env(0, 2, 0, O.K, 0, x), _env(1, 2, 0, O.K, 0, filler)])[0]
    assert torch.equal(solo, big)


@pytest.mark.parametrize("zero_copy", [0, 1 << 30])
def test_host_pipeline_pieces_keep_request_class(zero_copy):
    """Pinned-host requests through ss_compute_batch_host, split into many sub-batches
    (pipeline_rows 8): pieces of decode requests stay decode class, pieces of long requests stay
    single-chain; every row equals the device-resident dispatch bitwise."""
    d_in, d_out = 1024, 1536
    w, b = O.layer_params(37, 0, O.V, d_in, d_out)
    ex = _ex({(0, O.V): (w, b)})
    ex.pipeline_rows = 8
    ex.ctx.set_option("zero_copy_bytes", zero_copy)
    _clients(ex, 37, 0, O.V, d_in, d_out, 7)
    counts = [13, 3, 200, 16, 17, 1, 40]
    for pass_kind, (wi, wo) in ((0, (d_in, d_out)), (1, (d_out, d_in))):
        xs = [torch.randn(t, wi).to(torch.bfloat16) for t in counts]
        devr = ex._compute_batch(pass_kind, [_env(c, 50 + pass_kind, 0, O.V, pass_kind, x.to(ex.device))
                                             for c, x in enumerate(xs)])
        hin = [x.pin_memory() for x in xs]
        hout = [torch.empty(t, wo, dtype=torch.bfloat16).pin_memory() for t in counts]
        got = ex._compute_batch(pass_kind, [_env(c, 60 + pass_kind, 0, O.V, pass_kind, hin[c], reply_to=hout[c])
                                            for c in range(len(counts))])
        for c in range(len(counts)):
            assert torch.equal(got[c], devr[c].cpu()), (pass_kind, c)


def test_class_decode_flag_ignored_beyond_16_rows():
    """SS_SEGF_CLASS_DECODE on a segment of more than 16 rows is ignored (single-chain order,
    the rows of the same segment without the flag), through the C ABI."""
    import ctypes
    from paper_2507_03220_b200 import _lib as L
    lib = L.load()
    dev = torch.device("cuda:0")
    ctx = ctypes.c_void_p()
    L.check(None, lib.ss_ctx_create(0, 0, 1, ctypes.byref(ctx)))
    K, N, t = 1024, 768, 20
    W = (torch.randn(K, N, device=dev) / K ** 0.5).to(torch.bfloat16)
    L.check(ctx, lib.ss_load_layer(ctx, 0, 0, K, N, W.data_ptr(), N, None, L.SS_MEM_DEVICE | L.SS_DT_BF16))
    x = torch.randn(t, K, device=dev).to(torch.bfloat16)
    outs = []
    for extra in (0, L.SS_SEGF_CLASS_DECODE):
        out = torch.empty(t, N, device=dev, dtype=torch.bfloat16)
        arr = (L.SsSeg * 1)()
        s = arr[0]
        s.client_id, s.rows, s.width = 0, t, K
        s.flags = L.SS_SEGF_SRC_BF16 | L.SS_SEGF_DST_BF16 | extra
        s.src, s.src_ld, s.dst, s.dst_ld = x.data_ptr(), K, out.data_ptr(), N
        st = (ctypes.c_int32 * 1)()
        L.check(ctx, lib.ss_compute_batch(ctx, 0, 0, 0, 1, arr, torch.cuda.current_stream().cuda_stream, st))
        torch.cuda.synchronize()
        assert st[0] == 0
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    lib.ss_ctx_destroy(ctx)
