"""Host-side f32 -> bf16 conversion of pageable request rows (ss_compute_batch_host,
`host_convert`): numpy f32 payloads (the reference channels' payload type, transport.py:36, 78)
give bitwise the same replies with the conversion on the host threads as with the device gather's
own conversion, forward and backward, LoRA / IA3 / plain clients, ragged row counts; and rows
holding NaN / Inf / values that round across a bf16 binade convert exactly like the gather."""

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O
from tests.test_gpu_parity import _Adapter, _addr, _env, _ex

pytestmark = pytest.mark.gpu


def _run(ex, pass_kind, role, payloads, convert):
    ex.ctx.set_option("host_convert", convert)
    res = ex._compute_batch(pass_kind, [_env(c, 900 + convert, 0, role, pass_kind, p) for c, p in enumerate(payloads)])
    return [np.array(r, copy=True) for r in res]


@pytest.mark.parametrize("pass_kind", [0, 1])
@pytest.mark.parametrize("ia3", [False, True])
def test_numpy_f32_host_convert_bitwise(pass_kind, ia3):
    d_in, d_out, role = 1024, 1536, O.K
    w, b = O.layer_params(51, 0, role, d_in, d_out)
    ex = _ex({(0, role): (w, b)})
    ex.pipeline_rows = 256            # several sub-batches per dispatch (ring slots reused)
    for c, r in enumerate((8, 16, 64)):
        ad = O.lora_params(51, c, 0, role, d_in, d_out, r, 2.0 * r)
        ex.register_adapter(c, _Adapter(lora={_addr(0, role): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
    if ia3:
        ex.register_adapter(3, _Adapter(ia3={_addr(0, role): O.ia3_params(51, 3, 0, role, d_out).ia3}))
    rng = np.random.default_rng(51 + pass_kind)
    counts = [300, 17, 1024, 5, 640]
    width = d_out if pass_kind == 1 else d_in
    payloads = [rng.standard_normal((t, width)).astype(np.float32) for t in counts]
    payloads[1][3, :7] = [np.nan, np.inf, -np.inf, 1.00390625, 1.01171875, -0.0, 3.4e38]
    a = _run(ex, pass_kind, role, payloads, 0)
    b_ = _run(ex, pass_kind, role, payloads, 1)
    for c in range(len(counts)):
        assert a[c].shape == b_[c].shape
        assert np.array_equal(a[c], b_[c], equal_nan=True), c
    ex.close()


@pytest.mark.parametrize("pass_kind", [0, 1])
def test_numpy_f32_small_dispatch_host_convert_bitwise(pass_kind):
    """Decode-size numpy f32 dispatches (1-16 rows per client) take the host conversion into a
    page-locked slot and then the zero-copy path: replies bitwise those of the device gather's own
    conversion (host_convert 0), repeated (recurring-dispatch cache) and with changed values."""
    d_in, d_out, role = 2048, 1024, O.Q
    w, b = O.layer_params(53, 0, role, d_in, d_out)
    ex = _ex({(0, role): (w, b)})
    for c, r in enumerate((8, 16, 64, 32)):
        ad = O.lora_params(53, c, 0, role, d_in, d_out, r, 2.0 * r)
        ex.register_adapter(c, _Adapter(lora={_addr(0, role): (ad.a, ad.b)}, alpha=2.0 * r, rank=r))
    rng = np.random.default_rng(53 + pass_kind)
    counts = [2, 1, 16, 2, 5, 2]
    width = d_out if pass_kind == 1 else d_in
    for _ in range(2):
        payloads = [rng.standard_normal((t, width)).astype(np.float32) for t in counts]
        a = _run(ex, pass_kind, role, payloads, 0)
        b1 = _run(ex, pass_kind, role, payloads, 1)
        b2 = _run(ex, pass_kind, role, payloads, 1)
        for c in range(len(counts)):
            assert np.array_equal(a[c], b1[c]) and np.array_equal(a[c], b2[c]), c
    ex.close()
