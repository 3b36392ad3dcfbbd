"""Activation blinding composed with executor-fused adapters (privacy.py here; reference
privacy.py:1-12, 79-106). The NOISE pass of a fused client returns the noise
effect of the ADAPTED layer, (nW + s nAB) * l, so ``unblind`` recovers the fused reply.

Tolerance: the blinded payload x + n is rounded to bf16 before the GEMM, so the de-noised reply
carries bf16 rounding of |x + n| instead of |x|; with |n| <= 1 ~ |x| that is the same order as
the plain path: normwise max <= 2e-2, mean <= 5e-3 against the f32 oracle on the bf16 inputs."""

import numpy as np
import pytest
import torch

from oracle import splitserve_oracle as O

from .test_gpu_parity import _Adapter, _addr, _ex

pytestmark = pytest.mark.gpu


def _setup(d_in=256, d_out=512, role=O.FF_UP):
    w, b = O.layer_params(31, 0, role, d_in, d_out)
    ex = _ex({(0, role): (w, b)})
    addr = _addr(0, role)
    lo = O.lora_params(31, 0, 0, role, d_in, d_out, 16, 32.0)
    ia = O.ia3_params(31, 1, 0, role, d_out)
    ads = {0: (_Adapter(lora={addr: (lo.a, lo.b)}, alpha=32.0, rank=16),
               O.OracleAdapter(a=O.bf16_round(lo.a), b=O.bf16_round(lo.b), alpha=32.0, rank=16)),
           1: (_Adapter(ia3={addr: ia.ia3}), ia),
           2: (None, None)}
    for cid, (ad, _) in ads.items():
        if ad is not None:
            ex.register_adapter(cid, ad)
    return ex, w, b, addr, ads


def _channel(ex, cid, t, width):
    from paper_2507_03220_b200 import DeviceChannel
    ch = DeviceChannel(ex, cid, 1, t, width)
    ch.register(sends_backward=True)
    return ch


def test_zero_noise_blinded_path_is_bitwise_the_plain_path():
    from paper_2507_03220_b200 import VirtLayer
    from paper_2507_03220_b200.privacy import precompute_noise
    d_in, d_out, t = 256, 512, 64
    ex, w, b, addr, ads = _setup(d_in, d_out)
    with ex:
        for cid in ads:
            ch = _channel(ex, cid, t, d_out)
            ns = precompute_noise(ch, {addr: (d_in, d_out)}, k=2, scale=0.0, seed=3, t_max=t,
                                  device=ex.device)
            x = torch.randn(t, d_in, device=ex.device).to(torch.bfloat16)
            plain = VirtLayer(addr, d_in, d_out, ch).forward(x)
            blinded = VirtLayer(addr, d_in, d_out, ch, noise=ns).forward(x, iteration=5)
            assert torch.equal(plain.float(), blinded), cid
            ch.deregister()


@pytest.mark.parametrize("scale", [0.5, 1.0])
def test_blinded_fused_forward_matches_oracle(scale):
    """LoRA and IA3 clients (IA3 with y_base, which grad_l needs) and a plain client: blinded
    replies de-noised with the adapter-aware effect equal the oracle's unblinded fused output."""
    from paper_2507_03220_b200 import VirtLayer
    from paper_2507_03220_b200.privacy import precompute_noise
    d_in, d_out, t = 256, 512, 96
    ex, w, b, addr, ads = _setup(d_in, d_out)
    wr = O.bf16_round(w)
    rng = np.random.default_rng(7)
    with ex:
        for cid, (_, oad) in ads.items():
            ch = _channel(ex, cid, t, d_out)
            want_base = cid == 1
            ns = precompute_noise(ch, {addr: (d_in, d_out)}, k=3, scale=scale, seed=11, t_max=t,
                                  want_base=want_base, device=ex.device)
            layer = VirtLayer(addr, d_in, d_out, ch, noise=ns)
            for it in range(3):
                x = O.bf16_round(rng.standard_normal((t, d_in)).astype(np.float32))
                out = layer.forward(torch.as_tensor(x, device=ex.device), iteration=it, want_base=want_base)
                y, base = out if want_base else (out, None)
                y_base_ref = O.affine_forward(x, wr, b)
                ref = O.apply_adapter(oad, x, y_base_ref)
                mx, mn = O.normwise_errors(y.cpu().numpy(), ref)
                assert mx <= 2e-2 and mn <= 5e-3, (cid, it, mx, mn)
                if base is not None:
                    mx, mn = O.normwise_errors(base.cpu().numpy(), y_base_ref)
                    assert mx <= 2e-2 and mn <= 5e-3, ("base", it, mx, mn)
            ch.deregister()


def test_effect_is_adapter_aware_and_refresh_tracks_adapter_updates():
    from paper_2507_03220_b200 import VirtLayer
    from paper_2507_03220_b200.privacy import precompute_noise, refresh
    d_in, d_out, t = 256, 512, 32
    ex, w, b, addr, ads = _setup(d_in, d_out)
    wr = O.bf16_round(w)
    with ex:
        ch = _channel(ex, 0, t, d_out)
        ns = precompute_noise(ch, {addr: (d_in, d_out)}, k=2, scale=1.0, seed=5, t_max=t, device=ex.device)
        n0 = ns.noises[addr][0].cpu().numpy()
        # the effect includes the fused LoRA term: (nW + s nAB)
        ref_eff = O.bf16_round(n0) @ wr.astype(np.float64) + O.lora_forward(O.bf16_round(n0), *[ads[0][1].a, ads[0][1].b], 32.0, 16)
        mx, mn = O.normwise_errors(ns.effects[addr][0].cpu().numpy(), ref_eff)
        assert mx <= 2e-2 and mn <= 3e-3, (mx, mn)
        # an optimizer step changes B: refresh the effects, unblinding stays exact
        lo2 = O.lora_params(32, 0, 0, O.FF_UP, d_in, d_out, 16, 32.0)
        ex.register_adapter(0, _Adapter(lora={addr: (ads[0][1].a, lo2.b)}, alpha=32.0, rank=16))
        refresh(ns, ch, {addr: (d_in, d_out)})
        x = O.bf16_round(np.random.default_rng(1).standard_normal((t, d_in)).astype(np.float32))
        y = VirtLayer(addr, d_in, d_out, ch, noise=ns).forward(torch.as_tensor(x, device=ex.device), iteration=1)
        ref = O.apply_adapter(O.OracleAdapter(a=ads[0][1].a, b=O.bf16_round(lo2.b), alpha=32.0, rank=16),
                              x, O.affine_forward(x, wr, b))
        mx, mn = O.normwise_errors(y.cpu().numpy(), ref)
        assert mx <= 2e-2 and mn <= 5e-3, (mx, mn)
        ch.deregister()


def test_precompute_noise_needs_two_values():
    from paper_2507_03220_b200.errors import ConfigError
    from paper_2507_03220_b200.privacy import precompute_noise
    ex, w, b, addr, ads = _setup()
    with pytest.raises(ConfigError):
        precompute_noise(None, {addr: (256, 512)}, k=1, scale=1.0, seed=0, t_max=8)
    ex.close()
