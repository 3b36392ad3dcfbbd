"""Host-side blinding logic (privacy.py here) against the reference's own privacy.py outputs
(tests/golden/privacy.npz, made by tests/golden/make_golden.py privacy_golden): noise rotation
and noise draws bitwise; the reference's blind -> forward -> unblind round trip recovers the
plain affine output (pins the scheme the GPU tests build on). CPU only."""

import numpy as np
import torch

from oracle import splitserve_oracle as O
from paper_2507_03220_b200 import LayerAddress, Role
from paper_2507_03220_b200.privacy import DeviceNoiseSet, draw_noise, rotate


def test_rotate_and_draw_noise_match_reference(golden):
    g = golden("privacy")
    addrs = [LayerAddress(0, Role.Q), LayerAddress(3, Role.FF_UP), LayerAddress(2, Role.LM_HEAD)]
    got = np.array([[rotate(s, a, it, k) for a in addrs for it in range(6) for k in (2, 3, 5)]
                    for s in (0, 7)], dtype=np.int64)
    assert np.array_equal(got, g["rotate"])
    assert np.array_equal(draw_noise(4, addrs[0], 1, 5, 16, 1.0), g["noise_q"])
    assert np.array_equal(draw_noise(9, addrs[1], 0, 3, 24, 0.25), g["noise_up"])


def test_reference_round_trip_recovers_plain_output(golden):
    g = golden("privacy")
    plain = O.affine_forward(g["rt_x"], g["rt_W"], g["rt_b"])
    assert np.max(np.abs(g["rt_y"] - plain)) <= 1e-4 * max(1.0, float(np.max(np.abs(plain))))


def test_device_noise_set_blind_unblind_on_host_tensors(golden):
    """The same blind / unblind arithmetic on torch tensors (CPU here, device on the box)."""
    g = golden("privacy")
    addr = LayerAddress(0, Role.FF_UP)
    noise = torch.as_tensor(draw_noise(3, addr, int(g["rt_idx"]), 8, 16, 1.0))
    ns = DeviceNoiseSet(seed=3, k=2, t_max=8)
    ns.noises[addr] = [noise, noise]
    eff = torch.as_tensor(g["rt_effect"])
    ns.effects[addr] = [eff, eff]
    x = torch.as_tensor(g["rt_x"])
    payload, idx = ns.blind(addr, x, 4)
    assert idx == int(g["rt_idx"])
    y_noisy = torch.as_tensor(O.affine_forward(payload.numpy(), g["rt_W"], g["rt_b"]))
    y = ns.unblind(addr, y_noisy, idx)
    assert np.max(np.abs(y.numpy() - g["rt_y"])) <= 1e-4
