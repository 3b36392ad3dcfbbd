"""Cross-check the oracle against the live reference where it is importable (the build
container); skipped on the GPU box, where the golden vectors stand in."""

import sys

import numpy as np
import pytest

from oracle import splitserve_oracle as O
from tests.conftest import REFERENCE_SRC, reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import splitserve.adapters as adapters
    import splitserve.executor as executor
    import splitserve.model as model
    import splitserve.protocol as protocol
    import splitserve.tensor_ops as tensor_ops
    from splitserve.config import LayerAddress, ModelConfig, Role
    return dict(adapters=adapters, executor=executor, model=model, protocol=protocol,
                tensor_ops=tensor_ops, LayerAddress=LayerAddress, ModelConfig=ModelConfig, Role=Role)


@pytest.mark.parametrize("seed", range(6))
def test_random_batches_bitwise(ref, seed):
    rng = np.random.default_rng(100 + seed)
    d_in, d_out = int(rng.integers(4, 40)), int(rng.integers(4, 40))
    W = rng.standard_normal((d_in, d_out)).astype(np.float32)
    b = rng.standard_normal(d_out).astype(np.float32)
    addr = ref["LayerAddress"](0, ref["Role"].FF_UP)
    ex = ref["executor"].BaseExecutor({addr: ref["tensor_ops"].AffineParams(W, b)})
    rows = [int(r) for r in rng.integers(0, 9, size=int(rng.integers(1, 6)))]
    for pass_kind, width in ((0, d_in), (1, d_out), (2, d_in)):
        xs = [rng.standard_normal((r, width)).astype(np.float32) for r in rows]
        renvs = [ref["protocol"].Envelope(i, 1, 0, 4, pass_kind, x) for i, x in enumerate(xs)]
        oenvs = [O.OracleEnvelope(i, 1, 0, 4, pass_kind, x) for i, x in enumerate(xs)]
        got = O.compute_batch(pass_kind, oenvs, W, b)
        want = ref["executor"].BaseExecutor._compute_batch(ex, pass_kind, renvs)
        for g_, w_ in zip(got, want):
            assert np.array_equal(g_, w_)


def test_lora_and_layer_backward_match_reference(ref):
    rng = np.random.default_rng(7)
    x = rng.standard_normal((6, 12)).astype(np.float32)
    a = rng.standard_normal((12, 3)).astype(np.float32)
    b = rng.standard_normal((3, 10)).astype(np.float32)
    gy = rng.standard_normal((6, 10)).astype(np.float32)
    assert np.array_equal(O.lora_forward(x, a, b, 6.0, 3), ref["adapters"].lora_forward(x, a, b, 6.0, 3))
    for o, r in zip(O.lora_backward(x, gy, a, b, 6.0, 3), ref["adapters"].lora_backward(x, gy, a, b, 6.0, 3)):
        assert np.array_equal(o, r)
