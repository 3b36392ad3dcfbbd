"""CPU oracle for the base-executor hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference algorithm of the path the CUDA library
replaces (reference: /root/reference/pkg/src/splitserve, Python + numpy, f32, CPU). It is
the checker, never the product: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline leg / ``--impl reference`` arm may import it. The executor
package never imports it and has no CPU fallback.

Parity pinning: ``tests/golden/make_golden.py`` runs the reference itself (importable in the
build container) on seeded inputs and stores the outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks every function below against those vectors
(bitwise where the reference is bitwise, e.g. row independence and build_model).

Numerics follow the reference exactly: f32 arrays, ``np.einsum("ik,kj->ij", optimize=False)``
(the naive non-BLAS loop, single-threaded) for every product.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

DTYPE = np.float32

PASS_FORWARD = 0          # protocol.py:40
PASS_BACKWARD = 1         # protocol.py:41
PASS_NOISE_EFFECT = 2     # protocol.py:42

# Role ids, config.py:11-18
Q, K, V, O, FF_UP, FF_DOWN, LM_HEAD = range(7)
BLOCK_ROLES = (Q, K, V, O, FF_UP, FF_DOWN)          # config.py:21
IA3_ROLES = frozenset({K, V, FF_UP})                # config.py:24


class OracleProtocolError(Exception):
    """Stands in for splitserve.errors.ProtocolError in batch results (executor.py:203-213)."""


# ----------------------------------------------------------------------------- L0 kernels

def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """tensor_ops.py:26-36 — naive einsum, row-independent accumulation."""
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"matmul shapes {a.shape} @ {b.shape}")
    return np.einsum("ik,kj->ij", a, b, optimize=False)


def affine_forward(x: np.ndarray, weight: np.ndarray, bias: np.ndarray | None) -> np.ndarray:
    """tensor_ops.py:71-78 — y = x @ W (+ b)."""
    if x.ndim != 2 or x.shape[1] != weight.shape[0]:
        raise ValueError(f"affine_forward: input {x.shape} vs weight {weight.shape}")
    y = matmul(x, weight)
    if bias is not None:
        y = y + bias
    return y


def affine_backward_input(grad_y: np.ndarray, weight: np.ndarray) -> np.ndarray:
    """tensor_ops.py:81-89 — grad_x = grad_y @ W.T (no bias, no weight grad)."""
    if grad_y.ndim != 2 or grad_y.shape[1] != weight.shape[1]:
        raise ValueError(f"affine_backward_input: grad {grad_y.shape} vs weight {weight.shape}")
    return matmul(grad_y, weight.T)


def concat_rows(parts):
    """tensor_ops.py:145-146."""
    return np.concatenate(parts, axis=0)


def split_rows(x: np.ndarray, counts):
    """tensor_ops.py:149-156 — zero-copy views at prefix offsets."""
    out, pos = [], 0
    for c in counts:
        out.append(x[pos:pos + c])
        pos += c
    if pos != x.shape[0]:
        raise ValueError(f"split_rows: counts sum {pos} != rows {x.shape[0]}")
    return out


# ----------------------------------------------------------------------------- adapters

def lora_forward(x, a, b, alpha: float, rank: int) -> np.ndarray:
    """adapters.py:19-23 — (alpha/rank) * x @ A @ B, scale applied after both matmuls."""
    scale = np.asarray(alpha / rank, dtype=x.dtype)
    return matmul(matmul(x, a), b) * scale


def lora_backward(x_saved, grad_y, a, b, alpha: float, rank: int):
    """adapters.py:26-41 — returns (grad_a, grad_b, grad_x)."""
    scale = np.asarray(alpha / rank, dtype=x_saved.dtype)
    xa = matmul(x_saved, a)
    gyb = matmul(grad_y, b.T)
    grad_b = matmul(xa.T, grad_y) * scale
    grad_a = matmul(x_saved.T, gyb) * scale
    grad_x = matmul(gyb, a.T) * scale
    return grad_a, grad_b, grad_x


def lora_backward_dx(grad_y, a, b, alpha: float, rank: int) -> np.ndarray:
    """The grad_x term of lora_backward (adapters.py:37, 40) — the part the executor fuses."""
    scale = np.asarray(alpha / rank, dtype=grad_y.dtype)
    return matmul(matmul(grad_y, b.T), a.T) * scale


@dataclass
class OracleAdapter:
    """One client's adapter on one layer (the slice of AdapterState, adapters.py:44-115,
    that apply_adapter reads for a single address)."""

    a: np.ndarray | None = None      # LoRA A [d_in, r]
    b: np.ndarray | None = None      # LoRA B [r, d_out]
    alpha: float = 0.0
    rank: int = 0
    ia3: np.ndarray | None = None    # IA3 l [d_out]

    @property
    def scale(self) -> float:
        return self.alpha / self.rank if self.rank else 0.0


def apply_adapter(ad: OracleAdapter | None, x: np.ndarray, y_base: np.ndarray) -> np.ndarray:
    """adapters.py:127-145 — y = (y_base + lora(x)) * l."""
    if ad is None:
        return y_base
    if ad.a is not None:
        y_base = y_base + lora_forward(x, ad.a.astype(x.dtype, copy=False),
                                       ad.b.astype(x.dtype, copy=False), ad.alpha, ad.rank)
    if ad.ia3 is not None:
        y_base = y_base * ad.ia3.astype(x.dtype, copy=False)
    return y_base


def layer_backward_dx(ad: OracleAdapter | None, weight: np.ndarray, grad_y: np.ndarray) -> np.ndarray:
    """client.py:286-305 restricted to grad_x: g = dy * l (IA3), dx = g @ W.T (executor),
    dx += lora grad_x (LoRA, computed from the IA3-scaled g)."""
    g = grad_y
    if ad is not None and ad.ia3 is not None:
        g = g * ad.ia3
    dx = affine_backward_input(g, weight)
    if ad is not None and ad.a is not None:
        dx = dx + lora_backward_dx(g, ad.a, ad.b, ad.alpha, ad.rank)
    return dx


# ----------------------------------------------------------------------------- the batch

@dataclass
class OracleEnvelope:
    """protocol.py:55-76 (routing fields + payload)."""

    client_id: int
    request_id: int
    block: int
    role: int
    pass_kind: int
    payload: np.ndarray

    @property
    def token_count(self) -> int:
        return self.payload.shape[0]

    @property
    def width(self) -> int:
        return self.payload.shape[1] if self.payload.ndim == 2 else 0


ROLE_NAMES = ("Q", "K", "V", "O", "FF_UP", "FF_DOWN", "LM_HEAD")


def addr_repr(key) -> str:
    """repr of the reference's LayerAddress (config.py:27-33) for a (block, role) key."""
    return f"LayerAddress(block={key[0]}, role=<Role.{ROLE_NAMES[key[1]]}: {key[1]}>)"


def routing(pass_kind: int, envelopes, layer_key, d_in: int, d_out: int):
    """The routing part of executor.py:191-231: per-envelope validation against the first
    envelope's layer, then prefix offsets of the good ones in envelope order.

    Returns (results, good, offsets, counts) where results[i] is an OracleProtocolError for a
    rejected envelope and None otherwise; offsets/counts are split_rows' row ranges."""
    expected = d_out if pass_kind == PASS_BACKWARD else d_in
    results: list = [None] * len(envelopes)
    good: list[int] = []
    for i, env in enumerate(envelopes):
        if (env.block, env.role) != layer_key:
            results[i] = OracleProtocolError(
                f"layer mismatch in batch: {addr_repr((env.block, env.role))} != {addr_repr(layer_key)}")
        elif env.pass_kind != pass_kind:
            results[i] = OracleProtocolError(f"pass mismatch in batch: {env.pass_kind}")
        elif env.width != expected:
            results[i] = OracleProtocolError(
                f"row width {env.width} does not match layer {addr_repr(layer_key)} "
                f"expected {expected}")
        else:
            good.append(i)
    counts = [envelopes[i].token_count for i in good]
    offsets = list(np.cumsum([0] + counts[:-1])) if counts else []
    return results, good, [int(o) for o in offsets], counts


def compute_batch(pass_kind: int, envelopes, weight, bias):
    """executor.py:191-231 — concat -> one GEMM -> split; adapters NOT applied (reference)."""
    if not envelopes:
        return []
    key = (envelopes[0].block, envelopes[0].role)
    results, good, _, counts = routing(pass_kind, envelopes, key, weight.shape[0], weight.shape[1])
    if not good:
        return results
    x = concat_rows([envelopes[i].payload for i in good])
    if pass_kind == PASS_FORWARD:
        out = affine_forward(x, weight, bias)
    elif pass_kind == PASS_BACKWARD:
        out = affine_backward_input(x, weight)
    else:
        out = matmul(x, weight)
    for i, rows in zip(good, split_rows(out, counts)):
        results[i] = rows
    return results


def fused_compute_batch(pass_kind: int, envelopes, weight, bias, adapters: dict):
    """What the fused executor returns per envelope: the reference batch (executor.py:191-231)
    followed by each client's own adapter step (client.py:206-209 forward via
    adapters.py:127-145; client.py:286-305 backward grad_x). adapters maps client_id ->
    OracleAdapter (or is missing for plain clients). Forward also returns y_base per slot.

    Returns list of (out, y_base_or_None) or OracleProtocolError."""
    base = compute_batch(pass_kind, envelopes, weight, bias)
    out = []
    for env, r in zip(envelopes, base):
        if isinstance(r, OracleProtocolError):
            out.append(r)
            continue
        ad = adapters.get(env.client_id) if pass_kind != PASS_NOISE_EFFECT else None
        if pass_kind == PASS_FORWARD:
            out.append((apply_adapter(ad, env.payload, r), r))
        elif pass_kind == PASS_BACKWARD:
            out.append((layer_backward_dx(ad, weight, env.payload), None))
        else:
            out.append((r, None))
    return out


# ----------------------------------------------------------------------------- model init

@dataclass(frozen=True)
class OracleModelConfig:
    """config.py:36-56."""

    n_layers: int
    d_model: int
    n_heads: int
    d_ff: int
    vocab_size: int
    max_seq: int
    seed: int = 0


def layer_dims(cfg: OracleModelConfig, role: int) -> tuple[int, int]:
    """config.py:59-70."""
    d = cfg.d_model
    if role in (Q, K, V, O):
        return d, d
    if role == FF_UP:
        return d, cfg.d_ff
    if role == FF_DOWN:
        return cfg.d_ff, d
    if role == LM_HEAD:
        return d, cfg.vocab_size
    raise ValueError(role)


def base_addresses(cfg: OracleModelConfig):
    """config.py:73-77 — canonical order, LM_HEAD at block n_layers."""
    return [(b, r) for b in range(cfg.n_layers) for r in BLOCK_ROLES] + [(cfg.n_layers, LM_HEAD)]


def build_model_layers(cfg: OracleModelConfig):
    """model.py:65-85 — the exact reference init stream: embedding first, then per address
    W = N(0,1)/sqrt(d_in), b = 0.05 N(0,1). Returns ({(block, role): (W, b)}, embedding)."""
    rng = np.random.default_rng(cfg.seed)
    embedding = rng.standard_normal((cfg.vocab_size, cfg.d_model)).astype(DTYPE)
    layers = {}
    for addr in base_addresses(cfg):
        d_in, d_out = layer_dims(cfg, addr[1])
        w = (rng.standard_normal((d_in, d_out)) / np.sqrt(d_in)).astype(DTYPE)
        b = (0.05 * rng.standard_normal(d_out)).astype(DTYPE)
        layers[addr] = (w, b)
    return layers, embedding


def layers_checksum(cfg: OracleModelConfig, layers) -> str:
    """Same bytes as BaseModel.checksum's layer part (model.py:35-41)."""
    h = hashlib.sha256()
    for addr in base_addresses(cfg):
        w, b = layers[addr]
        h.update(w.tobytes())
        if b is not None:
            h.update(b.tobytes())
    return h.hexdigest()


def init_lora(cfg: OracleModelConfig, rank: int, alpha: float, targets, seed: int):
    """adapters.py:62-73 — A = N(0,1)/sqrt(d_in) per target address in sorted-role order,
    B = 0. Returns {(block, role): OracleAdapter}."""
    rng = np.random.default_rng(seed)
    out = {}
    for addr in _target_addresses(cfg, frozenset(targets)):
        d_in, d_out = layer_dims(cfg, addr[1])
        a = (rng.standard_normal((d_in, rank)) / np.sqrt(d_in)).astype(DTYPE)
        b = np.zeros((rank, d_out), dtype=DTYPE)
        out[addr] = OracleAdapter(a=a, b=b, alpha=alpha, rank=rank)
    return out


def init_ia3(cfg: OracleModelConfig, targets):
    """adapters.py:75-85 — l = 1 on K, V, FF_UP targets."""
    targets = frozenset(targets)
    if targets - IA3_ROLES:
        raise ValueError("IA3 targets must be within K, V, FF_UP")
    return {addr: OracleAdapter(ia3=np.ones(layer_dims(cfg, addr[1])[1], dtype=DTYPE))
            for addr in _target_addresses(cfg, targets)}


def _target_addresses(cfg: OracleModelConfig, targets):
    """adapters.py:118-124."""
    for role in sorted(targets):
        if role == LM_HEAD:
            yield (cfg.n_layers, role)
        else:
            for block in range(cfg.n_layers):
                yield (block, role)


# ----------------------------------------------------------------------------- synthetic data

def layer_params(seed: int, block: int, role: int, d_in: int, d_out: int):
    """Per-layer synthetic init for shapes too large for one build_model stream:
    same distributions as model.py:76-81 from default_rng([seed, block, role])."""
    rng = np.random.default_rng([seed, block, role])
    w = (rng.standard_normal((d_in, d_out), dtype=np.float32) / np.float32(np.sqrt(d_in)))
    b = (np.float32(0.05) * rng.standard_normal(d_out, dtype=np.float32))
    return w.astype(DTYPE), b.astype(DTYPE)


def lora_params(seed: int, client: int, block: int, role: int, d_in: int, d_out: int, rank: int,
                alpha: float):
    """A = N(0,1)/sqrt(d_in), B = 0.05 N(0,1) (non-zero so the delta is exercised,
    as test_acceptance.py:95-98 does)."""
    rng = np.random.default_rng([seed, 1000 + client, block, role])
    a = (rng.standard_normal((d_in, rank), dtype=np.float32) / np.float32(np.sqrt(d_in)))
    b = np.float32(0.05) * rng.standard_normal((rank, d_out), dtype=np.float32)
    return OracleAdapter(a=a.astype(DTYPE), b=b.astype(DTYPE), alpha=alpha, rank=rank)


def ia3_params(seed: int, client: int, block: int, role: int, d_out: int):
    """l = 1 + 0.1 N(0,1)."""
    rng = np.random.default_rng([seed, 2000 + client, block, role])
    return OracleAdapter(ia3=(1.0 + 0.1 * rng.standard_normal(d_out)).astype(DTYPE))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round f32 to the nearest bf16 (ties to even), returned as f32 — the values the GPU
    consumes, so the oracle can be fed identical inputs (SURVEY §8c parity protocol (3))."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = (rounded & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out.reshape(x.shape)


def normwise_errors(got: np.ndarray, ref: np.ndarray) -> tuple[float, float]:
    """(max|d|/max|ref|, mean|d|/mean|ref|) — the tolerance metric of SURVEY §8c."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.abs(got - ref)
    mx = float(np.max(np.abs(ref))) if ref.size else 0.0
    mn = float(np.mean(np.abs(ref))) if ref.size else 0.0
    return (float(d.max()) / mx if mx else float(d.max()),
            float(d.mean()) / mn if mn else float(d.mean()))


# Tolerances vs the f32 oracle fed the same bf16-rounded inputs (normwise, SURVEY §8c;
# measured per client kind in profiles/r02_precision.md, tools/precision_probe.py).
# bf16 activations in AND out: output rounding alone costs ~3e-3 max / ~1.4e-3 mean; the LoRA
# intermediate s*x.A is carried as a hi/lo bf16 pair (lora_hilo), so LoRA clients sit at the
# same floor.
TOL_MAX_REL = 2e-2
TOL_MEAN_REL = 2e-3
# IA3 backward with bf16 outputs: the operand g = dy*l (client.py:291-294, f32 in the
# reference) is itself rounded to bf16 once (the lo pass is reserved for f32 outputs, see
# below): measured 2.3e-3 mean.
TOL_IA3_BWD_MEAN_REL = 3e-3
# fp32 outputs (bf16 operands, fp32 accumulate): LoRA's s*x.A as hi + lo, IA3 backward's
# g*l as hi + lo with a second K pass (ia3_lo): measured <= 2e-5 max / 2e-5 mean at 13B
# shapes (vs ~1e-3 with a single bf16 intermediate).
TOL_F32_MAX_REL = 1e-3
TOL_F32_MEAN_REL = 1e-4
# LoRA weight gradients (ss_adapter_grads): the token contraction's operand s*x.A / s*g.B^T is
# a bf16 tensor-core operand (fp32 outputs).
TOL_GRAD_MEAN_REL = 3e-3
