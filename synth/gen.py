"""Seeded synthetic inputs for the LARS gradient-combine-and-update step.

This module is the ONLY code shared between the CUDA path's tests/bench and the oracle: it draws
random numbers and packs/unpacks flat buffers. It contains none of the method's arithmetic (no
schedule, no norms, no trust ratio, no update) — DESIGN.md §"Input recipe" states the recipe:

  * seed 100000 (``run_set_random_seed``), one independent NumPy stream per
    (purpose, rank, step, tensor) via ``SeedSequence([seed, purpose, rank, step, tensor])``;
  * weights: truncated normal, +-2 sigma, sigma = sqrt(2/fan_in) for weight-kind tensors
    ("initializer": "truncated_normal"; He scaling per SPEC.md:114);
    BN gamma = 1 + 0.1 N(0,1); BN beta / bias = 0.1 N(0,1) / 0.01 N(0,1);
  * gradients of rank r: N(0, (1e-2 sigma)^2) * 1024, rounded round-to-nearest-even to the wire
    dtype (fp16 per PAPER.md:183, bf16 optional, fp32 allowed at P=1); the library is then called
    with grad_scale s = 1/(1024 P) so the unscale is exact (power of two);
  * momentum: N(0, m_sigma^2) ("warmed-up" state) or zeros.
"""
from __future__ import annotations

import numpy as np

from .layouts import SEED, Tensor

PURPOSE_W, PURPOSE_G, PURPOSE_M, PURPOSE_INT = 1, 2, 3, 4
GRAD_PRESCALE = 1024.0


def _rng(purpose: int, rank: int, step: int, idx: int, seed: int = SEED) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed, purpose, rank, step, idx]))


def sigma_w(t: Tensor) -> float:
    return float(np.sqrt(2.0 / t.fan_in)) if t.kind == "weight" else 0.1


def _trunc_normal(rng: np.random.Generator, n: int, sigma: float) -> np.ndarray:
    x = rng.standard_normal(n)
    bad = np.abs(x) > 2.0
    while bad.any():
        x[bad] = rng.standard_normal(int(bad.sum()))
        bad = np.abs(x) > 2.0
    return x * sigma


def weights(layout: list[Tensor], seed: int = SEED) -> list[np.ndarray]:
    out = []
    for i, t in enumerate(layout):
        r = _rng(PURPOSE_W, 0, 0, i, seed)
        if t.kind == "weight":
            x = _trunc_normal(r, t.numel, sigma_w(t))
        elif t.kind == "bn_gamma":
            x = 1.0 + 0.1 * r.standard_normal(t.numel)
        elif t.kind == "bn_beta":
            x = 0.1 * r.standard_normal(t.numel)
        else:
            x = 0.01 * r.standard_normal(t.numel)
        out.append(x.astype(np.float32))
    return out


def to_bf16_bits(x32: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even (finite inputs)."""
    b = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return b.astype(np.uint16)


def _cast(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return x.astype(np.float32)
    if dtype == "f16":
        return x.astype(np.float32).astype(np.float16)  # numpy rounds RNE
    if dtype == "bf16":
        return to_bf16_bits(x.astype(np.float32))
    raise ValueError(dtype)


def grads(layout: list[Tensor], rank: int = 0, step: int = 0, dtype: str = "f32",
          seed: int = SEED, rel: float = 1e-2) -> list[np.ndarray]:
    """Rank ``rank``'s local gradient for ``step``: N(0,(rel*sigma_w)^2)*1024 in the wire dtype."""
    out = []
    for i, t in enumerate(layout):
        r = _rng(PURPOSE_G, rank, step, i, seed)
        out.append(_cast(r.standard_normal(t.numel) * (rel * sigma_w(t) * GRAD_PRESCALE), dtype))
    return out


def integer_grads(layout: list[Tensor], rank: int = 0, step: int = 0, dtype: str = "f16",
                  kmax: int = 64, seed: int = SEED) -> list[np.ndarray]:
    """Integer-valued gradients |k| <= kmax: any summation order is exact."""
    out = []
    for i, t in enumerate(layout):
        r = _rng(PURPOSE_INT, rank, step, i, seed)
        out.append(_cast(r.integers(-kmax, kmax + 1, t.numel).astype(np.float64), dtype))
    return out


def momentum(layout: list[Tensor], m_sigma: float = 0.0, seed: int = SEED) -> list[np.ndarray]:
    out = []
    for i, t in enumerate(layout):
        if m_sigma == 0.0:
            out.append(np.zeros(t.numel, np.float32))
        else:
            r = _rng(PURPOSE_M, 0, 0, i, seed)
            out.append((r.standard_normal(t.numel) * m_sigma * sigma_w(t)).astype(np.float32))
    return out


def pack(arrays: list[np.ndarray], offsets, padded_numel: int) -> np.ndarray:
    """Place per-tensor arrays into a zero-padded flat buffer at the library's offsets."""
    flat = np.zeros(int(padded_numel), dtype=arrays[0].dtype)
    for a, o in zip(arrays, offsets):
        flat[int(o):int(o) + a.size] = a
    return flat


def unpack(flat: np.ndarray, offsets, sizes) -> list[np.ndarray]:
    return [flat[int(o):int(o) + int(n)].copy() for o, n in zip(offsets, sizes)]
