"""Device-side seeded synthetic inputs for the very large layouts (configs[4]: 10^9 params), where
generating on the host would dominate the test time. Same recipe as synth/gen.py (no method arithmetic:
random numbers only), drawn with a seeded torch CUDA generator per (purpose, rank, step, tensor).
Sampled tensors are copied back to the host to feed the oracle."""
from __future__ import annotations

import math

from .gen import GRAD_PRESCALE, PURPOSE_G, PURPOSE_M, PURPOSE_W, sigma_w
from .layouts import SEED


def _gen(device, purpose: int, rank: int, step: int, idx: int, seed: int = SEED):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + purpose * 10_007 + rank * 101 + step) * 1_000_033 + idx)
    return g


def fill_weights(flat, layout, offsets, seed: int = SEED) -> None:
    import torch

    for i, t in enumerate(layout):
        x = flat[offsets[i]:offsets[i] + t.numel]
        gen = _gen(flat.device, PURPOSE_W, 0, 0, i, seed)
        if t.kind == "weight":
            s = sigma_w(t)
            torch.nn.init.trunc_normal_(x, 0.0, s, -2 * s, 2 * s, generator=gen)
        else:
            x.normal_(1.0 if t.kind == "bn_gamma" else 0.0, 0.1, generator=gen)


def fill_grads(flat, layout, offsets, rank: int = 0, step: int = 0, seed: int = SEED, rel: float = 1e-2) -> None:
    """flat: float32 / float16 / bfloat16 device tensor; values N(0, (rel*sigma)^2) * 1024 (RNE cast)."""
    import torch

    for i, t in enumerate(layout):
        gen = _gen(flat.device, PURPOSE_G, rank, step, i, seed)
        v = torch.empty(t.numel, device=flat.device, dtype=torch.float32)
        v.normal_(0.0, rel * sigma_w(t) * GRAD_PRESCALE, generator=gen)
        flat[offsets[i]:offsets[i] + t.numel] = v.to(flat.dtype)


def fill_momentum(flat, layout, offsets, m_sigma: float = 1e-3, seed: int = SEED) -> None:
    for i, t in enumerate(layout):
        gen = _gen(flat.device, PURPOSE_M, 0, 0, i, seed)
        flat[offsets[i]:offsets[i] + t.numel].normal_(0.0, m_sigma * sigma_w(t), generator=gen)


assert math.isfinite(GRAD_PRESCALE)
