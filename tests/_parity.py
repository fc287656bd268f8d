"""Shared helpers for GPU parity tests: run the CUDA path through the C ABI and gate it against the oracle.

Tolerance semantics (reading #17, north_star): an element passes when
    |gpu - oracle| <= tol * E
with E the oracle's magnitude envelope (E_m = mu|m| + |lr*lambda|(|s| sum_r |g_r| + beta_l |w|),
E_w = |w| + E_m: w - v is formed from |w| and every term of v); E >= |x| so this is plain relative
error whenever nothing cancels. Exact zeros
must be exact. Norms: relative 1e-6 against the oracle norm of the very buffer the kernel read.
"""
from __future__ import annotations

import numpy as np

import paper_1903_12650_b200 as P
from oracle import oracle as O
from synth import gen as G

TOL_F32 = 1e-5     # north_star: 1e-5 relative per element (fp32)
TOL_F16_DP = 2e-3  # north_star: 2e-3 when gradients are fp16 (P > 1: fp16 sums on the wire)
TOL_BF16_DP = 3e-2  # reading #18
TOL_NORM = 1e-6    # north_star: per-layer norms within 1e-6 relative


def torch_dtype(dtype: str):
    import torch

    return {"f32": torch.float32, "f16": torch.float16, "bf16": torch.int16}[dtype]


def to_dev(flat: np.ndarray, device: int = 0):
    import torch

    if flat.dtype == np.uint16:
        flat = flat.view(np.int16)
    return torch.from_numpy(np.ascontiguousarray(flat)).to(f"cuda:{device}")


def from_dev(t) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view(np.uint16) if a.dtype == np.int16 else a


def hp_kwargs(**kw):
    d = dict(base_lr=32.0, eta=1e-3, momentum=0.9, weight_decay=5e-5, eps=0.0, warmup_epochs=5.0, poly_power=2.0,
             global_batch=81920, grad_scale=1.0 / G.GRAD_PRESCALE, grad_dtype="f32")
    d.update(kw)
    return d


def oracle_hp(kw) -> O.HParams:
    import dataclasses

    names = {f.name for f in dataclasses.fields(O.HParams)}
    return O.HParams(**{k: v for k, v in kw.items() if k in names})


def gate(name: str, got, want, env, tol: float) -> float:
    """Max envelope error over all elements; asserts <= tol. Exact zeros are required to be exact."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    env = np.asarray(env, np.float64)
    diff = np.abs(got - want)
    with np.errstate(divide="ignore", invalid="ignore"):
        err = np.where(diff == 0, 0.0, diff / env)
    worst = float(np.max(err)) if err.size else 0.0
    assert np.all(np.isfinite(got)), f"{name}: non-finite output"
    assert worst <= tol, f"{name}: max envelope error {worst:.3e} > {tol:.1e} at {int(np.argmax(err))}"
    return worst


def gate_norms(name: str, got, want, tol: float = TOL_NORM) -> float:
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(got == want, 0.0, np.abs(got - want) / np.abs(want))
    worst = float(np.max(rel)) if rel.size else 0.0
    assert worst <= tol, f"{name}: norm rel error {worst:.3e} > {tol:.1e} at tensor {int(np.argmax(rel))}"
    return worst


class GpuStep:
    """One planned handle + device buffers for a layout."""

    def __init__(self, layout, device: int = 0, **kw):
        self.layout = layout
        self.kw = hp_kwargs(**kw)
        self.h = P.Lars([(t.numel, t.kind) for t in layout], device=device, **self.kw)
        self.device = device
        self.sizes = [t.numel for t in layout]
        self.kinds = [t.kind for t in layout]

    def upload(self, w, g, m):
        h = self.h
        self.w = to_dev(G.pack(w, h.offsets, h.padded_numel), self.device)
        self.g = to_dev(G.pack(g, h.offsets, h.padded_numel), self.device)
        self.m = to_dev(G.pack(m, h.offsets, h.padded_numel), self.device)

    def step(self, t: int):
        import torch

        self.h.lars_step(self.w, self.g, self.m, t)
        torch.cuda.synchronize(self.device)

    def state(self):
        h = self.h
        return (G.unpack(from_dev(self.w), h.offsets, self.sizes), G.unpack(from_dev(self.m), h.offsets, self.sizes))

    def check(self, t: int, w, g_ranks, m, tol: float = TOL_F32, tag: str = ""):
        """Runs the oracle on (w, g_ranks, m) — the exact pre-step state uploaded — and gates the GPU."""
        r = O.step(self.kinds, oracle_hp(self.kw), t, w, g_ranks, m)
        wg, mg = self.state()
        skipped = self.h.last_step_skipped()
        assert skipped == r.skipped, f"{tag}: skipped gpu={skipped} oracle={r.skipped}"
        wn, gn, lam, coef = self.h.last_norms()
        stats = {}
        if not r.skipped:
            stats["norm_w"] = gate_norms(f"{tag} ||w||", wn, r.w_norm)
            stats["norm_g"] = gate_norms(f"{tag} ||g||", gn, r.g_norm)
            stats["lambda"] = gate_norms(f"{tag} lambda", lam, r.lam, 1e-6)
            stats["m"] = gate(f"{tag} m", np.concatenate(mg), np.concatenate(r.m), np.concatenate(r.m_env), tol)
            stats["w"] = gate(f"{tag} w", np.concatenate(wg), np.concatenate(r.w), np.concatenate(r.w_env), tol)
        else:
            for a, b in zip(wg + mg, list(w) + list(m)):  # bitwise (a NaN weight stays the same NaN)
                assert np.array_equal(a.view(np.uint32), np.asarray(b, np.float32).view(np.uint32)), \
                    f"{tag}: skipped step modified state"
        return r, stats
