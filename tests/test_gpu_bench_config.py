"""Parity of the exact configuration bench.py times (BASELINE configs[1]) and of the step's degenerate
inputs, against the float64 oracle.

* bench.py's N = 1 handle — ResNet-50, 161 tensors, fp32 gradients, LARS_FLAG_CARRY_WNORM, the same
  hyper-parameters and the same one-tile-per-resident-CTA plan — chained over t = 719..721 with bench.py's
  inputs: the first step computes ||w|| from w, the next two consume the norms K2 carried. Every step is
  gated element by element (1e-5 envelope) and per layer (norms, lambda 1e-6) against the oracle run on the
  GPU's own pre-step state.
* a weight-kind layer with ||w|| = 0 (lambda = 1), a non-finite WEIGHT element (whole step
  skipped, SPEC.md:187 / reading #13), and eps > 0 including the zero-gradient fallback.
"""
from __future__ import annotations

import numpy as np
import pytest

from synth import gen as G
from synth import layouts as LY
from tests._parity import TOL_F32, GpuStep

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def test_benched_configuration_three_step_chain():
    torch = _torch()
    import bench
    import paper_1903_12650_b200 as PK

    lay = LY.resnet50()
    # bench.py's mk(FLAG_CARRY_WNORM) at N = 1, verbatim arguments
    kw = dict(grad_dtype="f32", nranks=1, grad_scale=1.0 / (G.GRAD_PRESCALE * 1), flags=PK.lars.FLAG_CARRY_WNORM,
              buckets=0, **bench.HP)
    s = GpuStep(lay, **kw)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert s.h.work_info()["tiles"] == sms * 4  # one tile per resident K1/K2 CTA (592 on B200)
    w, g, m = G.weights(lay), G.grads(lay, 0, 0, "f32"), G.momentum(lay, 1e-3)  # bench.py's inputs
    s.upload(w, g, m)
    for t in (bench.T0, bench.T0 + 1, bench.T0 + 2):
        pre_w, pre_m = s.state()
        s.step(t)
        r, st = s.check(t, pre_w, [g], pre_m, TOL_F32, tag=f"bench config t={t}")
        assert not r.skipped and st["w"] <= TOL_F32 and st["norm_w"] <= 1e-6
        print("bench config", t, st)


def test_zero_weight_layer_trust_ratio_one():
    """SURVEY P4(b) through the GPU: a weight-kind layer whose weights are all zero gets lambda = 1, so its
    update is the plain scheduled-lr momentum step on s*g (beta*w = 0)."""
    _torch()
    lay = [LY.Tensor("zero_conv", 4608, "weight", 512)] + LY.tiny()
    s = GpuStep(lay, grad_dtype="f16")
    w, g, m = G.weights(lay), G.grads(lay, 0, 4, "f16"), G.momentum(lay, 1e-3)
    w[0] = np.zeros(4608, np.float32)
    s.upload(w, g, m)
    s.step(300)
    r, _ = s.check(300, w, [g], m, TOL_F32, tag="zero weight layer")
    wn, _, lam, coef = s.h.last_norms()
    assert wn[0] == 0.0 and lam[0] == 1.0 and r.lam[0] == 1.0
    assert coef[0] == float(np.float32(s.h.lr_at(300)))


@pytest.mark.parametrize("bad", [np.nan, np.inf])
@pytest.mark.parametrize("flags", [0, 1])
def test_nonfinite_weight_skips_whole_step(bad, flags):
    """A non-finite master weight makes ||w|| non-finite: the whole step is skipped (w, m bitwise untouched)
    — also in carry mode, where the first step after a new w buffer recomputes ||w|| from w."""
    _torch()
    lay = LY.tiny() + LY.random_layout(np.random.default_rng(5), 9)
    s = GpuStep(lay, flags=flags)
    w, g, m = G.weights(lay), G.grads(lay, 0, 6, "f32"), G.momentum(lay, 1e-3)
    w[1] = w[1].copy()
    w[1][123] = bad
    s.upload(w, g, m)
    s.step(90)
    r, _ = s.check(90, w, [g], m, TOL_F32, tag="non-finite w")
    assert r.skipped and s.h.last_step_skipped()


@pytest.mark.parametrize("eps", [1e-8, 1e-3])
def test_eps_guard(eps):
    """eps > 0 (reading #1: lambda = eta*||w|| / (||G|| + beta*||w|| + eps)); with weight_decay = 0 a
    weight-kind layer with a zero gradient has denominator = eps and falls back to lambda = 1."""
    _torch()
    lay = LY.tiny() + LY.random_layout(np.random.default_rng(9), 12)
    for wd in (0.0, 5e-5):
        s = GpuStep(lay, grad_dtype="f16", eps=eps, weight_decay=wd)
        w, g, m = G.weights(lay), G.grads(lay, 0, 7, "f16"), G.momentum(lay, 1e-3)
        g[0] = np.zeros_like(g[0])  # conv1: weight kind, zero gradient
        s.upload(w, g, m)
        s.step(500)
        r, _ = s.check(500, w, [g], m, TOL_F32, tag=f"eps={eps} wd={wd}")
        lam = s.h.last_norms()[2]
        if wd == 0.0:
            assert lam[0] == 1.0 and r.lam[0] == 1.0
        else:
            assert lam[0] == pytest.approx(1e-3 / (wd + eps / r.w_norm[0]), rel=1e-12)
        s.h.close()
