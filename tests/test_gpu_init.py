"""Parallel deterministic initialization on the GPU (§III-B-1) against
the oracle's counter-based definition, plus the properties that make the broadcast unnecessary: the
weights are a pure function of (seed, layer, element) — independent of the launch configuration."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from synth import layouts as LY
from tests._parity import from_dev

pytestmark = pytest.mark.gpu


def _handle(lay, **kw):
    import paper_1903_12650_b200 as P

    return P.Lars([(t.numel, t.kind, t.fan_in) for t in lay], device=0, base_lr=32.0, **kw)


@pytest.mark.parametrize("name", ["tiny", "resnet50", "random"])
def test_init_weights_matches_oracle(name):
    import torch

    lay = LY.random_layout(np.random.default_rng(31), 40) if name == "random" else LY.by_name(name)
    if name == "resnet50":
        lay = lay[:60]  # the oracle's pure-Python Philox is slow; 60 layers cover every kind
    h = _handle(lay)
    w = torch.full((h.padded_numel,), float("nan"), dtype=torch.float32, device="cuda")
    h.init_weights(w, 100000)
    torch.cuda.synchronize()
    got = from_dev(w)
    want = O.init_weights([t.kind for t in lay], [t.numel for t in lay], [t.fan_in for t in lay], 100000)
    covered = np.zeros(h.padded_numel, bool)
    for l, t in enumerate(lay):
        g = got[h.offsets[l]:h.offsets[l] + t.numel].astype(np.float64)
        np.testing.assert_allclose(g, want[l], rtol=3e-7, atol=1e-30, err_msg=f"layer {l} ({t.kind})")
        covered[h.offsets[l]:h.offsets[l] + t.numel] = True
    assert np.isnan(got[~covered]).all()  # padding untouched


def test_init_weights_independent_of_launch_configuration():
    import torch

    lay = LY.resnet50()
    a, b = _handle(lay), _handle(lay, tile_elems=1 << 20)  # different tiles / grid
    assert a.work_info()["tiles"] != b.work_info()["tiles"]
    wa = torch.empty(a.padded_numel, dtype=torch.float32, device="cuda")
    wb = torch.empty(b.padded_numel, dtype=torch.float32, device="cuda")
    a.init_weights(wa, 7)
    b.init_weights(wb, 7)
    torch.cuda.synchronize()
    assert torch.equal(wa, wb)
    wc = torch.empty_like(wa)
    a.init_weights(wc, 8)
    torch.cuda.synchronize()
    assert not torch.equal(wa, wc)
    # statistics of the largest layer (2,359,296 weights, fan_in 4,608): truncated normal, sigma sqrt(2/4608)
    big = int(np.argmax([t.numel for t in lay]))
    z = wa[a.offsets[big]:a.offsets[big] + lay[big].numel].double() / np.sqrt(2.0 / lay[big].fan_in)
    assert float(z.abs().max()) <= 2.0 + 1e-6 and abs(float(z.mean())) < 2e-3
    assert abs(float(z.std()) - 0.8796256610342398) < 2e-3
