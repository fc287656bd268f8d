"""Work-list invariants the kernels rely on for in-bounds, race-free access (lars_check_work), checked on the
host for every layout family, rank count and shard policy: tiles partition the segments with no empty tile,
a tile's chunks fit the shared-memory partial arrays, segments and chunks tile every tensor piece exactly
(aligned for the 256-bit accesses), and nothing lies outside the rank's shard. The kernels index w, g and m
only through these chunks, so this is the host half of the memory-safety argument (the device half is the
-DLARS_DEVICE_CHECKS build, tools/checked_build.py). CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1903_12650_b200 as PK
from synth import layouts as LY


def _handle(lay, **kw):
    return PK.Lars([(t.numel, t.kind) for t in lay], device=-1, base_lr=1.0, **kw)


def _check_all(h, P):
    assert h.check_work(-1) == "ok"
    for r in range(P):
        assert h.check_work(r) == "ok", r


@pytest.mark.parametrize("name", ["tiny", "resnet50", "resnet152"])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("policy", ["contiguous", "lpt", "groups"])
def test_model_layouts(name, P, policy):
    h = _handle(LY.by_name(name), nranks=P, shard_policy=policy, grad_dtype="f16")
    _check_all(h, P)
    h.close()


@pytest.mark.parametrize("seed", range(12))
def test_random_ragged_layouts(seed):
    rng = np.random.default_rng(500 + seed)
    lay = LY.random_layout(rng, int(rng.integers(1, 200)), max_numel=int(rng.choice([70, 5000, 300000])))
    P = int(rng.choice([1, 2, 3, 5, 8]))
    policy = str(rng.choice(["contiguous", "lpt", "groups"]))
    h = _handle(lay, nranks=P, shard_policy=policy, tile_elems=int(rng.choice([0, 64, 512, 4096, 65536])),
                group_bytes=int(rng.choice([1 << 12, 1 << 16, 1 << 22])))
    _check_all(h, P)
    h.close()


@pytest.mark.parametrize("variant", ["uniform", "loguniform", "zipf", "giant"])
def test_skewed_1b_layouts(variant):
    """configs[4]: 1,000 tensors, 10^9 parameters (chunk-cap-bound tile budgets, huge split layers)."""
    lay = LY.skew1b(variant)
    for P in (1, 8):
        h = _handle(lay, nranks=P, grad_dtype="f16")
        _check_all(h, P)
        h.close()


def test_checker_rejects_nothing_it_should_not_and_reports_reason():
    h = _handle(LY.tiny())
    assert h.check_work() == "ok"
    with pytest.raises(PK.LarsError) as e:
        h.check_work(5)  # rank outside the plan
    assert e.value.status == 1
    h.close()
