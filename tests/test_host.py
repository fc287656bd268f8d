"""Host-side tests of the C-ABI library (no GPU): exports, planner, schedule, errors. CPU only."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_1903_12650_b200 as P
from oracle import oracle as O
from synth import layouts as LY


def desc(layout):
    return [(t.numel, t.kind) for t in layout]


def test_library_exports_every_declared_symbol():
    lib = P.load_library()
    names = P.declared_functions()
    assert {"lars_init", "lars_step", "dp_allreduce_lars_step", "lars_comm_init", "lars_destroy"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
        assert ctypes.cast(getattr(lib, n), ctypes.c_void_p).value


def test_library_is_sm100a_and_links_torch_nccl():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", P.lars.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", P.lars.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl.so.2" in ldd and "nvidia/nccl/lib" in ldd


@pytest.mark.parametrize("name,P_", [("tiny", 1), ("resnet50", 1), ("resnet50", 2), ("resnet50", 8),
                                     ("resnet152", 4), ("resnet50_4ch", 1)])
def test_layout_offsets_aligned_disjoint_and_shards(name, P_):
    lay = LY.by_name(name)
    h = P.Lars(desc(lay), device=-1, base_lr=32.0, nranks=P_, shard_policy="lpt")
    offs, n = np.array(h.offsets), np.array([t.numel for t in lay])
    assert (offs % 64 == 0).all()
    order = np.argsort(offs)
    ends = offs[order] + n[order]
    assert (ends[:-1] <= offs[order][1:]).all()            # non-overlapping
    assert ends.max() <= h.padded_numel
    owner = h.tensor_owner()
    S = h.padded_numel // P_
    assert h.padded_numel == S * P_ and S % 64 == 0
    for r in range(P_):
        b, e = h.shard_range(r)
        assert (b, e) == (r * S, (r + 1) * S)
    for l in range(len(lay)):                              # whole tensors inside their owner's shard
        b, e = h.shard_range(owner[l])
        assert b <= offs[l] and offs[l] + n[l] <= e
    assert h.padded_numel - n.sum() <= 63 * len(lay) + 64 * P_  # alignment padding only at P=1
    if P_ > 1 and name != "tiny":
        assert h.padded_numel / n.sum() - 1 < 1e-3         # LPT padding (0.008% at P=8)


def test_lpt_is_deterministic_and_hash_identifies_plan():
    lay = desc(LY.resnet50())
    a = P.Lars(lay, device=-1, base_lr=32.0, nranks=8)
    b = P.Lars(lay, device=-1, base_lr=32.0, nranks=8)
    assert a.offsets == b.offsets and a.layout_hash() == b.layout_hash()
    c = P.Lars(lay[:-1], device=-1, base_lr=32.0, nranks=8)
    d = P.Lars(lay, device=-1, base_lr=32.0, nranks=4)
    e = P.Lars(lay, device=-1, base_lr=16.0, nranks=8)
    assert len({a.layout_hash(), c.layout_hash(), d.layout_hash(), e.layout_hash()}) == 4


def test_schedule_matches_oracle_for_every_iteration():
    for kw in (dict(base_lr=32.0), dict(base_lr=8.0, poly_power=1.0), dict(base_lr=3.0, warmup_epochs=2.5),
               dict(base_lr=1.0, global_batch=32768, poly_power=0.0), dict(base_lr=0.5, warmup_epochs=0.0),
               dict(base_lr=8.0, decay="step", milestones=(30, 60, 80), step_gamma=0.1),
               dict(base_lr=2.0, decay="step", milestones=(0.5, 45.3), step_gamma=0.5, warmup_epochs=0.0)):
        h = P.Lars([(10, "weight")], device=-1, **kw)
        hp = O.HParams(**{k: v for k, v in kw.items()})
        ipe, T, W = O.schedule(hp)
        assert (h.ipe, h.total_iters, h.warmup_iters) == (ipe, T, W)
        lib = np.array([h.lr_at(t) for t in range(T)])
        ora = np.array([O.lr_at(hp, t) for t in range(T)])
        assert np.array_equal(lib, ora) or np.max(np.abs(lib - ora) / ora) < 4.5e-16


def test_schedule_paper_counts():
    h = P.Lars([(10, "weight")], device=-1, base_lr=32.0)
    assert (h.ipe, h.total_iters, h.warmup_iters) == (16, 1440, 80)
    assert h.lr_at(79) == 32.0 and h.lr_at(0) == 0.4


def test_error_codes():
    with pytest.raises(P.LarsError) as e:
        P.Lars([(10, "weight")], device=-1, base_lr=32.0).lr_at(1440)
    assert e.value.status == 3  # LARS_ERR_ITER_RANGE
    with pytest.raises(P.LarsError) as e:
        P.Lars([(0, "weight")], device=-1, base_lr=1.0)
    assert e.value.status == 2  # numel <= 0
    with pytest.raises(P.LarsError) as e:
        P.Lars([(5, 7)], device=-1, base_lr=1.0)
    assert e.value.status == 2  # unknown kind
    with pytest.raises(P.LarsError) as e:
        P.Lars([], device=-1, base_lr=1.0)
    assert e.value.status == 2  # empty layout
    for bad in (dict(base_lr=0.0), dict(base_lr=1.0, momentum=1.0), dict(base_lr=1.0, weight_decay=-1.0),
                dict(base_lr=1.0, global_batch=0), dict(base_lr=float("nan")), dict(base_lr=1.0, grad_scale=0.0), dict(base_lr=1.0, grad_scale=2.0 ** 65),
                dict(base_lr=1.0, warmup_epochs=1000.0), dict(base_lr=1.0, nranks=0)):
        with pytest.raises(P.LarsError) as e:
            P.Lars([(5, "weight")], device=-1, **bad)
        assert e.value.status == 1, bad
    h = P.Lars([(5, "weight")], device=-1, base_lr=1.0)
    with pytest.raises(P.LarsError) as e:
        h.lars_step(256, 256, 256, 0, stream=0)
    assert e.value.status == 9  # host-only handle
    with pytest.raises(P.LarsError) as e:
        h.shard_range(1)
    assert e.value.status == 1


def test_product_path_does_not_import_oracle():
    import pathlib
    import re

    pkg = pathlib.Path(P.__file__).parent
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cpp")) + list(pkg.rglob("*.h")):
        assert not re.search(r"^\s*(from|import)\s+oracle|#include.*oracle", f.read_text(), re.M), f


def test_half_weights_flag_validation():
    """LARS_FLAG_HALF_WEIGHTS needs a 16-bit wire dtype and excludes the group and bucket schedules (P = 1 is
    allowed: a one-rank communicator runs the data-parallel step)."""
    import paper_1903_12650_b200 as PK
    from synth import layouts as LY

    lay = [(t.numel, t.kind) for t in LY.tiny()]
    ok = PK.Lars(lay, device=-1, base_lr=1.0, nranks=2, grad_dtype="f16", flags=PK.lars.FLAG_HALF_WEIGHTS)
    assert ok.padded_numel > 0
    assert PK.Lars(lay, device=-1, base_lr=1.0, nranks=1, grad_dtype="f16", flags=PK.lars.FLAG_HALF_WEIGHTS).n == 3
    for kw in (dict(nranks=1, grad_dtype="f32"), dict(nranks=2, grad_dtype="f32"),
               dict(nranks=2, grad_dtype="bf16", shard_policy="groups"), dict(nranks=2, grad_dtype="f16", buckets=4)):
        with pytest.raises(PK.LarsError):
            PK.Lars(lay, device=-1, base_lr=1.0, flags=PK.lars.FLAG_HALF_WEIGHTS, **kw)
