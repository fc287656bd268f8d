"""Static backward-order groups (LARS_SHARD_GROUPS; §III-C): host-side plan
properties, checked on host-only handles (no GPU). The greedy rule and its worked examples are SPEC.md's
`make_buckets` (scheduler module): "greedy accumulation in backward order; a group closes when its byte total
first reaches >= threshold; trailing segments form a final residual group"."""
from __future__ import annotations

import numpy as np
import pytest

from synth import layouts as LY

MiB = 1 << 20


def _handle(sizes_bytes_fwd=None, thr=4 * MiB, P=1, dt="f16", layout=None, **kw):
    import paper_1903_12650_b200 as PK

    esz = 4 if dt == "f32" else 2
    tensors = [(t.numel, t.kind) for t in layout] if layout is not None else \
        [(b // esz, 0) for b in sizes_bytes_fwd]
    return PK.Lars(tensors, device=-1, base_lr=1.0, grad_dtype=dt, nranks=P, shard_policy="groups",
                   group_bytes=thr, **kw)


def _members(h):
    return [list(range(g["last"], g["first"] - 1, -1)) for g in h.groups()]  # backward order


def test_spec_worked_examples():
    # SPEC.md make_buckets: segments listed in BACKWARD order; the layout is given in forward order
    # sizes [1,1,1,5] MiB (backward), threshold 4 MiB -> a single group [s0..s3]
    h = _handle([5 * MiB, MiB, MiB, MiB])
    assert _members(h) == [[3, 2, 1, 0]]
    # sizes [5,1] MiB (backward) -> [[s0], [s1]]: s0 alone meets the threshold, s1 is the residual
    h = _handle([MiB, 5 * MiB])
    assert _members(h) == [[1], [0]]
    # threshold above the total -> one group with every segment
    h = _handle([MiB, 5 * MiB], thr=100 * MiB)
    assert _members(h) == [[1, 0]]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("thr", [64 << 10, MiB, 4 * MiB, 1 << 40])
def test_group_plan_invariants(P, thr):
    lay = LY.resnet50()
    h = _handle(layout=lay, thr=thr, P=P)
    groups = h.groups()
    L, esz = len(lay), 2
    # coverage: every tensor in exactly one group; groups in backward order, contiguous tensor ranges
    seen = []
    for g in groups:
        seen.extend(range(g["last"], g["first"] - 1, -1))
    assert seen == list(range(L - 1, -1, -1))
    # greedy: every group but the residual reaches the threshold, and only with its last-added tensor
    for k, g in enumerate(groups):
        nbytes = [lay[l].numel * esz for l in range(g["first"], g["last"] + 1)]
        if k < len(groups) - 1:
            assert sum(nbytes) >= thr and sum(nbytes) - nbytes[0] < thr  # nbytes[0] = tensor `first`
        else:
            assert sum(nbytes) - nbytes[0] < thr
    # spans: contiguous, disjoint, in flat order opposite to backward order, padded to 64*P, covering
    # [0, padded_numel) — byte conservation (every gradient element communicated exactly once)
    spans = sorted((g["begin"], g["len"]) for g in groups)
    pos = 0
    for b, n in spans:
        assert b == pos and n % (64 * P) == 0 and n > 0
        pos += n
    assert pos == h.padded_numel
    assert [g["begin"] for g in groups] == sorted([g["begin"] for g in groups], reverse=True)
    for g in groups:
        for l in range(g["first"], g["last"] + 1):
            o = h.offsets[l]
            assert o % 64 == 0 and g["begin"] <= o and o + lay[l].numel <= g["begin"] + g["len"]
    # ownership: rank r owns slice r of every group; owner = slice of the tensor's first element
    owner = h.tensor_owner()
    for g in groups:
        c = g["len"] // P
        for l in range(g["first"], g["last"] + 1):
            assert owner[l] == (h.offsets[l] - g["begin"]) // c
    if P > 1:
        import paper_1903_12650_b200 as PK

        with pytest.raises(PK.LarsError):
            h.shard_range(0)  # not contiguous under the group policy


def test_group_policy_validation_and_hash():
    import paper_1903_12650_b200 as PK

    lay = LY.resnet50()
    a = _handle(layout=lay, thr=4 * MiB, P=4)
    b = _handle(layout=lay, thr=4 * MiB, P=4)
    c = _handle(layout=lay, thr=1 * MiB, P=4)
    assert a.layout_hash() == b.layout_hash() != c.layout_hash()
    assert len(c.groups()) > len(a.groups()) > 1
    with pytest.raises(PK.LarsError):
        _handle(layout=lay, thr=0, P=2)
    with pytest.raises(PK.LarsError):
        _handle(layout=lay, thr=MiB, P=2, buckets=4)  # bucketed NCCL schedule and groups exclude each other
    # the other policies report one group = the whole flat buffer
    d = PK.Lars([(t.numel, t.kind) for t in lay], device=-1, base_lr=1.0, nranks=4)
    assert d.groups() == [{"begin": 0, "len": d.padded_numel, "first": 0, "last": len(lay) - 1}]


def test_group_slices_balance():
    """Every rank gets exactly padded/P elements (slices of equal length in every group)."""
    lay = LY.random_layout(np.random.default_rng(5), 60)
    for P in (2, 3, 8):
        h = _handle(layout=lay, thr=256 << 10, P=P)
        per_rank = [sum(g["len"] // P for g in h.groups()) for _ in range(P)]
        assert len(set(per_rank)) == 1 and per_rank[0] * P == h.padded_numel


def _toy_trace():
    groups = [{"begin": 128, "len": 128, "first": 2, "last": 3}, {"begin": 0, "len": 128, "first": 0, "last": 1}]
    bwd = {3: 0.1, 2: 0.2, 1: 0.5, 0: 0.6}
    lib = {"ready": [0.0, 0.4], "rs_start": [0.25, 0.65], "rs_end": [0.3, 0.7], "applied": 0.9}
    return groups, bwd, lib


def test_validate_trace_accepts_a_correct_schedule_and_catches_injected_faults():
    from tools.overlap_trace import validate_trace

    groups, bwd, lib = _toy_trace()
    assert validate_trace(groups, bwd, lib, 4, 256) == []
    # (a) reduction of group 0 before its member 2 was written
    g2, b2, l2 = _toy_trace()
    b2[2] = 0.3
    assert any(v.startswith("(a)") for v in validate_trace(g2, b2, l2, 4, 256))
    # (b) launches out of group order
    g3, b3, l3 = _toy_trace()
    l3["rs_start"] = [0.65, 0.62]
    b3[0] = b3[1] = 0.0
    assert any(v.startswith("(b)") for v in validate_trace(g3, b3, l3, 4, 256))
    # (c) applied before a reduction ended
    g4, b4, l4 = _toy_trace()
    l4["applied"] = 0.68
    assert any(v.startswith("(c)") for v in validate_trace(g4, b4, l4, 4, 256))
    # (d) a tensor in two groups (byte conservation)
    g5, b5, l5 = _toy_trace()
    g5[1]["last"] = 2
    assert any(v.startswith("(d)") for v in validate_trace(g5, b5, l5, 4, 256))
    # (d) a span gap
    g6, b6, l6 = _toy_trace()
    g6[0]["begin"] = 192
    assert any(v.startswith("(d)") for v in validate_trace(g6, b6, l6, 4, 256))


def test_validate_trace_on_a_real_plan():
    from tools.overlap_trace import validate_trace

    lay = LY.resnet50()
    h = _handle(layout=lay, thr=MiB, P=4)
    groups = h.groups()
    t, bwd = 0.0, {}
    for g in groups:  # members written in backward order, then the group starts
        for l in range(g["last"], g["first"] - 1, -1):
            t += 0.01
            bwd[l] = t
    rs = [bwd[g["first"]] + 0.001 for g in groups]
    lib = {"ready": rs, "rs_start": rs, "rs_end": [x + 0.05 for x in rs], "applied": rs[-1] + 0.2}
    assert validate_trace(groups, bwd, lib, len(lay), h.padded_numel) == []
