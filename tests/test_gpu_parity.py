"""Single-GPU parity: the CUDA path (through the C ABI) vs the float64 oracle on the same seeded inputs.

Covers BASELINE.json configs[0] (tiny, 5 iterations across the warm-up boundary) and configs[1]
(ResNet-50 layout, fp32 gradients, full size, the launch configuration bench.py times), random ragged
layouts, every gradient dtype, the degenerate cases (zero gradients, non-finite gradients, constant
tensors, 1-element tensors, one tensor spanning many tiles), determinism, CUDA-graph capture and the
host-gradient entry point.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from synth import gen as G
from synth import layouts as LY
from tests._parity import TOL_F32, GpuStep, from_dev, gate, hp_kwargs, oracle_hp, to_dev

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
def test_tiny_five_iterations_across_warmup(dtype):
    """configs[0]: 3 layers, t = 78..82 straddles W = 80; m = 0 at t = 78, then chained."""
    _torch()
    lay = LY.tiny()
    s = GpuStep(lay, grad_dtype=dtype)
    w0, m0 = G.weights(lay), G.momentum(lay)
    s.upload(w0, G.grads(lay, 0, 78, dtype), m0)
    ow, om = [x.astype(np.float64) for x in w0], [x.astype(np.float64) for x in m0]
    for t in range(78, 83):
        g = G.grads(lay, 0, t, dtype)
        pre_w, pre_m = s.state()
        s.g = to_dev(G.pack(g, s.h.offsets, s.h.padded_numel))
        s.step(t)
        r, st = s.check(t, pre_w, [g], pre_m, TOL_F32, tag=f"tiny {dtype} t={t}")
        assert r.lr == s.h.lr_at(t)
        chained = O.step(s.kinds, oracle_hp(s.kw), t, ow, [g], om)
        ow, om = chained.w, chained.m
    wg, mg = s.state()
    gate("chained w", np.concatenate(wg), np.concatenate(ow), np.concatenate(chained.w_env), 1e-4)


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LARS_TEST_SEEDS", "6"))))
def test_random_ragged_layouts(dtype, seed):
    _torch()
    rng = np.random.default_rng(1000 + seed)
    lay = LY.random_layout(rng, int(rng.integers(1, 60)), max_numel=int(rng.choice([70, 5000, 40000])))
    kw = dict(grad_dtype=dtype, momentum=float(rng.choice([0.0, 0.9])),
              weight_decay=float(rng.choice([0.0, 5e-5, 1e-4])), tile_elems=int(rng.choice([64, 512, 4096])))
    s = GpuStep(lay, **kw)
    w, g, m = G.weights(lay, seed=seed), G.grads(lay, 0, seed, dtype, seed=seed), G.momentum(lay, 1e-3, seed=seed)
    s.upload(w, g, m)
    t = int(rng.integers(0, 1440))
    s.step(t)
    s.check(t, w, [g], m, TOL_F32, tag=f"random seed={seed} {dtype} t={t}")


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_resnet50_full_size(dtype):
    """configs[1]: 161 tensors, 25,557,032 params, t = 719 with a warmed-up momentum buffer."""
    _torch()
    lay = LY.resnet50()
    s = GpuStep(lay, grad_dtype=dtype)
    w, g, m = G.weights(lay), G.grads(lay, 0, 719, dtype), G.momentum(lay, 1e-3)
    s.upload(w, g, m)
    s.step(719)
    _, st = s.check(719, w, [g], m, TOL_F32, tag=f"R50 {dtype}")
    print("R50", dtype, st)


def test_zero_gradient_zero_decay_leaves_weights_bitwise():
    """north_star invariant."""
    _torch()
    lay = LY.tiny() + LY.random_layout(np.random.default_rng(3), 20)
    s = GpuStep(lay, weight_decay=0.0)
    w = G.weights(lay)
    zeros = [np.zeros(t.numel, np.float32) for t in lay]
    for t in (0, 79, 80, 1439):
        s.upload(w, zeros, zeros)
        s.step(t)
        wg, mg = s.state()
        assert not s.h.last_step_skipped()
        for a, b in zip(wg, w):
            assert np.array_equal(a, b)
        assert not any(x.any() for x in mg)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_nonfinite_gradient_skips_whole_step(bad, dtype):
    _torch()
    lay = LY.tiny()
    s = GpuStep(lay, grad_dtype=dtype)
    w, g, m = G.weights(lay), G.grads(lay, 0, 5, dtype), G.momentum(lay, 1e-3)
    g[1] = g[1].copy()
    g[1][500] = bad
    s.upload(w, g, m)
    s.step(100)
    s.check(100, w, [g], m, tag="nonfinite")
    assert s.h.last_step_skipped()
    g2 = G.grads(lay, 0, 6, dtype)  # the next clean step is not stuck
    s.g = to_dev(G.pack(g2, s.h.offsets, s.h.padded_numel))
    s.step(101)
    assert not s.h.last_step_skipped()
    s.check(101, w, [g2], m, tag="after skip")


def test_constant_tensors_exact_norms_and_trust_ratio():
    """4,096 x 0.5 -> ||w|| = 32 bitwise; g = 2^-10 -> 1/16; lambda = 320/641."""
    _torch()
    lay = [LY.Tensor("c", 4096, "weight", 64)]
    s = GpuStep(lay, grad_dtype="f16", grad_scale=1.0)
    s.upload([np.full(4096, 0.5, np.float32)], [np.full(4096, 2.0 ** -10, np.float16)], [np.zeros(4096, np.float32)])
    s.step(0)
    wn, gn, lam, coef = s.h.last_norms()
    assert wn[0] == 32.0 and gn[0] == 0.0625
    assert abs(lam[0] - 320 / 641) <= 2 ** -52
    assert coef[0] == float(np.float32(0.4 * lam[0]))


def test_skip_kind_vanilla_sgd():
    """mu=0, lr=0.1, w=1, g=2 -> 0.8 (fp32, 1 ulp)."""
    _torch()
    lay = [LY.Tensor("b", 1, "bias", 1), LY.Tensor("bn", 3, "bn_gamma", 1)]
    s = GpuStep(lay, base_lr=0.1, warmup_epochs=0.0, poly_power=0.0, momentum=0.0, grad_scale=1.0)
    s.upload([np.ones(1, np.float32), np.ones(3, np.float32)], [np.full(1, 2.0, np.float32), np.full(3, 2.0, np.float32)],
             [np.zeros(1, np.float32), np.zeros(3, np.float32)])
    s.step(7)
    wg, _ = s.state()
    assert abs(float(wg[0][0]) - 0.8) <= np.spacing(np.float32(0.8)) and (wg[1] == wg[0][0]).all()


def test_single_tensor_spanning_many_tiles():
    _torch()
    lay = [LY.Tensor("big", (1 << 25) + 13, "weight", 4608), LY.Tensor("b", 1, "bias", 1),
           LY.Tensor("g", 77, "bn_gamma", 77)]
    s = GpuStep(lay, grad_dtype="f16")
    w, g, m = G.weights(lay), G.grads(lay, 0, 3, "f16"), G.momentum(lay, 1e-3)
    s.upload(w, g, m)
    s.step(900)
    s.check(900, w, [g], m, tag="big tensor")


def test_deterministic_bitwise_rerun():
    _torch()
    lay = LY.resnet50()[:60]
    outs = []
    for _ in range(2):
        s = GpuStep(lay, grad_dtype="f16")
        s.upload(G.weights(lay), G.grads(lay, 0, 1, "f16"), G.momentum(lay, 1e-3))
        s.step(300)
        outs.append((from_dev(s.w), from_dev(s.m), s.h.last_norms()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_cuda_graph_capture_matches_eager():
    torch = _torch()
    lay = LY.resnet50()[:40]
    a, b = GpuStep(lay), GpuStep(lay)
    w, g, m = G.weights(lay), G.grads(lay, 0, 2, "f32"), G.momentum(lay, 1e-3)
    a.upload(w, g, m)
    b.upload(w, g, m)
    a.step(500)
    stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            b.h.lars_step(b.w, b.g, b.m, 500, stream=stream)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(a.w, b.w) and torch.equal(a.m, b.m)


def test_host_gradient_entry_point():
    torch = _torch()
    lay = LY.resnet50()[:30]
    a, b = GpuStep(lay, grad_dtype="f16"), GpuStep(lay, grad_dtype="f16")
    w, g, m = G.weights(lay), G.grads(lay, 0, 2, "f16"), G.momentum(lay, 1e-3)
    a.upload(w, g, m)
    b.upload(w, g, m)
    a.step(81)
    g_host = torch.from_numpy(G.pack(g, b.h.offsets, b.h.padded_numel)).pin_memory()
    b.h.lars_step_host_grad(b.w, g_host, b.m, 81)
    torch.cuda.synchronize()
    assert torch.equal(a.w, b.w) and torch.equal(a.m, b.m)
    assert not b.h.last_step_skipped()
    # consecutive host-gradient steps, issued without synchronizing: the library's two staging buffers and
    # copy stream (the next step's copy overlaps this step) give bitwise the device-gradient result, and a
    # non-finite host gradient still skips its own step only
    hosts = [torch.from_numpy(G.pack(G.grads(lay, 0, 3 + k, "f16"), b.h.offsets, b.h.padded_numel)).pin_memory()
             for k in range(5)]
    hosts[3][b.h.offsets[2] + 1] = float("nan")
    for k in range(5):
        b.h.lars_step_host_grad(b.w, hosts[k], b.m, 82 + k)
    torch.cuda.synchronize()
    assert not b.h.last_step_skipped()
    for k in range(5):
        a.g.copy_(hosts[k])
        a.step(82 + k)
        torch.cuda.synchronize()
        assert a.h.last_step_skipped() == (k == 3)
    assert torch.equal(a.w, b.w) and torch.equal(a.m, b.m)


def test_device_argument_errors():
    torch = _torch()
    import paper_1903_12650_b200 as P

    lay = LY.tiny()
    s = GpuStep(lay)
    s.upload(G.weights(lay), G.grads(lay), G.momentum(lay))
    with pytest.raises(P.LarsError) as e:
        s.h.lars_step(s.w.data_ptr() + 4, s.g, s.m, 0)
    assert e.value.status == 4
    with pytest.raises(P.LarsError) as e:
        s.h.lars_step(s.w, s.g, s.m, 1440)
    assert e.value.status == 3
    with pytest.raises(P.LarsError) as e:
        s.h.dp_allreduce_lars_step(s.w, s.g, s.m, 0)
    assert e.value.status == 8
    with pytest.raises(P.LarsError) as e:
        s.h.comm_init(0, 2, bytes(128))
    assert e.value.status == 1  # planned for nranks = 1: nranks must match the plan
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_carried_weight_norms_chain(dtype):
    """LARS_FLAG_CARRY_WNORM: K2 leaves sum(w_new^2) per chunk, the next K1 reads only g. Each step of a
    5-step chain (first step recomputes, the rest carry) is checked against the oracle from the GPU's
    pre-step state, and against a non-carry handle fed the same inputs."""
    torch = _torch()
    lay = LY.resnet50()[:70] + LY.random_layout(np.random.default_rng(21), 15)
    a = GpuStep(lay, grad_dtype=dtype, flags=1)
    b = GpuStep(lay, grad_dtype=dtype)
    w, m = G.weights(lay), G.momentum(lay, 1e-3)
    a.upload(w, G.grads(lay, 0, 0, dtype), m)
    b.upload(w, G.grads(lay, 0, 0, dtype), m)
    for t in range(300, 305):
        g = G.grads(lay, 0, t, dtype)
        a.g = to_dev(G.pack(g, a.h.offsets, a.h.padded_numel))
        b.g = to_dev(G.pack(g, b.h.offsets, b.h.padded_numel))
        pre_w, pre_m = a.state()
        a.step(t)
        b.step(t)
        a.check(t, pre_w, [g], pre_m, TOL_F32, tag=f"carry {dtype} t={t}")
        wa, na = a.h.last_norms()[0], None
        wb = b.h.last_norms()[0]
        assert np.allclose(wa, wb, rtol=1e-13, atol=0)
    torch.cuda.synchronize()


def test_carried_norms_invalidation():
    torch = _torch()
    lay = LY.tiny()
    s = GpuStep(lay, flags=1)
    w, g, m = G.weights(lay), G.grads(lay, 0, 1, "f32"), G.momentum(lay, 1e-3)
    s.upload(w, g, m)
    s.step(100)
    s.step(101)
    with torch.no_grad():
        s.w.mul_(2.0)  # modified in place behind the library's back
    s.h.invalidate_carried_norms()
    pre_w, pre_m = s.state()
    s.step(102)
    s.check(102, pre_w, [g], pre_m, TOL_F32, tag="after invalidate")
    # a different weight buffer invalidates automatically
    s.w = s.w.clone() * 0.5
    pre_w, pre_m = s.state()
    s.step(103)
    s.check(103, pre_w, [g], pre_m, TOL_F32, tag="new w buffer")


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("form", ["velocity", "apply"])
def test_variants_step_decay_and_momentum_form(dtype, form):
    """NEXT-f3 variants: step decay across a milestone and SPEC.md:186's lr-at-apply
    momentum form, chained over 5 steps with carried norms; each step against the oracle."""
    _torch()
    lay = LY.tiny() + LY.random_layout(np.random.default_rng(41), 12)
    s = GpuStep(lay, grad_dtype=dtype, decay="step", milestones=(30, 60), step_gamma=0.1, momentum_form=form,
                flags=1)
    s.upload(G.weights(lay), G.grads(lay, 0, 0, dtype), G.momentum(lay, 1e-3))
    for t in range(478, 483):  # epoch-30 milestone at t = 480
        g = G.grads(lay, 0, t, dtype)
        s.g = to_dev(G.pack(g, s.h.offsets, s.h.padded_numel))
        pre_w, pre_m = s.state()
        s.step(t)
        r, _ = s.check(t, pre_w, [g], pre_m, TOL_F32, tag=f"{form} {dtype} t={t}")
        assert r.lr == s.h.lr_at(t) and r.lr == (32.0 if t < 480 else 32.0 * 0.1)


@pytest.mark.parametrize("layout", ["resnet50", "skew"])
def test_deferred_finish_matches_k1_finish(layout, monkeypatch):
    """The layer finish in K2's prologue (default for lars_step) and the finish in K1's tail
    (LARS_DEFER_FINISH=0) sum the same segment partials in the same fixed order: bitwise-equal w, m, norms,
    lambda and coefficients, over applied steps, carried norms, a device-iteration graph step at the end of
    the schedule and a skipped (NaN) step."""
    torch = _torch()
    import paper_1903_12650_b200 as PK

    rng = np.random.default_rng(77)
    lay = LY.resnet50() if layout == "resnet50" else LY.random_layout(rng, 40, max_numel=300000)
    runs = []
    for defer in ("1", "0"):
        monkeypatch.setenv("LARS_DEFER_FINISH", defer)
        s = GpuStep(lay, grad_dtype="f16", flags=PK.lars.FLAG_CARRY_WNORM)
        s.upload(G.weights(lay), G.grads(lay, 0, 5, "f16"), G.momentum(lay, 1e-3))
        out = []
        for t in (79, 80, 700):
            s.step(t)
            out.append(s.h.last_norms())
        it = torch.tensor([1439], dtype=torch.int64, device=s.w.device)
        s.h.lars_step_dev_iter(s.w, s.g, s.m, it)
        torch.cuda.synchronize()
        assert int(it.item()) == 1440 and not s.h.last_step_skipped()
        s.h.lars_step_dev_iter(s.w, s.g, s.m, it)  # t = T: out of range -> status 2, untouched
        torch.cuda.synchronize()
        assert s.h.last_step_status() == 2
        s.g.view(torch.float16)[s.h.offsets[len(lay) // 2]] = float("nan")
        s.step(701)
        torch.cuda.synchronize()
        assert s.h.last_step_skipped()
        runs.append((s.w.clone(), s.m.clone(), out))
        s.h.close()
    (wa, ma, na), (wb, mb, nb) = runs
    assert torch.equal(wa, wb) and torch.equal(ma, mb)
    for x, y in zip(na, nb):
        for u, v in zip(x, y):
            assert np.array_equal(np.asarray(u), np.asarray(v))
