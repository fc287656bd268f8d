"""BASELINE.json configs[3]: ResNet-152 layout (467 tensors, 60,192,808 params), full schedule replay at
global batch 81,920 — 16 updates/epoch x 90 epochs = 1,440 steps, warm-up then
polynomial decay — as CUDA-graph replays of lars_step_dev_iter (the device iteration advances itself).
Gradients come from a ring of 4 pre-generated buffers (graph k uses buffer k). At sampled iterations
{0, 79, 80, 719, 1439} the GPU pre-step state is snapshotted and the step is checked against the oracle;
the lr the kernels used is checked at every sample through a BN tensor (lambda = 1, coef = lr(t))."""
from __future__ import annotations

import time

import numpy as np
import pytest

from synth import gen as G
from synth import layouts as LY
from tests._parity import TOL_F32, GpuStep, to_dev

pytestmark = pytest.mark.gpu
SAMPLES = (0, 79, 80, 719, 1439)


def test_resnet152_full_schedule_graph_replay():
    import torch

    lay = LY.resnet152()
    s = GpuStep(lay, grad_dtype="f32")
    assert (s.h.ipe, s.h.total_iters, s.h.warmup_iters) == (16, 1440, 80)
    w0, m0 = G.weights(lay), G.momentum(lay)
    ring = [G.grads(lay, 0, k, "f32") for k in range(4)]
    s.upload(w0, ring[0], m0)
    g_dev = [to_dev(G.pack(gk, s.h.offsets, s.h.padded_numel)) for gk in ring]
    it = torch.zeros(1, dtype=torch.int64, device="cuda")
    stream = torch.cuda.Stream()
    graphs = []
    torch.cuda.synchronize()
    for k in range(4):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            s.h.lars_step_dev_iter(s.w, g_dev[k], s.m, it, stream=stream)
        graphs.append(gr)
    bn = next(i for i, t in enumerate(lay) if t.kind == "bn_gamma")
    t0 = time.perf_counter()
    for t in range(1440):
        if t in SAMPLES:
            pre_w, pre_m = s.state()
        graphs[t % 4].replay()
        if t in SAMPLES:
            torch.cuda.synchronize()
            assert int(it.item()) == t + 1
            _, _, lam, coef = s.h.last_norms()
            assert lam[bn] == 1.0 and coef[bn] == float(np.float32(s.h.lr_at(t)))
            s.check(t, pre_w, [ring[t % 4]], pre_m, TOL_F32, tag=f"R152 replay t={t}")
    torch.cuda.synchronize()
    print(f"R152 1,440-step replay incl. 5 oracle checks: {time.perf_counter() - t0:.2f} s")
    assert int(it.item()) == 1440
    # one step past the schedule: skipped on the device (status 2), state untouched, iteration advanced
    before = s.w.clone()
    graphs[0].replay()
    torch.cuda.synchronize()
    assert s.h.last_step_status() == 2 and torch.equal(before, s.w) and int(it.item()) == 1441


def test_device_iteration_matches_host_iteration():
    import torch

    lay = LY.resnet50()[:50]
    a, b = GpuStep(lay, grad_dtype="f16"), GpuStep(lay, grad_dtype="f16")
    w, g, m = G.weights(lay), G.grads(lay, 0, 1, "f16"), G.momentum(lay, 1e-3)
    a.upload(w, g, m)
    b.upload(w, g, m)
    it = torch.tensor([77], dtype=torch.int64, device="cuda")
    for t in range(77, 84):
        a.h.lars_step(a.w, a.g, a.m, t)
        b.h.lars_step_dev_iter(b.w, b.g, b.m, it)
    torch.cuda.synchronize()
    assert int(it.item()) == 84
    assert torch.equal(a.w, b.w) and torch.equal(a.m, b.m)
