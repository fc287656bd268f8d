"""BASELINE.json configs[4]: synthetic 10^9-parameter, 1,000-tensor layouts with skewed size mixes
(uniform, log-uniform [64, 2^24], Zipf 1.2, one 5x10^8 giant) — the norm kernel's load balance at full
size. Every layer's update depends only on its own norms, so the oracle checks a SAMPLE of layers
exactly (the smallest, a spread of medium ones); the largest layer is checked through properties that
hold at any size (its norms against float64 sums, and its update on 2^20 random elements against the
update formula with lambda from those norms)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from synth import gen_torch as GT
from synth import layouts as LY
from tests._parity import TOL_F32, gate, gate_norms, hp_kwargs, oracle_hp

pytestmark = pytest.mark.gpu


def _np(t):
    a = t.cpu().numpy()
    return a


@pytest.mark.parametrize("variant", ["loguniform", "zipf", "giant", "uniform"])
def test_skew1b_sampled_parity(variant):
    import torch

    import paper_1903_12650_b200 as P

    lay = LY.skew1b(variant)
    assert len(lay) == 1000 and sum(t.numel for t in lay) == 1_000_000_000
    kw = hp_kwargs(grad_dtype="f16")
    h = P.Lars([(t.numel, t.kind) for t in lay], device=0, **kw)
    dev = torch.device("cuda", 0)
    w = torch.zeros(h.padded_numel, dtype=torch.float32, device=dev)
    g = torch.zeros(h.padded_numel, dtype=torch.float16, device=dev)
    m = torch.zeros(h.padded_numel, dtype=torch.float32, device=dev)
    GT.fill_weights(w, lay, h.offsets)
    GT.fill_grads(g, lay, h.offsets, 0, 9)
    GT.fill_momentum(m, lay, h.offsets)
    sizes = np.array([t.numel for t in lay])
    order = np.argsort(sizes, kind="stable")
    rng = np.random.default_rng(4)
    medium = [int(i) for i in order if sizes[i] <= 4_000_000]
    sample = sorted(set([int(order[0]), int(order[1])] + list(rng.choice(medium, 6, replace=False))))
    big = int(order[-1])
    sl = lambda x, l: x[h.offsets[l]:h.offsets[l] + lay[l].numel]
    pre = {l: (_np(sl(w, l)), _np(sl(g, l)), _np(sl(m, l))) for l in sample}
    idx = np.sort(rng.choice(lay[big].numel, min(1 << 20, lay[big].numel), replace=False))
    big_w, big_g = sl(w, big), sl(g, big)
    wn_big = float(torch.sqrt((big_w.double() ** 2).sum()).item())  # float64 reductions, any order
    gn_big = float(torch.sqrt((big_g.double() ** 2).sum()).item()) * kw["grad_scale"]
    pre_big = (_np(big_w)[idx], _np(big_g)[idx], _np(sl(m, big))[idx])
    t = 719
    h.lars_step(w, g, m, t)
    torch.cuda.synchronize()
    assert not h.last_step_skipped()
    wn, gn, lam, coef = h.last_norms()
    hp = oracle_hp(kw)
    r = O.step([lay[l].kind for l in sample], hp, t, [pre[l][0] for l in sample], [[pre[l][1] for l in sample]],
               [pre[l][2] for l in sample])
    gate_norms(f"{variant} sampled ||w||", [wn[l] for l in sample], r.w_norm)
    gate_norms(f"{variant} sampled ||g||", [gn[l] for l in sample], r.g_norm)
    post_w = [_np(sl(w, l)) for l in sample]
    post_m = [_np(sl(m, l)) for l in sample]
    gate(f"{variant} sampled m", np.concatenate(post_m), np.concatenate(r.m), np.concatenate(r.m_env), TOL_F32)
    gate(f"{variant} sampled w", np.concatenate(post_w), np.concatenate(r.w), np.concatenate(r.w_env), TOL_F32)
    # largest layer: properties
    gate_norms(f"{variant} largest ||w||", [wn[big]], [wn_big], 1e-9)
    gate_norms(f"{variant} largest ||g||", [gn[big]], [gn_big], 1e-9)
    lam_big, beta = O.trust_ratio(wn_big, gn_big, lay[big].kind, hp.eta, hp.weight_decay, hp.eps)
    w0, g0, m0 = pre_big
    G0 = O.combine([g0], hp.grad_scale)
    w1, v1, env_m, env_w = O.update(hp, O.lr_at(hp, t), lam_big, beta, w0, G0, m0, np.abs(G0))
    gate(f"{variant} largest m sample", _np(sl(m, big))[idx], v1, env_m, TOL_F32)
    gate(f"{variant} largest w sample", _np(sl(w, big))[idx], w1, env_w, TOL_F32)
