"""Pins for the CPU oracle — each pins the oracle to something other than
itself: values printed in the paper, SPEC.md's worked examples, closed forms, exact rational
arithmetic and brute force on tiny inputs. CPU only (``-m "not gpu"``)."""
from __future__ import annotations

import math
import pathlib
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = pathlib.Path(__file__).parent / "golden"


def hp(**kw) -> O.HParams:
    d = dict(base_lr=32.0, eta=1e-3, momentum=0.9, weight_decay=5e-5, eps=0.0, warmup_epochs=5.0,
             poly_power=2.0, global_batch=81920)
    d.update(kw)
    return O.HParams(**d)


# ---------------------------------------------------------------- P1: update counts (printed)
def test_p1_update_count_printed_in_paper():
    # 1,280,000 images, 81,920 batch -> 16 updates/epoch, 1,440 in total
    assert O.iterations_per_epoch(1_280_000, 81_920) == 16
    ipe, T, W = O.schedule(hp())
    assert (ipe, T, W) == (16, 1440, 80)
    # 15.625 is rounded UP (reading #11): one more partial iteration, never fewer
    assert O.iterations_per_epoch(1_280_000, 81_921) == 16
    assert O.iterations_per_epoch(1_280_000, 80_000) == 16
    assert O.iterations_per_epoch(1_280_001, 80_000) == 17


# ---------------------------------------------------------------- P2: SPEC.md:162-164 examples
def test_p2_spec_lr_examples():
    h = hp(base_lr=8.0, warmup_epochs=1.0)  # W = 16
    assert O.schedule(h)[2] == 16
    assert O.lr_at(h, 15) == 8.0       # end of warm-up equals base
    assert O.lr_at(h, 3) == 2.0        # linear ramp
    h2 = hp(base_lr=8.0, warmup_epochs=0.0, dataset_size=100, global_batch=1, total_epochs=1)
    assert O.schedule(h2) == (100, 100, 0)
    assert O.lr_at(h2, 50) == 8.0 / 4  # p=2, T=100, W=0


# ---------------------------------------------------------------- P3: golden hand values
def _golden_lr():
    rows = []
    for line in (GOLDEN / "lr_schedule_b81920.txt").read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            b, t, n, d = line.split()
            rows.append((float(b), int(t), Fraction(int(n), int(d))))
    return rows


@pytest.mark.parametrize("base,t,exact", _golden_lr())
def test_p3_lr_golden(base, t, exact):
    got = O.lr_at(hp(base_lr=base), t)
    assert abs(Fraction(got) - exact) <= Fraction(4 * math.ulp(float(exact)))


def test_p3_lr_range_errors():
    h = hp()
    for bad in (-1, 1440, 10**6):
        with pytest.raises(ValueError):
            O.lr_at(h, bad)


def test_lr_shape_properties():
    h = hp()
    lrs = [O.lr_at(h, t) for t in range(1440)]
    assert all(b > a for a, b in zip(lrs[:79], lrs[1:80]))       # strictly rising warm-up
    assert all(b < a for a, b in zip(lrs[80:-1], lrs[81:]))      # strictly decaying after W
    assert min(lrs) > 0.0                                        # never zero (reading #6, #8)
    h1 = hp(poly_power=1.0)                                      # p=1 is linear decay
    d = [O.lr_at(h1, t) - O.lr_at(h1, t + 1) for t in range(80, 1439)]
    assert max(d) - min(d) < 1e-12
    h0 = hp(poly_power=0.0)                                      # p=0 is constant
    assert {O.lr_at(h0, t) for t in range(80, 1440)} == {32.0}


# ---------------------------------------------------------------- P4: trust ratio closed forms
def test_p4_trust_ratio_closed_forms():
    lam, beta = O.trust_ratio(1.0, 1.0, "weight", 1e-3, 0.0, 0.0)
    assert lam == pytest.approx(1e-3, rel=1e-15) and beta == 0.0          # (a) SPEC.md:180
    assert O.trust_ratio(0.0, 5.0, "weight", 1e-3, 5e-5, 0.0)[0] == 1.0  # (b) SPEC.md:181
    assert O.trust_ratio(0.0, 0.0, "weight", 1e-3, 0.0, 0.0)[0] == 1.0   # 0/0 guarded (#3)
    assert O.trust_ratio(2.0, 0.0, "weight", 1e-3, 0.0, 0.0)[0] == 1.0   # zero denominator
    for k in ("bias", "bn_gamma", "bn_beta"):                              # skip kinds (#4)
        assert O.trust_ratio(3.0, 4.0, k, 1e-3, 5e-5, 0.0) == (1.0, 0.0)
    # (c) homogeneity under joint scaling, beta > 0, eps = 0
    a = O.trust_ratio(1.7, 0.03, "weight", 1e-3, 5e-5, 0.0)[0]
    b = O.trust_ratio(1.7 * 7.3, 0.03 * 7.3, "weight", 1e-3, 5e-5, 0.0)[0]
    assert abs(a - b) <= 1e-12 * a
    # eps enters the denominator
    assert O.trust_ratio(1.0, 1.0, "weight", 1e-3, 0.0, 1.0)[0] == pytest.approx(5e-4, rel=1e-15)
    # "if w_norm = 0 or denominator <= epsilon_guard, returns 1" — with eps > 0 a zero
    # gradient of a layer without decay would otherwise get eta*||w||/eps (1e5 for eta = 1e-3, eps = 1e-8)
    assert O.trust_ratio(1.0, 0.0, "weight", 1e-3, 0.0, 1e-8)[0] == 1.0
    assert O.trust_ratio(1.0, 0.0, "weight", 1e-3, 5e-5, 1e-8)[0] == pytest.approx(1e-3 / (5e-5 + 1e-8), rel=1e-15)


def test_p4_eps_guard_zero_gradient_through_step():
    """eps > 0, g = 0, beta = 0 on a weight-kind layer: lambda = 1, so the update is exactly
    v = mu*m (no gradient, no decay) — not a 1e5-fold step."""
    w = [np.full(16, 0.25, np.float32)]
    m = [np.full(16, 2.0 ** -10, np.float32)]
    r = O.step(["weight"], hp(eps=1e-8, weight_decay=0.0), 100, w, [[np.zeros(16, np.float32)]], m)
    assert r.lam == [1.0] and not r.skipped
    assert np.array_equal(r.m[0], np.full(16, 0.9 * 2.0 ** -10)) and np.array_equal(r.w[0], 0.25 - r.m[0])


def test_p4d_constant_tensors_through_step():
    # golden/trust_ratio_closed_forms.txt (d): ||w|| = 32, ||g|| = 1/16, lambda = 320/641
    n = 4096
    w = [np.full(n, 0.5, np.float32)]
    g = [[np.full(n, 2.0 ** -10, np.float16)]]
    r = O.step(["weight"], hp(), 0, w, g, [np.zeros(n, np.float32)])
    assert r.w_norm == [32.0] and r.g_norm == [0.0625]
    assert abs(Fraction(r.lam[0]) - Fraction(320, 641)) <= Fraction(math.ulp(0.5))


# ---------------------------------------------------------------- P5: norms
def test_p5_norm_examples():
    assert O.l2norm(np.array([3.0, 4.0])) == 5.0
    assert O.l2norm(np.zeros(3)) == 0.0
    assert O.l2norm(np.full(4096, 0.5)) == 32.0           # exact case
    r = O.step(["weight", "weight"], hp(), 100, [np.array([3, 4], np.float32), np.zeros(3, np.float32)],
               [[np.array([0, 0], np.float32), np.array([0, 0, 0], np.float32)]],
               [np.zeros(2, np.float32), np.zeros(3, np.float32)])
    assert r.w_norm == [5.0, 0.0]


def test_p5_norms_brute_force_exact_rationals():
    rng = np.random.default_rng(5)
    for _ in range(30):
        sizes = rng.integers(1, 60, rng.integers(1, 8))
        w = [rng.standard_normal(n).astype(np.float32) for n in sizes]
        g = [(rng.standard_normal(n) * 3).astype(np.float16) for n in sizes]
        kinds = ["weight"] * len(sizes)
        r = O.step(kinds, hp(), 200, w, [g], [np.zeros(n, np.float32) for n in sizes])
        for l in range(len(sizes)):
            ew = sum(Fraction(float(x)) ** 2 for x in w[l])       # exact sum of squares
            eg = sum(Fraction(float(x)) ** 2 for x in g[l])
            assert r.w_norm[l] == pytest.approx(math.sqrt(ew), rel=2e-16, abs=0)
            assert r.g_norm[l] == pytest.approx(math.sqrt(eg), rel=2e-16, abs=0)


# ---------------------------------------------------------------- P6: invariants
def test_p6a_zero_grad_zero_decay_leaves_weights_bitwise():
    rng = np.random.default_rng(6)
    kinds = ["weight", "bn_gamma", "weight", "bias"]
    w = [rng.standard_normal(n).astype(np.float32) for n in (17, 8, 300, 5)]
    g = [[np.zeros(x.size, np.float16) for x in w]]
    for t in (0, 79, 80, 719, 1439):
        r = O.step(kinds, hp(weight_decay=0.0), t, w, g, [np.zeros(x.size, np.float32) for x in w])
        assert not r.skipped
        for a, b, m in zip(r.w, w, r.m):
            assert np.array_equal(a, b.astype(np.float64)) and not m.any()


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_p6b_nonfinite_gradient_skips_whole_step(bad):
    rng = np.random.default_rng(7)
    w = [rng.standard_normal(n).astype(np.float32) for n in (10, 20)]
    m = [rng.standard_normal(n).astype(np.float32) for n in (10, 20)]
    g = [[rng.standard_normal(10).astype(np.float32), rng.standard_normal(20).astype(np.float32)]]
    g[0][1][13] = bad
    r = O.step(["weight", "bn_beta"], hp(), 300, w, g, m)
    assert r.skipped
    for a, b in zip(r.w + r.m, w + m):
        assert np.array_equal(a, b.astype(np.float64))


# ---------------------------------------------------------------- P7: vanilla SGD reduction
def test_p7_skip_kind_no_momentum_is_plain_sgd():
    # mu=0, wd=0, LARS off, lr=0.1, w=1, g=2 -> 0.8
    h = hp(base_lr=0.1, warmup_epochs=0.0, poly_power=0.0, momentum=0.0)
    for kind in ("bias", "bn_gamma", "bn_beta"):
        r = O.step([kind], h, 500, [np.array([1.0], np.float32)], [[np.array([2.0], np.float32)]],
                   [np.zeros(1, np.float32)])
        assert r.lr == 0.1 and r.w[0][0] == pytest.approx(0.8, abs=1.2e-16)
    # skip kinds ignore weight decay (reading #4)
    r = O.step(["bn_gamma"], hp(base_lr=0.1, warmup_epochs=0.0, poly_power=0.0, momentum=0.0,
                                weight_decay=0.5), 3, [np.array([1.0], np.float32)],
               [[np.array([2.0], np.float32)]], [np.zeros(1, np.float32)])
    assert r.w[0][0] == pytest.approx(0.8, abs=1.2e-16)
    # grad_scale multiplies the combined gradient (reading #12): 1 - 0.1*0.5*2 = 0.9
    r = O.step(["bias"], hp(base_lr=0.1, warmup_epochs=0.0, poly_power=0.0, momentum=0.0,
                            grad_scale=0.5), 3, [np.array([1.0], np.float32)],
               [[np.array([2.0], np.float32)]], [np.zeros(1, np.float32)])
    assert r.w[0][0] == pytest.approx(0.9, abs=1.2e-16)


# ---------------------------------------------------------------- P8: first step, weight kind
def test_p8_first_weight_step_exact_rational():
    # constant tensors of test_p4d; t=0 -> lr = 32*1/80 = 2/5; lambda = 320/641
    # u = g + beta*w = 2^-10 + 5e-5*0.5 ; v = lr*lambda*u ; w1 = 0.5 - v ; m1 = v
    n = 4096
    r = O.step(["weight"], hp(), 0, [np.full(n, 0.5, np.float32)],
               [[np.full(n, 2.0 ** -10, np.float16)]], [np.zeros(n, np.float32)])
    u = Fraction(1, 1024) + Fraction(5e-5) * Fraction(1, 2)
    v = Fraction(2, 5) * Fraction(320, 641) * u
    assert float(r.m[0][0]) == pytest.approx(float(v), rel=4e-16)
    assert float(r.w[0][0]) == pytest.approx(float(Fraction(1, 2) - v), rel=4e-16)
    assert np.all(r.w[0] == r.w[0][0])


# ---------------------------------------------------------------- P9: closed-form recurrence
def test_p9_geometric_momentum_recurrence():
    mu, lr, g, w0 = 0.9, 0.25, 0.75, 3.0
    h = hp(base_lr=lr, warmup_epochs=0.0, poly_power=0.0, momentum=mu, weight_decay=0.0)
    w, m = [np.array([w0], np.float32)], [np.zeros(1, np.float32)]
    wd, md = w0, 0.0
    for k in range(1, 21):
        r = O.step(["bn_beta"], h, k, [np.array([wd])], [[np.array([g], np.float32)]], [np.array([md])])
        wd, md = float(r.w[0][0]), float(r.m[0][0])
        vk = lr * g * (1 - mu ** k) / (1 - mu)
        wk = w0 - lr * g * sum((1 - mu ** j) / (1 - mu) for j in range(1, k + 1))
        assert md == pytest.approx(vk, rel=1e-13) and wd == pytest.approx(wk, rel=1e-13)


def test_momentum_form_lr_inside_velocity():
    # reading #2: v <- mu v + lr*lambda*(g+beta w). Warm-up lr(0)=0.4, lr(1)=0.8 (base 32, W=80).
    # v1 = 0.4 g; w1 = w0 - 0.4 g; v2 = 0.9*0.4 g + 0.8 g = 1.16 g; w2 = w0 - 1.56 g.
    # (SPEC's lr-at-apply form would give w2 = w0 - 1.92 g; the two differ when lr changes.)
    g = np.array([0.5], np.float32)
    r1 = O.step(["bias"], hp(), 0, [np.array([1.0], np.float32)], [[g]], [np.zeros(1, np.float32)])
    r2 = O.step(["bias"], hp(), 1, r1.w, [[g]], r1.m)
    assert float(r2.m[0][0]) == pytest.approx(1.16 * 0.5, rel=1e-15)
    assert float(r2.w[0][0]) == pytest.approx(1.0 - 1.56 * 0.5, rel=1e-15)


# ---------------------------------------------------------------- P10: multi-rank summation
def test_p10_rank_sum_brute_force():
    # P=4 with [rank+1] -> [10]; P=1 identity
    assert O.combine([np.array([r + 1.0], np.float16) for r in range(4)], 1.0).tolist() == [10.0]
    x = np.array([1.5, -2.25, 65504.0], np.float16)
    assert O.combine([x], 1.0).tolist() == x.astype(np.float64).tolist()
    rng = np.random.default_rng(10)
    for P in (2, 3, 5, 8):  # matches a sequential-sum oracle, exactly for integer data
        gs = [rng.integers(-64, 65, 37).astype(np.float16) for _ in range(P)]
        brute = [sum(int(g[i]) for g in gs) for i in range(37)]
        assert O.combine(gs, 1.0).tolist() == [float(b) for b in brute]
        gr = [(rng.standard_normal(37)).astype(np.float16) for _ in range(P)]
        exact = [sum(Fraction(float(g[i])) for g in gr) for i in range(37)]
        assert O.combine(gr, 1.0).tolist() == [float(e) for e in exact]  # exact in double (O2)


def test_wire_overflow_thresholds_match_format_rounding():
    """Reading #29: the threshold is the smallest magnitude the format's round-to-nearest-even sends to
    infinity. Checked against numpy's own double -> fp16 / fp32 conversions and a bit-level fp32 -> bf16 RNE."""
    t16 = O.wire_overflow_threshold(np.zeros(1, np.float16))
    assert t16 == 65520.0
    assert np.isinf(np.float16(t16)) and np.float16(np.nextafter(t16, 0.0)) == 65504.0
    t32 = O.wire_overflow_threshold(np.zeros(1, np.float32))
    assert np.isinf(np.float32(t32)) and np.isfinite(np.float32(np.nextafter(t32, 0.0)))
    tb = O.wire_overflow_threshold(np.zeros(1, np.uint16))
    u = int(np.float32(tb).view(np.uint32))
    assert float(np.float32(tb)) == tb and u == 0x7F7F8000
    rne = lambda x: (x + 0x7FFF + ((x >> 16) & 1)) >> 16
    assert rne(u) == 0x7F80 and rne(u - 1) == 0x7F7F  # inf at the threshold, max finite just below


def test_wire_overflow_of_rank_sum_skips_step():
    """Reading #29: per-rank finite fp16 gradients whose exact sum overflows fp16 are an infinite combined
    gradient -> the whole step is skipped; a sum that stays below the threshold is applied."""
    kinds = ["weight", "bn_gamma"]
    w = [np.full(8, 0.5, np.float32), np.ones(3, np.float32)]
    m = [np.zeros(8, np.float32), np.zeros(3, np.float32)]
    for P in (2, 4, 8):
        over = [[np.full(8, 40000.0, np.float16), np.ones(3, np.float16)] for _ in range(P)]
        G = O.combine([g[0] for g in over], 1.0)
        assert np.isinf(G).all() and (G > 0).all()
        r = O.dp_step(kinds, hp(grad_scale=1.0 / P), 100, w, over, m)
        assert r.skipped and np.array_equal(r.w[0], w[0]) and np.array_equal(r.m[1], m[1])
        v = np.float16(65504.0 / (2 * P))  # exact: the sum 32752 is far below 65520
        under = [[np.full(8, v, np.float16), -np.ones(3, np.float16)] for _ in range(P)]
        assert O.combine([g[0] for g in under], 1.0).tolist() == [32752.0] * 8
        assert not O.dp_step(kinds, hp(grad_scale=1.0 / P), 100, w, under, m).skipped
    neg = O.combine([np.array([-65504.0], np.float16), np.array([-16.0], np.float16)], 1.0)
    assert neg.tolist() == [-np.inf]  # -65520 rounds to -inf (tie to even)
    assert O.combine([np.array([-65504.0], np.float16), np.array([-15.0], np.float16)], 1.0).tolist() == [-65519.0]


def test_dp_step_uses_exact_rank_sum():
    rng = np.random.default_rng(11)
    kinds = ["weight", "bn_gamma"]
    w = [rng.standard_normal(n).astype(np.float32) for n in (33, 7)]
    g_r = [[rng.standard_normal(n).astype(np.float16) for n in (33, 7)] for _ in range(4)]
    summed = [[np.sum([g_r[r][l].astype(np.float64) for r in range(4)], axis=0) for l in range(2)]]
    a = O.dp_step(kinds, hp(), 90, w, g_r, [np.zeros(n, np.float32) for n in (33, 7)])
    b = O.step(kinds, hp(), 90, w, summed, [np.zeros(n, np.float32) for n in (33, 7)])
    for x, y in zip(a.w + a.m, b.w + b.m):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------- P13: scale invariance
def test_p13_zero_decay_invariant_to_grad_scale():
    rng = np.random.default_rng(13)
    w = [rng.standard_normal(n).astype(np.float32) for n in (64, 9)]
    m = [rng.standard_normal(n).astype(np.float32) * 1e-3 for n in (64, 9)]
    g = [[rng.standard_normal(n).astype(np.float16) for n in (64, 9)]]
    base = O.step(["weight", "weight"], hp(weight_decay=0.0), 400, w, g, m)
    for k in (-10, -3, 4):
        r = O.step(["weight", "weight"], hp(weight_decay=0.0, grad_scale=2.0 ** k), 400, w, g, m)
        for a, b in zip(r.w, base.w):
            np.testing.assert_allclose(a, b, rtol=1e-14, atol=0)


# ---------------------------------------------------------------- P14: half formats
def _decode_half_bits(b: int) -> float:
    s, e, f = (b >> 15) & 1, (b >> 10) & 31, b & 1023
    v = (f / 1024.0) * 2.0 ** -14 if e == 0 else (1 + f / 1024.0) * 2.0 ** (e - 15)
    return -v if s else v


def test_p14_fp16_widening_exact_all_finite_patterns():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = ((bits >> 10) & 31) != 31
    assert int(finite.sum()) == 63488
    got = O.to_double(bits[finite].view(np.float16))
    want = np.array([_decode_half_bits(int(b)) for b in bits[finite]])
    assert np.array_equal(got, want)


def test_p14_bf16_widening():
    bits = np.array([0x3F80, 0xBF80, 0x0000, 0x4049, 0x0001, 0x7F7F], np.uint16)
    want = [1.0, -1.0, 0.0, 3.140625, 2.0 ** -133, (2 - 2.0 ** -7) * 2.0 ** 127]
    assert O.to_double(bits).tolist() == want


# ---------------------------------------------------------------- parallel initialization (NEXT-f4)
def test_philox4x64_known_answer():
    # Random123 known-answer vector (Salmon et al., SC'11): philox4x64-10, counter 0, key 0
    assert O.philox4x64_10((0, 0, 0, 0), (0, 0)) == (0x16554D9ECA36314C, 0xDB20FE9D672D0FDC,
                                                     0xD7E772CEE186176B, 0x7E68B68AEC7BA23B)


@pytest.mark.parametrize("key,ctr", [((0, 0), (0, 0, 0, 0)), ((100000, 0x4C415253), (7, 3, 0, 0)),
                                     ((2 ** 64 - 1, 12345), (2 ** 40, 2, 5, 9))])
def test_philox4x64_matches_numpy_library(key, ctr):
    # numpy.random.Philox is Philox4x64-10 and advances its counter before the first block
    bg = np.random.Philox(key=np.array(key, dtype=np.uint64), counter=np.array(ctr, dtype=np.uint64))
    got = tuple(int(x) for x in bg.random_raw(4))
    nxt = (ctr[0] + 1,) + tuple(ctr[1:])
    assert O.philox4x64_10(nxt, key) == got


def test_truncated_normal_transform_matches_scipy():
    from scipy.stats import truncnorm

    u = O.init_uniform(100000, 3, 4096)
    assert (u >= 0).all() and (u < 1).all()
    w = O.init_weights(["weight"], [4096], [2], 100000)[0]  # sigma = 1 (fan_in 2)
    # same u through a library truncated-normal quantile function
    ref = truncnorm(-2.0, 2.0).ppf(O.init_uniform(100000, 0, 4096))
    np.testing.assert_allclose(w, ref, rtol=1e-9, atol=1e-12)


def test_init_weights_distribution_and_constant_kinds():
    n = 65536
    w = O.init_weights(["weight", "bn_gamma", "bn_beta", "bias"], [n, 7, 7, 3], [147, 0, 0, 0], 100000)
    sigma = math.sqrt(2.0 / 147)
    z = w[0] / sigma
    assert np.abs(z).max() <= 2.0 and abs(z.mean()) < 0.02
    assert abs(z.std() - 0.8796256610342398) < 0.01  # std of N(0,1) truncated at +-2
    assert (w[1] == 1.0).all() and not w[2].any() and not w[3].any()
    # a different seed or layer gives different weights; the same seed gives the same
    assert not np.array_equal(w[0], O.init_weights(["weight"], [n], [147], 100001)[0])
    assert np.array_equal(w[0], O.init_weights(["weight"], [n], [147], 100000)[0])


# ---------------------------------------------------------------- optimizer variants (NEXT-f3)
def test_step_decay_hand_values():
    # PAPER.md:102 "step" decay: base 8, warm-up 1 epoch (W = 16), milestones 30/60/80 epochs, gamma 0.1
    h = hp(base_lr=8.0, warmup_epochs=1.0, decay="step", milestones=(30, 60, 80), step_gamma=0.1)
    want = {15: 8.0, 16: 8.0, 479: 8.0, 480: 0.8, 959: 0.8, 960: 0.08, 1279: 0.08, 1280: 0.008, 1439: 0.008}
    for t, v in want.items():
        assert O.lr_at(h, t) == pytest.approx(v, rel=1e-15), t
    assert O.lr_at(h, 3) == 2.0  # the warm-up is unchanged


def test_momentum_form_lr_at_apply():
    # SPEC.md:186 form: v <- mu v + (g + beta w); w <- w - lr lambda v. Warm-up lr(0) = 0.4, lr(1) = 0.8:
    # v1 = g, w1 = w0 - 0.4 g; v2 = 1.9 g, w2 = w1 - 0.8 * 1.9 g = w0 - 1.92 g (reading #2 gives 1.56 g)
    g = np.array([0.5], np.float32)
    h = hp(momentum_form="apply")
    r1 = O.step(["bias"], h, 0, [np.array([1.0], np.float32)], [[g]], [np.zeros(1, np.float32)])
    r2 = O.step(["bias"], h, 1, r1.w, [[g]], r1.m)
    assert float(r2.m[0][0]) == pytest.approx(1.9 * 0.5, rel=1e-15)
    assert float(r2.w[0][0]) == pytest.approx(1.0 - 1.92 * 0.5, rel=1e-15)
    # both forms agree on the first step from v = 0
    ra = O.step(["weight"], hp(), 5, [np.full(8, 0.3, np.float32)], [[np.full(8, 0.01, np.float32)]],
                [np.zeros(8, np.float32)])
    rb = O.step(["weight"], h, 5, [np.full(8, 0.3, np.float32)], [[np.full(8, 0.01, np.float32)]],
                [np.zeros(8, np.float32)])
    np.testing.assert_allclose(ra.w[0], rb.w[0], rtol=1e-15)
