"""CPU ORACLE for the LARS gradient-combine-and-update step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this module. The product path (``paper_1903_12650_b200``) never
imports, links or executes it, and this module imports nothing from the product path.

Plain, slow, obviously correct float64 NumPy following the paper's method step by step
(SURVEY.md §8(c) O1-O8). Passages followed (arxiv 1903.12650, /root/reference/PAPER.md):

  * PAPER.md:29-31 (§I)       "the weight gradients from all processes are combined to update
                               all the weights"                                   -> combine()
  * PAPER.md:96-98 (§III-A-1) warm-up "which raises learning rate gradually"      -> lr_at()
  * PAPER.md:99-100, 78-80    LARS "adjusts the learning rate of each layer according to the
                               norms weight and gradient"                         -> trust_ratio()
  * PAPER.md:102-103          decay patterns "step, polynomial, linear"           -> lr_at()
  * PAPER.md:130-135 (§III-B-2) per-layer norms for LARS                          -> l2norm()
  * PAPER.md:183 (§IV)        "compute and communicate using half precision ... update own
                               weights using single precision"                    -> to_double()
  * PAPER.md:184-185          "original optimizer ... warmup and LARS"            -> step()
  * PAPER.md:210-211          1,280,000 images / 81,920 batch -> 16 updates per epoch, 1,440
                               in total                                           -> schedule()

Where the paper is silent, the readings of SURVEY.md §8(c) are used and listed in DESIGN.md
§"Readings": LARS form lambda = eta*||w||/(||g|| + beta*||w|| + eps) (#1), lr*lambda inside the
velocity (#2), lambda = 1 fallback (#3), bias/BN skip kinds (#4), linear warm-up lr(t) =
base*(t+1)/W (#6), W = round-half-up(warmup_epochs*ipe) (#7), polynomial decay toward 0 over
[W,T) (#8), ipe = ceil(D/B) (#11), sum then multiply by grad_scale (#12), whole-step skip on a
non-finite norm (#13), lr(t) for the update performed at iteration t (#21).

Every function here is pinned by ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

WEIGHT, BIAS, BN_GAMMA, BN_BETA = "weight", "bias", "bn_gamma", "bn_beta"


@dataclass
class HParams:
    base_lr: float
    eta: float = 1e-3
    momentum: float = 0.9
    weight_decay: float = 5e-5
    eps: float = 0.0
    warmup_epochs: float = 5.0
    poly_power: float = 2.0
    global_batch: int = 81920
    dataset_size: int = 1_280_000
    total_epochs: int = 90         # PAPER.md:211; log epochs 0..89
    grad_scale: float = 1.0
    decay: str = "poly"            # "poly" or "step" ("step, polynomial, linear")
    step_gamma: float = 0.1        # step decay factor per milestone
    milestones: tuple = ()         # step decay milestones in epochs
    momentum_form: str = "velocity"  # reading #2 ("velocity") or SPEC.md:186's lr-at-apply ("apply")


# ----------------------------------------------------------------------------------------------
# O1. Schedule
# ----------------------------------------------------------------------------------------------
def iterations_per_epoch(dataset_size: int, global_batch: int) -> int:
    """ipe = ceil(D / B): "the number of updates in an epoch is only 16"."""
    return -(-dataset_size // global_batch)


def schedule(hp: HParams) -> tuple[int, int, int]:
    """(ipe, T, W): T = E * ipe (1,440 at B=81,920); W in iterations (reading #7)."""
    ipe = iterations_per_epoch(hp.dataset_size, hp.global_batch)
    T = hp.total_epochs * ipe
    W = int(math.floor(hp.warmup_epochs * ipe + 0.5))
    return ipe, T, W


def lr_at(hp: HParams, t: int) -> float:
    """Learning rate for the update performed at iteration t (0-based).

    Warm-up (reading #6): base * (t+1) / W for t < W.
    Polynomial decay (reading #8): base * (1 - (t-W)/(T-W))^p for W <= t < T,
    evaluated as base * ((T-t)/(T-W))^p — the same number, written without the cancellation of
    1 - (t-W)/(T-W) near t = T-1 (one rounding in the ratio instead of two).
    """
    ipe, T, W = schedule(hp)
    if not (0 <= t < T):
        raise ValueError(f"iteration {t} outside [0, {T})")
    if t < W:
        return hp.base_lr * (t + 1) / W
    if hp.decay == "step":  # base * gamma^(number of milestones reached); milestones in epochs -> iterations
        lr = hp.base_lr
        for m in hp.milestones:
            if t >= int(math.floor(m * ipe + 0.5)):
                lr *= hp.step_gamma
        return lr
    return hp.base_lr * ((T - t) / (T - W)) ** hp.poly_power


# ----------------------------------------------------------------------------------------------
# O2. Combine
# ----------------------------------------------------------------------------------------------
def to_double(g) -> np.ndarray:
    """Half/single precision wire values -> float64 (exact). bf16 arrives as uint16 bit patterns."""
    g = np.asarray(g)
    if g.dtype == np.uint16:  # bf16 bit patterns: the high half of an IEEE single
        return (g.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return g.astype(np.float64)


def wire_overflow_threshold(g) -> float:
    """Smallest magnitude that rounds (to nearest, ties to even) to infinity in g's wire format: halfway
    between the largest finite value (2 - 2^-p) 2^emax and 2^(emax+1), i.e. 2^(emax+1) (1 - 2^-(p+2)) for
    p stored significand bits. fp16 (p = 10, emax = 15): 65520; bf16 (uint16 bit patterns, p = 7,
    emax = 127): 2^128 (1 - 2^-9); fp32 (p = 23, emax = 127): 2^128 (1 - 2^-25)."""
    dt = np.asarray(g).dtype
    p, emax = {np.dtype(np.float16): (10, 15), np.dtype(np.uint16): (7, 127)}.get(dt, (23, 127))
    return math.ldexp(1.0 - math.ldexp(1.0, -(p + 2)), emax + 1)


def combine(g_ranks: list, grad_scale: float) -> np.ndarray:
    """G = s * sum_r g_r, summed in ascending rank order in float64.

    Reading #29 ("communicate using half precision"): the combined gradient is a value of the
    wire format, so an element whose exact rank sum rounds to infinity in that format is +-Inf (the step is
    then skipped, reading #13). A single rank's finite wire values never reach the threshold."""
    total = np.zeros(np.asarray(g_ranks[0]).shape, dtype=np.float64)
    for g in g_ranks:
        total = total + to_double(g)
    over = np.abs(total) >= wire_overflow_threshold(g_ranks[0])
    if over.any():
        total = np.where(over, np.copysign(np.inf, total), total)
    return grad_scale * total


# ----------------------------------------------------------------------------------------------
# O3. Norms
# ----------------------------------------------------------------------------------------------
def l2norm(x: np.ndarray) -> float:
    """sqrt of the correctly rounded sum of squares (math.fsum)."""
    x = np.asarray(x, dtype=np.float64)
    try:
        return math.sqrt(math.fsum((x * x).tolist()))
    except (OverflowError, ValueError):
        s = float(np.sum(x * x))
        return s if not math.isfinite(s) else math.sqrt(s)


# ----------------------------------------------------------------------------------------------
# O4. Trust ratio (reading #1, #3, #4)
# ----------------------------------------------------------------------------------------------
def trust_ratio(w_norm: float, g_norm: float, kind: str, eta: float, weight_decay: float,
                eps: float) -> tuple[float, float]:
    """Returns (lambda_l, beta_l). Skip kinds: (1, 0)."""
    if kind != WEIGHT:
        return 1.0, 0.0
    denom = g_norm + weight_decay * w_norm + eps
    # fallback 1 when ||w|| = 0 or the denominator does not exceed the guard (reading #3)
    if w_norm > 0.0 and denom > eps:
        return eta * w_norm / denom, weight_decay
    return 1.0, weight_decay


# ----------------------------------------------------------------------------------------------
# O5-O7. The step
# ----------------------------------------------------------------------------------------------
@dataclass
class StepResult:
    w: list            # float64 per tensor
    m: list            # float64 per tensor
    w_norm: list       # ||w_l||
    g_norm: list       # ||G_l|| (G = s * sum_r g_r)
    lam: list          # lambda_l
    lr: float
    skipped: bool
    m_env: list = field(default_factory=list)  # magnitude envelopes (tolerance reading #17)
    w_env: list = field(default_factory=list)


def step(kinds: list, hp: HParams, t: int, w: list, g_ranks: list, m: list) -> StepResult:
    """One LARS momentum-SGD update at iteration t.

    kinds:   per-tensor kind strings
    w, m:    per-tensor float32 (or float64) arrays — master weights / momentum
    g_ranks: g_ranks[r][l] = rank r's gradient for tensor l (fp16/bf16-bits/fp32)
    """
    lr = lr_at(hp, t)
    L = len(kinds)
    W64 = [np.asarray(x, dtype=np.float64) for x in w]
    M64 = [np.asarray(x, dtype=np.float64) for x in m]
    G = [combine([g_ranks[r][l] for r in range(len(g_ranks))], hp.grad_scale) for l in range(L)]
    absg = [abs(hp.grad_scale) * sum(np.abs(to_double(g_ranks[r][l])) for r in range(len(g_ranks)))
            for l in range(L)]
    w_norm = [l2norm(W64[l]) for l in range(L)]
    g_norm = [l2norm(G[l]) for l in range(L)]
    lam, beta = zip(*[trust_ratio(w_norm[l], g_norm[l], kinds[l], hp.eta, hp.weight_decay, hp.eps)
                      for l in range(L)]) if L else ((), ())

    # O5: any non-finite norm -> the whole step is skipped (reading #13)
    if not all(math.isfinite(x) for x in w_norm + g_norm):
        return StepResult([x.copy() for x in W64], [x.copy() for x in M64], w_norm, g_norm,
                          list(lam), lr, True)

    w_new, m_new, m_env, w_env = [], [], [], []
    for l in range(L):
        a, b, c, d = update(hp, lr, lam[l], beta[l], W64[l], G[l], M64[l], absg[l], hp.momentum_form)
        w_new.append(a)
        m_new.append(b)
        m_env.append(c)
        w_env.append(d)
    return StepResult(w_new, m_new, w_norm, g_norm, list(lam), lr, False, m_env, w_env)


def update(hp: HParams, lr: float, lam: float, beta: float, w, G, m, abs_g_sum, form: str = "velocity"):
    """O6 for one layer (or any subset of its elements) given its trust ratio lambda and decay beta_l.
    form "velocity" (reading #2): u = G + beta*w; v = mu*m + lr*lambda*u; w_new = w - v.
    form "apply":   u = G + beta*w; v = mu*m + u;           w_new = w - lr*lambda*v.
    G is the combined, scaled gradient and abs_g_sum = |s| sum_r |g_r| (for the magnitude envelopes of
    reading #17). Returns (w_new, v, E_m, E_w) in float64."""
    w = np.asarray(w, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    u = G + beta * w                                   # g + beta*w
    if form == "apply":
        v = hp.momentum * m + u                        # v <- mu*v + (g + beta*w)
        e_m = abs(hp.momentum) * np.abs(m) + abs_g_sum + abs(beta) * np.abs(w)
        return w - lr * lam * v, v, e_m, np.abs(w) + abs(lr * lam) * e_m
    v = hp.momentum * m + lr * lam * u                 # v <- mu*v + lr*lambda*(g + beta*w)
    e_m = abs(hp.momentum) * np.abs(m) + abs(lr * lam) * (abs_g_sum + abs(beta) * np.abs(w))
    # w - v is computed from |w| and every term of v: its envelope is |w| + E_m (reading #17)
    return w - v, v, e_m, np.abs(w) + e_m


def dp_step(kinds: list, hp: HParams, t: int, w: list, g_ranks: list, m: list) -> StepResult:
    """O8: P simulated ranks. The data-parallel result is O1-O7 with the exact rank sum."""
    return step(kinds, hp, t, w, g_ranks, m)


# ----------------------------------------------------------------------------------------------
# Parallel deterministic initialization (§III-B-1; NEXT-f4): "every process has the
# same seed and initializes weights in parallel" — a counter-based generator makes every weight a pure
# function of (seed, layer, element), so no broadcast is needed. "truncated_normal".
# ----------------------------------------------------------------------------------------------
PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
INIT_KEY1 = 0x4C415253  # "LARS"
_M64 = (1 << 64) - 1


def philox4x64_10(counter, key) -> tuple:
    """Philox4x64-10 (Salmon et al., SC'11) on one 256-bit counter, Python integers (reference)."""
    c, k = list(counter), list(key)
    for r in range(10):
        if r:
            k = [(k[0] + PHILOX_W[0]) & _M64, (k[1] + PHILOX_W[1]) & _M64]
        p0, p1 = PHILOX_M[0] * c[0], PHILOX_M[1] * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & _M64, (p0 >> 64) ^ c[3] ^ k[1], p0 & _M64]
    return tuple(c)


def init_uniform(seed: int, layer: int, n: int) -> np.ndarray:
    """u_i = (x_i >> 11) 2^-53, x_i = word (i mod 4) of Philox4x64-10((i // 4, layer, 0, 0), (seed, "LARS"))."""
    words = []
    for blk in range((n + 3) // 4):
        words.extend(philox4x64_10((blk, layer, 0, 0), (seed & _M64, INIT_KEY1)))
    x = np.array(words[:n], dtype=np.uint64)
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def init_weights(kinds: list, numels: list, fan_ins: list, seed: int) -> list:
    """Weight kind: sigma * sqrt(2) * erfinv(2p - 1), p = Phi(-2) + u (1 - 2 Phi(-2)), sigma = sqrt(2/fan_in)
    (truncated at +-2 sigma); BN gamma 1; BN beta and biases 0. Returns float64 arrays."""
    from scipy.special import erfinv

    phi_m2 = 0.5 * math.erfc(math.sqrt(2.0))  # Phi(-2)
    out = []
    for l, (kind, n) in enumerate(zip(kinds, numels)):
        if kind == WEIGHT:
            u = init_uniform(seed, l, n)
            p = phi_m2 + u * (1.0 - 2.0 * phi_m2)
            sigma = math.sqrt(2.0 / (fan_ins[l] or n))
            out.append(sigma * (math.sqrt(2.0) * erfinv(2.0 * p - 1.0)))
        elif kind == BN_GAMMA:
            out.append(np.ones(n))
        else:
            out.append(np.zeros(n))
    return out
