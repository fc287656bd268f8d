"""Synthetic parameter layouts (input descriptions only — no LARS arithmetic here).

Shared by the tests, ``bench.py`` and ``__graft_entry__.smoke()`` to describe *what* tensors a
workload has. Neither the CUDA path nor the oracle imports anything else from here; this module
holds none of the method's arithmetic (DESIGN.md §"Input recipe").

A layout is a list of :class:`Tensor` (name, numel, kind, fan_in). ``kind`` is one of
``weight`` (LARS + weight decay), ``bias``, ``bn_gamma``, ``bn_beta`` (skip kinds) — the
per-tensor classification of SURVEY.md §8(c) reading #4 (SPEC.md:33-36 ParamSegment kinds).

Layouts:
  * ``tiny``      — 3 tensors, 10,471 params (BASELINE.json configs[0]).
  * ``resnet50``  — torchvision ResNet-50 order, 161 tensors, 25,557,032 params
                    (``in_ch=4`` gives the paper's 4-channel conv1 variant).
  * ``resnet152`` — 467 tensors, 60,192,808 params (configs[3]).
  * ``skew1b``    — 1,000 tensors summing to 1e9 params (configs[4]); variants
                    ``uniform``, ``loguniform``, ``zipf``, ``giant``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KINDS = ("weight", "bias", "bn_gamma", "bn_beta")
KIND_CODE = {k: i for i, k in enumerate(KINDS)}  # matches lars_kind_t in include/lars.h

SEED = 100000  # run_set_random_seed: 100000 (Appendix log)


@dataclass(frozen=True)
class Tensor:
    name: str
    numel: int
    kind: str
    fan_in: int


def tiny() -> list[Tensor]:
    """BASELINE.json configs[0]: conv1-like 7x7x3x64, an odd-sized weight, a BN gamma."""
    return [
        Tensor("conv1.weight", 9408, "weight", 147),
        Tensor("odd.weight", 999, "weight", 999),
        Tensor("bn.weight", 64, "bn_gamma", 64),
    ]


def _resnet(blocks, in_ch=3) -> list[Tensor]:
    t = [Tensor("conv1.weight", 64 * in_ch * 49, "weight", in_ch * 49),
         Tensor("bn1.weight", 64, "bn_gamma", 64), Tensor("bn1.bias", 64, "bn_beta", 64)]
    inpl = 64
    for li, (nb, pl) in enumerate(zip(blocks, (64, 128, 256, 512))):
        for b in range(nb):
            p = f"layer{li + 1}.{b}."
            t += [Tensor(p + "conv1.weight", pl * inpl, "weight", inpl),
                  Tensor(p + "bn1.weight", pl, "bn_gamma", pl), Tensor(p + "bn1.bias", pl, "bn_beta", pl),
                  Tensor(p + "conv2.weight", pl * pl * 9, "weight", pl * 9),
                  Tensor(p + "bn2.weight", pl, "bn_gamma", pl), Tensor(p + "bn2.bias", pl, "bn_beta", pl),
                  Tensor(p + "conv3.weight", pl * 4 * pl, "weight", pl),
                  Tensor(p + "bn3.weight", pl * 4, "bn_gamma", pl * 4),
                  Tensor(p + "bn3.bias", pl * 4, "bn_beta", pl * 4)]
            if b == 0:
                t += [Tensor(p + "downsample.0.weight", pl * 4 * inpl, "weight", inpl),
                      Tensor(p + "downsample.1.weight", pl * 4, "bn_gamma", pl * 4),
                      Tensor(p + "downsample.1.bias", pl * 4, "bn_beta", pl * 4)]
            inpl = pl * 4
    t += [Tensor("fc.weight", 1000 * 2048, "weight", 2048), Tensor("fc.bias", 1000, "bias", 2048)]
    return t


def resnet50(in_ch: int = 3) -> list[Tensor]:
    return _resnet((3, 4, 6, 3), in_ch)


def resnet152(in_ch: int = 3) -> list[Tensor]:
    return _resnet((3, 8, 36, 3), in_ch)


def skew1b(variant: str = "loguniform", n_tensors: int = 1000, total: int = 1_000_000_000,
           seed: int = SEED) -> list[Tensor]:
    """1,000 weight-kind tensors summing exactly to ``total`` (configs[4])."""
    rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(1)[0])
    if variant == "uniform":
        sizes = np.full(n_tensors, total // n_tensors, dtype=np.int64)
    elif variant == "loguniform":
        sizes = np.exp(rng.uniform(np.log(64), np.log(2 ** 24), n_tensors))
    elif variant == "zipf":
        sizes = 1.0 / np.arange(1, n_tensors + 1) ** 1.2
    elif variant == "giant":
        sizes = np.concatenate([[total / 2], np.full(n_tensors - 1, total / 2 / (n_tensors - 1))])
    else:
        raise ValueError(variant)
    sizes = np.maximum(64, np.floor(sizes / sizes.sum() * total)).astype(np.int64)
    sizes[int(np.argmax(sizes))] += total - int(sizes.sum())  # exact total
    return [Tensor(f"t{i}.weight", int(n), "weight", max(1, int(np.sqrt(n)))) for i, n in enumerate(sizes)]


def by_name(name: str) -> list[Tensor]:
    if name == "tiny":
        return tiny()
    if name == "resnet50":
        return resnet50()
    if name == "resnet50_4ch":
        return resnet50(4)
    if name == "resnet152":
        return resnet152()
    if name.startswith("skew1b"):
        return skew1b(name.split(":", 1)[1] if ":" in name else "loguniform")
    raise ValueError(f"unknown layout {name!r}")


def random_layout(rng: np.random.Generator, n: int, max_numel: int = 5000) -> list[Tensor]:
    """Random odd-sized layouts for parity sweeps (ragged tails, tiny tensors, all kinds)."""
    out = []
    for i in range(n):
        numel = int(rng.integers(1, max_numel + 1))
        kind = KINDS[int(rng.integers(0, 4))] if i % 3 else "weight"
        out.append(Tensor(f"r{i}", numel, kind, max(1, numel // 3)))
    return out
