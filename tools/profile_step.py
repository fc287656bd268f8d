#!/usr/bin/env python
"""Short single-GPU run of lars_step for ncu / compute-sanitizer captures (no timing printed as a result).

    python tools/profile_step.py --layout resnet50 --dtype f32 --warmup 3 --steps 3
    ncu --set full -k regex:lars_ -s 6 -c 2 -o gpurun_out/prof python tools/profile_step.py ...
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--flags", type=int, default=0, help="lars_hparams_t.flags (1 = carry weight norms)")
    a = ap.parse_args()
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    lay = LY.by_name(a.layout)
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype=a.dtype, base_lr=32.0,
                grad_scale=1.0 / G.GRAD_PRESCALE, flags=a.flags)
    dev = torch.device("cuda", 0)
    w = torch.from_numpy(G.pack(G.weights(lay), h.offsets, h.padded_numel)).to(dev)
    g = torch.from_numpy(G.pack(G.grads(lay, 0, 0, a.dtype), h.offsets, h.padded_numel)).to(dev)
    m = torch.from_numpy(G.pack(G.momentum(lay, 1e-3), h.offsets, h.padded_numel)).to(dev)
    for i in range(a.warmup + a.steps):
        h.lars_step(w, g, m, 719 + i)
    torch.cuda.synchronize()
    assert not h.last_step_skipped()
    print("ok", a.layout, a.dtype, a.warmup + a.steps, "steps")


if __name__ == "__main__":
    main()
