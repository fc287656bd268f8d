#!/usr/bin/env python
"""A short fused data-parallel loop through a ONE-rank communicator (F1 reduce+norms, F2 update+gather on a
single GPU: no peer traffic, every other instruction of the kernels), ResNet-50 layout, fp16 gradients,
carried norms — for ncu captures of the fused kernels, which cannot be profiled in a multi-rank run.

    ncu --set full -k regex:lars_dp_ -s 6 -c 2 -o gpurun_out/prof_dp1 python tools/profile_dp1.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    lay = LY.resnet50()
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype="f16", base_lr=32.0, nranks=1,
                grad_scale=1.0 / G.GRAD_PRESCALE, flags=PK.lars.FLAG_CARRY_WNORM)
    h.comm_init(0, 1, PK.get_unique_id())
    w, g = h.dp_buffers()
    w.copy_(torch.from_numpy(G.pack(G.weights(lay), h.offsets, h.padded_numel)))
    g.copy_(torch.from_numpy(G.pack(G.grads(lay, 0, 0, "f16"), h.offsets, h.padded_numel)))
    m = torch.from_numpy(G.pack(G.momentum(lay, 1e-3), h.offsets, h.padded_numel)).to(w.device)
    for i in range(6):
        h.dp_allreduce_lars_step(w, g, m, 719 + i)
    torch.cuda.synchronize()
    assert h.last_step_status() == 0
    print("ok fused 1-rank steps", flush=True)
    h.close()


if __name__ == "__main__":
    main()
