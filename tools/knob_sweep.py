#!/usr/bin/env python
"""Single-GPU lars_step timing over environment knobs read at lars_init (e.g. LARS_DEFER_FINISH).

    python tools/knob_sweep.py --knob LARS_DEFER_FINISH --values 0,1 --dtype f32,f16

Each (dtype, value) gets a fresh handle on the same device buffers (ResNet-50 layout by default, carried
weight norms as in bench.py); the step is timed with CUDA events over --steps steps, --reps times,
interleaved across values so clock drift hits every value alike. One JSON line per (dtype, value):
median / min ms per step and the K1 / K2 phase split (library profiling events, separate pass).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--knob", default="LARS_DEFER_FINISH")
    ap.add_argument("--values", default="0,1")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--layout", default="resnet50")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--flags", type=int, default=1, help="lars_hparams_t.flags (1 = carry weight norms)")
    a = ap.parse_args()
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    lay = LY.by_name(a.layout)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    for dtype in a.dtype.split(","):
        handles = {}
        for v in a.values.split(","):
            os.environ[a.knob] = v
            handles[v] = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype=dtype, base_lr=32.0,
                                 grad_scale=1.0 / G.GRAD_PRESCALE, flags=a.flags)
        os.environ.pop(a.knob, None)
        h0 = next(iter(handles.values()))
        w = torch.from_numpy(G.pack(G.weights(lay), h0.offsets, h0.padded_numel)).to(dev)
        g = torch.from_numpy(G.pack(G.grads(lay, 0, 0, dtype), h0.offsets, h0.padded_numel)).to(dev)
        m = torch.from_numpy(G.pack(G.momentum(lay, 1e-3), h0.offsets, h0.padded_numel)).to(dev)
        times = {v: [] for v in handles}
        for rep in range(a.reps):
            for v, h in handles.items():
                h.invalidate_carried_norms()
                for i in range(20):
                    h.lars_step(w, g, m, 719 + i, stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                for i in range(a.steps):
                    h.lars_step(w, g, m, (719 + i) % 1440, stream)
                e1.record(stream)
                torch.cuda.synchronize()
                assert not h.last_step_skipped()
                times[v].append(e0.elapsed_time(e1) / a.steps)
        for v, h in handles.items():
            h.invalidate_carried_norms()
            h.profile_enable(True)
            for i in range(a.steps):
                h.lars_step(w, g, m, (719 + i) % 1440, stream)
            ph, n = h.profile_read()
            h.profile_enable(False)
            print(json.dumps({"knob": a.knob, "value": v, "dtype": dtype, "layout": a.layout,
                              "ms_median": round(statistics.median(times[v]), 5), "ms_min": round(min(times[v]), 5),
                              "phases_ms": {k: round(x / max(1, n), 5) for k, x in ph.items()}}), flush=True)
            h.close()


if __name__ == "__main__":
    main()
