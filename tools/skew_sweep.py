#!/usr/bin/env python
"""configs[4] measurement: 10^9-param, 1,000-tensor skewed layouts on one B200 — K1 (norms) and K2
(update) algorithmic GB/s per size mix, and the flatness across mixes (load balance). One JSON line per
(variant, grad dtype) plus a summary line. Timing: lars_profile_* CUDA events on the launching stream,
after warm-up; inputs (12 GB) far exceed L2."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1903_12650_b200 as P
    from synth import gen_torch as GT
    from synth import layouts as LY

    steps = int(os.environ.get("SKEW_STEPS", "20"))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rows = []
    dev = torch.device("cuda", 0)
    for dtype in ("f32", "f16"):
        for variant in ("uniform", "loguniform", "zipf", "giant"):
            lay = LY.skew1b(variant)
            E = sum(t.numel for t in lay)
            h = P.Lars([(t.numel, t.kind) for t in lay], device=0, base_lr=32.0, grad_dtype=dtype,
                       grad_scale=1.0 / 1024)
            w = torch.zeros(h.padded_numel, dtype=torch.float32, device=dev)
            g = torch.zeros(h.padded_numel, dtype=torch.float32 if dtype == "f32" else torch.float16, device=dev)
            m = torch.zeros(h.padded_numel, dtype=torch.float32, device=dev)
            GT.fill_weights(w, lay, h.offsets)
            GT.fill_grads(g, lay, h.offsets)
            GT.fill_momentum(m, lay, h.offsets)
            for i in range(3):
                h.lars_step(w, g, m, 700 + i)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(steps):
                h.lars_step(w, g, m, 710 + i)
            e1.record()
            torch.cuda.synchronize()
            step_ms = e0.elapsed_time(e1) / steps
            h.profile_enable(True)
            for i in range(steps):
                h.lars_step(w, g, m, 740 + i)
            ph, n = h.profile_read()
            h.profile_enable(False)
            assert not h.last_step_skipped()
            gb = 4 if dtype == "f32" else 2
            k1, k2 = ph["norms"] / n, ph["update"] / n
            row = {"variant": variant, "grad_dtype": dtype, "params": E, "max_tensor": max(t.numel for t in lay),
                   "step_ms": round(step_ms, 4), "k1_ms": round(k1, 4), "k2_ms": round(k2, 4),
                   "k1_GBps": round((4 + gb) * E / (k1 * 1e-3) / 1e9, 1),
                   "k2_GBps": round((16 + gb) * E / (k2 * 1e-3) / 1e9, 1),
                   "step_alg_GBps": round((16 + gb) * E / (step_ms * 1e-3) / 1e9, 1)}
            row["k2_frac_of_peak"] = round(row["k2_GBps"] / peak, 4)
            row["step_frac_of_peak"] = round(row["step_alg_GBps"] / peak, 4)
            rows.append(row)
            print(json.dumps(row), flush=True)
            del w, g, m
            h.close()
            torch.cuda.empty_cache()
    for dtype in ("f32", "f16"):
        r = [x for x in rows if x["grad_dtype"] == dtype]
        print(json.dumps({"summary": dtype, "hbm_peak_GBps": peak,
                          "k1_flatness_min_over_max": round(min(x["k1_GBps"] for x in r) / max(x["k1_GBps"] for x in r), 4),
                          "k2_flatness_min_over_max": round(min(x["k2_GBps"] for x in r) / max(x["k2_GBps"] for x in r), 4)}))


if __name__ == "__main__":
    main()
