#!/usr/bin/env python
"""Per-CTA timeline of K1/K2 from the diagnostics library (tools/trace_build.py)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1903_12650_b200 as PK
    from synth import gen as G
    from synth import layouts as LY

    lib = PK.load_library(os.path.join(ROOT, "build", f"liblars_trace{os.environ.get('TRACE_TAG', '')}.so"))
    layout = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
    lay = LY.by_name(layout)
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype=dtype, base_lr=32.0, grad_scale=1 / 1024,
                flags=int(os.environ.get("TRACE_FLAGS", "0")))
    dev = torch.device("cuda", 0)
    w = torch.from_numpy(G.pack(G.weights(lay), h.offsets, h.padded_numel)).to(dev)
    g = torch.from_numpy(G.pack(G.grads(lay, 0, 0, dtype), h.offsets, h.padded_numel)).to(dev)
    m = torch.from_numpy(G.pack(G.momentum(lay, 1e-3), h.offsets, h.padded_numel)).to(dev)
    buf = torch.zeros(2 * 4096 * 4, dtype=torch.int64, device=dev)
    lib.lars_trace_arm.argtypes = [ctypes.c_void_p]
    for i in range(30):
        h.lars_step(w, g, m, 719 + i)
    torch.cuda.synchronize()
    assert lib.lars_trace_arm(buf.data_ptr()) == 0
    for i in range(3):
        h.lars_step(w, g, m, 800 + i)
        torch.cuda.synchronize()
    tr = buf.view(2, 4096, 4).cpu().numpy()
    for k, name in enumerate(["K1 norms", "K2 update"]):
        n = int(tr[k, 0, 3])
        t = tr[k, :n]
        t0 = t[:, 0].min()
        st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        dur = en - st
        print(f"{name}: ctas={n} span={en.max():.1f}us start[min,max]=({st.min():.1f},{st.max():.1f}) "
              f"end[min,p50,max]=({en.min():.1f},{np.median(en):.1f},{en.max():.1f}) dur[min,p50,max]=("
              f"{dur.min():.1f},{np.median(dur):.1f},{dur.max():.1f})")
        slow = np.argsort(-en)[:8]
        print("  slowest CTAs (cta, sm, start, end):", [(int(c), int(t[c, 2]), round(st[c], 1), round(en[c], 1)) for c in slow])
        sms = t[:, 2]
        per_sm = {}
        for c in range(n):
            per_sm.setdefault(int(sms[c]), []).append(c)
        load = sorted(((len(v), s) for s, v in per_sm.items()), reverse=True)
        print("  CTAs per SM (max, min, #SMs):", load[0][0], load[-1][0], len(per_sm))


if __name__ == "__main__":
    main()
