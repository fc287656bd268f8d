import os, sys
sys.path.insert(0, ".")
import torch, paper_1903_12650_b200 as PK
from synth import layouts as LY
lay = LY.resnet50()
for dt in ("f32", "f16"):
    os.environ["LARS_K1_BULK"] = "1"
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype=dt, base_lr=32.0, flags=1); h.close()
for npt in ("2", "4", "8"):
    os.environ["LARS_DP_BULK"] = "1"; os.environ["LARS_DP_NP"] = npt
    h = PK.Lars([(t.numel, t.kind) for t in lay], device=0, grad_dtype="f16", base_lr=32.0, nranks=1, flags=1)
    h.comm_init(0, 1, PK.get_unique_id()); h.close()
