"""Multi-GPU parity of dp_allreduce_lars_step (BASELINE configs[2]): torchrun one process per GPU over
NCCL; every rank runs tests/dp_worker.py and reports. Skipped on a box with fewer than 2 GPUs."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus() -> int:
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_dp_step_parity_and_replica_consistency(nproc, tmp_path):
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs, have {_ngpus()}")
    env = dict(os.environ, DP_REPORT_DIR=str(tmp_path), NCCL_DEBUG="WARN")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + nproc}", os.path.join(ROOT, "tests", "dp_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    for rk in range(nproc):
        rep = json.loads((tmp_path / f"rank{rk}.json").read_text())
        assert rep["layout_mismatch_rejected"]
        names = [c["name"] for c in rep["cases"]]
        assert "r50-f16" in names and "nan-on-rank1" in names
        print(rk, rep["cases"])


def test_dp_fused_p8_kernel_instance(tmp_path):
    """The fused F1 instance for 8 peers (used at P = 8) run at P = 2 or 4 with the absent peers predicated
    off (LARS_DP_NP=8): the P = 8 kernel code is exercised on a box with fewer GPUs."""
    n = min(4, _ngpus())
    if n < 2:
        pytest.skip(f"needs 2 GPUs, have {_ngpus()}")
    env = dict(os.environ, DP_REPORT_DIR=str(tmp_path), NCCL_DEBUG="WARN", LARS_DP_NP="8", DP_CASES="^fused")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29519", os.path.join(ROOT, "tests", "dp_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    for rk in range(n):
        rep = json.loads((tmp_path / f"rank{rk}.json").read_text())
        names = [c["name"] for c in rep["cases"]]
        assert names and all(x.startswith("fused") for x in names), names
        assert "fused-r50-f16-carry" in names and "fused-nan-in-split-layer" in names
