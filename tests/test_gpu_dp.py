"""Data-parallel parity of dp_allreduce_lars_step (BASELINE configs[2]): torchrun one process per GPU over
NCCL; every rank runs tests/dp_worker.py and reports. nproc = 1 runs the whole case list on ONE GPU through a
one-rank communicator (the fused F1/F2 kernels, the NCCL reduce-scatter/all-gather path, buckets, groups,
half-precision compute weights); larger worlds are skipped on a box with fewer GPUs."""
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


@pytest.mark.parametrize("nproc", [1, 2, 4, 8])
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
        assert rep["layout_mismatch_rejected"] is (None if nproc == 1 else True)
        assert not rep["failures"]
        names = [c["name"] for c in rep["cases"]]
        assert "r50-f16" in names and "nan-on-rank1" in names and "fused-r50-f16-carry" in names
        assert "fused-overflow-sum-f16" in names and "groups-r50-f16" in names
        assert "fused-tiny-graph-replay" in names  # 1,000 graph replays of the fused handshake, bitwise
        # fp32 sums (fused path) and P = 1 are gated at the fp32 tolerance
        for c in rep["cases"]:
            if c.get("reduced_dtype") == "f32" or nproc == 1:
                assert c.get("tol", 1e-5) == 1e-5, c
        print(rk, rep["cases"])


@pytest.mark.parametrize("np_template", [4, 8])
def test_dp_fused_wide_kernel_instance(np_template, tmp_path):
    """The fused F1 instances for 4 and 8 peers (used at P = 3-4 and 5-8) run on the GPUs this box has (one
    is enough) with the absent peers predicated off (LARS_DP_NP): the P = 8 kernel code is exercised and
    gated against the oracle on a box with fewer GPUs."""
    n = min(4, _ngpus())
    if n < 1:
        pytest.skip("needs a GPU")
    env = dict(os.environ, DP_REPORT_DIR=str(tmp_path), NCCL_DEBUG="WARN", LARS_DP_NP=str(np_template),
               DP_CASES="^fused")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29519 + np_template}",
           os.path.join(ROOT, "tests", "dp_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    for rk in range(n):
        rep = json.loads((tmp_path / f"rank{rk}.json").read_text())
        names = [c["name"] for c in rep["cases"]]
        assert names and all(x.startswith("fused") for x in names), names
        assert "fused-r50-f16-carry" in names and "fused-nan-in-split-layer" in names
