"""The boundary driven from plain C (examples/c_abi_demo.c, compiled here with gcc against include/lars.h and the
in-tree library): no Python on the product side. CPU: planning, schedule and error codes.
GPU: one lars_step at t = 80 on exactly representable inputs, checked against the oracle."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "c_abi_demo.c")
LIBDIR = os.path.join(ROOT, "paper_1903_12650_b200")
TINY = [(9408, O.WEIGHT), (999, O.WEIGHT), (64, O.BN_GAMMA)]


def _compile(tmp_path, cuda: bool) -> str:
    exe = str(tmp_path / ("demo_gpu" if cuda else "demo"))
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR, "-llars_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    if cuda:
        cmd[1:1] = ["-DWITH_CUDA", "-I", "/usr/local/cuda/include"]
        cmd += ["-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def _run(exe, *args) -> list[list[str]]:
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return [ln.split() for ln in r.stdout.splitlines()]


def test_c_program_plans_and_reports_errors(tmp_path):
    out = _run(_compile(tmp_path, cuda=False))
    kv = {ln[0]: ln[1:] for ln in out}
    assert kv["err_layout"] == ["2"] and kv["err_no_base_lr"] == ["1"] and kv["err_iter_range"] == ["3"]
    assert kv["schedule"] == ["ipe=16", "T=1440", "W=80"]
    assert kv["layout"] == ["0", "9408", "10432", "padded=10496"]  # 64-element aligned offsets
    hp = O.HParams(base_lr=32.0)
    for ln in out:
        if ln[0] == "lr":
            assert float(ln[2]) == O.lr_at(hp, int(ln[1])), ln  # printed with 17 digits: exact double


def _inputs():
    w, g, m = [], [], []
    for l, (n, _) in enumerate(TINY):
        i = np.arange(n, dtype=np.int64)
        w.append(((i * 37 + l * 11) % 2001 - 1000) * 2.0 ** -16 + (1.0 if l == 2 else 0.0))
        g.append(((i * 53 + l * 7) % 1999 - 999) * 2.0 ** -20)
        m.append(((i * 29 + l * 3) % 997 - 498) * 2.0 ** -24)
    f32 = lambda xs: [x.astype(np.float32) for x in xs]  # exact: small integers times powers of two
    return f32(w), f32(g), f32(m)


@pytest.mark.gpu
def test_c_program_step_matches_oracle(tmp_path):
    from tests._parity import TOL_F32, TOL_NORM, gate, gate_norms

    out = _run(_compile(tmp_path, cuda=True), "gpu")
    kv = {ln[0]: ln[1:] for ln in out}
    assert kv["skipped"] == ["0"]
    w, g, m = _inputs()
    hp = O.HParams(base_lr=32.0)
    ref = O.step([k for _, k in TINY], hp, 80, w, [g], m)
    for ln in out:
        if ln[0] == "norms":
            l = int(ln[1])
            gate_norms(f"||w|| {l}", [float(ln[2])], [ref.w_norm[l]], TOL_NORM)
            gate_norms(f"||g|| {l}", [float(ln[3])], [ref.g_norm[l]], TOL_NORM)
            gate_norms(f"lambda {l}", [float(ln[4])], [ref.lam[l]], 1e-6)
    got_w, got_m, want_w, want_m, env_w, env_m = [], [], [], [], [], []
    for ln in out:
        if ln[0] == "wm":
            l, i = int(ln[1]), int(ln[2])
            got_w.append(float(ln[3]))
            got_m.append(float(ln[4]))
            want_w.append(ref.w[l][i])
            want_m.append(ref.m[l][i])
            env_w.append(ref.w_env[l][i])
            env_m.append(ref.m_env[l][i])
    assert len(got_w) > 100
    # printed with 9 significant digits: exact for float32
    gate("C step w", got_w, want_w, env_w, TOL_F32)
    gate("C step m", got_m, want_m, env_m, TOL_F32)
