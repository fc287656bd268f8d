#!/bin/bash
# Device-checked run (tools/checked_step.py docstring): every kernel path with -DLARS_DEVICE_CHECKS bounds
# and invariant checks, plus the whole GPU test suite against the checked library. One GPU.
# Usage (GPU box, repo root, after `python -m paper_1903_12650_b200.build --checked` here): tools/checked_round.sh OUT
out=${1:-gpurun_out/checked}
mkdir -p "$out"
export LARS_LIB=build/checked/liblars_b200_checked.so
for lay in tiny resnet50 resnet152; do
  timeout 600 python tools/checked_step.py --layout $lay > "$out/step_${lay}.log" 2>&1
  echo "checked_step $lay rc=$?" >> "$out/status"
done
timeout 600 python tools/sanitize_cases.py > "$out/sanitize_cases.log" 2>&1
echo "sanitize_cases (every kernel path incl. the 8-peer F1 instance) rc=$?" >> "$out/status"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > "$out/pytest_checked.log" 2>&1
echo "pytest -m gpu (checked library) rc=$?" >> "$out/status"
