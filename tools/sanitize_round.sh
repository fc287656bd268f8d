#!/bin/bash
# compute-sanitizer over every kernel path of the library (tools/sanitize_cases.py), ONE tool per call
# (B200_PROFILING.md: several tools in one call have left the GPU unusable). Only the library's kernels are
# checked (NCCL's own kernels excluded by the name filter). One GPU.
# Usage (GPU box, repo root): bash tools/sanitize_round.sh memcheck|racecheck|synccheck|initcheck OUTDIR [--small]
tool=${1:?tool}
out=${2:-gpurun_out/sanitize}
mkdir -p "$out"
extra=""
[ "$tool" = memcheck ] && extra="--leak-check no --padding 0"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$tool" $extra --kernel-name kns=lars_ \
  --kernel-name kns=empty_step_kernel --error-exitcode 17 --print-limit 50 \
  python tools/sanitize_cases.py $3 > "$out/${tool}.log" 2>&1
echo "compute-sanitizer --tool $tool rc=$?" >> "$out/status"
grep -E "ERROR SUMMARY|========= (Invalid|Race|Barrier|Uninitialized)" "$out/${tool}.log" | sort | uniq -c | head -20 >> "$out/status"
