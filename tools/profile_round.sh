#!/bin/bash
# Round profiling bundle (run under gpurun, 1 GPU): bench line, ncu launch list of the bench command,
# and one `ncu --set full` capture of K1/K2 on the bench workload. Outputs land in gpurun_out/.
set -u
TAG=${1:-r01}
python bench.py --steps 200 --warmup 20 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --soak-s 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --soak-s 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
python tools/profile_step.py > gpurun_out/plain_step_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lars_ -s 6 -c 2 -o gpurun_out/prof_${TAG} \
    python tools/profile_step.py > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
