#!/bin/bash
# Round profiling bundle (run under gpurun, 1 GPU): the default bench line, the ncu launch list of the bench
# command, one `ncu --set full` capture of K1/K2 on the bench workload (carried weight norms, as the bench
# runs) and a warm-cache DRAM pass. Outputs land in gpurun_out/; copy what is judged into profiles/.
set -u
TAG=${1:-r01}
python bench.py > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --soak-s 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --soak-s 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
python tools/profile_step.py --flags 1 > gpurun_out/plain_step_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lars_ -s 6 -c 2 -o gpurun_out/prof_${TAG}_carry \
    python tools/profile_step.py --flags 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    -k regex:lars_ -s 6 -c 4 --csv python tools/profile_step.py --flags 1 > gpurun_out/ncu_warm_${TAG}.csv 2>&1
echo "ncu warm rc=$?"
# configs[3] and configs[4] at P = 1 with the round's code (no profiler)
timeout 600 python tools/schedule_replay.py > gpurun_out/r152_replay_${TAG}.jsonl 2> gpurun_out/r152_replay_${TAG}.err
echo "schedule_replay rc=$?"
timeout 900 python tools/skew_sweep.py > gpurun_out/skew_sweep_${TAG}.jsonl 2> gpurun_out/skew_sweep_${TAG}.err
echo "skew_sweep rc=$?"
# the fused data-parallel kernels F1/F2 through a one-rank communicator (ncu cannot replay a multi-rank run)
python tools/profile_dp1.py > gpurun_out/plain_dp1_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lars_dp_ -s 6 -c 2 -o gpurun_out/prof_${TAG}_dp1 \
    python tools/profile_dp1.py > gpurun_out/ncu_dp1_${TAG}.log 2>&1
echo "ncu dp1 rc=$?"
