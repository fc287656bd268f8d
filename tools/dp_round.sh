#!/bin/bash
# Multi-GPU evidence bundle (GPU box, repo root, N GPUs): the whole dp_worker.py case list at P = N (per-rank
# reports), the fused cases with the bulk-copy F1 (LARS_DP_BULK=1) and with the 8-peer F1 instance
# (LARS_DP_NP=8), then bench.py at --gpus N on the default path and with LARS_DP_BULK=1, then the per-CTA
# fused-path trace. Usage: bash tools/dp_round.sh N OUTDIR
N=${1:?N}
out=${2:-gpurun_out/dp$N}
mkdir -p "$out"
run() {  # name, env..., then torchrun args
  local name=$1; shift
  env "$@" NCCL_DEBUG=WARN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
    --master-addr=127.0.0.1 --master-port=$((29600 + RANDOM % 300)) tests/dp_worker.py > "$out/$name.log" 2>&1
  echo "dp_worker $name rc=$?" >> "$out/status"
}
if [ "${DP_ROUND_ONLY:-}" != bench ]; then  # DP_ROUND_ONLY=bench: bench lines and traces only
  mkdir -p "$out/cases" "$out/cases_bulk" "$out/cases_np8"
  run cases DP_REPORT_DIR=$out/cases
  run cases_bulk DP_REPORT_DIR=$out/cases_bulk LARS_DP_BULK=1 DP_CASES=^fused
  run cases_np8 DP_REPORT_DIR=$out/cases_np8 LARS_DP_NP=8 DP_CASES=^fused
fi
for v in 0 1; do
  LARS_DP_BULK=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
    --master-addr=127.0.0.1 --master-port=$((29900 + v)) bench.py --gpus $N > "$out/bench_bulk$v.json" 2> "$out/bench_bulk$v.err"
  echo "bench --gpus $N LARS_DP_BULK=$v rc=$?" >> "$out/status"
done
# the 8-peer F1 instance through bench.py's whole argument/launch/JSON path (absent peers predicated off)
LARS_DP_NP=8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
  --master-addr=127.0.0.1 --master-port=29910 bench.py --gpus $N --steps 100 --warmup 10 --e2e-steps 5 \
  > "$out/bench_np8.json" 2> "$out/bench_np8.err"
echo "bench --gpus $N LARS_DP_NP=8 rc=$?" >> "$out/status"
if [ -f build/liblars_trace.so ]; then
  for v in 0 1; do
    LARS_DP_BULK=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
      --master-addr=127.0.0.1 --master-port=$((29950 + v)) tools/trace_dp.py > "$out/trace_dp_bulk$v.txt" 2>&1
    echo "trace_dp LARS_DP_BULK=$v rc=$?" >> "$out/status"
  done
fi
python - > "$out/nvlink_probe.txt" 2>&1 <<'PY'
import sys, time; sys.path.insert(0, ".")
from tools.nvlink_counters import NvlinkCounters
n = NvlinkCounters(0)
print(n.describe())
n.start(); time.sleep(0.2); print(n.stop())
PY
# configs[3] and configs[4] at P = N (fused NVLink path; --nccl for the NCCL path)
if [ "${DP_ROUND_EXTRA:-0}" = 1 ]; then
  for extra in "" "--nccl"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
      --master-port=29960 tools/schedule_replay.py $extra >> "$out/r152_replay.jsonl" 2>> "$out/r152_replay.err"
    echo "schedule_replay $extra rc=$?" >> "$out/status"
  done
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29961 tools/skew_dp.py > "$out/skew_dp_1b.jsonl" 2> "$out/skew_dp_1b.err"
  echo "skew_dp rc=$?" >> "$out/status"
fi
