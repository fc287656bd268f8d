#!/bin/bash
# Repeated bench runs at P = N, each under its own timeout, to catch an intermittent stall (GPU box).
# Usage: bash tools/repeat_bench.sh N OUTDIR REPS
N=${1:?N}; out=${2:?out}; reps=${3:-6}
mkdir -p $out
for i in $(seq $reps); do
  timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=$((29700 + i)) bench.py --gpus $N --steps 200 --warmup 20 --e2e-steps 2 --no-cpu-baseline \
    > $out/run$i.json 2> $out/run$i.err
  echo "run $i rc=$?" >> $out/status
done
