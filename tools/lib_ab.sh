#!/bin/bash
# A/B of two library builds on the bench at P = N (GPU box): alternating runs, 100 steps each.
# Usage: bash tools/lib_ab.sh N OUTDIR LIB_B [reps]
N=${1:?N}; out=${2:?out}; libb=${3:?lib}; reps=${4:-2}
mkdir -p $out
for i in $(seq $reps); do
  for tag in a b; do
    if [ $tag = b ]; then export LARS_LIB=$libb; else unset LARS_LIB; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
      --master-port=$((29800 + i)) bench.py --gpus $N --steps 200 --warmup 20 --e2e-steps 2 --no-cpu-baseline \
      >> $out/bench_$tag.jsonl 2>> $out/bench_$tag.err
  done
done
