#!/bin/bash
# F1 instance / bulk-copy A/B at P = N (GPU box, N GPUs): bench lines (100 steps) and fused-path traces for
# the register and bulk-copy F1 of the native peer-count instance and of the 8-peer instance (LARS_DP_NP=8).
N=${1:-4}
out=${2:-gpurun_out/np8}
mkdir -p $out
for cfg in "LARS_DP_NP=0 LARS_DP_BULK=0" "LARS_DP_NP=0 LARS_DP_BULK=1" "LARS_DP_NP=8 LARS_DP_BULK=0" "LARS_DP_NP=8 LARS_DP_BULK=1"; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg LARS_VERBOSE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29931 bench.py --gpus $N --steps 100 --warmup 10 --e2e-steps 2 --no-cpu-baseline \
    > $out/bench_$tag.json 2> $out/bench_$tag.err
  echo "$cfg rc=$?" >> $out/status
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29932 tools/trace_dp.py > $out/trace_$tag.txt 2>&1
done
