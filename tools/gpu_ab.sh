#!/bin/bash
# A/B sweep of env knobs at N = 2 and N = #GPUs: AB_VARS="HETCCL_WS=0 HETCCL_WS=1" x TKB
TAG=${TAG:-ab}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
for n in ${AB_N:-2 $NG}; do
for v in ${AB_VARS:-HETCCL_WS=1}; do for tkb in ${AB_TKB:-256}; do
  env ${v//,/ } HETCCL_TILE_KB=$tkb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null \
    | sed "s/^/n=$n $v tkb=$tkb /" >> $O/ab.txt
done; done; done
