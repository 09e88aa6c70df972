#!/bin/bash
TAG=${TAG:-q7}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
SKIP_SWEEP=1 bash tools/gpu_quick.sh
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2980$n tools/report.py --what ar_sweep --out $O/sweep_n$n.jsonl > $O/sweep_n$n.log 2>&1
done
