#!/bin/bash
# multi-GPU per-iteration traces: trace_run.py under torchrun on $N GPUs for each env combination in $ENVS
O=gpurun_out/${TAG:-tracen}; mkdir -p $O
for e in ${ENVS:-NONE=1}; do
  env ${e//,/ } timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-4} --master-addr 127.0.0.1 \
    --master-port 29$((RANDOM%800+100)) tools/trace_run.py --sym --out $O/t_$e > $O/trace_$e.txt 2>&1
done
