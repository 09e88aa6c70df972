#!/bin/bash
TAG=${TAG:-q6}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
bash tools/gpu_quick.sh
for n in 2 4; do
  for os in 1024 8192; do
    HETCCL_ONESHOT_KB=$os timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2980$n tools/report.py --what ar_sweep --out $O/sweep_os${os}_n$n.jsonl > $O/sweep_os${os}_n$n.log 2>&1
  done
done
AB_VARS="HETCCL_NSLOTS=8 HETCCL_WS=2,HETCCL_NSLOTS=12" AB_TKB="256 384" bash tools/gpu_ab.sh
