#!/bin/bash
# multi-GPU A/B of bench.py under torchrun: for each N in $NS and env combo in $ENVS (commas separate vars)
O=gpurun_out/${TAG:-mab}; mkdir -p $O
NGPU=$(python -c 'import torch; print(torch.cuda.device_count())')
for n in ${NS:-4}; do
  [ "$NGPU" -ge "$n" ] || continue
  for e in ${ENVS:-NONE=1}; do
    env ${e//,/ } timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2970$n bench.py --gpus $n --no-cpu-baseline ${BARGS} > $O/b${n}_$e.json 2> $O/b${n}_$e.err
    echo "n=$n $e $(tail -1 $O/b${n}_$e.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['nccl_flat'], d['staged_recv']['busbw'], d['roofline']['frac'])" 2>&1 | tail -1)" >> $O/mab.txt
  done
done
