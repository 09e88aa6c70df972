#!/bin/bash
TAG=${TAG:-q12}; O=gpurun_out/$TAG; mkdir -p $O
SKIP_SWEEP=1 bash tools/gpu_quick.sh
AB_VARS="HETCCL_NSLOTS=8" AB_TKB="128 192 256 384" bash tools/gpu_ab.sh
for t in 128 256; do HETCCL_TILE_KB=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | sed "s/^/tkb=$t /" >> $O/mux.txt; done
for n in 2 4; do
  HETCCL_TRACE_ITERS=256 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2990$n tools/trace_run.py --sym --out $O/trace_n$n >> $O/trace.txt 2>&1
done
