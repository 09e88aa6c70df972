#!/bin/bash
# P0 box probe: GPUs, P2P matrix, push/pull NVLink bandwidth, NCCL flat baselines. Output -> gpurun_out/probe/
mkdir -p gpurun_out/probe
nvidia-smi > gpurun_out/probe/nvidia-smi.txt 2>&1
nvidia-smi topo -m > gpurun_out/probe/topo.txt 2>&1
nproc > gpurun_out/probe/nproc.txt
timeout 300 ./tools/p2p_probe > gpurun_out/probe/p2p.jsonl 2>&1
N=$(nvidia-smi -L | wc -l)
for tag in default ring nonvls; do
  env=""
  [ $tag = ring ] && env="NCCL_ALGO=Ring"
  [ $tag = nonvls ] && env="NCCL_NVLS_ENABLE=0"
  for n in 2 $N; do
    [ $n -gt $N ] && continue
    env $env PROBE_TAG=$tag timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/nccl_probe.py >> gpurun_out/probe/nccl.jsonl 2>> gpurun_out/probe/nccl.err
  done
done
NCCL_DEBUG=INFO timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/nccl_probe.py > gpurun_out/probe/nccl_debug.log 2>&1
grep -iE "nvls|multicast|NCCL version" gpurun_out/probe/nccl_debug.log | head -40 > gpurun_out/probe/nvls_grep.txt
echo done
