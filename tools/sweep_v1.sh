#!/bin/bash
# knob sweep of the current kernel at N=2 + copy-engine probe
O=gpurun_out/sweep1; mkdir -p $O
timeout 300 ./tools/tma_probe > $O/tma_probe.jsonl 2>&1; echo "probe rc=$?" >> $O/tma_probe.jsonl
for nch in 32 64; do for tkb in 256 1024 4096; do
 HETCCL_NCHANNELS=$nch HETCCL_TILE_KB=$tkb HETCCL_SLOT_KB=$((tkb*3)) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 bench.py --gpus 2 --steps 10 --warmup 3 2>/dev/null | sed "s/^/nch=$nch tkb=$tkb /" >> $O/bench2.txt
done; done
