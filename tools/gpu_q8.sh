#!/bin/bash
TAG=${TAG:-q8}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --maxfail=30 --timeout 180 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for n in 2 4; do
  for mt in 1 4 8; do
    HETCCL_MIN_TILES=$mt timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2980$n tools/report.py --what ar_sweep --out $O/sweep_mt${mt}_n$n.jsonl > $O/sweep_mt${mt}_n$n.log 2>&1
  done
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2981$n tools/report.py --what collectives --out $O/coll_n$n.jsonl > $O/coll_n$n.log 2>&1
done
