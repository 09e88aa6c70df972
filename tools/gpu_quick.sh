#!/bin/bash
# quick correctness + perf pass: build, gpu tests (all failures listed), bench at N=1 and N=#GPUs
TAG=${TAG:-q}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 1500 python -m pytest tests -m gpu -q --maxfail=30 --timeout 180 ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err
for n in 2 4; do
  [ $n -gt $NG ] && continue
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2960$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench$n.json 2> $O/bench$n.err
  echo "bench$n rc=$?" >> $O/bench$n.err
done
for nch in ${SWEEP_NCH:-}; do for tkb in ${SWEEP_TKB:-256}; do
  HETCCL_NCHANNELS=$nch HETCCL_TILE_KB=$tkb timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG \
    --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null \
    | sed "s/^/nch=$nch tkb=$tkb /" >> $O/sweep.txt
done; done
