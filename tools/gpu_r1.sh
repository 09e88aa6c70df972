#!/bin/bash
# One GPU session: build check, gpu tests, smoke, bench N=1 (+ N=2/4 if visible), ncu launch list and
# one full capture of the top kernel. Output under gpurun_out/$TAG.
TAG=${TAG:-r}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -L > $O/gpus.txt 2>&1
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err
for n in 2 4; do
  [ $n -gt $NG ] && continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench$n.json 2> $O/bench$n.err
  echo "bench$n rc=$?" >> $O/bench$n.err
done
if [ "${SKIP_NCU:-0}" != 1 ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 300 $CMD > $O/plain_ncu_cmd.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
  echo "ncu list rc=$?" >> $O/ncu_list.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 \
    -o $O/ar_full $CMD > $O/ncu_full.log 2>&1
  echo "ncu full rc=$?" >> $O/ncu_full.log
fi
