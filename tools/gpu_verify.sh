#!/bin/bash
# end-of-round verification: build, every GPU test, smoke, bench N=1/2/4, the ncu captures of the N=1 kernel
TAG=${TAG:-verify}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err
for n in 2 4; do
  [ $n -gt $NG ] && continue
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2960$n bench.py --gpus $n > $O/bench$n.json 2> $O/bench$n.err; echo "bench$n rc=$?" >> $O/bench$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29804 tools/report.py --what splits --out $O/report_n4.jsonl > $O/report_splits_n4.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > $O/plain_ncu_cmd.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
echo "ncu list rc=$?" >> $O/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 -o $O/ar_full $CMD > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
