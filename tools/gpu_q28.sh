#!/bin/bash
# verification of the cp.async-staged folds on 4 GPUs: every GPU test, smoke, bench N=1/2/4 (A/B vs
# register loads at N=2/4), collectives, ncu launch list + full capture of the N=1 kernel
TAG=${TAG:-q28}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2960$n bench.py --gpus $n > $O/bench$n.json 2> $O/bench$n.err; echo "bench$n rc=$?" >> $O/bench$n.err
  HETCCL_LIB=libhetccl_st0.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2961$n bench.py --gpus $n --no-cpu-baseline > $O/bench${n}_st0.json 2>/dev/null
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29814 tools/report.py --what collectives --out $O/coll_n4.jsonl > $O/coll_n4.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
echo "ncu list rc=$?" >> $O/ncu_list.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 -o $O/ar_full $CMD > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
