#!/bin/bash
# one GPU session: smoke, bench N=1 (+ncu launch list), bench N=2/4 via torchrun
mkdir -p gpurun_out/r
O=gpurun_out/r
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err
NG=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -gt $NG ] && continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 10 --warmup 3 > $O/bench$n.json 2> $O/bench$n.err; echo "bench$n rc=$?" >> $O/bench$n.err
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_ncu_cmd.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_list.log 2>&1
echo "ncu rc=$?" >> $O/ncu_list.log
