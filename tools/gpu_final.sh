#!/bin/bash
# final measurement session of the round: tests, smoke, bench N=1/2/4, reference arm (N=1), report rows,
# a trace and the ncu captures of the N=1 bench kernel. Output under gpurun_out/$TAG.
TAG=${TAG:-final}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
nvidia-smi > $O/nvidia-smi.txt 2>&1; nproc > $O/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err
timeout 600 python bench.py --impl reference > $O/ref1.json 2> $O/ref1.err
for n in 2 4; do
  [ $n -gt $NG ] && continue
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2960$n bench.py --gpus $n > $O/bench$n.json 2> $O/bench$n.err; echo "bench$n rc=$?" >> $O/bench$n.err
done
for w in ${REPORT4:-splits ar_sweep collectives c5 c4}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29804 tools/report.py --what $w --out $O/report_n4.jsonl > $O/report_${w}_n4.log 2>&1
  echo "report $w n=4 rc=$?" >> $O/report_rc.txt
done
for w in ${REPORT2:-splits ar_sweep}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29802 tools/report.py --what $w --out $O/report_n2.jsonl > $O/report_${w}_n2.log 2>&1
  echo "report $w n=2 rc=$?" >> $O/report_rc.txt
done
HETCCL_TRACE_ITERS=256 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29904 tools/trace_run.py --sym --out $O/trace_n4 >> $O/trace.txt 2>&1
HETCCL_TRACE_ITERS=256 timeout 300 python tools/trace_run.py --out $O/trace_mux >> $O/trace.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > $O/plain_ncu_cmd.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
echo "ncu list rc=$?" >> $O/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 -o $O/ar_full $CMD > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
