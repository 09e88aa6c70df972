#!/bin/bash
# perf pass: traces at N=2/4, tile sweep at N=#GPUs, then ncu (launch list + full) on the 1-GPU mux bench
TAG=${TAG:-p}; O=gpurun_out/$TAG; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
for n in 2 4; do
  [ $n -gt $NG ] && continue
  for tkb in ${TRACE_TKB:-256}; do
  HETCCL_TILE_KB=$tkb HETCCL_SLOT_KB=$((tkb*4)) HETCCL_NCHANNELS=148 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2970$n tools/trace_run.py --out $O/trace_n${n}_t$tkb >> $O/trace.txt 2>&1
  done
done
for tkb in ${SWEEP_TKB:-}; do for nch in ${SWEEP_NCH:-148}; do
  HETCCL_NCHANNELS=$nch HETCCL_TILE_KB=$tkb HETCCL_SLOT_KB=$((tkb*4)) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG \
    --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null \
    | sed "s/^/nch=$nch tkb=$tkb /" >> $O/sweep.txt
done; done
if [ "${NCU:-1}" = 1 ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 300 $CMD > $O/plain_ncu_cmd.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
  echo "ncu list rc=$?" >> $O/ncu_list.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 \
    -o $O/ar_full $CMD > $O/ncu_full.log 2>&1
  echo "ncu full rc=$?" >> $O/ncu_full.log
fi
