#!/bin/bash
TAG=${TAG:-q9}; O=gpurun_out/$TAG; mkdir -p $O
SKIP_SWEEP=1 bash tools/gpu_quick.sh
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > $O/plain_ncu_cmd.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
echo "ncu list rc=$?" >> $O/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 -o $O/ar_full $CMD > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/ncu_full.log
