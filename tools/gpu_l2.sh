#!/bin/bash
# L2-policy A/B of the N=1 bench: time (bench) and DRAM bytes (ncu metrics) per HETCCL_L2HINT value in $HS
O=gpurun_out/${TAG:-l2}; mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for h in ${HS:-1 3 7}; do
  HETCCL_L2HINT=$h timeout 300 python bench.py --no-cpu-baseline > $O/ab_$h.json 2>$O/ab_$h.err
  echo "$h $(tail -1 $O/ab_$h.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])")" >> $O/ab.txt
done
$CMD > $O/plain.log 2>&1
for h in ${HS:-1 3 7}; do
  HETCCL_L2HINT=$h timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_allreduce -s 3 -c 1 --csv $CMD > $O/ncu_$h.csv 2>&1
done
