O=gpurun_out/r02n; mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for h in 0 1 2 4 6 7; do
  HETCCL_L2HINT=$h timeout 300 python bench.py --no-cpu-baseline --steps 20 > $O/ab_$h.json 2>$O/ab_$h.err
  echo "$h $(python -c "import json; d=json.load(open('$O/ab_$h.json')); print(d['value'], d['roofline']['frac'])")" >> $O/ab.txt
done
$CMD > $O/plain.log 2>&1
for h in 0 6 7; do
  HETCCL_L2HINT=$h timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_allreduce -s 3 -c 1 --csv $CMD > $O/ncu_$h.csv 2>&1
done
