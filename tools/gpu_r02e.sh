O=gpurun_out/r02e; mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for v in tma reg; do
  t=1; [ $v = reg ] && t=0
  HETCCL_TMA=$t $CMD > $O/plain_$v.log 2>&1 && HETCCL_TMA=$t timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_allreduce -s 3 -c 1 -o /tmp/$v $CMD > $O/ncu_$v.log 2>&1
  ncu -i /tmp/$v.ncu-rep --page raw --csv > $O/raw_$v.csv 2>&1
  ncu -i /tmp/$v.ncu-rep --page details --csv > $O/details_$v.csv 2>&1
  ncu -i /tmp/$v.ncu-rep --page source --csv > $O/source_$v.csv 2>&1
  ls -la /tmp/$v.ncu-rep >> $O/sizes.txt
done
echo done > $O/done.txt
