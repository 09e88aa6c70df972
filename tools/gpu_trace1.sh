O=gpurun_out/${TAG:-trace}; mkdir -p $O
for e in ${ENVS:-NONE=1}; do
  env ${e//,/ } timeout 300 python tools/trace_run.py --out $O/t_$e > $O/trace_$e.txt 2>&1
done
