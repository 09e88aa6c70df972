#!/bin/bash
# Profile one library variant / env of the N=1 bench: per-iteration trace + ncu --set full (CSV exports only,
# the .ncu-rep stays on the box unless KEEP_REP=1).   TAG=... LIBV=c4 ENVX="HETCCL_FLAT_AG=1" bash tools/gpu_prof.sh
O=gpurun_out/${TAG:-prof}; mkdir -p $O
LIB=libhetccl.so; [ -n "$LIBV" ] && LIB=libhetccl_$LIBV.so
export HETCCL_LIB=$LIB; for e in ${ENVX//,/ }; do export $e; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 python tools/trace_run.py --out $O/trace > $O/trace.txt 2>&1
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_allreduce} -s 3 -c 1 -o /tmp/prof $CMD > $O/ncu.log 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > $O/raw.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page details --csv > $O/details.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page source --csv > $O/source.csv 2>&1
[ "$KEEP_REP" = 1 ] && cp /tmp/prof.ncu-rep $O/
echo done > $O/done.txt
