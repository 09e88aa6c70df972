#!/bin/bash
# cp.async-staged fold sources: single-GPU tests + mux A/B against register loads (libhetccl_st0.so)
TAG=${TAG:-q27}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "not multi and not nccl and not ddp and not shim" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for rep in 1 2; do
  for lib in libhetccl.so libhetccl_st0.so; do
    HETCCL_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>$O/err.txt | sed "s/^/$lib /" >> $O/mux.txt
  done
done
HETCCL_LIB=libhetccl.so timeout 300 python tools/trace_run.py --out $O/trace > $O/trace.txt 2>&1
