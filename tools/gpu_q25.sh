#!/bin/bash
# GPU-scope flag operations for rank-multiplexed comms: mux tests + A/B against .sys
TAG=${TAG:-q25}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "not multi and not nccl and not ddp and not shim" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for rep in 1 2; do
  for v in HETCCL_SYS_SCOPE=0 HETCCL_SYS_SCOPE=1; do
    env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | sed "s/^/$v /" >> $O/mux.txt
  done
done
for v in HETCCL_SYS_SCOPE=0 HETCCL_SYS_SCOPE=1; do
  env $v timeout 300 python tools/trace_run.py --out $O/trace_$v > $O/trace_$v.txt 2>&1
done
