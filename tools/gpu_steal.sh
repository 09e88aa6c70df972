#!/bin/bash
# chunk-stealing session: the protocol tests that cover it, N=1 bench A/B over $ENVS and a trace with $TRACE_ENV
O=gpurun_out/${TAG:-steal}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mux_protocol.py -q -p no:cacheprovider --timeout 300 -k steal > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for e in ${ENVS:-HETCCL_STEAL=0 HETCCL_STEAL=100}; do
  env ${e//,/ } timeout 300 python bench.py --no-cpu-baseline > $O/ab.json 2> $O/ab.err
  echo "$e $(tail -1 $O/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1)" >> $O/ab.txt
done
env ${TRACE_ENV:-HETCCL_STEAL=25} timeout 300 python tools/trace_run.py --out $O/t > $O/trace.txt 2>&1
