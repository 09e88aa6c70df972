#!/bin/bash
TAG=${TAG:-q11}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_shim.py tests/test_gpu_ddp.py -q --timeout 600 > $O/pytest_shim.log 2>&1; echo "rc=$?" >> $O/pytest_shim.log
for n in 2 4; do
  for w in ar_sweep splits; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2980$n tools/report.py --what $w --out $O/report_n$n.jsonl > $O/${w}_n$n.log 2>&1
  done
done
