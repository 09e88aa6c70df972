#!/bin/bash
# one-shot A/B: AR sweep at 2+2 (4 GPUs) and 1+1 for each env combination in $ENVS, plus the one-shot tests
O=gpurun_out/${TAG:-os}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_oneshot.py tests/test_gpu_mux.py -q -p no:cacheprovider --timeout 300 > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for e in ${ENVS:-NONE=1}; do
  env ${e//,/ } timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29$((RANDOM%800+100)) tools/report.py --what ar_sweep --mibs ${MIBS:-2,4,8,16,32} --out $O/sweep4_$e.jsonl > /dev/null 2>> $O/err.log
done
