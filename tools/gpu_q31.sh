#!/bin/bash
# NVLS mode after the fixed chunk partition: tests (twice, to catch races) + bench
TAG=${TAG:-q31}; O=gpurun_out/$TAG; mkdir -p $O
for rep in 1 2; do
timeout 400 python -m pytest tests/test_gpu_nvls.py -m gpu -q --timeout 120 > $O/pytest_nvls_$rep.log 2>&1; echo "pytest rc=$?" >> $O/pytest_nvls_$rep.log
done
timeout 300 python tools/nvls_bench.py --gpus 4 --maps 2,4,2+2 --mibs 16,64,256 > $O/nvls_bench.jsonl 2> $O/nvls_bench.err; echo "bench rc=$?" >> $O/nvls_bench.err
