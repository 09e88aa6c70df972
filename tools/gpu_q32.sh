#!/bin/bash
# NVLS: per-thread alias fence after the copy-in; tests + bench
TAG=${TAG:-q32}; O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_nvls.py -m gpu -q --timeout 120 > $O/pytest_nvls.log 2>&1; echo "pytest rc=$?" >> $O/pytest_nvls.log
timeout 200 python tools/nvls_bench.py --gpus 4 --maps 4,2+2 --mibs 64,256 > $O/nvls_bench.jsonl 2> $O/nvls_bench.err; echo "bench rc=$?" >> $O/nvls_bench.err
