#!/bin/bash
# NVLS mode (NEXT-1): tests + NVLS vs P2P single-process bench
TAG=${TAG:-q29}; O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi -q | grep -i -A3 "fabric\|multicast" > $O/smi_fabric.txt 2>&1
timeout 400 python -m pytest tests/test_gpu_nvls.py -m gpu -x -q --timeout 120 > $O/pytest_nvls.log 2>&1; echo "pytest rc=$?" >> $O/pytest_nvls.log
timeout 300 python tools/nvls_bench.py --gpus 4 --maps 2,4,2+2 --mibs 16,64,256 > $O/nvls_bench.jsonl 2> $O/nvls_bench.err; echo "bench rc=$?" >> $O/nvls_bench.err
