#!/bin/bash
# NVLS session: the NVLS test file (single- and multi-process), the single-process NVLS bench, and the
# multi-process bench.py with HETCCL_NVLS=1 (fp32-staged and native 16-bit) for each $ENVX setting
O=gpurun_out/${TAG:-nvls}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nvls.py -q -p no:cacheprovider --timeout 300 > $O/pytest_nvls.log 2>&1; echo rc=$? >> $O/pytest_nvls.log
timeout 600 python tools/nvls_bench.py --gpus 4 --maps 4,2+2 --mibs 16,256 > $O/nvls_bench.jsonl 2>&1
NS="4" ENVS="${ENVX:-HETCCL_NVLS=1 HETCCL_NVLS=1,HETCCL_NVLS_WIDE=0}" TAG=${TAG:-nvls} bash tools/gpu_mab.sh
