O=gpurun_out/r02be; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nvls.py -q -p no:cacheprovider --timeout 300 > $O/pytest_nvls.log 2>&1; echo rc=$? >> $O/pytest_nvls.log
NS="4 2" ENVS="HETCCL_NVLS=1 HETCCL_NVLS=1,HETCCL_NVLS_WIDE=0 HETCCL_NVLS=1,HETCCL_NVLS_WIDE=0,HETCCL_NVLS_NCH=296" TAG=r02be bash tools/gpu_mab.sh
