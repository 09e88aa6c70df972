O=gpurun_out/r02at; mkdir -p $O
HETCCL_S2G=1 timeout 600 python -m pytest tests/test_gpu_mux.py tests/test_gpu_mux_protocol.py -q -p no:cacheprovider --timeout 300 -x > $O/pytest_mux_s2g.log 2>&1; echo rc=$? >> $O/pytest_mux_s2g.log
HETCCL_LEGACY=0 HETCCL_S2G=1 timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_collectives.py -q -p no:cacheprovider --timeout 300 -x > $O/pytest_multi_s2g.log 2>&1; echo rc=$? >> $O/pytest_multi_s2g.log
HETCCL_S2G=1 timeout 300 python bench.py --no-cpu-baseline > $O/mux_s2g.json 2>&1
NS="4 2" ENVS="HETCCL_LEGACY=0,HETCCL_S2G=1,HETCCL_NCHANNELS=64 HETCCL_LEGACY=0,HETCCL_S2G=1,HETCCL_NCHANNELS=148 HETCCL_LEGACY=0,HETCCL_S2G=1,HETCCL_NCHANNELS=296 HETCCL_LEGACY=0,HETCCL_S2G=1 HETCCL_LEGACY=0,HETCCL_NCHANNELS=148 NONE=1" TAG=r02at bash tools/gpu_mab.sh
echo done > $O/done.txt
