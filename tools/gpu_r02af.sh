O=gpurun_out/r02af; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist_backend.py tests/test_gpu_shim.py -q -p no:cacheprovider --timeout 300 > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29444 tools/report.py --what overlap --out $O/overlap_n4.jsonl > /dev/null 2>> $O/err.log
echo done > $O/done.txt
