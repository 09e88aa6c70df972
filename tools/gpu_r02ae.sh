O=gpurun_out/r02ae; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist_backend.py tests/test_gpu_ddp.py tests/test_gpu_shim.py tests/test_gpu_special.py tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 300 > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
run 4 --what channels --out $O/channels_n4.jsonl
run 2 --what channels --out $O/channels_n2.jsonl
run 4 --what overlap --out $O/overlap_n4.jsonl
echo done > $O/done.txt
