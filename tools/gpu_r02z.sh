O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
for e in NONE=1 HETCCL_LEGACY=0; do
  env $e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --no-cpu-baseline > $O/bench4_$e.json 2> $O/bench4_$e.err
  env $e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --no-cpu-baseline > $O/bench2_$e.json 2> $O/bench2_$e.err
done
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
run --what splits --out $O/splits_n4.jsonl
run --what collectives --out $O/coll_n4.jsonl
HETCCL_LEGACY=0 run --what collectives --out $O/coll_n4_tma.jsonl
timeout 300 python bench.py --no-cpu-baseline > $O/bench1.json 2> $O/bench1.err
echo done > $O/done.txt
