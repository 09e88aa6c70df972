O=gpurun_out/r02y; mkdir -p $O
run() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
run 2 --what ar_sweep --kibs 1,4,16,64,256,1024 --out $O/lat_n2.jsonl
run 4 --what ar_sweep --kibs 1,4,16,64,256,1024 --out $O/lat_n4.jsonl
run 4 --what splits --out $O/splits_n4.jsonl
run 4 --what collectives --out $O/coll_n4.jsonl
run 4 --what c4 --out $O/c4_n4.jsonl
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 4 > $O/bench4.json 2> $O/bench4.err
echo done > $O/done.txt
