O=gpurun_out/r02ar; mkdir -p $O
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
HETCCL_TILE_KB=512 run --what collectives --out $O/coll_t512.jsonl
HETCCL_TILE_KB=1024 run --what collectives --out $O/coll_t1024.jsonl
HETCCL_TILE_KB=512 run --what splits --out $O/splits_t512.jsonl
echo done > $O/done.txt
