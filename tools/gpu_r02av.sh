O=gpurun_out/r02av; mkdir -p $O
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
HETCCL_LEGACY=0 run --what collectives --out $O/coll_k4s2g.jsonl
HETCCL_LEGACY=0 run --what splits --out $O/splits_k4s2g.jsonl
HETCCL_LEGACY=0 run --what channels --out $O/channels_k4s2g.jsonl
echo done > $O/done.txt
