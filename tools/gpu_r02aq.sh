O=gpurun_out/r02aq; mkdir -p $O
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
HETCCL_LEGACY=0 HETCCL_NCHANNELS=296 run --what collectives --out $O/coll_k4_296.jsonl
run --what collectives --out $O/coll_legacy.jsonl
echo done > $O/done.txt
