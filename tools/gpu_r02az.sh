O=gpurun_out/r02az; mkdir -p $O
run() { n=$1; shift; timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
HETCCL_ONESHOT_KB=16384 run 4 --what ar_sweep --mibs 2,4,8,16 --out $O/sweep_os16_n4.jsonl
HETCCL_LEGACY=0 run 4 --what ar_sweep --mibs 4,8,16,32,64,128 --out $O/sweep_k4_n4.jsonl
echo done > $O/done.txt
