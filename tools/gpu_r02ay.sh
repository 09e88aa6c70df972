O=gpurun_out/r02ay; mkdir -p $O
run() { n=$1; shift; timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((RANDOM%800+100)) tools/report.py "$@" > /dev/null 2>> $O/err.log; }
run 4 --what ar_sweep --out $O/sweep_n4.jsonl
run 2 --what ar_sweep --out $O/sweep_n2.jsonl
run 4 --what c4 --out $O/c4_n4.jsonl
run 4 --what c5 --out $O/c5_n4.jsonl
run 2 --what c5 --out $O/c5_n2.jsonl
echo done > $O/done.txt
