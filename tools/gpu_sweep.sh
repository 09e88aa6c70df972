#!/bin/bash
# AR size sweep (tools/report.py --what ar_sweep) on $N GPUs for each env combination in $ENVS (commas separate
# vars): one JSONL per combination, rows = sizes in $MIBS
O=gpurun_out/${TAG:-sweep}; mkdir -p $O
for e in ${ENVS:-NONE=1}; do
  env ${e//,/ } timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-4} --master-addr 127.0.0.1 \
    --master-port 29$((RANDOM%800+100)) tools/report.py --what ar_sweep --mibs ${MIBS:-2,4,8,16,32,64,128} ${RARGS} \
    --out $O/s_$e.jsonl > $O/s_$e.txt 2>&1
  echo "$e" >> $O/sweep.txt
  python - "$O/s_$e.jsonl" >> $O/sweep.txt <<'EOF'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(" ", {k: d[k] for k in d if k in ("bytes", "us", "nccl_us", "busbw", "nccl_busbw", "vs_nccl", "staged_busbw", "r7_gate")})
EOF
done
