#!/bin/bash
# One parameterised gpurun session (replaces round 1's per-session gpu_q*.sh scripts).
#
#   gpurun --timeout 1800 -- 'TAG=r02a STEPS="tests smoke bench1 ncu_list ncu_full" bash tools/gpu.sh'
#
# TAG   : output directory gpurun_out/$TAG
# STEPS : any of
#   build       rebuild libhetccl.so in place (normally built here and shipped)
#   tests       pytest -m gpu (every GPU test the box's GPU count allows)
#   tests_k     pytest -m gpu -k "$K" (a subset)
#   smoke       __graft_entry__.py smoke
#   bench1      bench.py N=1 (the driver's line)
#   benchN      bench.py under torchrun for N in $NS (default "2 4"; skipped when fewer GPUs)
#   ref1        bench.py --impl reference N=1
#   ncu_list    ncu launch list of the N=1 bench (cold-cache per-launch times)
#   ncu_full    ncu --set full of the N=1 bench's k_allreduce (one launch)
#   report      tools/report.py --what $WHAT under torchrun on $NR GPUs (default: collectives on 4)
#   mux_ab      bench.py N=1 for each build variant in $LIBS (libhetccl_<v>.so) and env set in $ENVS
#   cmd         eval "$CMD" (anything else; output in $O/cmd.log)
TAG=${TAG:-s}; O=gpurun_out/$TAG; mkdir -p $O
NGPU=$(python -c 'import torch; print(torch.cuda.device_count())' 2>/dev/null || echo 0)
echo "ngpu=$NGPU tag=$TAG steps=$STEPS" > $O/session.txt
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv >> $O/session.txt 2>&1
NCUCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for s in $STEPS; do
  case $s in
    build) python -c "from paper_2601_22585_b200 import build as b; b.build(force=True); b.build_shim(force=True)" > $O/build.log 2>&1 ;;
    tests) timeout ${TTEST:-1500} python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log ;;
    tests_k) timeout ${TTEST:-1500} python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "$K" > $O/pytest_k.log 2>&1; echo "pytest rc=$?" >> $O/pytest_k.log ;;
    smoke) timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log ;;
    bench1) timeout 600 python bench.py ${BARGS} > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?" >> $O/bench1.err ;;
    ref1) timeout 600 python bench.py --impl reference > $O/ref1.json 2> $O/ref1.err; echo "ref1 rc=$?" >> $O/ref1.err ;;
    benchN)
      for n in ${NS:-2 4}; do
        [ "$NGPU" -ge "$n" ] || continue
        timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port 2960$n bench.py --gpus $n ${BARGS} > $O/bench$n.json 2> $O/bench$n.err; echo "bench$n rc=$?" >> $O/bench$n.err
      done ;;
    ncu_list)
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_list.log 2>&1 && \
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $NCUCMD > $O/ncu_list.log 2>&1
      echo "ncu list rc=$?" >> $O/ncu_list.log ;;
    ncu_full)
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_full.log 2>&1 && \
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_allreduce} -s 3 -c 1 -o $O/ar_full $NCUCMD > $O/ncu_full.log 2>&1
      echo "ncu full rc=$?" >> $O/ncu_full.log ;;
    report)
      NR=${NR:-4}; [ "$NGPU" -ge "$NR" ] || NR=$NGPU
      timeout ${TREP:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $NR --master-addr 127.0.0.1 \
        --master-port 2981$NR tools/report.py --what ${WHAT:-collectives} ${RARGS} --out $O/report_${WHAT:-collectives}_n$NR.jsonl > $O/report_${WHAT:-collectives}_n$NR.log 2>&1 ;;
    mux_ab)
      for v in ${LIBS:-default}; do
        for e in ${ENVS:-NONE=1}; do
          lib=libhetccl.so; [ "$v" = default ] || lib=libhetccl_$v.so
          env ${e//,/ } HETCCL_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps ${ABSTEPS:-20} ${BARGS} > $O/ab_${v}_${e}.json 2> $O/ab_${v}_${e}.err
          echo "$v $e $(python -c "import json,sys; d=json.load(open('$O/ab_${v}_${e}.json')); print(d['value'], d['roofline']['frac'])" 2>&1)" >> $O/mux_ab.txt
        done
      done ;;
    cmd) eval "$CMD" > $O/cmd.log 2>&1; echo "cmd rc=$?" >> $O/cmd.log ;;
  esac
done
echo done >> $O/session.txt
