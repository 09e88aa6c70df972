O=gpurun_out/${TAG:-r02am}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "mux or oneshot or special or collectives" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for e in HETCCL_STEAL=0 HETCCL_STEAL=1 HETCCL_STEAL=0,HETCCL_TILE_KB=1024 HETCCL_STEAL=1,HETCCL_TILE_KB=1024; do
  env ${e//,/ } timeout 300 python bench.py --no-cpu-baseline > $O/ab_$e.json 2> $O/ab_$e.err
  echo "$e $(tail -1 $O/ab_$e.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1)" >> $O/ab.txt
done
HETCCL_STEAL=1 timeout 300 python tools/trace_run.py --out $O/t > $O/trace.txt 2>&1
echo done > $O/done.txt
