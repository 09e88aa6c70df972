#!/bin/bash
# flat cross all-gather by default for <= 32 MiB (R20) + mid-size tile experiments (balanced tiles)
TAG=${TAG:-q24}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout 900 python -m pytest tests/test_gpu_mux.py tests/test_gpu_multi.py tests/test_gpu_oneshot.py -m gpu -q --timeout 300 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
MIBS=4,8,16,32,64,128
for n in 4 2; do
  for cfg in "dflt" "flat0" "mt2f16" "mt4f8"; do
    case $cfg in
      dflt) E="";; flat0) E="HETCCL_FLAT_AG=0";; mt2f16) E="HETCCL_MIN_TILES=2 HETCCL_TILE_FLOOR_KB=16";;
      mt4f8) E="HETCCL_MIN_TILES=4 HETCCL_TILE_FLOOR_KB=8";;
    esac
    env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2990$n tools/report.py --what ar_sweep --mibs $MIBS --out $O/sweep_${cfg}_n$n.jsonl > $O/sweep_${cfg}_n$n.log 2>&1
  done
done
