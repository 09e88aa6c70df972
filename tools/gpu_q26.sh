#!/bin/bash
# mux A/B of build variants: CTAs per SM (3, 4) and L2 prefetch distance (4 batches)
TAG=${TAG:-q26}; O=gpurun_out/$TAG; mkdir -p $O
for rep in 1 2; do
  for lib in libhetccl.so libhetccl_c3.so libhetccl_c4.so libhetccl_pf4.so libhetccl_c3pf4.so; do
    HETCCL_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>$O/err.txt | sed "s/^/$lib /" >> $O/mux.txt
  done
done
