#!/bin/bash
cfg=$1; n=$2
for i in $(seq 1 $n); do
  RSVD_BENCH_VERBOSE=1 python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "step device" 
done
