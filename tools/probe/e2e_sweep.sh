#!/bin/bash
# Usage: tools/probe/e2e_sweep.sh CONFIG "ENV1" "ENV2" ...   (results in gpurun_out/sweep_*.log)
cfg=$1; shift
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --config $cfg --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$i.log 2>&1
  echo "$e" > gpurun_out/sweep_$i.env
  i=$((i+1))
done
