#!/bin/bash
# Usage: tools/probe/var_sweep.sh CONFIG STEPS "ENV" ... : 3 runs each, value and ms/step
cfg=$1; steps=$2; shift 2
for e in "$@"; do
  for i in 1 2 3; do
    env $e python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value'],2), round(d['ms_per_step'],2))"
  done
done
