#!/bin/bash
for c in C1 C2 C3 C5; do
  for e in "X=1" "RSVD_NO_GRAPH=1" "X=1" "RSVD_NO_GRAPH=1"; do
    env $e python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $e', round(d['value'],2), round(d['ms_per_step'],3))"
  done
done
