#!/bin/bash
cfg=$1; shift
for e in "$@"; do
  out=""
  for i in 1 2 3 4 5 6; do
    v=$(env $e python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']))")
    out="$out $v"
  done
  echo "$cfg $e:$out"
done
