#!/bin/bash
for i in 1 2 3; do
  python bench.py --config C2 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps30', round(d['value']), round(d['ms_per_step'],2), d['clocks'])"
  python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps5 ', round(d['value']), round(d['ms_per_step'],2), d['clocks'])"
done
