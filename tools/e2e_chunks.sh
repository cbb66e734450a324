#!/bin/bash
# e2e (host buffers) of C4 against the chunk count of the pipelined host path.
out=gpurun_out/${1:-e2e}
mkdir -p $out
for n in 7 8 11 16; do
  RSVD_HOST_CHUNKS=$n timeout 300 python bench.py --no-cpu-baseline --no-gpu-tsvd --steps 5 --warmup 3 > $out/bench_C4_chunks$n.json 2>/dev/null
  python - <<PY
import json
d=json.loads(open("$out/bench_C4_chunks$n.json").read().strip().splitlines()[-1])
print("chunks $n: value", round(d["value"],1), "e2e", round(d["e2e"]["value"],1))
PY
done
