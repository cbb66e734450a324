#!/bin/bash
# Check of the 128 x 32 tile / path rule: Ozaki + config tests, C3 / C3q3 / C4 / C5 bench lines, launch list of C3.
out=gpurun_out/${1:-oz14}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "ozaki or c3 or c4 or c5 or acceptance or sweep" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for c in C3 C3q3 C4 C5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
done
RSVD_FP64_GEMM=dmma timeout 300 python bench.py --config C3 --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_C3_dmma.json 2>/dev/null
timeout 600 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file $out/launches_C3.csv python tools/probe/one_call.py C3 > $out/launches_C3.log 2>&1
tail -3 $out/pytest.log
python tools/ncu_launch_shares.py $out/launches_C3.csv 2>/dev/null | head -12
