#!/bin/bash
# Quick check of an Ozaki-kernel change (tools/oz_check.sh <name>): kernel + C4/C5 parity tests, C4 / C5 / C2 bench lines, one C4 launch list.
out=gpurun_out/${1:-oz7}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "ozaki or c4 or c5 or acceptance" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_C4.json 2> $out/bench_C4.err
timeout 300 python bench.py --config C5 --no-cpu-baseline --no-gpu-tsvd --steps 5 --warmup 3 > $out/bench_C5.json 2> $out/bench_C5.err
timeout 300 python bench.py --config C2 --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_C2.json 2> $out/bench_C2.err
timeout 600 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file $out/launches_C4.csv python tools/probe/one_call.py C4 > $out/launches_C4.log 2>&1
tail -3 $out/pytest.log
python tools/ncu_launch_shares.py $out/launches_C4.csv > $out/launch_shares_C4.txt 2>&1; head -12 $out/launch_shares_C4.txt
