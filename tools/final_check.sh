#!/bin/bash
# Last check of the shipped build, as the driver runs it: smoke(), pytest -m gpu, the default bench line and the reference arm.
out=gpurun_out/${1:-final_check}
mkdir -p $out
timeout 300 python __graft_entry__.py smoke > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench_default.json 2> $out/bench_default.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
tail -2 $out/smoke.log; tail -2 $out/pytest_gpu.log; cut -c1-400 $out/bench_default.json
