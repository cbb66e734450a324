mkdir -p gpurun_out/oz3
timeout 900 python -m pytest tests -m gpu -q -x -k "ozaki or configs or acceptance" > gpurun_out/oz3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/oz3/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/oz3/bench_C4.json 2> gpurun_out/oz3/bench_C4.err
timeout 300 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/oz3/bench_C5.json 2> gpurun_out/oz3/bench_C5.err
