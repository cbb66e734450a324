mkdir -p gpurun_out/oz6
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/oz6/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/oz6/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/oz6/bench_C4.json 2> gpurun_out/oz6/bench_C4.err
timeout 300 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/oz6/bench_C5.json 2> gpurun_out/oz6/bench_C5.err
