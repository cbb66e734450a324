set -u
out=gpurun_out/val1
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for c in C4 C1 C2 C3 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
done
