#!/bin/bash
# Round-2 final measurements on the GPU box (run from the repo root under
# gpurun): GPU test suite, bench lines of every config (driver-style command),
# the reference arm, complex and TEBD throughput, the host-buffer probe and
# the per-GPU batch sweep that the strong batch split runs at 2/4/8 GPUs.
set -u
out=gpurun_out/final
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > $out/bench_C4.json 2> $out/bench_C4.err
for c in C1 C2 C3 C3q3 C5; do
  python bench.py --config $c --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
done
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference_C4.json 2> $out/bench_reference_C4.err
for b in 4 8 16; do
  python bench.py --batch $b --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_C4_batch$b.json 2>/dev/null
done
for c in C4 C3 C2 C1; do python tools/complex_bench.py --config $c >> $out/complex_bench.jsonl 2>/dev/null; done
for c in 32 64 128 256; do python tools/tebd_bench.py --chi $c --layers 4 --random-state >> $out/tebd_layer.jsonl 2>/dev/null; done
python tools/probe/e2e_probe.py 7 > $out/e2e_probe.txt 2>&1
ls -la $out
