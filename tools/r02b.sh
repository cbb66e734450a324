#!/bin/bash
# Round-2 measurements after the emulated-FP64 (INT8 tcgen05) A-pass: smoke,
# GPU tests, bench lines of every config, reference arm, launch lists of one
# call (C4, C5) and ncu --set full of the three Ozaki kernels.  Run from the
# repo root under gpurun; outputs under gpurun_out/r02b/.
set -u
out=gpurun_out/r02b
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 300 python __graft_entry__.py smoke > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > $out/bench_C4.json 2> $out/bench_C4.err
for c in C1 C2 C3 C3q3 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
done
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference_C4.json 2> $out/bench_reference_C4.err
for b in 4 8 16; do
  timeout 200 python bench.py --batch $b --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_C4_batch$b.json 2>/dev/null
done
RSVD_FP64_GEMM=dmma timeout 300 python bench.py --no-cpu-baseline --no-gpu-tsvd --steps 10 --warmup 3 > $out/bench_C4_dmma.json 2>/dev/null
NCU="ncu --clock-control none --profile-from-start off"
for c in C4 C5; do
  timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file $out/launches_$c.csv \
    python tools/probe/one_call.py $c > $out/launches_$c.log 2>&1
done
full() {  # name config kernel-regex [launch-skip]
  timeout 900 $NCU --set full --import-source on -k "regex:$3" --launch-skip ${4:-0} -c 1 \
    -o $out/$1 python tools/probe/one_call.py $2 > $out/$1.log 2>&1
}
full ozgemm_c4 C4 oz_gemm 0
full ozgemm_tn_c4 C4 oz_gemm 1
full ozslicea_c4 C4 oz_slice_a_kernel 0
full ozsliceb_c4 C4 oz_slice_b_kernel 0
full ozexp_c4 C4 oz_exp_kernel 0
full ozgemm_c5 C5 oz_gemm 0
ls -la $out
