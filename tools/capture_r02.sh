#!/bin/bash
# Round-2 evidence capture on the GPU box (run from the repo root under gpurun):
# launch lists of one pipeline call per config and ncu --set full captures of
# the dominant / latency-bound kernels.  Outputs go to gpurun_out/cap/.
set -u
out=gpurun_out/cap
mkdir -p $out
NCU="ncu --clock-control none --profile-from-start off"
for c in C1 C2 C3 C4 C5; do
  timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file $out/launches_$c.csv \
    python tools/probe/one_call.py $c > $out/launches_$c.log 2>&1
done
full() {  # name config kernel-regex [launch-skip]
  timeout 900 $NCU --set full --import-source on -k "regex:$3" --launch-skip ${4:-0} -c 1 \
    -o $out/$1 python tools/probe/one_call.py $2 > $out/$1.log 2>&1
}
full apass_c4 C4 'dgemm_tma_kernel<128, 96, 4, 2, 3, 0>' 0
full gram_c4 C4 'dgemm_tma_kernel<96, 96' 0
full jdf_c4 C4 jacobi_df_kernel 0
full gchol_c4 C4 'gchol_kernel' 0
full jdf_c2 C2 jacobi_df_kernel 0
full fcqr_c2 C2 fcqr_kernel 0
full fcqr_c1 C1 fcqr_kernel 0
full jclug_c3 C3 jacobi_clug_kernel 0
full gchol_c3 C3 'gchol_kernel' 0
ls -la $out
