#!/bin/bash
# ncu --set full of the Ozaki GEMM launches: C4 NN / TN (mixed 64 + 32 tiles), C5 first launch, C3 (32-wide tiles).
out=gpurun_out/${1:-ozncu}
mkdir -p $out
NCU="ncu --clock-control none --profile-from-start off --set full --import-source on"
timeout 900 $NCU -k "regex:oz_gemm" -c 1 -o $out/ozgemm_c4 python tools/probe/one_call.py C4 > $out/ozgemm_c4.log 2>&1
timeout 900 $NCU -k "regex:oz_gemm" --launch-skip 1 -c 1 -o $out/ozgemm_tn_c4 python tools/probe/one_call.py C4 > $out/ozgemm_tn_c4.log 2>&1
timeout 900 $NCU -k "regex:oz_gemm" -c 1 -o $out/ozgemm_c5 python tools/probe/one_call.py C5 > $out/ozgemm_c5.log 2>&1
timeout 900 $NCU -k "regex:oz_gemm" -c 1 -o $out/ozgemm_c3 python tools/probe/one_call.py C3 > $out/ozgemm_c3.log 2>&1
for c in C1 C2 C3; do
  timeout 600 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file $out/launches_$c.csv python tools/probe/one_call.py $c > $out/launches_$c.log 2>&1
done
ls -la $out
