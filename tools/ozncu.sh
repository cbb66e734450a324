#!/bin/bash
# ncu --set full of the Ozaki GEMM (first NN launch of one C4 call).
out=gpurun_out/${1:-ozncu}
mkdir -p $out
timeout 900 ncu --clock-control none --profile-from-start off --set full --import-source on -k "regex:oz_gemm" -c 1 -o $out/ozgemm_c4 python tools/probe/one_call.py C4 > $out/ozgemm_c4.log 2>&1
timeout 900 ncu --clock-control none --profile-from-start off --set full --import-source on -k "regex:oz_slice_a_kernel" -c 1 -o $out/ozslicea_c4 python tools/probe/one_call.py C4 > $out/ozslicea_c4.log 2>&1
ls -la $out
