#!/bin/bash
# ncu --set full of one c5 TF32 weight-gradient launch (persistent MN/MN EpiGrad) and one forward launch
# usage: tools/ncu_c5_grad.sh <out-prefix>
set -e
OUT=${1:-gpurun_out/ncu_c5}
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_persistent -s 8 -c 4 \
    -o $OUT python tools/kernel_times.py 5 tf32 2 > ${OUT}.log 2>&1 || true
ncu -i $OUT.ncu-rep --page details --csv > ${OUT}_details.csv 2>/dev/null || true
