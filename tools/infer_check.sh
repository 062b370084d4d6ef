#!/bin/bash
# Inference kernel check: parity tests of the tcgen05 inference kernel, then nf_output timing over
# config 2's 50,000 rows for each formulation (NF_INFER_TC_FORM) and the timing experiments.
# Usage (under gpurun): bash tools/infer_check.sh [tag]
set -u
tag=${1:-infer}
out=gpurun_out/$tag
mkdir -p $out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "inference or output or accuracy or loss" > $out/pytest.log 2>&1
echo "pytest rc=$?" >> $out/pytest.log; tail -4 $out/pytest.log
{
for f in 2 1 0; do echo "form $f"; NF_INFER_TC_FORM=$f timeout 120 python tools/infer_probe.py 100; done
for e in 2 4 6; do echo "form 2 exp $e"; NF_INFER_TC_FORM=2 NF_ITC_EXP=$e timeout 120 python tools/infer_probe.py 100; done
echo "simt"; NF_INFER_SIMT=1 timeout 120 python tools/infer_probe.py 100
} > $out/probe.txt 2>&1
cat $out/probe.txt
