#!/bin/bash
# One GPU-box pass: build, GPU parity tests, smoke, bench, launch list of the bench command.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
set -u
tag=${1:-check}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -5 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
tail -3 $out/smoke.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
cat $out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $out/launches.csv \
  python bench.py --steps 500 --warmup 3 --no-cpu-baseline --no-e2e --min-seconds 0 > $out/ncu_bench.log 2>&1; echo "ncu rc=$?"
