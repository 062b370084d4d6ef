#!/bin/bash
# One GPU-box pass: build, GPU parity tests, smoke, default bench (c2), wide-config benches,
# launch list of the default bench and a full ncu capture of its kernel.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
set -u
tag=${1:-check}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
for c in 5 3 4; do for m in tf32 fp32; do
  timeout 600 python bench.py --config $c --math $m --steps 10 --warmup 3 --no-e2e --min-seconds 0.5 > $out/bench_c${c}_$m.json 2> $out/bench_c${c}_$m.err
done; done
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
  python bench.py --steps 500 --warmup 3 --no-cpu-baseline --no-e2e --min-seconds 0 > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
# one ncu tool per gpurun call: the full capture runs separately (NCU_FULL=1 or tools/ncu_full.sh)
if [ "${NCU_FULL:-0}" = 1 ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o $out/prof_fused \
  python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e --min-seconds 0 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
