# out-layer kernel check: focused GPU tests, c3/c4 step times (graph-replay protocol) with the
# register-resident output layer and with NF_OUT_V1=1, ncu per-launch times of both kernels
set -u
out=gpurun_out/${1:-olt}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { tail -20 $out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "full_size or out_layer or c3 or c4 or fused_out or train_batch" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log; tail -3 $out/pytest.log
for v in 0 1; do
  if [ $v = 1 ]; then export NF_OUT_V1=1; else unset NF_OUT_V1; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --min-seconds 0.2 --configs 3:tf32,3:fp32,4:tf32,4:fp32 > $out/b_v$v.json 2> $out/b_v$v.err
  python -c "
import json; d=json.loads(open('$out/b_v$v.json').read().splitlines()[-1])
for k,c in d['configs'].items(): print('v$v', k, round(c['ms_per_step']*1000,1), 'us', round(c['roofline']['frac'],4))"
done
unset NF_OUT_V1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:out_layer --csv python bench.py --config 3 --math tf32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --min-seconds 0 > $out/ncu_c3.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:out_layer --csv python bench.py --config 4 --math tf32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --min-seconds 0 > $out/ncu_c4.csv 2>&1
