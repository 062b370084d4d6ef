#!/bin/bash
# Re-measure the tiling / overlap switches of the wide configs (bench.py --config N --math M, one
# line each): usage (under gpurun) bash tools/switch_sweep.sh [tag]
set -u
tag=${1:-sweep}
out=gpurun_out/$tag
mkdir -p $out
run() {  # name config math env...
  local name=$1 c=$2 m=$3; shift 3
  env "$@" timeout 300 python bench.py --config $c --math $m --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --min-seconds 0.5 > $out/$name.json 2> $out/$name.err
  python - "$out/$name.json" "$name" <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:28s} {d['ms_per_step']*1e3:10.1f} us/step  frac {d['roofline']['frac']:.4f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
P
}
run c4_tf32_base 4 tf32 NF_X=0
run c4_tf32_bn32 4 tf32 NF_TC_BN32=1
run c4_fp32_base 4 fp32 NF_X=0
run c3_tf32_base 3 tf32 NF_X=0
run c3_tf32_ew8 3 tf32 NF_TC_EW8=1
run c3_tf32_dual 3 tf32 NF_TC_DUAL=1
run c3_fp32_base 3 fp32 NF_X=0
run c3_fp32_narrow 3 fp32 NF_TC3_NARROW=1
run c5_tf32_base 5 tf32 NF_X=0
run c5_tf32_overlap 5 tf32 NF_BWD_OVERLAP=1
run c5_tf32_noper 5 tf32 NF_TC_NO_PERSISTENT=1
run c5_tf32_dual 5 tf32 NF_TC_DUAL=1
run c5_fp32_base 5 fp32 NF_X=0
run c5_fp32_deep256 5 fp32 NF_TC3_DEEP256=1
run c5_fp32_tpose2 5 fp32 NF_TPOSE=2
