run() { name=$1; cfgs=$2; shift 2; env "$@" python bench.py --configs $cfgs --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['configs'].items(): print('$name', k, round(v['ms_per_step']*1e3,1), 'us', round(v['roofline']['frac'],4), v.get('clocks',{}).get('sm_mhz'))
"; }
run base 5:tf32 NF_X=0
run tpose0 5:tf32 NF_TPOSE=0
run base 5:tf32 NF_X=0
run tpose0 5:tf32 NF_TPOSE=0
run base 5:tf32 NF_X=0
run tpose0 5:tf32 NF_TPOSE=0
