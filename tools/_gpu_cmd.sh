O=gpurun_out
for cfg in "UL_TC_GRID_DX=0" "UL_TC_GRID_DX=74" "UL_TC_GRID_DX=96" "UL_TC_GRID_DX=74 UL_GROUP_BWD=0"; do env $cfg timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('$cfg', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['roofline']['phase_ms_per_update'].items()}, 'e2e', round(d['e2e']['ms_per_step'],2))"; done
