O=gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
UL_GROUP=1 timeout 600 python -m pytest tests/test_gpu_ppo.py tests/test_gpu_bf16.py -q -x -m gpu 2>&1 | tail -1
for cfg in "UL_GROUP_BWD=0" "UL_GROUP_BWD=1" "UL_GROUP_BWD=0" "UL_GROUP_BWD=1"; do env $cfg timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('$cfg', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['roofline']['phase_ms_per_update'].items()}, 'e2e', round(d['e2e']['ms_per_step'],2))"; done
