O=gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
for v in 1 0; do UL_GATHER_AHEAD=$v timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('ahead=$v', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['phase_ms_per_update'].items()})"; done
