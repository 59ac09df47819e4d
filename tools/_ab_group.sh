for g in 0 1; do for pr in bf16 tf32; do UL_GROUP=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision $pr > gpurun_out/bench_${pr}_g$g.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/bench_${pr}_g$g.log').read().strip().splitlines()[-1])
print('group=$g $pr', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M/s e2e', round(d['e2e']['ms_per_step'],2))"; done; done
