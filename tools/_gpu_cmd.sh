O=gpurun_out
for b in 4 8 16; do UL_GATHER_BLOCKS_PER_SM=$b timeout 300 python tools/bench_kernels.py > $O/kernels.json 2>&1; python -c "
import json; d=json.load(open('$O/kernels.json')); print('bpsm=$b', {k:(round(v['gbs']),round(v['frac'],3)) for k,v in d.items() if 'gather' in k})"
UL_GATHER_BLOCKS_PER_SM=$b timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), 'ms gather', round(d['roofline']['phase_ms_per_update']['gather'],3))"; done
