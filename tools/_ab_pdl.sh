for pdl in 1 0; do for pr in bf16 tf32; do UL_PDL=$pdl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision $pr > gpurun_out/bench_${pr}_pdl$pdl.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/bench_${pr}_pdl$pdl.log').read().strip().splitlines()[-1])
print('pdl=$pdl $pr', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'M/s e2e', round(d['e2e']['ms_per_step'],2), 'parity', round(d['parity_mode']['update_ms'],2))"; done; done
