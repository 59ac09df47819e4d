O=gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
timeout 300 python tools/_e2e_probe.py 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['ms_per_step'],3), 'serial', round(d['e2e']['serial_gae_ppo_update_ms'],2), 'parity', round(d['parity_mode']['update_ms'],2))"; done
