O=gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/lb.csv python tools/profile_ppo.py bf16 > /dev/null 2>&1
python tools/launch_summary.py $O/lb.csv | head -12
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['roofline']['phase_ms_per_update'].items()})"; done
