# A/B of runtime switches on one box: bench.py bf16 update ms for each combination
for rep in 1 2; do
for pair in 1 0; do for g in 0 1; do
UL_TC_PAIR=$pair UL_GROUP=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision ${PREC:-bf16} > gpurun_out/ab.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('rep=$rep pair=$pair group=$g', round(d['ms_per_step'],3), 'ms', 'e2e', round(d['e2e']['ms_per_step'],2))"
done; done; done
