for ts in 0 1; do UL_TC_TMASTORE=$ts BENCH_DT=1 timeout 120 python tools/bench_gemm.py > gpurun_out/g.json 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1])
print('tmastore=$ts', ' '.join(f\"{k}={v['us']:.1f}\" for k,v in d.items() if isinstance(v,dict)), 'total', round(d['total_us'],1))"; done
for ts in 0 1; do UL_TC_TMASTORE=$ts timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('tmastore=$ts', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['ms_per_step'],2))"; done
