O=gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
for v in 1 0; do echo "bnwaves=$v"; UL_TC_BN_WAVES=$v BENCH_DT=1 timeout 120 python tools/bench_gemm.py | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' '.join(f\"{k}={v['us']:.1f}\" for k,v in d.items() if isinstance(v,dict)), 'total', round(d['total_us'],1))"
UL_TC_BN_WAVES=$v timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['roofline']['phase_ms_per_update'].items()})"; done
