O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bf16.py -q -x > $O/t_gemm.log 2>&1; tail -2 $O/t_gemm.log
for v in "UL_TC_PAIR=0" "UL_TC_TMASTORE=0"; do echo "== $v"; env $v BENCH_DT=1 timeout 120 python tools/bench_gemm.py | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' '.join(f\"{k}={v['us']:.1f}\" for k,v in d.items() if isinstance(v,dict)), 'total', round(d['total_us'],1))"; done
timeout 120 python tools/trace_gemm.py > $O/trace.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/b.log 2>&1; python -c "
import json
d=json.loads(open('$O/b.log').read().strip().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), 'ms', d['roofline']['phase_ms_per_update'], 'e2e', round(d['e2e']['ms_per_step'],2))"
