for cfg in "UL_TC_CLUSTER=1" "UL_TC_CLUSTER=1 UL_TC_DBG=1" "UL_TC_CLUSTER=1 UL_TC_DBG=2" "UL_TC_CLUSTER=1 UL_TC_DBG=4" "UL_TC_CLUSTER=1 UL_TC_DBG=5" "UL_TC_CLUSTER=1 UL_TC_DBG=7" "UL_TC_CLUSTER=1 UL_TC_BN=128" "UL_TC_CLUSTER=2 UL_TC_BN=128" "UL_TC_CLUSTER=1 UL_TC_BN=128 UL_TC_DBG=4"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/bench_gemm.py 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' '.join(f\"{k}={v['us']:.1f}\" for k,v in d.items() if isinstance(v,dict)), 'total', round(d['total_us'],1))"
done
