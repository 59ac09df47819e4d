O=gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
timeout 300 python tools/bench_kernels.py > $O/kernels.json 2>&1; python -c "
import json; d=json.load(open('$O/kernels.json')); print({k:(round(v['gbs']),round(v['frac'],3)) for k,v in d.items()})"
